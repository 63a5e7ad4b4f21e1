"""Float64 CPU restatement of the reference DSP train step -- TEST INFRASTRUCTURE.

Every function cites the reference file:line it restates (paths relative to
/root/reference/pkg/src/stalepipe/). Bit-level conventions that the parity
tests depend on are kept: ascending-k `matmul`, the IEEE op order of the
optimizers, the FIFO prefill tags and the TrainLog checksum format.

The CNN layer kinds (conv_bn_relu, basic_unit, bottleneck, avgpool, maxpool)
are not in the reference; their float64 math lives in
oracle/cnn.py and plugs into the same Block/engine machinery.
"""

from __future__ import annotations

import hashlib
from collections import deque
from dataclasses import dataclass, field

import numpy as np

from . import cnn

# ============================================================ rng (rng.py)
_GOLDEN = 0x9E3779B97F4A7C15
_MIX1 = 0xBF58476D1CE4E5B9
_MIX2 = 0x94D049BB133111EB
_MASK64 = (1 << 64) - 1


def mix64(z: int) -> int:
    """splitmix64 finaliser (rng.py:30-35)."""
    z &= _MASK64
    z = ((z ^ (z >> 30)) * _MIX1) & _MASK64
    z = ((z ^ (z >> 27)) * _MIX2) & _MASK64
    return z ^ (z >> 31)


def derive_seed(seed: int, stream: int) -> int:
    """Child seed for a named sub-stream (rng.py:38-44)."""
    return mix64((seed & _MASK64) + _GOLDEN * (stream + 1))


class SeededRng:
    """Counter-based splitmix64 (rng.py:47-88): draw i of seed s hashes s+(i+1)*golden."""

    def __init__(self, seed: int):
        self.seed = seed & _MASK64
        self.counter = 0

    def _raw(self, n: int) -> np.ndarray:
        i = np.arange(self.counter + 1, self.counter + 1 + n, dtype=np.uint64)
        self.counter += n
        with np.errstate(over="ignore"):
            z = np.uint64(self.seed) + i * np.uint64(_GOLDEN)
            z = (z ^ (z >> np.uint64(30))) * np.uint64(_MIX1)
            z = (z ^ (z >> np.uint64(27))) * np.uint64(_MIX2)
            return z ^ (z >> np.uint64(31))

    def uniform(self, n: int, low: float = 0.0, high: float = 1.0) -> np.ndarray:
        u = (self._raw(n) >> np.uint64(11)).astype(np.float64) * 2.0**-53
        return low + (high - low) * u

    def normal(self, n: int) -> np.ndarray:
        """Box-Muller on consecutive uniform pairs (rng.py:71-83)."""
        half = (n + 1) // 2
        u = (self._raw(2 * half) >> np.uint64(11)).astype(np.float64) * 2.0**-53
        u1, u2 = u[0::2], u[1::2]
        u1 = np.where(u1 == 0.0, 2.0**-53, u1)
        rad = np.sqrt(-2.0 * np.log(u1))
        ang = 2.0 * np.pi * u2
        out = np.empty(2 * half)
        out[0::2] = rad * np.cos(ang)
        out[1::2] = rad * np.sin(ang)
        return out[:n]

    def permutation(self, n: int) -> np.ndarray:
        return np.argsort(self._raw(n), kind="stable")


# ============================================================ tensor.py
class ShapeError(ValueError):
    pass


class NonFiniteError(ArithmeticError):
    pass


def check_finite(a: np.ndarray, what: str) -> np.ndarray:
    """tensor.py:34-37."""
    if not np.isfinite(a).all():
        raise NonFiniteError(f"non-finite values in {what}")
    return a


def matmul_exact(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """Ascending-k rank-1 accumulation, bitwise equal to tensor.py:40-56."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    if a.ndim != 2 or b.ndim != 2 or a.shape[1] != b.shape[0]:
        raise ShapeError(f"matmul shapes {a.shape} x {b.shape}")
    acc = np.zeros((a.shape[0], b.shape[1]))
    with np.errstate(over="ignore", invalid="ignore"):
        for t in range(a.shape[1]):
            acc += a[:, t:t + 1] * b[t]
    return check_finite(acc, "matmul output")


def act_fwd(kind: str, x: np.ndarray) -> np.ndarray:
    """tensor.py:59-67."""
    out = np.maximum(x, 0.0) if kind == "relu" else np.tanh(x)
    return check_finite(out, f"{kind} output")


def act_vjp(kind: str, x: np.ndarray, u: np.ndarray) -> np.ndarray:
    """tensor.py:70-83 (relu subgradient 0 at 0)."""
    if kind == "relu":
        out = u * (x > 0.0)
    else:
        t = np.tanh(x)
        out = u * (1.0 - t * t)
    return check_finite(out, f"{kind} vjp")


def softmax_xent(logits: np.ndarray, labels: np.ndarray) -> tuple[float, np.ndarray]:
    """Row-max-stabilised mean cross-entropy and (softmax-onehot)/B (tensor.py:86-111)."""
    logits = np.asarray(logits, dtype=np.float64)
    n, c = logits.shape
    labels = np.asarray(labels)
    if labels.shape != (n,):
        raise ShapeError("labels shape")
    if labels.min(initial=0) < 0 or labels.max(initial=0) >= c:
        raise ValueError(f"label out of range [0, {c})")
    z = logits - logits.max(axis=1, keepdims=True)
    ez = np.exp(z)
    den = ez.sum(axis=1, keepdims=True)
    rows = np.arange(n)
    loss = float(-(z - np.log(den))[rows, labels].sum() / n)
    grad = ez / den
    grad[rows, labels] -= 1.0
    grad /= n
    if not np.isfinite(loss):
        raise NonFiniteError("non-finite cross-entropy loss")
    return loss, check_finite(grad, "cross-entropy gradient")


# ============================================================ blocks.py
KINDS_REF = ("dense", "relu", "tanh")
KINDS_CNN = ("conv_bn_relu", "basic_unit", "bottleneck", "avgpool", "maxpool")


@dataclass(frozen=True)
class LayerSpec:
    """blocks.py:21-39, extended with the CNN kinds (shape-carrying)."""

    kind: str
    in_dim: int = 0
    out_dim: int = 0
    bias: bool = True
    in_shape: tuple = ()      # (C, H, W) for CNN kinds
    out_c: int = 0
    mid_c: int = 0
    stride: int = 1
    ksize: int = 3

    @property
    def out_shape(self) -> tuple:
        if self.kind == "dense":
            return (self.out_dim,)
        if self.kind in ("relu", "tanh"):
            return ()  # shape-preserving
        return cnn.out_shape(self)

    @property
    def param_count(self) -> int:
        if self.kind == "dense":
            return self.in_dim * self.out_dim + (self.out_dim if self.bias else 0)
        if self.kind in ("relu", "tanh"):
            return 0
        return cnn.param_count(self)


def dense(i, o, bias=True):
    return LayerSpec("dense", i, o, bias)


def relu():
    return LayerSpec("relu")


def tanh():
    return LayerSpec("tanh")


def conv_bn_relu(in_shape, out_c, ksize=3, stride=1):
    return LayerSpec("conv_bn_relu", in_shape=tuple(in_shape), out_c=out_c, ksize=ksize, stride=stride)


def basic_unit(in_shape, out_c, stride=1):
    return LayerSpec("basic_unit", in_shape=tuple(in_shape), out_c=out_c, stride=stride)


def bottleneck(in_shape, mid_c, out_c, stride=1):
    return LayerSpec("bottleneck", in_shape=tuple(in_shape), mid_c=mid_c, out_c=out_c, stride=stride)


def avgpool(in_shape):
    return LayerSpec("avgpool", in_shape=tuple(in_shape))


def maxpool(in_shape):
    return LayerSpec("maxpool", in_shape=tuple(in_shape), ksize=3, stride=2)


class Tape:
    """Single-use forward record (blocks.py:54-62): one entry per layer."""

    def __init__(self, entries):
        self.entries = entries
        self.consumed = False


class Block:
    """Consecutive layers owning one flat float64 vector (blocks.py:65-93)."""

    def __init__(self, index: int, layers: list[LayerSpec]):
        self.index = index
        self.layers = list(layers)
        self.is_last = False
        self.offsets = []
        n = 0
        for s in self.layers:
            self.offsets.append(n)
            n += s.param_count
        self.params = np.zeros(n)

    @property
    def param_count(self) -> int:
        return self.params.size

    def slice(self, i: int, vec: np.ndarray | None = None) -> np.ndarray:
        v = self.params if vec is None else vec
        return v[self.offsets[i]:self.offsets[i] + self.layers[i].param_count]

    def dense_views(self, i: int):
        """(W[in][out], b) views exactly as blocks.py:79-93."""
        s = self.layers[i]
        p = self.slice(i)
        w = p[: s.in_dim * s.out_dim].reshape(s.in_dim, s.out_dim)
        b = p[s.in_dim * s.out_dim:] if s.bias else None
        return w, b


def block_forward(block: Block, h_in: np.ndarray, record: bool = False):
    """blocks.py:96-118; CNN kinds reshape the 2-D packet to NCHW internally."""
    h = np.asarray(h_in, dtype=np.float64)
    entries = []
    for i, s in enumerate(block.layers):
        if s.kind == "dense":
            if h.ndim != 2 or h.shape[1] != s.in_dim:
                raise ShapeError(f"block {block.index} layer {i}: input {h.shape} vs dense({s.in_dim},{s.out_dim})")
            if record:
                entries.append(h)
            w, b = block.dense_views(i)
            h = matmul_exact(h, cnn.q(w))
            if b is not None:
                h = h + b
            if not (block.is_last and i == len(block.layers) - 1):
                h = cnn.q(h)  # logits stay fp32 on the device
        elif s.kind in ("relu", "tanh"):
            if record:
                entries.append(h)
            h = cnn.q(act_fwd(s.kind, h))
        else:
            h, ent = cnn.layer_forward(s, block.slice(i), h)
            if record:
                entries.append(ent)
    check_finite(h, f"block {block.index} output")
    return h, (Tape(entries) if record else None)


def block_backward(block: Block, tape: Tape, upstream: np.ndarray):
    """blocks.py:121-154: reverse layer loop, flat grad laid out like params."""
    if tape.consumed:
        raise RuntimeError("forward tape already consumed")
    tape.consumed = True
    u = np.asarray(upstream, dtype=np.float64)
    grad = np.zeros_like(block.params)
    for i in range(len(block.layers) - 1, -1, -1):
        s = block.layers[i]
        ent = tape.entries[i]
        if s.kind == "dense":
            w, b = block.dense_views(i)
            off = block.offsets[i]
            grad[off:off + w.size] = matmul_exact(ent.T, u).reshape(-1)
            if b is not None:
                grad[off + w.size:off + w.size + s.out_dim] = u.sum(axis=0)
            u = cnn.q(matmul_exact(u, cnn.q(w).T))
        elif s.kind in ("relu", "tanh"):
            u = cnn.q(act_vjp(s.kind, ent, u))
        else:
            g, u = cnn.layer_backward(s, block.slice(i), ent, u)
            grad[block.offsets[i]:block.offsets[i] + s.param_count] = g
    return grad, u


def _flat_width(shape) -> int:
    return int(np.prod(shape)) if shape else 0


def layer_in_width(s: LayerSpec, width: int) -> int:
    if s.kind == "dense":
        return s.in_dim
    if s.kind in ("relu", "tanh"):
        return width
    return _flat_width(s.in_shape)


def layer_out_width(s: LayerSpec, width: int) -> int:
    if s.kind in ("relu", "tanh"):
        return width
    return _flat_width(s.out_shape)


class Model:
    """blocks.py:157-214."""

    def __init__(self, blocks, layers, boundaries):
        self.blocks = blocks
        self.layers = layers
        self.boundaries = list(boundaries)
        self.block_input_dims = block_input_dims(layers, boundaries)

    @property
    def k(self) -> int:
        return len(self.blocks)

    @property
    def param_count(self) -> int:
        return sum(b.param_count for b in self.blocks)

    def forward(self, x):
        h = x
        for b in self.blocks:
            h, _ = block_forward(b, h)
        return h

    def param_snapshot(self):
        return [b.params.copy() for b in self.blocks]

    def flat_params(self):
        return np.concatenate([b.params for b in self.blocks])

    def load_params(self, snap):
        for b, p in zip(self.blocks, snap):
            b.params[:] = p

    def clone(self):
        m = build_model(self.layers, self.boundaries)
        m.load_params(self.param_snapshot())
        return m


def block_input_dims(layers, boundaries) -> list[int]:
    """Flat input width of every block (blocks.py:217-226)."""
    cuts = [0, *boundaries, len(layers)]
    width = layer_in_width(layers[0], 0)
    dims = []
    for a, b in zip(cuts[:-1], cuts[1:]):
        dims.append(width)
        for s in layers[a:b]:
            width = layer_out_width(s, width)
    return dims


def build_model(layers, boundaries) -> Model:
    """blocks.py:229-252 with shape checks for the CNN kinds."""
    layers = list(layers)
    if not layers:
        raise ValueError("model needs at least one layer")
    if layers[0].kind in ("relu", "tanh"):
        raise ValueError("first layer must fix the input width")
    prev = 0
    for b in boundaries:
        if b <= prev or b >= len(layers):
            raise ValueError(f"boundaries must be strictly increasing inside (0, {len(layers)}), got {boundaries}")
        prev = b
    width = layer_in_width(layers[0], 0)
    for i, s in enumerate(layers):
        need = layer_in_width(s, width)
        if need != width:
            raise ShapeError(f"layer {i} ({s.kind}) expects width {need}, got {width}")
        width = layer_out_width(s, width)
    cuts = [0, *boundaries, len(layers)]
    blocks = [Block(k, layers[a:b]) for k, (a, b) in enumerate(zip(cuts[:-1], cuts[1:]))]
    blocks[-1].is_last = True
    return Model(blocks, layers, boundaries)


def init_params(model: Model, seed: int) -> None:
    """One SeededRng stream over all layers, independent of the cuts (blocks.py:278-302).

    dense: He-uniform if followed by relu else Glorot-uniform, zero bias (as the
    reference).  CNN kinds: cnn.init_layer (He-uniform convs, BN gamma=1, beta=0).
    """
    rng = SeededRng(seed)
    flat = 0
    for block in model.blocks:
        for i, s in enumerate(block.layers):
            if s.kind == "dense":
                nxt = model.layers[flat + 1].kind if flat + 1 < len(model.layers) else None
                lim = np.sqrt(6.0 / s.in_dim) if nxt == "relu" else np.sqrt(6.0 / (s.in_dim + s.out_dim))
                w, b = block.dense_views(i)
                w[:] = rng.uniform(w.size, -lim, lim).reshape(w.shape)
                if b is not None:
                    b[:] = 0.0
            elif s.kind not in ("relu", "tanh"):
                cnn.init_layer(s, block.slice(i), rng)
            flat += 1


# ============================================================ optim.py
@dataclass
class LrSchedule:
    base: float
    decays: tuple = ()


def lr_at(schedule: LrSchedule, n: int) -> float:
    """base * every factor whose step has passed, in list order (optim.py:38-45)."""
    if n < 0:
        raise ValueError("step must be non-negative")
    lr = schedule.base
    for step, factor in schedule.decays:
        if n >= step:
            lr *= factor
    return lr


def sgd_step(x, g, lr):
    """optim.py:48-55."""
    if not np.isfinite(g).all():
        raise NonFiniteError("non-finite gradient in sgd_step")
    return x - lr * g


@dataclass
class OptimizerState:
    """optim.py:58-83; 'adam' is this repo's unpinned extension (BASELINE C3)."""

    rule: str
    beta: float = 0.0
    s: float = 1.0
    y: np.ndarray | None = None
    ys: np.ndarray | None = None
    n: int = 0
    # adam (unpinned: the reference rejects it, optim.py:70-71)
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8
    m1: np.ndarray | None = None
    m2: np.ndarray | None = None

    @classmethod
    def for_params(cls, rule, x0, beta=0.0, s=1.0):
        st = cls(rule=rule, beta=beta, s=s)
        if rule == "sum":
            st.y = x0.copy()
            st.ys = x0.copy()
        elif rule == "adam":
            st.m1 = np.zeros_like(x0)
            st.m2 = np.zeros_like(x0)
        elif rule != "sgd":
            raise ValueError(f"unknown optimizer rule: {rule!r}")
        return st


def sum_step(st: OptimizerState, x, g, lr):
    """Unified momentum, y/ys form (optim.py:86-99), same IEEE op order."""
    if not np.isfinite(g).all():
        raise NonFiniteError("non-finite gradient in sum_step")
    y_new = x - lr * g
    ys_new = x - (st.s * lr) * g
    x_new = y_new if st.beta == 0.0 else y_new + st.beta * (ys_new - st.ys)
    st.y = y_new
    st.ys = ys_new
    return x_new


def adam_step(st: OptimizerState, x, g, lr):
    """Bias-corrected Adam per block (unpinned extension)."""
    t = st.n + 1
    st.m1 = st.beta1 * st.m1 + (1.0 - st.beta1) * g
    st.m2 = st.beta2 * st.m2 + (1.0 - st.beta2) * (g * g)
    mhat = st.m1 / (1.0 - st.beta1 ** t)
    vhat = st.m2 / (1.0 - st.beta2 ** t)
    return x - lr * mhat / (np.sqrt(vhat) + st.eps)


def apply_update(st: OptimizerState, x, g, lr):
    """optim.py:102-109."""
    if st.rule == "sgd":
        out = sgd_step(x, g, lr)
    elif st.rule == "sum":
        out = sum_step(st, x, g, lr)
    else:
        out = adam_step(st, x, g, lr)
    st.n += 1
    return out


# ============================================================ pipeline.py
WARMUP_POLICIES = ("faithful_zero_updates", "discard_warmup_updates")


class ConfigError(ValueError):
    def __init__(self, constraint, index, message):
        super().__init__(message)
        self.constraint = constraint
        self.index = index


class ProtocolError(AssertionError):
    pass


@dataclass(frozen=True)
class PipelineConfig:
    k: int
    p: tuple
    m: tuple
    q: tuple
    warmup: str = "faithful_zero_updates"
    overlap_recompute: bool = True


def validate_config(p, m, warmup="faithful_zero_updates", overlap_recompute=True) -> PipelineConfig:
    """Eq.(5) checks in the reference's order; derives q (pipeline.py:85-128)."""
    p = tuple(int(v) for v in p)
    m = tuple(int(v) for v in m)
    if not p or len(p) != len(m):
        raise ConfigError("length", 0, f"p and m must be equal-length, non-empty: p={p}, m={m}")
    K = len(p)
    if warmup not in WARMUP_POLICIES:
        raise ConfigError("warmup", 0, f"warmup must be one of {WARMUP_POLICIES}, got {warmup!r}")
    if p[-1] != 0:
        raise ConfigError("p_last_zero", K - 1,
                          f"p[{K - 1}] = {p[-1]} must be 0 (the last block sends no activations upward)")
    for k in range(K - 1):
        if p[k] <= 0:
            raise ConfigError("p_positive", k, f"p[{k}] = {p[k]} must be > 0")
    for k in range(K - 1):
        if m[k] <= 0:
            raise ConfigError("m_positive", k, f"m[{k}] = {m[k]} must be > 0")
    if m[-1] < 0:
        raise ConfigError("m_last_nonneg", K - 1, f"m[{K - 1}] = {m[-1]} must be >= 0")
    q = [0]
    for k in range(1, K):
        qk = m[k - 1] - p[k - 1] - m[k]
        if qk <= 0:
            raise ConfigError("q_positive", k,
                              f"q[{k}] = m[{k - 1}]-p[{k - 1}]-m[{k}] = {m[k - 1]}-{p[k - 1]}-{m[k]} = {qk} <= 0")
        q.append(qk)
    return PipelineConfig(K, p, m, tuple(q), warmup, overlap_recompute)


class Fifo:
    """Bounded FIFO whose misuse is a ProtocolError (pipeline.py:148-169)."""

    def __init__(self, name, capacity):
        self.name = name
        self.capacity = capacity
        self.items = deque()

    def put(self, pkt):
        if len(self.items) >= self.capacity:
            raise ProtocolError(f"push to full queue {self.name} (capacity {self.capacity})")
        self.items.append(pkt)

    def get(self):
        if not self.items:
            raise ProtocolError(f"pop from empty queue {self.name}")
        return self.items.popleft()


@dataclass
class Record:
    step: int
    block: int
    batch_index: int
    grad_norm: float
    loss: float | None = None


def log_checksum(records) -> str:
    """SHA-256 of step|block|batch|loss.hex|grad_norm.hex, sorted (pipeline.py:230-236)."""
    h = hashlib.sha256()
    for r in sorted(records, key=lambda r: (r.step, r.block)):
        lh = "-" if r.loss is None else float(r.loss).hex()
        h.update(f"{r.step}|{r.block}|{r.batch_index}|{lh}|{float(r.grad_norm).hex()}\n".encode())
    return h.hexdigest()


class Engine:
    """Serial DSP engine (pipeline.py:443-618): identical FP sequence to the
    reference's serial (and parallel) backends."""

    def __init__(self, model: Model, config: PipelineConfig, stream, schedule: LrSchedule, rule="sgd",
                 beta=0.0, s=1.0, weight_decay=0.0, loss_fn=softmax_xent):
        if config.k != model.k:
            raise ConfigError("k", 0, f"config K={config.k} but model has {model.k} blocks")
        self.model = model
        self.config = config
        self.schedule = schedule
        self.wd = weight_decay
        self.loss_fn = loss_fn
        self._stream = stream
        self._first = next(stream)
        self._first_pending = True
        B = self._first[0].shape[0]
        K = config.k
        self.cum_p = [0] * (K + 1)
        for k in range(K):
            self.cum_p[k + 1] = self.cum_p[k] + config.p[k]
        dims = model.block_input_dims
        zero = lambda tag, d: (tag, np.zeros((B, d)), np.zeros(B, dtype=np.int64))  # noqa: E731
        # prefill tags (pipeline.py:493-512)
        self.out_q = []
        for k in range(K - 1):
            q = Fifo(f"out[{k}]", 1 + config.p[k])
            for t in range(config.p[k]):
                q.put(zero(t - self.cum_p[k + 1], dims[k + 1]))
            self.out_q.append(q)
        self.in_q = []
        for k in range(K):
            q = Fifo(f"in[{k}]", 1 + config.m[k])
            for t in range(config.m[k]):
                q.put(zero(t - self.cum_p[k] - config.m[k], dims[k]))
            self.in_q.append(q)
        self.grad_q = [None]
        for k in range(1, K):
            q = Fifo(f"grad[{k}]", 1 + config.q[k])
            for t in range(config.q[k]):
                q.put((t - self.cum_p[k - 1] - config.m[k - 1], np.zeros((B, dims[k]))))
            self.grad_q.append(q)
        self.opt = [OptimizerState.for_params(rule, b.params, beta=beta, s=s) for b in model.blocks]
        self.steps = [0] * K
        self.records: list[Record] = []
        self.trace = []  # (step, block, fresh_tag, stale_tag) for index-parity checks

    def _batch(self):
        if self._first_pending:
            self._first_pending = False
            return self._first
        return next(self._stream)

    def iterate(self, k: int) -> None:
        """One Algorithm-2 body (pipeline.py:538-606)."""
        n = self.steps[k]
        cfg = self.config
        blk = self.model.blocks[k]
        last = cfg.k - 1
        if k == 0:
            x, lab = self._batch()
            fresh = (n, cnn.q(np.asarray(x, dtype=np.float64)), lab)
        else:
            fresh = self.out_q[k - 1].get()
        self.in_q[k].put(fresh)
        stale = self.in_q[k].get()
        loss = None
        if k < last:
            h, _ = block_forward(blk, fresh[1])
            self.out_q[k].put((fresh[0], h, fresh[2]))
            _, tape = block_forward(blk, stale[1], record=True)
            gtag, up = self.grad_q[k + 1].get()
            if gtag != stale[0]:
                raise ProtocolError(f"block {k} step {n}: gradient batch {gtag} does not meet activation batch {stale[0]}")
        else:
            top, tape = block_forward(blk, stale[1], record=True)
            loss, up = self.loss_fn(top, stale[2])
            up = cnn.q(up)
        gp, gin = block_backward(blk, tape, up)
        if k > 0:
            self.grad_q[k].put((stale[0], gin))
        g = gp
        if self.wd != 0.0:
            g = g + self.wd * blk.params
        if not (cfg.warmup == "discard_warmup_updates" and stale[0] < 0):
            blk.params = apply_update(self.opt[k], blk.params, g, lr_at(self.schedule, n))
            if cnn.STORAGE["mode"] == "bf16":  # fp32 master weights on the device
                blk.params = blk.params.astype(np.float32).astype(np.float64)
        self.records.append(Record(n, k, stale[0], float(np.sqrt((gp ** 2).sum())), loss))
        self.trace.append((n, k, fresh[0], stale[0]))
        self.steps[k] = n + 1

    def run(self, n_steps: int) -> None:
        for _ in range(n_steps):
            for k in range(self.config.k):
                self.iterate(k)

    def checksum(self) -> str:
        return log_checksum(self.records)

    def realized_staleness(self) -> list[int]:
        """pipeline.py:682-694."""
        out = []
        for k in range(self.config.k):
            rows = [r for r in self.records if r.block == k and r.batch_index >= 0]
            lags = {(r.step - self.cum_p[k]) - r.batch_index for r in rows}
            if len(lags) > 1:
                raise ProtocolError(f"block {k} staleness drifted: {sorted(lags)}")
            out.append(lags.pop() if lags else 0)
        return out


def bp_gradient(model: Model, x, labels):
    """Chained BP at current params (pipeline.py:256-267)."""
    tapes = []
    h = x
    for b in model.blocks:
        h, t = block_forward(b, h, record=True)
        tapes.append(t)
    loss, u = softmax_xent(h, labels)
    grads = [None] * model.k
    for k in range(model.k - 1, -1, -1):
        grads[k], u = block_backward(model.blocks[k], tapes[k], u)
    return grads, loss


def stale_gradient(model: Model, fwd, bwd, x, labels, loss_and_grad=softmax_xent):
    """Eq.(4) operator (pipeline.py:270-305)."""
    work = model.clone()
    K = work.k
    inputs = []
    h = x
    for k, b in enumerate(work.blocks):
        b.params[:] = fwd[k]
        inputs.append(h)
        if k < K - 1:
            h, _ = block_forward(b, h)
    for k, b in enumerate(work.blocks):
        b.params[:] = bwd[k]
    top, tape = block_forward(work.blocks[-1], inputs[-1], record=True)
    loss, u = loss_and_grad(top, labels)
    grads = [None] * K
    for k in range(K - 1, -1, -1):
        if k < K - 1:
            _, tape = block_forward(work.blocks[k], inputs[k], record=True)
        grads[k], u = block_backward(work.blocks[k], tape, u)
    return grads, loss


class storage:
    """Context manager selecting the oracle's storage emulation ("f64", "f32" or "bf16") and the
    conv accumulation precision ("f64", or "f32" for the noise-floor measurement of cnn._mm)."""

    def __init__(self, mode: str, acc: str = "f64"):
        if mode not in ("f64", "f32", "bf16") or acc not in ("f64", "f32"):
            raise ValueError((mode, acc))
        self.mode, self.acc = mode, acc

    def __enter__(self):
        self.prev = dict(cnn.STORAGE)
        cnn.STORAGE.update(mode=self.mode, acc=self.acc)
        return self

    def __exit__(self, *exc):
        cnn.STORAGE.clear()
        cnn.STORAGE.update(self.prev)
        return False


# ============================================================ data (data.py + SURVEY §8d)
def synthetic_batches(n_batches: int, batch: int, in_shape, num_classes: int, seed: int = 0):
    """Pool of batches: x ~ N(0,1) from SeededRng(seed).normal (NCHW-flattened),
    labels = floor(uniform * C) from SeededRng(derive_seed(seed, 1))."""
    width = int(np.prod(in_shape))
    rx = SeededRng(seed)
    rl = SeededRng(derive_seed(seed, 1))
    out = []
    for _ in range(n_batches):
        x = rx.normal(batch * width).reshape(batch, width)
        lab = np.minimum((rl.uniform(batch) * num_classes).astype(np.int64), num_classes - 1)
        out.append((x, lab))
    return out


def cycle(pool):
    while True:
        for b in pool:
            yield b
