"""Layer specs, block partitioning and parameter layout (reference: blocks.py).

Same surface as the reference -- ``LayerSpec``, ``dense``/``relu``/``tanh``,
``Block`` (flat parameter vector + offsets), ``Model``, ``build_model``,
``init_params``, ``suggest_boundaries`` (/root/reference/pkg/src/stalepipe/
blocks.py:21-302) -- plus the CNN layer kinds the BASELINE configs need
(SURVEY.md G1): ``conv_bn_relu``, ``basic_unit``, ``bottleneck``, ``avgpool``,
``maxpool``. CNN activations cross block boundaries as flat (B, C*H*W) packets
in (C,H,W) order on the host API, exactly as the reference's 2-D packets
(pipeline.py:494, 524-528); on the device they live as padded NHWC bf16.

A ``Block`` starts host-resident (float64 numpy ``params``, like the reference)
and becomes device-resident when a B200 engine binds it: ``params`` then reads
back a float64 copy of the fp32 master weights and writes upload + re-pack.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib as L
from .rng import SeededRng

BN_EPS = 1e-5
REF_KINDS = ("dense", "relu", "tanh")
CNN_KINDS = ("conv_bn_relu", "basic_unit", "bottleneck", "avgpool", "maxpool")


class ShapeError(ValueError):
    """Operand shapes are incompatible (reference: tensor.py:19-20)."""


@dataclass(frozen=True)
class LayerSpec:
    kind: str
    in_dim: int = 0
    out_dim: int = 0
    bias: bool = True
    in_shape: tuple = ()
    out_c: int = 0
    mid_c: int = 0
    stride: int = 1
    ksize: int = 3

    def __post_init__(self):
        if self.kind == "dense":
            if self.in_dim <= 0 or self.out_dim <= 0:
                raise ValueError(f"dense dims must be positive, got {self.in_dim}x{self.out_dim}")
        elif self.kind in ("relu", "tanh"):
            pass
        elif self.kind in CNN_KINDS:
            if len(self.in_shape) != 3 or min(self.in_shape) <= 0:
                raise ValueError(f"{self.kind} needs a positive (C, H, W) in_shape, got {self.in_shape}")
            if self.kind in ("conv_bn_relu", "basic_unit", "bottleneck") and self.out_c <= 0:
                raise ValueError(f"{self.kind} needs out_c > 0")
            if self.kind == "bottleneck" and self.mid_c <= 0:
                raise ValueError("bottleneck needs mid_c > 0")
            if self.stride not in (1, 2):
                raise ValueError("stride must be 1 or 2")
        else:
            raise ValueError(f"unknown layer kind: {self.kind!r}")

    # ---- shapes -------------------------------------------------------------
    @property
    def out_shape(self) -> tuple:
        if self.kind == "dense":
            return (self.out_dim,)
        if self.kind in ("relu", "tanh"):
            return ()
        c, h, w = self.in_shape
        if self.kind == "conv_bn_relu":
            p = self.ksize // 2
            return (self.out_c, _co(h, self.ksize, self.stride, p), _co(w, self.ksize, self.stride, p))
        if self.kind in ("basic_unit", "bottleneck"):
            return (self.out_c, _co(h, 3, self.stride, 1), _co(w, 3, self.stride, 1))
        if self.kind == "avgpool":
            return (c,)
        return (c, _co(h, 3, 2, 1), _co(w, 3, 2, 1))

    @property
    def projection(self) -> bool:
        return self.kind in ("basic_unit", "bottleneck") and (self.stride != 1 or self.in_shape[0] != self.out_c)

    def convs(self) -> list[tuple]:
        """(name, c_out, k, c_in, stride, pad) in parameter order."""
        if self.kind not in ("conv_bn_relu", "basic_unit", "bottleneck"):
            return []
        c = self.in_shape[0]
        if self.kind == "conv_bn_relu":
            return [("c", self.out_c, self.ksize, c, self.stride, self.ksize // 2)]
        if self.kind == "basic_unit":
            lst = [("c1", self.out_c, 3, c, self.stride, 1), ("c2", self.out_c, 3, self.out_c, 1, 1)]
        else:
            lst = [("c1", self.mid_c, 1, c, 1, 0), ("c2", self.mid_c, 3, self.mid_c, self.stride, 1),
                   ("c3", self.out_c, 1, self.mid_c, 1, 0)]
        if self.projection:
            lst.append(("sc", self.out_c, 1, c, self.stride, 0))
        return lst

    @property
    def param_count(self) -> int:
        if self.kind == "dense":
            return self.in_dim * self.out_dim + (self.out_dim if self.bias else 0)
        return sum(co * k * k * ci + 2 * co for _, co, k, ci, _, _ in self.convs())

    def flops(self, width_hint: int = 0) -> float:
        """Forward multiply-adds x2 per sample (dense / conv only)."""
        if self.kind == "dense":
            return 2.0 * self.in_dim * self.out_dim
        total = 0.0
        if not self.convs():
            return 0.0
        c, h, w = self.in_shape
        prev = (h, w)
        for name, co, k, ci, st, pad in self.convs():
            ih, iw = (h, w) if name in ("c", "c1", "sc") else prev
            p, q = _co(ih, k, st, pad), _co(iw, k, st, pad)
            if name != "sc":
                prev = (p, q)
            total += 2.0 * p * q * co * k * k * ci
        return total


def _co(h: int, k: int, s: int, p: int) -> int:
    return (h + 2 * p - k) // s + 1


def dense(in_dim: int, out_dim: int, bias: bool = True) -> LayerSpec:
    return LayerSpec("dense", in_dim, out_dim, bias)


def relu() -> LayerSpec:
    return LayerSpec("relu")


def tanh() -> LayerSpec:
    return LayerSpec("tanh")


def conv_bn_relu(in_shape, out_c: int, ksize: int = 3, stride: int = 1) -> LayerSpec:
    return LayerSpec("conv_bn_relu", in_shape=tuple(in_shape), out_c=out_c, ksize=ksize, stride=stride)


def basic_unit(in_shape, out_c: int, stride: int = 1) -> LayerSpec:
    return LayerSpec("basic_unit", in_shape=tuple(in_shape), out_c=out_c, stride=stride)


def bottleneck(in_shape, mid_c: int, out_c: int, stride: int = 1) -> LayerSpec:
    return LayerSpec("bottleneck", in_shape=tuple(in_shape), mid_c=mid_c, out_c=out_c, stride=stride)


def avgpool(in_shape) -> LayerSpec:
    return LayerSpec("avgpool", in_shape=tuple(in_shape))


def maxpool(in_shape) -> LayerSpec:
    return LayerSpec("maxpool", in_shape=tuple(in_shape), ksize=3, stride=2)


# ------------------------------------------------------------------ shapes through a layer list
def _in_width(s: LayerSpec, width: int) -> int:
    if s.kind == "dense":
        return s.in_dim
    if s.kind in ("relu", "tanh"):
        return width
    return int(np.prod(s.in_shape))


def _out_width(s: LayerSpec, width: int) -> int:
    if s.kind in ("relu", "tanh"):
        return width
    return int(np.prod(s.out_shape))


def tensor_shape_after(layers: list[LayerSpec]) -> tuple:
    """(C, H, W) of the activation after `layers` (dense widths are (D, 1, 1))."""
    shape = None
    for s in layers:
        if s.kind == "dense":
            shape = (s.out_dim, 1, 1)
        elif s.kind in ("relu", "tanh"):
            continue
        else:
            o = s.out_shape
            shape = (o[0], 1, 1) if len(o) == 1 else tuple(o)
    return shape


def layer_in_shape(s: LayerSpec, prev: tuple | None) -> tuple:
    if s.kind == "dense":
        return (s.in_dim, 1, 1)
    if s.kind in ("relu", "tanh"):
        return prev
    return tuple(s.in_shape)


class Block:
    """A consecutive run of layers owning one flat parameter vector (blocks.py:65-93)."""

    def __init__(self, index: int, layers: list[LayerSpec], in_shape: tuple):
        self.index = index
        self.layers = list(layers)
        self.in_shape = in_shape
        self._offsets = []
        total = 0
        for spec in self.layers:
            self._offsets.append(total)
            total += spec.param_count
        self._host = np.zeros(total)
        self.dev = None  # runtime.DeviceBlock once bound to a B200 engine

    @property
    def offsets(self) -> list[int]:
        return list(self._offsets)

    @property
    def param_count(self) -> int:
        return int(sum(s.param_count for s in self.layers))

    @property
    def params(self) -> np.ndarray:
        if self.dev is not None:
            return self.dev.read_params()
        return self._host

    @params.setter
    def params(self, value) -> None:
        value = np.asarray(value, dtype=np.float64)
        if value.shape != (self.param_count,):
            raise ShapeError(f"block {self.index}: expected {self.param_count} params, got {value.shape}")
        if self.dev is not None:
            self.dev.write_params(value)
        else:
            self._host = value.copy()

    def layer_params(self, i: int):
        """(W[in][out], b) views for a dense layer of a host-resident block (blocks.py:79-93)."""
        spec = self.layers[i]
        if spec.kind != "dense":
            return None, None
        p = self.params[self._offsets[i]:self._offsets[i] + spec.param_count]
        w = p[: spec.in_dim * spec.out_dim].reshape(spec.in_dim, spec.out_dim)
        b = p[spec.in_dim * spec.out_dim:] if spec.bias else None
        return w, b

    @property
    def out_shape(self) -> tuple:
        return tensor_shape_after(self.layers) or self.in_shape

    def layer_descs(self):
        """Layer program for dsp_block_create (include/dsp_b200.h)."""
        kinds = {"dense": L.DSP_LAYER_DENSE, "relu": L.DSP_LAYER_RELU, "tanh": L.DSP_LAYER_TANH,
                 "conv_bn_relu": L.DSP_LAYER_CONV_BN_RELU, "basic_unit": L.DSP_LAYER_BASIC_UNIT,
                 "bottleneck": L.DSP_LAYER_BOTTLENECK, "avgpool": L.DSP_LAYER_AVGPOOL,
                 "maxpool": L.DSP_LAYER_MAXPOOL}
        arr = (L.LayerDesc * len(self.layers))()
        cur = self.in_shape
        for i, s in enumerate(self.layers):
            d = arr[i]
            d.kind = kinds[s.kind]
            ish = layer_in_shape(s, cur)
            d.in_c, d.in_h, d.in_w = ish
            if s.kind == "dense":
                d.out_c, d.out_h, d.out_w = s.out_dim, 1, 1
                d.bias = 1 if s.bias else 0
            elif s.kind in ("relu", "tanh"):
                d.out_c, d.out_h, d.out_w = ish
            else:
                o = s.out_shape
                d.out_c, d.out_h, d.out_w = (o[0], 1, 1) if len(o) == 1 else o
            d.mid_c = s.mid_c
            d.stride = s.stride
            d.ksize = s.ksize
            d.param_offset = self._offsets[i]
            d.param_count = s.param_count
            cur = (d.out_c, d.out_h, d.out_w)
        return arr


class Model:
    """K consecutive blocks (blocks.py:157-214)."""

    def __init__(self, blocks: list[Block], layers: list[LayerSpec], boundaries: list[int]):
        self.blocks = blocks
        self.layers = layers
        self.boundaries = list(boundaries)
        self.block_input_dims = block_input_dims(layers, boundaries)

    @property
    def k(self) -> int:
        return len(self.blocks)

    @property
    def input_dim(self) -> int:
        return _in_width(self.layers[0], 0)

    @property
    def input_shape(self) -> tuple:
        return self.blocks[0].in_shape

    @property
    def output_dim(self) -> int:
        for s in reversed(self.layers):
            if s.kind == "dense":
                return s.out_dim
        raise ValueError("model has no dense layer")

    @property
    def param_count(self) -> int:
        return sum(b.param_count for b in self.blocks)

    def param_snapshot(self) -> list[np.ndarray]:
        return [b.params.copy() for b in self.blocks]

    def flat_params(self) -> np.ndarray:
        return np.concatenate([b.params for b in self.blocks]) if self.blocks else np.zeros(0)

    def set_flat_params(self, vec: np.ndarray) -> None:
        if vec.size != self.param_count:
            raise ShapeError(f"expected {self.param_count} params, got {vec.size}")
        off = 0
        for b in self.blocks:
            b.params = vec[off:off + b.param_count]
            off += b.param_count

    def load_params(self, snapshot: list[np.ndarray]) -> None:
        for b, p in zip(self.blocks, snapshot):
            b.params = p

    def clone(self) -> "Model":
        m = build_model(self.layers, self.boundaries)
        m.load_params(self.param_snapshot())
        return m

    def forward(self, x: np.ndarray) -> np.ndarray:
        """Evaluation forward through every block on the device (returns host logits)."""
        from .pipeline import model_forward

        return model_forward(self, x)


def block_input_dims(layers: list[LayerSpec], boundaries: list[int]) -> list[int]:
    cuts = [0, *boundaries, len(layers)]
    width = _in_width(layers[0], 0)
    dims = []
    for a, b in zip(cuts[:-1], cuts[1:]):
        dims.append(width)
        for s in layers[a:b]:
            width = _out_width(s, width)
    return dims


def build_model(layers: list[LayerSpec], boundaries: list[int]) -> Model:
    """Cut a layer list at K-1 strictly increasing indices (blocks.py:229-252)."""
    layers = list(layers)
    if not layers:
        raise ValueError("model needs at least one layer")
    if layers[0].kind in ("relu", "tanh"):
        raise ValueError("first layer must be dense (or a CNN kind) so the input width is known")
    boundaries = list(boundaries)
    prev = 0
    for b in boundaries:
        if b <= prev or b >= len(layers):
            raise ValueError(f"boundaries must be strictly increasing inside (0, {len(layers)}), got {boundaries}")
        prev = b
    width = _in_width(layers[0], 0)
    shape = layer_in_shape(layers[0], None)
    shapes = []
    for i, s in enumerate(layers):
        need = _in_width(s, width)
        if need != width:
            raise ShapeError(f"layer {i}: {s.kind} expects width {need}, got {width}")
        if s.kind in CNN_KINDS and tuple(s.in_shape) != tuple(shape):
            raise ShapeError(f"layer {i}: {s.kind} expects input {s.in_shape}, got {shape}")
        shapes.append(layer_in_shape(s, shape))
        width = _out_width(s, width)
        after = tensor_shape_after([s])
        if after is not None:
            shape = after
    cuts = [0, *boundaries, len(layers)]
    blocks = [Block(k, layers[a:b], shapes[a]) for k, (a, b) in enumerate(zip(cuts[:-1], cuts[1:]))]
    return Model(blocks, layers, boundaries)


def suggest_boundaries(layers: list[LayerSpec], k: int) -> list[int]:
    """Parameter-balanced cuts, advisory (blocks.py:255-275)."""
    if k < 1 or k > len(layers):
        raise ValueError(f"cannot split {len(layers)} layers into {k} blocks")
    total = sum(s.param_count for s in layers)
    cuts = []
    running = 0
    nxt = 1
    for i, s in enumerate(layers):
        running += s.param_count
        if len(cuts) < k - 1 and running >= nxt * total / k and i + 1 < len(layers):
            cuts.append(i + 1)
            nxt += 1
    while len(cuts) < k - 1:
        cand = len(layers) - (k - 1 - len(cuts))
        cuts.append(max(cand, (cuts[-1] if cuts else 0) + 1))
    return cuts


def flop_balanced_boundaries(layers: list[LayerSpec], k: int) -> list[int]:
    """Cuts at layer (residual-unit) granularity minimising the max per-block
    DSP cost. Cost of block j: (3 if j<K-1 else 2) x fwd FLOPs
    (fresh + recompute + ~2x backward for non-last blocks)."""
    n = len(layers)
    if k < 1 or k > n:
        raise ValueError(f"cannot split {n} layers into {k} blocks")
    f = [max(s.flops(), 1.0) for s in layers]
    pre = np.concatenate([[0.0], np.cumsum(f)])

    def cost(a, b, last):
        return (pre[b] - pre[a]) * (3.0 if last else 4.0)

    best = {}

    def solve(start, parts):
        key = (start, parts)
        if key in best:
            return best[key]
        if parts == 1:
            r = (cost(start, n, True), [])
        else:
            r = (float("inf"), [])
            for cut in range(start + 1, n - parts + 2):
                c0 = cost(start, cut, False)
                if c0 >= r[0]:
                    break
                sub, cuts = solve(cut, parts - 1)
                m = max(c0, sub)
                if m < r[0]:
                    r = (m, [cut] + cuts)
        best[key] = r
        return r

    return solve(0, k)[1]


def init_params(model: Model, seed: int) -> None:
    """One SeededRng stream over all layers, independent of the cuts (blocks.py:278-302).

    dense: He-uniform (limit sqrt(6/in)) when followed by relu, Glorot-uniform
    otherwise, zero bias -- exactly the reference. CNN kinds: He-uniform conv
    weights (limit sqrt(6/fan_in)) conv by conv, BatchNorm gamma=1, beta=0.
    """
    rng = SeededRng(seed)
    flat = 0
    for block in model.blocks:
        vec = np.zeros(block.param_count)
        for i, s in enumerate(block.layers):
            off = block._offsets[i]
            if s.kind == "dense":
                nxt = model.layers[flat + 1].kind if flat + 1 < len(model.layers) else None
                lim = np.sqrt(6.0 / s.in_dim) if nxt == "relu" else np.sqrt(6.0 / (s.in_dim + s.out_dim))
                vec[off:off + s.in_dim * s.out_dim] = rng.uniform(s.in_dim * s.out_dim, -lim, lim)
            elif s.kind not in ("relu", "tanh"):
                o = off
                for _, co, k, ci, _, _ in s.convs():
                    nw = co * k * k * ci
                    lim = np.sqrt(6.0 / (k * k * ci))
                    vec[o:o + nw] = rng.uniform(nw, -lim, lim)
                    o += nw
                    vec[o:o + co] = 1.0
                    o += 2 * co
            flat += 1
        block.params = vec


# ------------------------------------------------------------------ ResNet layer lists
def resnet_cifar_layers(depth: int, num_classes: int = 10, width: int = 16, in_shape=(3, 32, 32)) -> list[LayerSpec]:
    """ResNet-(6n+2) for CIFAR (basic units, post-activation, 1x1-projection shortcuts)."""
    if (depth - 2) % 6:
        raise ValueError("CIFAR ResNet depth must be 6n+2")
    n = (depth - 2) // 6
    layers = [conv_bn_relu(in_shape, width)]
    shape = layers[-1].out_shape
    for stage, c in enumerate((width, 2 * width, 4 * width)):
        for u in range(n):
            stride = 2 if (stage > 0 and u == 0) else 1
            layers.append(basic_unit(shape, c, stride))
            shape = layers[-1].out_shape
    layers.append(avgpool(shape))
    layers.append(dense(shape[0], num_classes))
    return layers


def resnet_cifar_bottleneck_layers(depth: int, num_classes: int = 100, width: int = 16,
                                   in_shape=(3, 32, 32)) -> list[LayerSpec]:
    """ResNet-(9n+2) with bottleneck units (ResNet-164: n=18), expansion 4."""
    if (depth - 2) % 9:
        raise ValueError("bottleneck CIFAR ResNet depth must be 9n+2")
    n = (depth - 2) // 9
    layers = [conv_bn_relu(in_shape, width)]
    shape = layers[-1].out_shape
    for stage, mid in enumerate((width, 2 * width, 4 * width)):
        for u in range(n):
            stride = 2 if (stage > 0 and u == 0) else 1
            layers.append(bottleneck(shape, mid, 4 * mid, stride))
            shape = layers[-1].out_shape
    layers.append(avgpool(shape))
    layers.append(dense(shape[0], num_classes))
    return layers


def resnet50_layers(num_classes: int = 1000, in_shape=(3, 224, 224)) -> list[LayerSpec]:
    """ResNet-50 (v1.5: stride on the 3x3 conv)."""
    layers = [conv_bn_relu(in_shape, 64, ksize=7, stride=2)]
    layers.append(maxpool(layers[-1].out_shape))
    shape = layers[-1].out_shape
    for stage, (mid, reps) in enumerate(((64, 3), (128, 4), (256, 6), (512, 3))):
        for u in range(reps):
            stride = 2 if (stage > 0 and u == 0) else 1
            layers.append(bottleneck(shape, mid, 4 * mid, stride))
            shape = layers[-1].out_shape
    layers.append(avgpool(shape))
    layers.append(dense(shape[0], num_classes))
    return layers
