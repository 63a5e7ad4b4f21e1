"""DSP pipeline: queue sizing, FIFO schedule and the train-step driver
(reference: /root/reference/pkg/src/stalepipe/pipeline.py).

The host side mirrors the reference exactly -- ``validate_config`` (Eq. 5),
the three bounded FIFO families with their zero-packet prefill tags, the
Algorithm-2 loop body ``_iterate_block``, the per-(step, block) ``TrainLog``
and its checksum, ``realized_staleness`` -- while every tensor operation of the
loop body runs on the B200 through the block runtime (``runtime.DeviceBlock``
-> ``libdsp_b200.so``). Packets carry device tensors by reference, like the
reference's immutable packets.

Multi-GPU: blocks are placed on ranks (one process per GPU). An edge whose
producer and consumer live on different ranks is carried by point-to-point
send/recv (torch.distributed: NCCL on GPUs, gloo in the CPU tests) at the end
of each step; since p_k >= 1 and q_k >= 1 every packet is consumed at least one
step after it is produced, so the per-rank schedule is identical, value for
value, to the single-process serial schedule (pipeline.py:538-606).
"""

from __future__ import annotations

import hashlib
import json
import os
import time
from collections import deque
from dataclasses import dataclass
from typing import Iterator

import numpy as np

from .blocks import Model, ShapeError
from .optim import RULES, LrSchedule, OptimizerState, lr_at
from .rng import mix64

WARMUP_POLICIES = ("faithful_zero_updates", "discard_warmup_updates")
BACKENDS = ("b200",)


class ConfigError(ValueError):
    """A queue-sizing constraint is violated; names the constraint and block (pipeline.py:49-55)."""

    def __init__(self, constraint: str, index: int, message: str):
        super().__init__(message)
        self.constraint = constraint
        self.index = index


class ProtocolError(AssertionError):
    """Queue protocol violation (pipeline.py:58-59)."""


class DeadlockError(RuntimeError):
    """Workers stopped making progress (pipeline.py:62-63)."""


@dataclass(frozen=True)
class PipelineConfig:
    k: int
    p: tuple
    m: tuple
    q: tuple
    warmup: str = "faithful_zero_updates"
    overlap_recompute: bool = True

    def describe(self) -> str:
        return f"(p={','.join(map(str, self.p))}; m={','.join(map(str, self.m))})"


@dataclass(frozen=True)
class StalenessProfile:
    per_block: tuple
    max: int


def validate_config(p, m, warmup: str = "faithful_zero_updates", overlap_recompute: bool = True) -> PipelineConfig:
    """Eq.(5) constraints in the reference's order; derives q (pipeline.py:85-128).

      p_last_zero, p_positive, m_positive, m_last_nonneg, q_positive
      with q[k] = m[k-1] - p[k-1] - m[k] for 1 <= k <= K-1, q[0] = 0.
    """
    p = tuple(int(v) for v in p)
    m = tuple(int(v) for v in m)
    if len(p) != len(m) or not p:
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


def staleness_of(config: PipelineConfig) -> StalenessProfile:
    return StalenessProfile(per_block=config.m, max=max(config.m))


def default_queue_config(k: int, warmup: str = "faithful_zero_updates") -> PipelineConfig:
    """p_k = 1, m_k = 2(K-1-k): q = (0,1,...,1), DSP(1,1,0;4,2,0) at K=3."""
    p = [1] * (k - 1) + [0]
    m = [2 * (k - 1 - i) for i in range(k)]
    return validate_config(p, m, warmup=warmup)


@dataclass(frozen=True)
class ActivationPacket:
    batch_index: int
    tensor: object
    labels: object


@dataclass(frozen=True)
class GradPacket:
    batch_index: int
    tensor: object


class _Fifo:
    """Bounded FIFO; overflow / underflow are bugs (pipeline.py:148-169)."""

    __slots__ = ("name", "capacity", "items")

    def __init__(self, name: str, capacity: int):
        self.name = name
        self.capacity = capacity
        self.items = deque()

    def put(self, pkt) -> None:
        if len(self.items) >= self.capacity:
            raise ProtocolError(f"push to full queue {self.name} (capacity {self.capacity})")
        self.items.append(pkt)

    def get(self):
        if not self.items:
            raise ProtocolError(f"pop from empty queue {self.name}")
        return self.items.popleft()

    def __len__(self) -> int:
        return len(self.items)


@dataclass
class LogRecord:
    step: int
    block: int
    batch_index: int
    grad_norm: float
    loss: float | None = None
    grad_deviation: float | None = None
    wall_nanos: int = 0


class TrainLog:
    """Per-(step, block) records with the reference's content checksum (pipeline.py:208-253)."""

    SCHEMA_VERSION = 1

    def __init__(self, records=None):
        self.records = records or []

    def sorted(self):
        return sorted(self.records, key=lambda r: (r.step, r.block))

    def checksum(self) -> str:
        h = hashlib.sha256()
        for r in self.sorted():
            lh = "-" if r.loss is None else float(r.loss).hex()
            h.update(f"{r.step}|{r.block}|{r.batch_index}|{lh}|{float(r.grad_norm).hex()}\n".encode())
        return h.hexdigest()

    def index_checksum(self) -> str:
        """Checksum of the FIFO/staleness schedule alone (step, block, batch_index)."""
        h = hashlib.sha256()
        for r in self.sorted():
            h.update(f"{r.step}|{r.block}|{r.batch_index}\n".encode())
        return h.hexdigest()

    def to_jsonl(self, path) -> None:
        with open(path, "w") as f:
            f.write(json.dumps({"schema_version": self.SCHEMA_VERSION, "kind": "train_log"}) + "\n")
            for r in self.sorted():
                f.write(json.dumps({"step": r.step, "block": r.block, "batch_index": r.batch_index,
                                    "loss": r.loss, "grad_norm": r.grad_norm,
                                    "grad_deviation": r.grad_deviation, "wall_nanos": r.wall_nanos}) + "\n")

    def losses(self):
        return [(r.step, r.loss) for r in self.sorted() if r.loss is not None]


@dataclass
class RuntimeStraggler:
    """Seeded host sleeps; changes timing only (pipeline.py:429-440)."""

    prob: float = 1 / 3
    delay_s: float = 0.001
    seed: int = 0

    def sleep_maybe(self, block: int, step: int, phase: int) -> None:
        z = mix64(self.seed ^ mix64((block + 1) * 0x9E37 + step * 2 + phase))
        if (z >> 11) * 2.0**-53 < self.prob:
            time.sleep(self.delay_s)


@dataclass
class DeviceStraggler(RuntimeStraggler):
    """RuntimeStraggler's seeded decisions, with the delay injected on the block's device stream
    (dsp_device_sleep) -- it slows the GPU work itself, like a straggling worker, and never changes
    values. Runs with eager steps: the per-step decisions vary."""

    def hits(self, block: int, step: int, phase: int) -> bool:
        z = mix64(self.seed ^ mix64((block + 1) * 0x9E37 + step * 2 + phase))
        return (z >> 11) * 2.0**-53 < self.prob

    def sleep_maybe(self, block: int, step: int, phase: int, rt=None) -> None:
        if not self.hits(block, step, phase):
            return
        if rt is None:
            time.sleep(self.delay_s)
        else:
            rt.device_sleep(block, self.delay_s)


def default_placement(k: int, world: int) -> list[int]:
    """Contiguous blocks per rank: K blocks over `world` ranks (one block per GPU when K == world)."""
    if world <= 1:
        return [0] * k
    if world > k:
        raise ConfigError("placement", 0, f"{world} ranks but only {k} blocks")
    return [min(world - 1, (i * world) // k) for i in range(k)]


class TrainEngine:
    """Resumable K-block DSP training pipeline (pipeline.py:443-694), backend "b200".

    ``run(n)`` advances every (local) block by n iterations and may be called
    repeatedly; queue contents persist across calls. ``placement[k]`` is the
    rank that owns block k (default: all local, or contiguous over the
    initialised torch.distributed world).
    """

    def __init__(self, model: Model, config: PipelineConfig, data_stream: Iterator, schedule: LrSchedule,
                 rule: str = "sgd", beta: float = 0.0, s: float = 1.0, weight_decay: float = 0.0,
                 backend: str = "b200", deviation_every: int = 0, straggler: RuntimeStraggler | None = None,
                 watchdog_s: float = 120.0, placement=None, device=None, precision: str = "bf16", _runtime=None,
                 _transport=None):
        if config.k != model.k:
            raise ConfigError("k", 0, f"config K={config.k} but model has {model.k} blocks")
        if backend not in BACKENDS:
            raise ValueError(f"backend must be one of {BACKENDS} (this package is the B200 backend; "
                             f"'serial'/'parallel' are the reference's CPU backends), got {backend!r}")
        if rule not in RULES:
            raise ValueError(f"unknown optimizer rule: {rule!r}")
        OptimizerState(rule=rule, beta=beta, s=s)  # validates beta / s like the reference
        self.model = model
        self.config = config
        self.schedule = schedule
        self.rule = rule
        self.beta = beta
        self.s = s
        self.weight_decay = weight_decay
        self.backend = backend
        self.straggler = straggler
        self.watchdog_s = watchdog_s
        self._data = data_stream
        self._first_batch = next(data_stream)  # peeked to size the warmup packets (pipeline.py:479)
        self._pending_first = True
        x0 = self._first_batch[0]
        self.batch_size = int(x0.shape[0] if hasattr(x0, "shape") else np.asarray(x0).shape[0])

        K = config.k
        self._transport = _transport
        if self._transport is None:
            from .transport import default_transport

            self._transport = default_transport()
        rank = self._transport.rank
        world = self._transport.world
        self.placement = list(placement) if placement is not None else default_placement(K, world)
        if len(self.placement) != K or any(not (0 <= r < world) for r in self.placement):
            raise ConfigError("placement", 0, f"bad placement {self.placement} for K={K}, world={world}")
        self.rank = rank
        self.local = [k for k in range(K) if self.placement[k] == rank]

        self._cum_p = [0] * (K + 1)
        for k in range(K):
            self._cum_p[k + 1] = self._cum_p[k] + config.p[k]

        if _runtime is None:
            from .engine_b200 import B200Runtime

            _runtime = B200Runtime(model, self.local, self.batch_size, rule=rule, beta=beta, s=s, config=config,
                                   weight_decay=weight_decay, device=device, precision=precision)
        self.rt = _runtime

        # queues: a FIFO lives on the consumer's rank (pipeline.py:483-513)
        cp = self._cum_p
        self.out_queues = [None] * max(K - 1, 0)
        for k in range(K - 1):
            if self.placement[k + 1] != rank:
                continue
            q = _Fifo(f"out[{k}]", 1 + config.p[k])
            for t in range(config.p[k]):
                q.put(ActivationPacket(t - cp[k + 1], self.rt.zero_act(k + 1), self.rt.zero_labels()))
            self.out_queues[k] = q
        self.in_queues = [None] * K
        for k in self.local:
            q = _Fifo(f"in[{k}]", 1 + config.m[k])
            for t in range(config.m[k]):
                q.put(ActivationPacket(t - cp[k] - config.m[k], self.rt.zero_act(k), self.rt.zero_labels()))
            self.in_queues[k] = q
        self.grad_queues = [None] * K
        for k in range(1, K):
            if self.placement[k - 1] != rank:
                continue
            q = _Fifo(f"grad[{k}]", 1 + config.q[k])
            for t in range(config.q[k]):
                q.put(GradPacket(t - cp[k - 1] - config.m[k - 1], self.rt.zero_grad(k)))
            self.grad_queues[k] = q
        # outgoing cross-rank packets produced during the current step
        self._outbox_act = {}
        self._outbox_grad = {}

        # gradient-deviation diagnostics on the device (pipeline.py:520; deviation.py). Needs
        # every block in this process; tracked runs take eager steps (snapshots are conditional).
        self.tracker = None
        if deviation_every:
            if len(self.local) != K:
                raise ValueError("deviation diagnostics need all blocks in one process")
            from .deviation import DeviationTracker

            self.tracker = DeviationTracker(deviation_every, model, self.batch_size, device=self.rt.device,
                                            stream=self.rt.stream, dtype=getattr(self.rt, "dtype_code", 0))
            self.rt.eager_concurrent = False  # snapshots are taken on the main stream

        self.opt_states = [self.rt.opt_state(k) if k in self.local else None for k in range(K)]
        self.block_steps = [0] * K
        self._block_logs = [[] for _ in range(K)]
        self._pending = []  # (record, loss_handle, gsq_handle)

    # ------------------------------------------------------------------ data
    def _next_batch(self):
        if self._pending_first:
            self._pending_first = False
            return self._first_batch
        return next(self._data)

    # ------------------------------------------------------------------ Algorithm-2 loop body
    def _iterate_block(self, k: int) -> None:
        """One step of block k (pipeline.py:538-606)."""
        n = self.block_steps[k]
        cfg = self.config
        last = cfg.k - 1
        rt = self.rt

        if k == 0:
            x, labels = self._next_batch()
            act, lab = rt.make_input(x, labels, n)
            fresh = ActivationPacket(n, act, lab)
        else:
            fresh = self.out_queues[k - 1].get()
        self.in_queues[k].put(fresh)
        stale = self.in_queues[k].get()

        if isinstance(self.straggler, DeviceStraggler):
            self.straggler.sleep_maybe(k, n, 0, rt)
        elif self.straggler is not None:
            self.straggler.sleep_maybe(k, n, 0)

        tr = self.tracker
        track_fresh = tr is not None and tr.wants(fresh.batch_index)
        track_stale = tr is not None and tr.wants(stale.batch_index)
        if track_fresh and k == 0:
            tr.on_input(fresh.batch_index, fresh.tensor, fresh.labels)
        if track_fresh and k < last:
            tr.on_forward(k, fresh.batch_index, rt.params_tensor(k))

        loss_h = None
        up_norm = None
        if k < last:
            h_out = rt.forward(k, fresh.tensor, n)
            pkt = ActivationPacket(fresh.batch_index, h_out, fresh.labels)
            if self.placement[k + 1] == self.rank:
                self.out_queues[k].put(pkt)
            else:
                self._outbox_act[k] = pkt
            rt.forward_record(k, stale.tensor, n)
            gpkt = self.grad_queues[k + 1].get()
            if gpkt.batch_index != stale.batch_index:
                raise ProtocolError(f"block {k} step {n}: gradient batch {gpkt.batch_index} "
                                    f"does not meet activation batch {stale.batch_index}")
            upstream = gpkt.tensor
            if track_stale:
                up_norm = rt.vector_norm(upstream)
        else:
            logits = None
            if track_stale:
                logits = rt.logits_buffer(k)
                rt.forward_record(k, stale.tensor, n, y=logits)
            else:
                rt.forward_record(k, stale.tensor, n)
            loss_h = rt.loss(k, stale.labels, n)
            upstream = None
            if track_stale:
                up_norm = rt.xent_grad_norm(logits, stale.labels)

        if isinstance(self.straggler, DeviceStraggler):
            self.straggler.sleep_maybe(k, n, 1, rt)
        elif self.straggler is not None:
            self.straggler.sleep_maybe(k, n, 1)

        grad_in = rt.backward(k, upstream, k > 0, n)
        if track_stale:  # backward-time parameters (before the update) and the runtime gradient
            tr.on_backward(k, stale.batch_index, rt.params_tensor(k), rt.grads_tensor(k), up_norm, n)
        if k > 0:
            gp = GradPacket(stale.batch_index, grad_in)
            if self.placement[k - 1] == self.rank:
                self.grad_queues[k].put(gp)
            else:
                self._outbox_grad[k] = gp

        discard = cfg.warmup == "discard_warmup_updates" and stale.batch_index < 0
        lr = lr_at(self.schedule, n)
        gsq_h = rt.update(k, lr, self.s * lr, not discard, n)
        st = self.opt_states[k]
        if st is not None and not discard:
            st.n += 1
        rec = LogRecord(step=n, block=k, batch_index=stale.batch_index, grad_norm=float("nan"), loss=None,
                        wall_nanos=time.monotonic_ns())
        self._block_logs[k].append(rec)
        self._pending.append((rec, loss_h, gsq_h))
        self.block_steps[k] = n + 1

    # ------------------------------------------------------------------ cross-rank exchange
    def _exchange(self, n: int | None = None) -> None:
        """Ship this step's boundary packets to their consumers and receive the packets the
        neighbours produced this step (consumed >= 1 step later).

        Packets land in the consumer runtime's per-phase receive rings (``recv_buffers``: slot
        n mod R, the same periodic addresses the step graphs bake in). Their batch tags follow the
        closed forms of SURVEY Appendix A (fresh tag n - cum_p[k], stale tag n - cum_p[k] - m_k),
        so the consumer queues the expected tag at once and verifies the received header on the
        device (``check_tag``), raising ProtocolError at the next sync point -- no per-step
        device->host read."""
        if self._transport.world <= 1:
            return
        K = self.config.k
        if n is None:
            n = self.block_steps[self.local[0]] - 1 if self.local else 0
        cp, m = self._cum_p, self.config.m
        sends, recvs = [], []
        for k in range(K - 1):
            prod, cons = self.placement[k], self.placement[k + 1]
            if prod == cons:
                continue
            if prod == self.rank:
                pkt = self._outbox_act.pop(k)
                sends.append((cons, self.rt.act_header(pkt.batch_index, pkt.labels), pkt.tensor))
            elif cons == self.rank:
                recvs.append(("act", k, prod, n - cp[k]))
        for k in range(1, K):
            prod, cons = self.placement[k], self.placement[k - 1]
            if prod == cons:
                continue
            if prod == self.rank:
                pkt = self._outbox_grad.pop(k)
                sends.append((cons, self.rt.grad_header(pkt.batch_index), pkt.tensor))
            elif cons == self.rank:
                recvs.append(("grad", k, prod, n - cp[k] - m[k]))
        bufs = []
        ring = getattr(self.rt, "recv_buffers", None)
        for kind, k, src, _ in recvs:
            if ring is not None:
                hdr, ten = ring(kind, k + 1 if kind == "act" else k, n)
            elif kind == "act":
                hdr, ten = self.rt.empty_act_header(), self.rt.empty_act(k + 1)
            else:
                hdr, ten = self.rt.empty_grad_header(), self.rt.empty_grad(k)
            bufs.append((src, hdr, ten))
        try:
            self._transport.exchange(sends, bufs, timeout_s=self.watchdog_s)
        except TimeoutError as exc:  # the reference's watchdog (pipeline.py:644-657)
            raise self._deadlock() from exc
        check = getattr(self.rt, "check_tag", None)
        for (kind, k, _, tag), (_, hdr, ten) in zip(recvs, bufs):
            if check is not None:  # device-side comparison, read at the next sync point
                check(hdr, tag)
                labels = hdr[1:] if kind == "act" else None
            elif kind == "act":
                tag, labels = self.rt.parse_act_header(hdr)
            else:
                tag = self.rt.parse_grad_header(hdr)
            if kind == "act":
                self.out_queues[k].put(ActivationPacket(tag, ten, labels))
            else:
                self.grad_queues[k].put(GradPacket(tag, ten))

    def _deadlock(self) -> DeadlockError:
        occupancy = {q.name: len(q) for q in self.out_queues if q is not None}
        occupancy.update({q.name: len(q) for q in self.grad_queues[1:] if q is not None})
        return DeadlockError(f"workers stalled after {self.watchdog_s}s; queue occupancy {occupancy} "
                             f"steps {self.block_steps}")

    # ------------------------------------------------------------------ drivers
    def run(self, n_steps: int) -> None:
        if n_steps < 0:
            raise ValueError("n_steps must be non-negative")
        # multi-rank: the local blocks' step is graph-replayed too; the NCCL exchange follows the
        # graph launch on the same stream (packets received into periodic per-phase ring slots)
        graphs = (getattr(self.rt, "use_graphs", False) and self.tracker is None
                  and not isinstance(self.straggler, DeviceStraggler)
                  and (self._transport.world <= 1 or os.environ.get("DSP_B200_MULTIRANK_GRAPHS", "1") != "0"))
        scope = getattr(self.rt, "scope", None)
        with scope() if scope is not None else _nullctx():
            for _ in range(n_steps):
                self._run_one(graphs)

    def _run_one(self, graphs: bool) -> None:
        n = self.block_steps[self.local[0]] if self.local else 0
        if graphs and n >= self._graph_horizon():
            self.rt.graph_step(n, self._step_signature(n), self._issue_local)
            self._exchange(n)
        else:
            self._issue_step()
            end = getattr(self.rt, "end_step", None)
            if end is not None:
                end(n)

    def _issue_step(self) -> None:
        self._issue_local()
        self._exchange()

    def _issue_local(self) -> None:
        fork = getattr(self.rt, "fork_blocks", None)
        if fork is not None:
            fork()
        for k in self.local:
            if self._transport.world <= 1:
                self._iterate_block(k)
                continue
            try:  # one process per GPU stands in for the reference's worker threads (pipeline.py:658-660)
                self._iterate_block(k)
            except (DeadlockError, ProtocolError, ConfigError):
                raise
            except Exception as exc:
                raise RuntimeError(f"worker for block {k} failed") from exc
        join = getattr(self.rt, "join_blocks", None)
        if join is not None:
            join()

    def _graph_horizon(self) -> int:
        """First step from which every queued packet is a ring slot (zero prefill drained)."""
        c = self.config
        return max(c.m) + max(c.p) + max(c.q) + 1

    def _step_signature(self, n: int) -> tuple:
        """Everything a step graph bakes in besides ring-slot addresses."""
        sig = []
        for k in self.local:
            lr = lr_at(self.schedule, n)
            tag = n - self._cum_p[k] - self.config.m[k]
            discard = self.config.warmup == "discard_warmup_updates" and tag < 0
            sig.append((lr, self.s * lr, not discard))
        return tuple(sig)

    def synchronize(self) -> None:
        try:
            self._transport.drain(self.watchdog_s)
        except TimeoutError as exc:
            raise self._deadlock() from exc
        self.rt.synchronize()
        bad = getattr(self.rt, "tag_errors", None)
        if bad is not None and bad():
            raise ProtocolError("a received packet's batch tag does not match the closed-form FIFO schedule "
                                "(gradient batch does not meet activation batch, pipeline.py:567-572)")

    def last_loss(self) -> float | None:
        """Loss of the most recent last-block step on this rank (a 4-byte device->host read)."""
        K = self.config.k
        if (K - 1) not in self.local or not self._block_logs[K - 1]:
            return None
        for rec, lh, _ in reversed(self._pending):
            if rec.block == K - 1:
                return self.rt.read_scalar(lh)
        return self._block_logs[K - 1][-1].loss

    def _materialize(self) -> None:
        if not self._pending:
            return
        self.synchronize()
        vals = self.rt.read_scalars([(l, g) for _, l, g in self._pending])
        for (rec, _, _), (lv, gv) in zip(self._pending, vals):
            rec.grad_norm = float(np.sqrt(gv))
            rec.loss = None if lv is None else float(lv)
        self._pending = []

    # ------------------------------------------------------------------ results
    @property
    def log(self) -> TrainLog:
        self._materialize()
        merged = []
        for rows in self._block_logs:
            merged.extend(rows)
        log = TrainLog(sorted(merged, key=lambda r: (r.step, r.block)))
        if self.tracker is not None:  # pipeline.py:670-677
            by_key = {}
            for row in self.tracker.rows():
                for k, step in enumerate(row.steps):
                    by_key[(step, k)] = row.per_param[k]
            for r in log.records:
                r.grad_deviation = by_key.get((r.step, r.block))
        return log

    def deviation_rows(self) -> list:
        return self.tracker.rows() if self.tracker is not None else []

    def realized_staleness(self) -> list[int]:
        """Fresh-vs-backward lag per block over non-warmup records (pipeline.py:682-694)."""
        lags = []
        for k in range(self.config.k):
            rows = [r for r in self._block_logs[k] if r.batch_index >= 0]
            if not rows:
                lags.append(0)
                continue
            lag = {(r.step - self._cum_p[k]) - r.batch_index for r in rows}
            if len(lag) != 1:
                raise ProtocolError(f"block {k} staleness drifted: {sorted(lag)}")
            lags.append(lag.pop())
        return lags


class _nullctx:
    def __enter__(self):
        return self

    def __exit__(self, *exc):
        return False


def model_forward(model: Model, x: np.ndarray) -> np.ndarray:
    """Evaluation forward (blocks.py:182-186) through device-bound blocks."""
    from .engine_b200 import eval_forward

    return eval_forward(model, x)


__all__ = [
    "ActivationPacket", "ConfigError", "DeadlockError", "GradPacket", "LogRecord", "PipelineConfig",
    "ProtocolError", "RuntimeStraggler", "DeviceStraggler", "ShapeError", "StalenessProfile", "TrainEngine", "TrainLog",
    "WARMUP_POLICIES", "default_placement", "default_queue_config", "model_forward", "staleness_of",
    "validate_config",
]
