"""B200 runtime behind ``TrainEngine``: the device half of ``_iterate_block``.

One ``DeviceBlock`` per local block. Packets live in fixed device rings: the
packet a block produces at step n occupies slot n mod R of its ring, where R
exceeds every packet's lifetime in steps (an out-packet of block k lives
p_k + m_{k+1} steps, an input packet m_0, a gradient packet q_k), so the
buffers a step touches depend only on n mod R.

That makes a step's device work periodic, and the runtime turns it into CUDA
graphs (``graph_step``): once the zero prefill packets have drained, step n is
captured once per phase n mod R -- each of the K local blocks on its own forked
stream, since within a step the blocks are independent (every packet they read
was produced in an earlier step) -- and afterwards replayed with one graph
launch. A phase is re-captured if its learning rates / update flags change
(lr decay). The per-step loss and squared grad norm land in per-phase slots
that are copied into a device log after each replay; the host reads them
lazily, so the training loop never synchronises.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import _lib as L
from .optim import RULES, OptimizerState
from .runtime import DeviceBlock, pack_input, ptr, require_cuda, stream_ptr, torch_mod


def _pad8(c: int) -> int:
    return (c + 7) // 8 * 8


def act_elems(batch: int, shape: tuple) -> int:
    c, h, w = shape
    return batch * h * w * _pad8(c)


def block_priorities(model, local) -> dict:
    """CUDA stream priority per local block (lower = scheduled first).

    All K blocks of a step run concurrently on their own streams. Default: equal
    priorities -- measured on B200 (ResNet-56, K=4), ranking blocks by FLOPs or favouring
    block 0 made the step 3-7% slower. DSP_B200_BLOCK_PRIORITY="p0,p1,..." sets them
    (lower = dispatched first; "flops" = heaviest block first)."""
    env = os.environ.get("DSP_B200_BLOCK_PRIORITY")
    if not env or env == "none":
        return {k: 0 for k in local}
    if env != "flops":
        vals = [int(v) for v in env.split(",")]
        return {k: vals[k] if k < len(vals) else 0 for k in local}
    flops = {k: sum(sp.flops() for sp in model.blocks[k].layers) for k in local}
    order = sorted(local, key=lambda k: -flops[k])
    return {k: -min(3, len(order) - 1 - order.index(k)) if len(order) > 1 else 0 for k in local}


def use_twins(n_local: int) -> bool:
    """Forward twins (up to 8 blocks per rank). Measured on B200 (tools/block_step_latency.py,
    profiles/r01_twins.md): a GPU owning one block steps 11-22% faster on the CIFAR ResNets
    (ResNet-56 block 0 905 -> 775 us). With round-2 grid sizing (one CTA per SM for the CIFAR
    convs) they also pay when one GPU runs all blocks: ResNet-56 K=4 82.8k vs 74.2k samples/s,
    ResNet-164 K=4 22.6k vs 21.7k, ResNet-110 K=8 46.3k vs 45.8k (round 1: -3% at K=8).
    DSP_B200_TWIN=0/1 overrides."""
    env = os.environ.get("DSP_B200_TWIN")
    if env is not None:
        return env == "1"
    return n_local <= 8


class B200Runtime:
    LOG_CHUNK = 4096

    def __init__(self, model, local, batch: int, rule: str = "sgd", beta: float = 0.0, s: float = 1.0,
                 weight_decay: float = 0.0, device=None, config=None, use_graphs: bool = True,
                 precision: str = "bf16"):
        torch = torch_mod()
        self.torch = torch
        self.precision = precision
        self.dtype_code = L.storage_dtype(precision)
        self.act_dtype = L.torch_storage(self.dtype_code)
        self.device = require_cuda(device)
        if self.device.index is None:
            self.device = torch.device("cuda", torch.cuda.current_device())
        with torch.cuda.device(self.device):  # the library creates its streams / events on the current device
            self._init(model, local, batch, rule, beta, s, weight_decay, config, use_graphs)

    def scope(self):
        """Context making this runtime's device current: every library call that creates CUDA
        objects (block side streams, events) or launches kernels runs under it."""
        return self.torch.cuda.device(self.device)

    def _init(self, model, local, batch, rule, beta, s, weight_decay, config, use_graphs):
        torch = self.torch
        self.stream = torch.cuda.current_stream(self.device)
        self.model = model
        self.B = batch
        self.K = model.k
        self.local = list(local)
        self.rule = rule
        self.rule_code = RULES[rule]
        self.beta = beta
        self.s = s
        self.wd = weight_decay
        self.num_classes = model.output_dim
        self.dev = {}
        self.ys = {}
        self.adam = OptimizerState(rule="adam")  # Adam hyper-parameters (extension; defaults of the oracle)
        for k in self.local:
            blk = model.blocks[k]
            db = DeviceBlock(blk, batch, is_last=(k == self.K - 1), device=self.device, stream=self.stream,
                             dtype=self.dtype_code)
            blk.dev = db
            self.dev[k] = db
            if rule == "sum":
                with torch.cuda.stream(self.stream):
                    self.ys[k] = db.params.clone()
            elif rule == "adam":  # [m | v | int64 step counter] (DSP_ADAM_STATE_BYTES), zero = fresh
                n = db.params.numel()
                self.ys[k] = torch.zeros(2 * n + 2, dtype=torch.float32, device=self.device)
        # ---- rings (slot = step mod R) -------------------------------------------
        if config is not None:
            p, m, q = config.p, config.m, config.q
            life = [m[0] + 1] + [p[k] + m[k + 1] + 1 for k in range(self.K - 1)] + [q[k] + 1 for k in range(1, self.K)]
            self.R = max(life) + 1
        else:
            self.R = 8
        R = self.R
        self.ring_out = {k: [self._empty(self.dev[k].out_elems) for _ in range(R)]
                         for k in self.local if k < self.K - 1}
        self.ring_gin = {k: [self._empty(self.dev[k].in_elems) for _ in range(R)] for k in self.local if k > 0}
        self.ring_in = [self._empty(self.in_elems(0)) for _ in range(R)] if 0 in self.local else []
        self.ring_lab = [self._empty(batch, dtype=torch.int64, zero=True) for _ in range(R)] if 0 in self.local else []
        self._pinned = {}
        # ---- scalar slots: per phase, per block: [loss, grad_sq] ------------------
        self.slots = self._empty(R * self.K * 2, dtype=torch.float32, zero=True)
        self._log = []          # device chunks [LOG_CHUNK][K][2]
        self._log_rows = 0
        self._row_of_step = {}
        # ---- graphs -----------------------------------------------------------------
        self.use_graphs = use_graphs and torch.cuda.is_available()
        self.graphs = {}        # phase -> (CUDAGraph, signature, kernels, cudaGraphExec_t)
        self.mode = "eager"     # eager | capture | replay
        self._cur_stream = self.stream
        prio = block_priorities(model, self.local)
        self._block_streams = {k: torch.cuda.Stream(self.device, priority=prio[k]) for k in self.local}
        self.eager_concurrent = True  # eager steps: local blocks on their own streams too
        # forward twins: block k's fresh forward (pipeline.py:564) runs on a twin with its own
        # workspace and stream, overlapping the recompute + backward; joined before the update
        self.twins, self._fwd_streams, self._fwd_pending = {}, {}, {}
        if use_twins(len(self.local)):
            for k in self.local:
                if k < self.K - 1:
                    self.twins[k] = self.dev[k].make_twin()
                    self._fwd_streams[k] = torch.cuda.Stream(self.device, priority=prio[k])
        self.replayed_kernels = 0  # library kernels executed through graph replays
        self._recv = {}  # multi-rank receive rings (recv_buffers)
        self._tagbad = self._empty(1, dtype=torch.int64, zero=True)

    def kernels_executed(self) -> int:
        """Library kernels run so far: eager launches (dsp_launch_count, which also counts
        the launches recorded while capturing) plus every graph replay's kernels."""
        return int(L.load().dsp_launch_count()) + self.replayed_kernels

    # ---------------------------------------------------------------- buffers
    def _empty(self, n, dtype=None, zero=False):
        torch = self.torch
        dtype = dtype or self.act_dtype
        with torch.cuda.stream(self.stream):
            return (torch.zeros if zero else torch.empty)(max(n, 1), dtype=dtype, device=self.device)

    def in_elems(self, k: int) -> int:
        return act_elems(self.B, self.model.blocks[k].in_shape)

    def _s(self, k):
        """Stream for block k's work: its own forked stream while capturing a step graph, and in
        eager steps too (eager_concurrent) so the local blocks of a step run concurrently."""
        if self.mode == "capture" or (self.mode == "eager" and self.eager_concurrent):
            return self._block_streams[k]
        return self.stream

    def device_sleep(self, k: int, seconds: float) -> None:
        """Straggler delay on block k's stream (DeviceStraggler)."""
        L.check(L.load().dsp_device_sleep(int(seconds * 1e9), stream_ptr(self._s(k))))

    def fork_blocks(self) -> None:
        """Eager step start: every block stream waits for the main stream (inputs staged, the
        previous step and its exchange done)."""
        if self.mode != "eager" or not self.eager_concurrent:
            return
        ev = self.torch.cuda.Event()
        ev.record(self.stream)
        for k in self.local:
            self._block_streams[k].wait_event(ev)

    def join_blocks(self) -> None:
        """Eager step end: the main stream waits for every block stream (before the exchange)."""
        if self.mode != "eager" or not self.eager_concurrent:
            return
        for k in self.local:
            self.stream.wait_stream(self._block_streams[k])

    def make_input(self, x, labels, n: int = 0):
        from .data import DeviceBatch

        torch = self.torch
        slot = n % self.R
        act, lab = self.ring_in[slot], self.ring_lab[slot]
        if isinstance(x, DeviceBatch):
            if x.act.dtype != self.act_dtype:
                raise ValueError(f"device batch holds {x.act.dtype}, engine precision {self.precision!r} stores "
                                 f"{self.act_dtype}")
            if self.mode == "eager":
                self._copy_device_batch(x, slot, self._s(0))
            else:  # graph steps copy the batch in right before the launch
                self._pending_input = (x, slot)
            return act, lab
        if x.shape[0] != self.B:
            raise ValueError(f"batch of {x.shape[0]} rows, engine sized for {self.B}")
        width = int(np.prod(x.shape[1:]))
        shape0 = self.model.blocks[0].in_shape
        if width != int(np.prod(shape0)):
            from .blocks import ShapeError

            raise ShapeError(f"batch width {width} does not match the model input {tuple(shape0)}")
        lab_h = np.asarray(labels, dtype=np.int64)
        if lab_h.shape != (self.B,):
            raise ValueError(f"labels must have shape ({self.B},), got {lab_h.shape}")
        if lab_h.size and (lab_h.min() < 0 or lab_h.max() >= self.num_classes):
            raise ValueError(f"label out of range [0, {self.num_classes})")
        # host batch -> pinned staging slot -> device (H2D + pack run on the stream).
        # Graph steps defer all of it to just before the launch (no syncs in capture).
        if self.mode == "eager":
            self._stage_host_input(x, lab_h, slot)
            self._issue_host_input(slot, self._s(0))
        else:
            self._pending_input = ("host", slot, x, lab_h)
        return act, lab

    def _stage_host_input(self, x, lab_h, slot):
        torch = self.torch
        ev = self._pinned.get(("ev", slot))
        if ev is not None:
            ev.synchronize()  # the previous H2D out of this pinned slot has completed
        xs = self._pinned.get(("x", slot))
        if xs is None:
            xs = torch.empty(x.shape, dtype=torch.float32).pin_memory()
            ls = torch.empty(self.B, dtype=torch.int64).pin_memory()
            xd = self._empty(int(np.prod(x.shape)), dtype=torch.float32)
            self._pinned[("x", slot)], self._pinned[("l", slot)], self._pinned[("xd", slot)] = xs, ls, xd
        xs.numpy()[...] = x
        self._pinned[("l", slot)].numpy()[...] = lab_h

    def _copy_device_batch(self, db, slot, stream):
        with self.torch.cuda.stream(stream):
            self.ring_in[slot].copy_(db.act, non_blocking=True)
            self.ring_lab[slot].copy_(db.labels, non_blocking=True)

    def _issue_host_input(self, slot, stream):
        torch = self.torch
        xs, ls, xd = self._pinned[("x", slot)], self._pinned[("l", slot)], self._pinned[("xd", slot)]
        c, h, w = self.model.blocks[0].in_shape
        with torch.cuda.stream(stream):
            xd.copy_(xs.view(-1), non_blocking=True)
            self.ring_lab[slot].copy_(ls, non_blocking=True)
        L.check(L.load().dsp_pack_input(ptr(xd), ptr(self.ring_in[slot]), self.B, c, h, w, _pad8(c),
                                        self.dtype_code, 1, stream_ptr(stream)))
        ev = self._pinned.get(("ev", slot)) or torch.cuda.Event()
        ev.record(stream)
        self._pinned[("ev", slot)] = ev

    def zero_act(self, k: int):
        return self._empty(self.in_elems(k), zero=True)

    def zero_labels(self):
        return self._empty(self.B, dtype=self.torch.int64, zero=True)

    def zero_grad(self, k: int):
        return self._empty(self.in_elems(k), zero=True)

    def empty_act(self, k: int):
        return self._empty(self.in_elems(k))

    def empty_grad(self, k: int):
        return self._empty(self.in_elems(k))

    def act_header(self, tag: int, labels):
        torch = self.torch
        with torch.cuda.stream(self.stream):
            return torch.cat([torch.tensor([tag], dtype=torch.int64, device=self.device), labels])

    def grad_header(self, tag: int):
        return self.torch.tensor([tag], dtype=self.torch.int64, device=self.device)

    def empty_act_header(self):
        return self._empty(1 + self.B, dtype=self.torch.int64)

    def empty_grad_header(self):
        return self._empty(1, dtype=self.torch.int64)

    # ---- multi-rank receive rings (graph-safe: slot n mod R) and lazy tag checks ------------
    def recv_buffers(self, kind: str, k: int, n: int):
        """(header, tensor) slot n mod R of the receive ring for block k's cross-rank input
        packets (kind "act": header = [tag, labels...]; "grad": header = [tag]). A packet lives at
        most p_k + m_k (act) / q_k (grad) steps < R, so slots are never overwritten early."""
        key = (kind, k, n % self.R)
        buf = self._recv.get(key)
        if buf is None:
            torch = self.torch
            hdr = self._empty(1 + self.B if kind == "act" else 1, dtype=torch.int64, zero=True)
            buf = (hdr, self._empty(self.in_elems(k), zero=True))
            self._recv[key] = buf
        return buf

    def check_tag(self, hdr, tag: int) -> None:
        """Compare a received header's batch tag with the closed-form one on the device; any
        mismatch is counted in a device flag that synchronize() turns into ProtocolError."""
        with self.torch.cuda.stream(self.stream):
            self._tagbad.add_((hdr[:1] != tag).to(self.torch.int64))

    def tag_errors(self) -> int:
        return int(self._tagbad.item())

    def parse_act_header(self, hdr):
        return int(hdr[0].item()), hdr[1:]

    def parse_grad_header(self, hdr) -> int:
        return int(hdr[0].item())

    # ---------------------------------------------------------------- compute
    def _slot(self, n: int, k: int, which: int):
        return ("slot", n, k, which)

    def _slot_tensor(self, n: int, k: int, which: int):
        i = ((n % self.R) * self.K + k) * 2 + which
        return self.slots[i:i + 1]

    def forward(self, k: int, x, n: int = 0):
        y = self.ring_out[k][n % self.R]
        if self.mode != "replay":
            tw = self.twins.get(k)
            if tw is None:
                self.dev[k].forward(x, y, record=False, stream=self._s(k))
            else:  # fork onto the twin's stream; joined in update() before the weights change
                fs = self._fwd_streams[k]
                fs.wait_stream(self._s(k))
                tw.forward(x, y, record=False, stream=fs)
                self._fwd_pending[k] = fs
        return y

    def forward_record(self, k: int, x, n: int = 0, y=None) -> None:
        if self.mode != "replay":
            self.dev[k].forward(x, y, record=True, stream=self._s(k))

    # ---- deviation diagnostics (eager steps only) ---------------------------
    def params_tensor(self, k: int):
        return self.dev[k].params[: self.model.blocks[k].param_count]

    def grads_tensor(self, k: int):
        return self.dev[k].grads[: self.model.blocks[k].param_count]

    def logits_buffer(self, k: int):
        """fp32 [B][C_pad] buffer the last block's recorded forward copies its logits into."""
        with self.torch.cuda.stream(self.stream):
            return self.torch.empty(self.B * _pad8(self.num_classes), dtype=self.torch.float32, device=self.device)

    def vector_norm(self, t):
        with self.torch.cuda.stream(self.stream):
            return self.torch.linalg.vector_norm(t.float())

    def xent_grad_norm(self, logits, labels):
        """||(softmax(z) - onehot) / B|| of the recorded logits: the upstream error gradient
        the last block differentiates (tensor.py:86-111)."""
        torch = self.torch
        with torch.cuda.stream(self.stream):
            z = logits.view(self.B, -1)[:, : self.num_classes].double()
            g = torch.softmax(z, dim=1)
            g[torch.arange(self.B, device=self.device), labels] -= 1.0
            return torch.linalg.vector_norm(g / self.B)

    def loss(self, k: int, labels, n: int = 0):
        if self.mode != "replay":
            self.dev[k].loss(labels, self._slot_tensor(n, k, 0), stream=self._s(k))
        return self._slot(n, k, 0)

    def backward(self, k: int, upstream, need_grad_in: bool, n: int = 0):
        gin = self.ring_gin[k][n % self.R] if need_grad_in else None
        if self.mode != "replay":
            self.dev[k].backward(upstream, gin, stream=self._s(k))
        return gin

    def update(self, k: int, lr: float, slr: float, apply: bool, n: int = 0):
        fs = self._fwd_pending.pop(k, None)
        if fs is not None:
            self._s(k).wait_stream(fs)
        if self.mode != "replay" and self.rule == "adam":
            st = self.adam
            self.dev[k].update_adam(self.ys[k], lr, st.beta1, st.beta2, st.eps, self.wd, apply,
                                    self._slot_tensor(n, k, 1), stream=self._s(k))
        elif self.mode != "replay":
            self.dev[k].update(self.rule_code, self.ys.get(k), lr, slr, self.beta, self.wd, apply,
                               self._slot_tensor(n, k, 1), stream=self._s(k))
        return self._slot(n, k, 1)

    def opt_state(self, k: int) -> OptimizerState:
        st = OptimizerState(rule=self.rule, beta=self.beta, s=self.s)
        if self.rule == "adam":
            torch = self.torch
            n = self.dev[k].params.numel()
            self.synchronize()
            state = self.ys[k]
            st.m1, st.m2 = state[:n], state[n:2 * n]
            st.n = int(state[2 * n:2 * n + 2].view(torch.int64)[0].item())  # applied updates
        else:
            st.ys = self.ys.get(k)
        return st

    # ---------------------------------------------------------------- graph steps
    def graph_step(self, n: int, signature, issue) -> None:
        """Run step n's device work through the phase graph (capture on first use).

        issue(): runs the engine's host-side loop body for all local blocks; in
        capture mode it issues kernels, in replay mode it only does bookkeeping."""
        torch = self.torch
        phase = n % self.R
        entry = self.graphs.get(phase)
        if entry is not None and entry[1] == signature:
            self.mode = "replay"
            try:
                issue()
            finally:
                self.mode = "eager"
            self._pre_replay()
            L.check(L.load().dsp_graph_launch(entry[3], self.torch.cuda.current_stream(self.device).cuda_stream))
            self.replayed_kernels += entry[2]
        else:
            lib = L.load()
            before = lib.dsp_launch_count()
            g = torch.cuda.CUDAGraph(keep_graph=True)
            cs = torch.cuda.Stream(self.device)
            cs.wait_stream(self.stream)
            self.mode = "capture"
            saved = self.stream
            try:
                with torch.cuda.graph(g, stream=cs):
                    fork = torch.cuda.Event()
                    fork.record(cs)
                    for k in self.local:
                        self._block_streams[k].wait_event(fork)
                    issue_stream = cs
                    self.stream = issue_stream
                    issue()
                    for k in self.local:
                        cs.wait_stream(self._block_streams[k])
            finally:
                self.mode = "eager"
                self.stream = saved
            self.stream.wait_stream(cs)
            captured = lib.dsp_launch_count() - before
            # instantiate through the library so each kernel node keeps its block stream's
            # priority (torch's own instantiate ignores node priorities)
            exe = C.c_void_p()
            L.check(lib.dsp_graph_instantiate(C.c_void_p(g.raw_cuda_graph()), L.DSP_GRAPH_NODE_PRIORITY,
                                              C.byref(exe)))
            old = self.graphs.get(phase)
            if old is not None:
                lib.dsp_graph_destroy(old[3])
            self.graphs[phase] = (g, signature, captured, exe)
            self._pre_replay()  # this step's input batch -> its ring slot, outside the graph
            # (its kernels were counted once by dsp_launch_count while capturing)
            L.check(lib.dsp_graph_launch(exe, self.torch.cuda.current_stream(self.device).cuda_stream))
        self._post_step(n)

    def _pre_replay(self):
        pend = getattr(self, "_pending_input", None)
        self._pending_input = None
        if pend is None:
            return
        if pend[0] == "host":  # graph steps: staged on the main stream the graph launch follows
            _, slot, x, lab_h = pend
            self._stage_host_input(x, lab_h, slot)
            self._issue_host_input(slot, self.stream)
        else:
            self._copy_device_batch(pend[0], pend[1], self.stream)

    def _post_step(self, n: int) -> None:
        """Copy phase slots of step n into the device log (eager steps write slots too)."""
        torch = self.torch
        row = self._log_rows
        if row % self.LOG_CHUNK == 0:
            self._log.append(self._empty(self.LOG_CHUNK * self.K * 2, dtype=torch.float32, zero=True))
        chunk = self._log[row // self.LOG_CHUNK]
        r = row % self.LOG_CHUNK
        ph = n % self.R
        with torch.cuda.stream(self.stream):
            chunk[r * self.K * 2:(r + 1) * self.K * 2].copy_(self.slots[ph * self.K * 2:(ph + 1) * self.K * 2],
                                                             non_blocking=True)
        self._row_of_step[n] = row
        self._log_rows += 1

    def end_step(self, n: int) -> None:
        """Eager step finished (no graph): log its slots."""
        self._pending_input = None
        self._post_step(n)

    def synchronize(self) -> None:
        self.stream.synchronize()
        self.check_finite()

    def check_finite(self) -> None:
        """The reference raises NonFiniteError inside the step (tensor.py:34-37, optim.py:53 / 89);
        the device sets sticky per-block flags (dsp_block_nonfinite) that every sync point checks."""
        lib = L.load()
        for k in self.local:
            f = C.c_int(0)
            L.check(lib.dsp_block_nonfinite(self.dev[k].h, 0, C.byref(f), stream_ptr(self.stream)))
            if f.value:
                from .optim import NonFiniteError

                if f.value & L.DSP_NONFINITE_LOSS:
                    raise NonFiniteError(f"non-finite values in softmax_xent (block {k})")
                step = {"sgd": "sgd_step", "sum": "sum_step"}.get(self.rule, "update")
                raise NonFiniteError(f"non-finite gradient in {step} (block {k})")

    def _value(self, h, host_chunks):
        _, n, k, which = h
        row = self._row_of_step[n]
        return float(host_chunks[row // self.LOG_CHUNK][((row % self.LOG_CHUNK) * self.K + k) * 2 + which])

    def read_scalar(self, h) -> float:
        self.synchronize()
        _, n, k, which = h
        row = self._row_of_step.get(n)
        if row is None:  # not yet copied into the log: read the live slot
            return float(self._slot_tensor(n, k, which).item())
        c = self._log[row // self.LOG_CHUNK]
        i = ((row % self.LOG_CHUNK) * self.K + k) * 2 + which
        return float(c[i:i + 1].item())

    def read_scalars(self, pairs):
        self.synchronize()
        host = [c.cpu().numpy() for c in self._log]
        return [(None if lh is None else self._value(lh, host), self._value(gh, host)) for lh, gh in pairs]


def eval_forward(model, x: np.ndarray) -> np.ndarray:
    """Host batch -> host logits through device blocks (binds temporary DeviceBlocks if needed)."""
    torch = torch_mod()
    device = require_cuda()
    stream = torch.cuda.current_stream(device)
    B = x.shape[0]
    bound = [blk.dev for blk in model.blocks if blk.dev is not None]
    dtype = bound[0].dtype if bound else L.DSP_DTYPE_BF16
    h = pack_input(np.asarray(x), model.blocks[0].in_shape, device, stream, dtype=dtype)
    K = model.k
    for k, blk in enumerate(model.blocks):
        db = blk.dev
        if db is None or db.batch != B or db.dtype != dtype:
            db = DeviceBlock(blk, B, is_last=(k == K - 1), device=device, stream=stream, dtype=dtype)
        if k < K - 1:
            y = db.new_activation(db.out_elems)
            db.forward(h, y, record=False, stream=stream)
            h = y
        else:
            cp = _pad8(model.output_dim)
            with torch.cuda.stream(stream):
                logits = torch.empty(B * cp, dtype=torch.float32, device=device)
            db.forward(h, logits, record=False, stream=stream)
            stream.synchronize()
            return logits.view(B, cp)[:, : model.output_dim].double().cpu().numpy()
    raise L.DspError(1, "empty model")
