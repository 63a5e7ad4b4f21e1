"""Gradient-deviation diagnostics on the device.

Device counterparts of the reference's standalone operators and tracker
(/root/reference/pkg/src/stalepipe/pipeline.py:256-427):

* ``DeviceOperators.bp_gradient``   -- plain chained backprop at given parameters (256-267);
* ``DeviceOperators.stale_gradient`` -- the recompute-based gradient from forward-time and
  backward-time snapshots (270-305): the operator the runtime realises through its queues;
* ``DeviceOperators.grad_deviation`` -- per-block ||g_runtime - g_BP|| (308-326);
* ``DeviationTracker`` -- snapshots at fresh-forward / backward time and scores every
  sampled batch (345-427), feeding ``DeviationRow`` and ``LogRecord.grad_deviation``.

The operators run the same block kernels as the engine on a second set of block
executors (their own workspaces), so on identical snapshots they reproduce the
runtime bit for bit (tests/test_deviation_gpu.py). Snapshots, gradients and norms stay
on the device; a row's scalars are read when the row is scored.
"""

from __future__ import annotations

from dataclasses import dataclass, field

from .runtime import DeviceBlock, torch_mod


@dataclass
class DeviationRow:
    batch_index: int
    raw: list            # ||g_k - bp_k|| with BP at the backward snapshot
    per_param: list      # raw / d_k
    raw_fwd: list        # ||g_k - bp_k|| with BP at the forward snapshot
    diffs: list          # ||x_k(bwd) - x_k(fwd)||
    upstream_norms: list
    steps: list          # iteration at which block k ran this batch's backward


@dataclass
class DeviationSample:
    batch_index: int
    x: object = None
    labels: object = None
    fwd: dict = field(default_factory=dict)
    bwd: dict = field(default_factory=dict)
    grads: dict = field(default_factory=dict)
    upstream: dict = field(default_factory=dict)
    steps: dict = field(default_factory=dict)


class DeviceOperators:
    """bp_gradient / stale_gradient / grad_deviation on device block executors."""

    def __init__(self, model, batch: int, device=None, stream=None, dtype: int = 0):
        torch = torch_mod()
        self.torch = torch
        self.model = model
        self.K = model.k
        self.B = batch
        self.stream = stream if stream is not None else torch.cuda.current_stream(device)
        self.blocks = [DeviceBlock(blk, batch, is_last=(k == self.K - 1), device=device, stream=self.stream,
                                   dtype=dtype) for k, blk in enumerate(model.blocks)]
        self.n = [blk.param_count for blk in model.blocks]
        with torch.cuda.stream(self.stream):
            self.inputs = [None] + [db.new_activation(db.in_elems) for db in self.blocks[1:]]
            self.gins = [None] + [db.new_activation(db.in_elems) for db in self.blocks[1:]]
            self.loss = torch.zeros(1, device=self.blocks[0].device)

    def _load(self, params):
        """params[k]: device fp32 vectors of block k's parameters (snapshots)."""
        from . import _lib as L
        from .runtime import stream_ptr

        for k, (db, p) in enumerate(zip(self.blocks, params)):
            with self.torch.cuda.stream(self.stream):
                db.params[: self.n[k]].copy_(p[: self.n[k]])
            L.check(L.load().dsp_block_pack(db.h, stream_ptr(self.stream)))

    def _chain_inputs(self, x):
        """inputs[k] of every block under the currently loaded parameters (fresh forwards)."""
        h = x
        ins = [x]
        for k in range(self.K - 1):
            y = self.inputs[k + 1]
            self.blocks[k].forward(h, y, record=False, stream=self.stream)
            ins.append(y)
            h = y
        return ins

    def _backward_chain(self, ins, labels, recompute_all: bool):
        """Last block: forward(record) + loss; then blocks K-1..0 backward, chaining grad_input.
        recompute_all: re-record blocks < K-1 right before their backward (stale_gradient)."""
        K = self.K
        last = self.blocks[K - 1]
        last.forward(ins[K - 1], None, record=True, stream=self.stream)
        last.loss(labels, self.loss, stream=self.stream)
        upstream = None
        grads = [None] * K
        for k in range(K - 1, -1, -1):
            db = self.blocks[k]
            if k < K - 1 and recompute_all:
                db.forward(ins[k], None, record=True, stream=self.stream)
            gin = self.gins[k] if k > 0 else None
            db.backward(upstream, gin, stream=self.stream)
            with self.torch.cuda.stream(self.stream):
                grads[k] = db.grads[: self.n[k]].clone()
            upstream = gin
        return grads

    def bp_gradient(self, params, x, labels):
        """Plain chained BP at ``params`` on the packed device batch x (pipeline.py:256-267)."""
        self._load(params)
        K = self.K
        h = x
        for k in range(K - 1):  # record every block's tape on the way up
            y = self.inputs[k + 1]
            self.blocks[k].forward(h, y, record=False, stream=self.stream)
            self.blocks[k].forward(h, None, record=True, stream=self.stream)
            h = y
        ins = [x] + self.inputs[1:]
        return self._backward_chain(ins, labels, recompute_all=False)

    def stale_gradient(self, fwd_params, bwd_params, x, labels):
        """Inputs by a forward chain under fwd_params, every block re-run under bwd_params and
        differentiated, chaining the error gradient downward (pipeline.py:270-305)."""
        self._load(fwd_params)
        ins = self._chain_inputs(x)
        self._load(bwd_params)
        return self._backward_chain(ins, labels, recompute_all=True)

    def grad_deviation(self, bwd_params, x, labels, pipeline_grads):
        """Per block {block, raw, per_param} vs BP at the backward snapshot (pipeline.py:308-326)."""
        bp = self.bp_gradient(bwd_params, x, labels)
        rows = []
        for k, (gp, gb) in enumerate(zip(pipeline_grads, bp)):
            raw = float(self.torch.linalg.vector_norm((gp.double() - gb.double())).item())
            rows.append({"block": k, "raw": raw, "per_param": raw / max(1, self.n[k])})
        return rows


class DeviationTracker:
    """Collects per-batch snapshots during a run and scores them against BP on the device
    (pipeline.py:345-427). Block k contributes when it fresh-forwards a sampled batch
    (forward-time parameters) and when it backward-processes it (backward-time parameters,
    runtime gradient, upstream norm); the last block's backward covers both."""

    def __init__(self, every: int, model, batch: int, device=None, stream=None, dtype: int = 0):
        if every <= 0:
            raise ValueError("sampling interval must be positive")
        self.every = every
        self.K = model.k
        self.ops = DeviceOperators(model, batch, device=device, stream=stream, dtype=dtype)
        self.torch = self.ops.torch
        self._pending = {}
        self._rows = []

    def wants(self, batch_index: int) -> bool:
        return batch_index >= 0 and batch_index % self.every == 0

    def _sample(self, b):
        return self._pending.setdefault(b, DeviationSample(b))

    def on_input(self, batch_index: int, x, labels) -> None:
        s = self._sample(batch_index)
        s.x, s.labels = x.clone(), labels.clone()

    def on_forward(self, k: int, batch_index: int, params) -> None:
        self._sample(batch_index).fwd[k] = params.clone()

    def on_backward(self, k: int, batch_index: int, params, grad, upstream_norm, step: int) -> None:
        s = self._sample(batch_index)
        s.bwd[k] = params.clone()
        if k == self.K - 1:
            s.fwd.setdefault(k, s.bwd[k])
        s.grads[k] = grad.clone()
        s.upstream[k] = upstream_norm
        s.steps[k] = step
        if len(s.bwd) == self.K and s.x is not None:
            del self._pending[batch_index]
            self._rows.append(self._score(s))

    def _score(self, s: DeviationSample) -> DeviationRow:
        torch = self.torch
        K = self.K
        bwd = [s.bwd[k] for k in range(K)]
        fwd = [s.fwd[k] for k in range(K)]
        grads = [s.grads[k] for k in range(K)]
        rows = self.ops.grad_deviation(bwd, s.x, s.labels, grads)
        bp_fwd = self.ops.bp_gradient(fwd, s.x, s.labels)
        raw_fwd = [float(torch.linalg.vector_norm(g.double() - b.double()).item()) for g, b in zip(grads, bp_fwd)]
        diffs = [float(torch.linalg.vector_norm(s.bwd[k].double() - s.fwd[k].double()).item()) for k in range(K)]
        ups = [float(s.upstream[k].item()) if hasattr(s.upstream[k], "item") else float(s.upstream[k])
               for k in range(K)]
        return DeviationRow(batch_index=s.batch_index, raw=[r["raw"] for r in rows],
                            per_param=[r["per_param"] for r in rows], raw_fwd=raw_fwd, diffs=diffs,
                            upstream_norms=ups, steps=[s.steps[k] for k in range(K)])

    def rows(self) -> list:
        return sorted(self._rows, key=lambda r: r.batch_index)
