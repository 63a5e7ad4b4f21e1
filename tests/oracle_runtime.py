"""Test double: the product TrainEngine's runtime interface backed by the CPU oracle.

Lets the CPU suite drive the real engine (FIFOs, prefill tags, warmup policy,
log, cross-rank exchange over gloo) with float64 oracle math, so the
schedule / transport logic is checked bitwise against the oracle engine
without a GPU. Packets are torch CPU float64 tensors (gloo can ship them).
"""

from __future__ import annotations

import numpy as np
import torch

import oracle.dsp_ref as R


class OracleRuntime:
    def __init__(self, omodel, local, batch, rule="sgd", beta=0.0, s=1.0, weight_decay=0.0):
        self.m = omodel
        self.B = batch
        self.local = list(local)
        self.wd = weight_decay
        self.dims = omodel.block_input_dims
        self.opt = {k: R.OptimizerState.for_params(rule, omodel.blocks[k].params, beta=beta, s=s) for k in local}
        self.tapes, self.tops, self.grads, self.vals = {}, {}, {}, []

    # packets
    def make_input(self, x, labels, n=0):
        return torch.from_numpy(np.asarray(x, dtype=np.float64)), torch.from_numpy(np.asarray(labels, dtype=np.int64))

    def zero_act(self, k):
        return torch.zeros(self.B, self.dims[k], dtype=torch.float64)

    def zero_labels(self):
        return torch.zeros(self.B, dtype=torch.int64)

    def zero_grad(self, k):
        return torch.zeros(self.B, self.dims[k], dtype=torch.float64)

    def empty_act(self, k):
        return torch.empty(self.B, self.dims[k], dtype=torch.float64)

    empty_grad = empty_act

    def act_header(self, tag, labels):
        return torch.cat([torch.tensor([tag], dtype=torch.int64), labels])

    def grad_header(self, tag):
        return torch.tensor([tag], dtype=torch.int64)

    def empty_act_header(self):
        return torch.empty(1 + self.B, dtype=torch.int64)

    def empty_grad_header(self):
        return torch.empty(1, dtype=torch.int64)

    def parse_act_header(self, hdr):
        return int(hdr[0]), hdr[1:].clone()

    def parse_grad_header(self, hdr):
        return int(hdr[0])

    # compute
    def _h(self, v):
        self.vals.append(v)
        return len(self.vals) - 1

    def forward(self, k, x, n=0):
        h, _ = R.block_forward(self.m.blocks[k], x.numpy())
        return torch.from_numpy(h)

    def forward_record(self, k, x, n=0):
        self.tops[k], self.tapes[k] = R.block_forward(self.m.blocks[k], x.numpy(), record=True)

    def loss(self, k, labels, n=0):
        loss, up = R.softmax_xent(self.tops[k], labels.numpy())
        self._up = up
        return self._h(loss)

    def backward(self, k, upstream, need_grad_in, n=0):
        up = self._up if upstream is None else upstream.numpy()
        g, gin = R.block_backward(self.m.blocks[k], self.tapes.pop(k), up)
        self.grads[k] = g
        return torch.from_numpy(gin) if need_grad_in else None

    def update(self, k, lr, slr, apply, n=0):
        blk = self.m.blocks[k]
        g0 = self.grads.pop(k)
        h = self._h(float((g0 ** 2).sum()))
        g = g0 + self.wd * blk.params if self.wd != 0.0 else g0
        if apply:
            blk.params = R.apply_update(self.opt[k], blk.params, g, lr)
            self.opt[k].n -= 1  # the engine counts opt_states[k].n itself
        return h

    def opt_state(self, k):
        return self.opt[k]

    def synchronize(self):
        pass

    def read_scalar(self, h):
        return self.vals[h]

    def read_scalars(self, pairs):
        return [(None if lh is None else self.vals[lh], self.vals[gh]) for lh, gh in pairs]
