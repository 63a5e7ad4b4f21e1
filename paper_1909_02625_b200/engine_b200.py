"""B200 runtime behind ``TrainEngine``: the device half of ``_iterate_block``.

One ``DeviceBlock`` per local block, all issued on one CUDA stream per
process (blocks of one step are independent -- every packet they consume was
produced in an earlier step -- so a single in-order stream is race-free and
the GPU overlaps back-to-back kernels). Packets are device tensors; the
per-(step, block) loss and squared gradient norm stay on the device until the
log is read, so the training loop never synchronises with the host.
"""

from __future__ import annotations

import numpy as np

from . import _lib as L
from .optim import RULES, OptimizerState
from .runtime import DeviceBlock, pack_input, require_cuda, torch_mod


def _pad8(c: int) -> int:
    return (c + 7) // 8 * 8


def act_elems(batch: int, shape: tuple) -> int:
    c, h, w = shape
    return batch * h * w * _pad8(c)


class B200Runtime:
    SLOTS = 4096

    def __init__(self, model, local, batch: int, rule: str = "sgd", beta: float = 0.0, s: float = 1.0,
                 weight_decay: float = 0.0, device=None):
        torch = torch_mod()
        self.torch = torch
        self.device = require_cuda(device)
        self.stream = torch.cuda.current_stream(self.device)
        self.model = model
        self.B = batch
        self.K = model.k
        self.rule = rule
        self.rule_code = RULES[rule]
        self.beta = beta
        self.s = s
        self.wd = weight_decay
        self.dev = {}
        self.ys = {}
        self.num_classes = model.output_dim
        for k in local:
            blk = model.blocks[k]
            db = DeviceBlock(blk, batch, is_last=(k == self.K - 1), device=self.device, stream=self.stream)
            blk.dev = db
            self.dev[k] = db
            if rule == "sum":
                with torch.cuda.stream(self.stream):
                    self.ys[k] = db.params.clone()
        self._chunks = []
        self._fill = self.SLOTS
        self.launches = 0

    # ---------------------------------------------------------------- packets
    def _empty(self, n, dtype=None, zero=False):
        torch = self.torch
        dtype = dtype or torch.bfloat16
        with torch.cuda.stream(self.stream):
            return (torch.zeros if zero else torch.empty)(n, dtype=dtype, device=self.device)

    def in_elems(self, k: int) -> int:
        return act_elems(self.B, self.model.blocks[k].in_shape)

    def make_input(self, x, labels):
        from .data import DeviceBatch

        if isinstance(x, DeviceBatch):  # already packed in HBM
            return x.act, x.labels
        if x.shape[0] != self.B:
            raise ValueError(f"batch of {x.shape[0]} rows, engine sized for {self.B}")
        lab = np.asarray(labels, dtype=np.int64)
        if lab.shape != (self.B,):
            raise ValueError(f"labels must have shape ({self.B},), got {lab.shape}")
        if lab.size and (lab.min() < 0 or lab.max() >= self.num_classes):
            raise ValueError(f"label out of range [0, {self.num_classes})")
        act = pack_input(np.asarray(x), self.model.blocks[0].in_shape, self.device, self.stream)
        torch = self.torch
        with torch.cuda.stream(self.stream):
            labd = torch.from_numpy(lab).pin_memory().to(self.device, non_blocking=True)
        return act, labd

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

    def parse_act_header(self, hdr):
        return int(hdr[0].item()), hdr[1:]

    def parse_grad_header(self, hdr) -> int:
        return int(hdr[0].item())

    # ---------------------------------------------------------------- compute
    def _slot(self):
        if self._fill >= self.SLOTS:
            self._chunks.append(self._empty(self.SLOTS, dtype=self.torch.float32, zero=True))
            self._fill = 0
        h = (len(self._chunks) - 1, self._fill)
        self._fill += 1
        return h

    def _slot_tensor(self, h):
        return self._chunks[h[0]][h[1]:h[1] + 1]

    def forward(self, k: int, x):
        db = self.dev[k]
        y = db.new_activation(db.out_elems)
        db.forward(x, y, record=False)
        return y

    def forward_record(self, k: int, x) -> None:
        self.dev[k].forward(x, None, record=True)

    def loss(self, k: int, labels):
        h = self._slot()
        self.dev[k].loss(labels, self._slot_tensor(h))
        return h

    def backward(self, k: int, upstream, need_grad_in: bool):
        db = self.dev[k]
        gin = db.new_activation(db.in_elems) if need_grad_in else None
        db.backward(upstream, gin)
        return gin

    def update(self, k: int, lr: float, slr: float, apply: bool):
        h = self._slot()
        self.dev[k].update(self.rule_code, self.ys.get(k), lr, slr, self.beta, self.wd, apply, self._slot_tensor(h))
        return h

    def opt_state(self, k: int) -> OptimizerState:
        st = OptimizerState(rule=self.rule, beta=self.beta, s=self.s)
        st.ys = self.ys.get(k)
        return st

    def synchronize(self) -> None:
        self.stream.synchronize()

    def read_scalar(self, h) -> float:
        return float(self._chunks[h[0]][h[1]].item())

    def read_scalars(self, pairs):
        self.stream.synchronize()
        host = [c.cpu().numpy() for c in self._chunks]
        out = []
        for lh, gh in pairs:
            lv = None if lh is None else float(host[lh[0]][lh[1]])
            gv = float(host[gh[0]][gh[1]])
            out.append((lv, gv))
        return out


def eval_forward(model, x: np.ndarray) -> np.ndarray:
    """Host batch -> host logits through device blocks (binds temporary DeviceBlocks if needed)."""
    torch = torch_mod()
    device = require_cuda()
    stream = torch.cuda.current_stream(device)
    B = x.shape[0]
    h = pack_input(np.asarray(x), model.blocks[0].in_shape, device, stream)
    K = model.k
    for k, blk in enumerate(model.blocks):
        db = blk.dev
        if db is None or db.batch != B:
            db = DeviceBlock(blk, B, is_last=(k == K - 1), device=device, stream=stream)
        if k < K - 1:
            y = db.new_activation(db.out_elems)
            db.forward(h, y, record=False)
            h = y
        else:
            cp = _pad8(model.output_dim)
            with torch.cuda.stream(stream):
                logits = torch.empty(B * cp, dtype=torch.float32, device=device)
            db.forward(h, logits, record=False)
            stream.synchronize()
            return logits.view(B, cp)[:, : model.output_dim].double().cpu().numpy()
    raise L.DspError(1, "empty model")
