"""Device-side block runtime: one ``dsp_block_t`` (include/dsp_b200.h) per block.

PyTorch is plumbing here: it owns the device memory (workspace, fp32 master
params, grads, activation packets) and the streams; every FLOP runs in
``libdsp_b200.so``. There is no CPU fallback -- constructing a DeviceBlock
without CUDA or without the library raises ``B200Unavailable``.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib as L


def torch_mod():
    import torch

    return torch


def require_cuda(device=None):
    torch = torch_mod()
    if not torch.cuda.is_available():
        raise L.B200Unavailable("no CUDA device: the DSP B200 backend has no CPU fallback")
    L.load()
    dev = torch.device(device if device is not None else "cuda")
    major, minor = torch.cuda.get_device_capability(dev)
    if major < 10:
        raise L.B200Unavailable(f"device {dev} is sm_{major}{minor}; libdsp_b200.so targets sm_100a")
    return dev


def ptr(t) -> C.c_void_p:
    return C.c_void_p(t.data_ptr()) if t is not None else C.c_void_p(0)


def stream_ptr(stream) -> C.c_void_p:
    return C.c_void_p(stream.cuda_stream)


class DeviceBlock:
    """Owns a planned block, its workspace, fp32 params / grads (and the
    optimizer's ys vector when the SUM rule is used)."""

    def __init__(self, block, batch: int, is_last: bool, device=None, stream=None, dtype: int = L.DSP_DTYPE_BF16):
        torch = torch_mod()
        self.device = require_cuda(device)
        self.lib = L.load()
        self.dtype = dtype
        self.block = block
        self.batch = batch
        self.is_last = is_last
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        descs = block.layer_descs()
        h = C.c_void_p()
        L.check(self.lib.dsp_block_create(descs, len(descs), batch, dtype, int(is_last), C.byref(h)))
        self.h = h
        self.ws_bytes = int(self.lib.dsp_block_workspace_bytes(h))
        self.in_elems = int(self.lib.dsp_block_in_elems(h))
        self.out_elems = int(self.lib.dsp_block_out_elems(h))
        n = int(self.lib.dsp_block_param_count(h))
        if n != block.param_count:
            raise L.DspError(1, f"block {block.index}: library counts {n} params, layout says {block.param_count}")
        with torch.cuda.stream(self.stream):
            self.ws = torch.empty(max(self.ws_bytes, 1), dtype=torch.uint8, device=self.device)
            self.params = torch.tensor(np.asarray(block.params, dtype=np.float32), device=self.device)
            if self.params.numel() == 0:
                self.params = torch.zeros(1, device=self.device)
            self.grads = torch.zeros_like(self.params)
        L.check(self.lib.dsp_block_bind(h, ptr(self.ws), ptr(self.params), ptr(self.grads), stream_ptr(self.stream)))

    def make_twin(self) -> "DeviceBlock":
        """A forward twin (dsp_block_share_weights): same program, own workspace, this block's
        params and packed weights -- runs the fresh forward beside this block's recompute."""
        torch = torch_mod()
        tw = DeviceBlock.__new__(DeviceBlock)
        tw.device, tw.lib, tw.block, tw.batch, tw.is_last = self.device, self.lib, self.block, self.batch, False
        tw.dtype = self.dtype
        tw.stream = self.stream
        descs = self.block.layer_descs()
        h = C.c_void_p()
        L.check(self.lib.dsp_block_create(descs, len(descs), self.batch, self.dtype, 0, C.byref(h)))
        tw.h = h
        tw.ws_bytes = int(self.lib.dsp_block_workspace_bytes(h))
        tw.in_elems, tw.out_elems = self.in_elems, self.out_elems
        with torch.cuda.stream(self.stream):
            tw.ws = torch.empty(max(tw.ws_bytes, 1), dtype=torch.uint8, device=self.device)
        tw.params, tw.grads = self.params, self.grads
        L.check(self.lib.dsp_block_bind(h, ptr(tw.ws), ptr(tw.params), ptr(tw.grads), stream_ptr(self.stream)))
        L.check(self.lib.dsp_block_share_weights(h, self.h))
        return tw

    def __del__(self):
        h = getattr(self, "h", None)
        if h is not None and h.value:
            try:
                self.lib.dsp_block_destroy(h)
            except Exception:
                pass
            self.h = None

    # ---- parameters -------------------------------------------------------
    def read_params(self) -> np.ndarray:
        self.stream.synchronize()
        return self.params[: self.block.param_count].double().cpu().numpy()

    def write_params(self, value: np.ndarray) -> None:
        torch = torch_mod()
        src = torch.tensor(np.asarray(value, dtype=np.float32))
        with torch.cuda.stream(self.stream):
            self.params[: self.block.param_count].copy_(src, non_blocking=False)
        L.check(self.lib.dsp_block_pack(self.h, stream_ptr(self.stream)))

    # ---- step pieces --------------------------------------------------------
    def new_activation(self, n_elems: int, zero: bool = False):
        torch = torch_mod()
        dt = L.torch_storage(self.dtype)
        with torch.cuda.stream(self.stream):
            if zero:
                return torch.zeros(n_elems, dtype=dt, device=self.device)
            return torch.empty(n_elems, dtype=dt, device=self.device)

    def forward(self, x, y=None, record: bool = False, stream=None) -> None:
        st = stream_ptr(stream or self.stream)
        L.check(self.lib.dsp_block_forward(self.h, ptr(x), ptr(y), int(record), st))

    def loss(self, labels, loss_out, stream=None) -> None:
        L.check(self.lib.dsp_block_loss(self.h, ptr(labels), ptr(loss_out), stream_ptr(stream or self.stream)))

    def backward(self, upstream, grad_in, stream=None) -> None:
        L.check(self.lib.dsp_block_backward(self.h, ptr(upstream), ptr(grad_in), stream_ptr(stream or self.stream)))

    def update(self, rule: int, ys, lr: float, slr: float, beta: float, wd: float, apply: bool, grad_sq_out,
               stream=None) -> None:
        L.check(self.lib.dsp_block_update(self.h, rule, ptr(ys), C.c_double(lr), C.c_double(slr), C.c_double(beta),
                                          C.c_double(wd), int(apply), ptr(grad_sq_out),
                                          stream_ptr(stream or self.stream)))


    def update_adam(self, state, lr: float, b1: float, b2: float, eps: float, wd: float, apply: bool, grad_sq_out,
                    stream=None) -> None:
        L.check(self.lib.dsp_block_update_adam(self.h, ptr(state), C.c_double(lr), C.c_double(b1), C.c_double(b2),
                                               C.c_double(eps), C.c_double(wd), int(apply), ptr(grad_sq_out),
                                               stream_ptr(stream or self.stream)))

def pack_input(x_host: np.ndarray, shape: tuple, device, stream, dtype: int = L.DSP_DTYPE_BF16):
    """Host float batch (B, C*H*W) in (C,H,W) order -> padded NHWC device packet (storage dtype)."""
    torch = torch_mod()
    lib = L.load()
    B = x_host.shape[0]
    c, h, w = shape
    cp = (c + 7) // 8 * 8
    with torch.cuda.stream(stream):
        src = torch.from_numpy(np.ascontiguousarray(x_host, dtype=np.float32)).pin_memory()
        dev = src.to(device, non_blocking=True)
        out = torch.empty(B * h * w * cp, dtype=L.torch_storage(dtype), device=device)
    L.check(lib.dsp_pack_input(ptr(dev), ptr(out), B, c, h, w, cp, dtype, 1, stream_ptr(stream)))
    dev.record_stream(stream)
    return out


def unpack_output(t, batch: int, shape: tuple, stream, dtype: int = L.DSP_DTYPE_BF16) -> np.ndarray:
    """Padded NHWC device tensor -> host float64 (B, C*H*W) in (C,H,W) order."""
    torch = torch_mod()
    lib = L.load()
    c, h, w = shape
    cp = (c + 7) // 8 * 8
    with torch.cuda.stream(stream):
        out = torch.empty(batch * c * h * w, dtype=torch.float32, device=t.device)
    L.check(lib.dsp_unpack_output(ptr(t), ptr(out), batch, c, h, w, cp, dtype, 1, stream_ptr(stream)))
    stream.synchronize()
    return out.double().cpu().numpy().reshape(batch, c * h * w)
