"""ctypes binding of ``libdsp_b200.so`` (the C ABI in include/dsp_b200.h).

This is the only way the package reaches its CUDA kernels. There is no CPU
fallback: if the library is missing or no CUDA device is present, the
product path raises ``B200Unavailable`` instead of silently running elsewhere.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

LIB_PATH = Path(os.environ.get("DSP_B200_LIB", Path(__file__).resolve().parent / "libdsp_b200.so"))

DSP_DTYPE_BF16 = 0
DSP_OK = 0
DSP_E_INVALID = 1
DSP_E_CUDA = 2
DSP_E_STATE = 3
DSP_E_NONFINITE = 4
DSP_GRAPH_NODE_PRIORITY = 1
DSP_NONFINITE_LOSS = 1
DSP_NONFINITE_GRAD = 2
DSP_DTYPE_F32 = 1
# engine precisions (storage dtype + tensor-core arithmetic):
#   "bf16": bf16 activations / weight shadow, kind::f16 MMA -- the performance mode;
#   "fp32": fp32 activations / weight shadow, 3xTF32 on kind::tf32 (each operand split into a
#           tf32 hi part and an fp32 remainder, three MMAs) -- fp32-faithful, the parity mode.
# Accumulation, BatchNorm statistics, master weights and optimizer state are fp32 in both.
PRECISIONS = {"bf16": DSP_DTYPE_BF16, "fp32": DSP_DTYPE_F32}


def storage_dtype(precision: str) -> int:
    if precision not in PRECISIONS:
        raise ValueError(f"precision must be one of {sorted(PRECISIONS)}, got {precision!r}")
    return PRECISIONS[precision]


def torch_storage(dtype_code: int):
    import torch

    return torch.float32 if dtype_code == DSP_DTYPE_F32 else torch.bfloat16

DSP_IGEMM_FPROP = 0
DSP_IGEMM_DGRAD = 1
DSP_IGEMM_WGRAD = 2

DSP_LAYER_DENSE = 0
DSP_LAYER_RELU = 1
DSP_LAYER_TANH = 2
DSP_LAYER_CONV_BN_RELU = 10
DSP_LAYER_BASIC_UNIT = 11
DSP_LAYER_BOTTLENECK = 12
DSP_LAYER_AVGPOOL = 13
DSP_LAYER_MAXPOOL = 14

DSP_RULE_SGD = 0
DSP_RULE_SUM = 1
DSP_RULE_ADAM = 2  # extension (BASELINE configs[2]); the reference rejects 'adam'


class B200Unavailable(RuntimeError):
    """The CUDA library or a CUDA device is missing; there is no fallback."""


class DspError(RuntimeError):
    def __init__(self, code: int, message: str):
        super().__init__(f"[dsp error {code}] {message}")
        self.code = code


class ConvGeom(C.Structure):
    _fields_ = [(n, C.c_int32) for n in ("nimg", "H", "W", "C", "P", "Q", "K", "R", "S", "stride", "pad")]


class BnbTarget(C.Structure):
    _fields_ = [("y", C.c_void_p), ("stat", C.c_void_p), ("gamma", C.c_void_p), ("dgamma", C.c_void_p),
                ("dbeta", C.c_void_p), ("coef", C.c_void_p)]


class IgemmArgs(C.Structure):
    _fields_ = [
        ("geom", ConvGeom),
        ("M", C.c_int32), ("N", C.c_int32), ("Kd", C.c_int32),
        ("A", C.c_void_p), ("B", C.c_void_p), ("D", C.c_void_p),
        ("ldd", C.c_int32), ("out_f32", C.c_int32),
        ("residual", C.c_void_p), ("bias", C.c_void_p), ("stats", C.c_void_p),
        ("kb_per_split", C.c_int32),
        ("n_valid", C.c_int32),
        ("stat_out", C.c_void_p), ("gamma", C.c_void_p), ("beta", C.c_void_p), ("sem", C.c_void_p),
        ("trace", C.c_void_p),
        ("bnb_mask", C.c_void_p), ("bnb_count", C.c_int32), ("bnb_c_real", C.c_int32),
        ("bnb", BnbTarget * 2),
        ("B_t", C.c_void_p),
        ("bnb_mask_bits", C.c_void_p),
    ]


IGEMM_MAX_CTAS = 444
IGEMM_SEM_INTS = 1024  # DSP_IGEMM_SEM_INTS


class LayerDesc(C.Structure):
    _fields_ = [
        ("kind", C.c_int32),
        ("in_c", C.c_int32), ("in_h", C.c_int32), ("in_w", C.c_int32),
        ("out_c", C.c_int32), ("out_h", C.c_int32), ("out_w", C.c_int32),
        ("mid_c", C.c_int32), ("stride", C.c_int32), ("ksize", C.c_int32),
        ("bias", C.c_int32), ("reserved", C.c_int32),
        ("param_offset", C.c_int64), ("param_count", C.c_int64),
    ]


DSP_MAX_BLOCKS = 8
DSP_WARMUP_FAITHFUL = 0
DSP_WARMUP_DISCARD = 1


class EngineConfig(C.Structure):
    _fields_ = [
        ("K", C.c_int32),
        ("p", C.c_int32 * DSP_MAX_BLOCKS), ("m", C.c_int32 * DSP_MAX_BLOCKS),
        ("warmup", C.c_int32), ("batch", C.c_int32), ("dtype", C.c_int32),
        ("in_c", C.c_int32), ("in_h", C.c_int32), ("in_w", C.c_int32),
        ("num_classes", C.c_int32),
        ("n_layers", C.c_int32 * DSP_MAX_BLOCKS),
        ("layers", C.POINTER(LayerDesc)),
        ("use_graphs", C.c_int32), ("device", C.c_int32),
        ("multi_device", C.c_int32), ("device_of_block", C.c_int32 * DSP_MAX_BLOCKS),
    ]


class LogRecordC(C.Structure):
    _fields_ = [("step", C.c_int64), ("block", C.c_int32), ("has_loss", C.c_int32), ("batch_index", C.c_int64),
                ("loss", C.c_double), ("grad_norm", C.c_double)]


# name -> (restype, argtypes); mirrors include/dsp_b200.h exactly
_P = C.c_void_p
_SIGNATURES = {
    "dsp_igemm": (C.c_int, [C.c_int, C.c_int, C.POINTER(IgemmArgs), C.c_int, _P]),
    "dsp_update_f64": (C.c_int, [C.c_int, C.c_int64, _P, _P, _P, _P, C.c_double, C.c_double, C.c_double,
                                 C.c_double, _P, _P]),
    "dsp_update_f32": (C.c_int, [C.c_int, C.c_int64, _P, _P, _P, C.c_double, C.c_double, C.c_double,
                                 C.c_double, _P, _P]),
    "dsp_block_create": (C.c_int, [C.POINTER(LayerDesc), C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(_P)]),
    "dsp_block_destroy": (None, [_P]),
    "dsp_block_workspace_bytes": (C.c_int64, [_P]),
    "dsp_block_in_elems": (C.c_int64, [_P]),
    "dsp_block_out_elems": (C.c_int64, [_P]),
    "dsp_block_param_count": (C.c_int64, [_P]),
    "dsp_block_bind": (C.c_int, [_P, _P, _P, _P, _P]),
    "dsp_block_pack": (C.c_int, [_P, _P]),
    "dsp_block_share_weights": (C.c_int, [_P, _P]),
    "dsp_block_forward": (C.c_int, [_P, _P, _P, C.c_int, _P]),
    "dsp_block_loss": (C.c_int, [_P, _P, _P, _P]),
    "dsp_block_backward": (C.c_int, [_P, _P, _P, _P]),
    "dsp_update_adam_f64": (C.c_int, [C.c_int64, _P, _P, _P, _P, _P, C.c_double, C.c_double, C.c_double,
                                      C.c_double, C.c_double, C.c_double, C.c_double, _P, _P]),
    "dsp_update_adam_f32": (C.c_int, [C.c_int64, _P, _P, _P, _P, _P, C.c_double, C.c_double, C.c_double,
                                      C.c_double, C.c_double, C.c_double, C.c_double, _P, _P]),
    "dsp_block_update_adam": (C.c_int, [_P, _P, C.c_double, C.c_double, C.c_double, C.c_double, C.c_double,
                                        C.c_int, _P, _P]),
    "dsp_set_adam": (C.c_int, [_P, C.c_double, C.c_double, C.c_double]),
    "dsp_block_update": (C.c_int, [_P, C.c_int, _P, C.c_double, C.c_double, C.c_double, C.c_double, C.c_int,
                                   _P, _P]),
    "dsp_block_nonfinite": (C.c_int, [_P, C.c_int, C.POINTER(C.c_int), _P]),
    "dsp_pack_input": (C.c_int, [_P, _P, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _P]),
    "dsp_unpack_output": (C.c_int, [_P, _P, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _P]),
    "dsp_last_error": (C.c_char_p, []),
    "dsp_abi_version": (C.c_int, []),
    "dsp_launch_count": (C.c_int64, []),
    "dsp_graph_instantiate": (C.c_int, [C.c_void_p, C.c_int, C.POINTER(C.c_void_p)]),
    "dsp_graph_launch": (C.c_int, [C.c_void_p, C.c_void_p]),
    "dsp_graph_destroy": (C.c_int, [C.c_void_p]),
    "dsp_probe_arm": (C.c_int, [C.c_int, C.c_int, C.c_int64, C.POINTER(C.c_void_p), C.c_int]),
    "dsp_probe_reset": (C.c_int, []),
    "dsp_create": (C.c_int, [C.POINTER(EngineConfig), C.POINTER(C.c_void_p)]),
    "dsp_set_params": (C.c_int, [_P, C.c_int, _P, C.c_size_t, C.c_int]),
    "dsp_get_params": (C.c_int, [_P, C.c_int, C.POINTER(C.c_double), C.c_size_t]),
    "dsp_param_count": (C.c_size_t, [_P, C.c_int]),
    "dsp_set_optimizer": (C.c_int, [_P, C.c_int, C.c_double, C.c_double, C.c_double, C.c_double,
                                    C.POINTER(C.c_int64), C.POINTER(C.c_double), C.c_int]),
    "dsp_run": (C.c_int, [_P, C.c_int, C.POINTER(C.c_float), C.POINTER(C.c_int64)]),
    "dsp_read_log": (C.c_int, [_P, C.POINTER(LogRecordC), C.c_size_t, C.POINTER(C.c_size_t)]),
    "dsp_steps_done": (C.c_int64, [_P]),
    "dsp_destroy": (None, [_P]),
    "dsp_device_sleep": (C.c_int, [C.c_int64, _P]),
    "dsp_synth_batch": (C.c_int, [C.c_uint64, C.c_int64, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                  C.c_int, _P, C.POINTER(C.c_int64), _P]),
}

_lib = None


def exported_symbols() -> list[str]:
    return list(_SIGNATURES)


def load(require_symbols: bool = True):
    """Load libdsp_b200.so (no device needed). Raises B200Unavailable if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise B200Unavailable(
            f"{LIB_PATH} is missing: run __graft_entry__.build() (nvcc, sm_100a). "
            "There is no CPU fallback for the DSP B200 path."
        )
    lib = C.CDLL(os.fspath(LIB_PATH))
    for name, (res, args) in _SIGNATURES.items():
        try:
            fn = getattr(lib, name)
        except AttributeError:
            if require_symbols:
                raise B200Unavailable(f"{LIB_PATH} does not export {name}")
            continue
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(rc: int) -> None:
    if rc != 0:
        msg = load().dsp_last_error()
        msg = msg.decode() if msg else "unknown"
        if rc == DSP_E_NONFINITE:  # the reference's NonFiniteError (tensor.py:34-37, optim.py:53 / 89)
            from .optim import NonFiniteError

            raise NonFiniteError(msg)
        raise DspError(rc, msg)


def lib():
    return load()
