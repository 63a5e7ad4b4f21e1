"""Optimizer surface (reference: optim.py:1-109) over the CUDA update kernels.

``LrSchedule`` / ``lr_at`` are host arithmetic identical to the reference
(the learning rate is a per-step scalar handed to the kernel). ``sgd_step``,
``sum_step`` and ``apply_update`` run on the device:

  * float64 inputs (numpy arrays or CUDA fp64 tensors) go through
    ``dsp_update_f64``, which reproduces the reference's IEEE operation order
    without FMA contraction -- results are bitwise equal to optim.py;
  * CUDA fp32 tensors (the engine's master weights) go through ``dsp_update_f32``.

The SUM state keeps ``ys`` on the device; ``y`` (written but never read by the
reference, optim.py:97) is materialised only on the float64 path.

``rule="adam"`` is this package's EXTENSION for BASELINE configs[2] (ResNet-110,
Adam): the reference rejects it (optim.py:70-71), so its parity is pinned only
against the restatement ``oracle/dsp_ref.py`` ``adam_step`` (bias-corrected
Adam, beta1 0.9, beta2 0.999, eps 1e-8; ``beta`` / ``s`` are unused by it).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib as L
from .runtime import ptr, require_cuda, torch_mod


class NonFiniteError(ArithmeticError):
    """An operation produced NaN or Inf (reference: tensor.py:23-24)."""


@dataclass
class LrSchedule:
    """Piecewise-constant schedule (optim.py:23-35)."""

    base: float
    decays: tuple = ()

    def __post_init__(self):
        if self.base <= 0:
            raise ValueError("base learning rate must be positive")
        for _, factor in self.decays:
            if factor <= 0:
                raise ValueError("decay factors must be positive")


def lr_at(schedule: LrSchedule, n: int) -> float:
    """base * every factor whose step has passed, multiplied in list order (optim.py:38-45)."""
    if n < 0:
        raise ValueError("step must be non-negative")
    lr = schedule.base
    for step, factor in schedule.decays:
        if n >= step:
            lr *= factor
    return lr


RULES = {"sgd": L.DSP_RULE_SGD, "sum": L.DSP_RULE_SUM, "adam": L.DSP_RULE_ADAM}


@dataclass
class OptimizerState:
    """Per-block update state (optim.py:58-83). ``ys`` lives on the device."""

    rule: str
    beta: float = 0.0
    s: float = 1.0
    y: object = None
    ys: object = None
    n: int = 0
    # adam (extension; unpinned against the reference, which rejects it)
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8
    m1: object = None
    m2: object = None

    def __post_init__(self):
        if self.rule not in RULES:
            raise ValueError(f"unknown optimizer rule: {self.rule!r}")
        if not (0.0 <= self.beta < 1.0):
            raise ValueError("beta must lie in [0, 1)")
        if self.s < 0.0:
            raise ValueError("s must be non-negative")

    @classmethod
    def for_params(cls, rule: str, x0, beta: float = 0.0, s: float = 1.0) -> "OptimizerState":
        st = cls(rule=rule, beta=beta, s=s)
        if rule == "sum":
            st.ys = _clone(x0)  # ys[0] = x[0]: first momentum correction is zero
            st.y = _clone(x0)
        elif rule == "adam":
            st.m1 = np.zeros_like(x0) if isinstance(x0, np.ndarray) else x0.new_zeros(x0.shape)
            st.m2 = _clone(st.m1)
        return st


def _clone(x):
    if isinstance(x, np.ndarray):
        return x.copy()
    return x.clone()


def _to_dev64(x):
    torch = torch_mod()
    if isinstance(x, np.ndarray):
        return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64)).to(require_cuda()), True
    if x.dtype != torch.float64:
        raise TypeError("float64 path expects float64 tensors")
    return x, False


def _update64(rule: int, x, g, ys, y, lr: float, slr: float, beta: float):
    """Device fp64 update; returns (x_new, ys_new, y_new) in the caller's container type."""
    torch = torch_mod()
    xd, host = _to_dev64(x)
    gd, _ = _to_dev64(g)
    if not bool(torch.isfinite(gd).all()):
        raise NonFiniteError("non-finite gradient in update")
    xo = xd.clone()
    ysd = _to_dev64(ys)[0].clone() if ys is not None else None
    yd = torch.empty_like(xd) if ys is not None else None
    stream = torch.cuda.current_stream()
    L.check(L.load().dsp_update_f64(rule, xo.numel(), ptr(xo), ptr(gd), ptr(ysd), ptr(yd), C.c_double(lr),
                                    C.c_double(slr), C.c_double(beta), C.c_double(0.0), None,
                                    C.c_void_p(stream.cuda_stream)))
    if host:
        cv = lambda t: None if t is None else t.cpu().numpy()  # noqa: E731
        return cv(xo), cv(ysd), cv(yd)
    return xo, ysd, yd


def sgd_step(x, g, lr: float):
    """x - lr*g on the device (optim.py:48-55), bitwise equal to the reference in fp64."""
    if tuple(np.shape(x)) != tuple(np.shape(g)):
        raise ValueError(f"shape mismatch: x {np.shape(x)}, g {np.shape(g)}")
    if lr <= 0:
        raise ValueError("learning rate must be positive")
    out, _, _ = _update64(L.DSP_RULE_SGD, x, g, None, None, lr, lr, 0.0)
    return out


def sum_step(state: OptimizerState, x, g, lr: float):
    """Unified momentum (optim.py:86-99) on the device."""
    if state.rule != "sum" or state.ys is None:
        raise RuntimeError("momentum state not initialized; use OptimizerState.for_params")
    out, ys, y = _update64(L.DSP_RULE_SUM, x, g, state.ys, state.y, lr, state.s * lr, state.beta)
    state.ys = ys
    state.y = y
    return out


def adam_step(state: OptimizerState, x, g, lr: float):
    """Bias-corrected Adam on the device (extension; oracle/dsp_ref.py adam_step, same op order).

    Float64 inputs are bitwise equal to the restatement: bc_i = 1 - beta_i**t is formed here
    exactly as the oracle forms it and handed to ``dsp_update_adam_f64``."""
    if state.rule != "adam" or state.m1 is None:
        raise RuntimeError("adam state not initialized; use OptimizerState.for_params")
    torch = torch_mod()
    xd, host = _to_dev64(x)
    gd, _ = _to_dev64(g)
    if not bool(torch.isfinite(gd).all()):
        raise NonFiniteError("non-finite gradient in update")
    xo = xd.clone()
    m1 = _to_dev64(state.m1)[0].clone()
    m2 = _to_dev64(state.m2)[0].clone()
    t = state.n + 1
    bc1 = 1.0 - state.beta1 ** t
    bc2 = 1.0 - state.beta2 ** t
    stream = torch.cuda.current_stream()
    L.check(L.load().dsp_update_adam_f64(xo.numel(), ptr(xo), ptr(gd), ptr(m1), ptr(m2), None, C.c_double(bc1),
                                         C.c_double(bc2), C.c_double(lr), C.c_double(state.beta1),
                                         C.c_double(state.beta2), C.c_double(state.eps), C.c_double(0.0), None,
                                         C.c_void_p(stream.cuda_stream)))
    if host:
        xo, m1, m2 = xo.cpu().numpy(), m1.cpu().numpy(), m2.cpu().numpy()
    state.m1, state.m2 = m1, m2
    return xo


def apply_update(state: OptimizerState, x, g, lr: float):
    """Advance one step under the state's rule (optim.py:102-109)."""
    if state.rule == "sgd":
        out = sgd_step(x, g, lr)
    elif state.rule == "sum":
        out = sum_step(state, x, g, lr)
    else:
        out = adam_step(state, x, g, lr)
    state.n += 1
    return out
