"""``NativeEngine``: the DSP train step through the engine-level C-ABI.

The whole schedule (rings, zero prefill, per-phase CUDA graphs, optimizer, log)
runs inside ``libdsp_b200.so`` (csrc/engine.cu); this wrapper only builds the
``dsp_config_t`` from a ``Model`` + ``PipelineConfig`` and converts host arrays.
It is the single-GPU drop-in for the reference's serial ``TrainEngine``
(/root/reference/pkg/src/stalepipe/pipeline.py:451-620) that a C, cgo or ctypes
caller would bind; ``TrainEngine(backend="b200")`` stays the
Python-orchestrated path (multi-GPU placement, arbitrary data iterators).
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib as L
from .optim import RULES, LrSchedule
from .pipeline import LogRecord, PipelineConfig, TrainLog


class NativeEngine:
    def __init__(self, model, config: PipelineConfig, batch: int, schedule: LrSchedule, rule: str = "sgd",
                 beta: float = 0.0, s: float = 1.0, weight_decay: float = 0.0, use_graphs: bool = True,
                 device: int = 0, precision: str = "bf16", devices=None):
        """devices: optional CUDA ordinal per block (one GPU per block, packets stored into the
        consumer's ring over NVLink); default: every block on `device`."""
        lib = L.load()
        self.lib = lib
        self.model = model
        self.config = config
        self.B = batch
        K = config.k
        if model.k != K:
            raise ValueError(f"model has {model.k} blocks, config {K}")
        if K > L.DSP_MAX_BLOCKS:
            raise ValueError(f"at most {L.DSP_MAX_BLOCKS} blocks")
        cfg = L.EngineConfig()
        cfg.K = K
        for k in range(K):
            cfg.p[k], cfg.m[k] = config.p[k], config.m[k]
        cfg.warmup = L.DSP_WARMUP_DISCARD if config.warmup == "discard_warmup_updates" else L.DSP_WARMUP_FAITHFUL
        cfg.batch = batch
        cfg.dtype = L.storage_dtype(precision)
        c, h, w = model.blocks[0].in_shape
        cfg.in_c, cfg.in_h, cfg.in_w = c, h, w
        cfg.num_classes = model.output_dim
        descs = [blk.layer_descs() for blk in model.blocks]
        flat = (L.LayerDesc * sum(len(d) for d in descs))()
        i = 0
        for k, d in enumerate(descs):
            cfg.n_layers[k] = len(d)
            for e in d:
                flat[i] = e
                i += 1
        self._layers = flat  # keep alive for the call
        cfg.layers = C.cast(flat, C.POINTER(L.LayerDesc))
        cfg.use_graphs = int(use_graphs)
        cfg.device = device
        if devices is not None:
            if len(devices) != K:
                raise ValueError(f"devices names {len(devices)} devices for {K} blocks")
            cfg.multi_device = 1
            for k, d in enumerate(devices):
                cfg.device_of_block[k] = int(d)
        # ring depth and graph horizon exactly as csrc/engine.cu derives them (steps >= horizon
        # replay per-phase graphs; the first replay of each of the ring phases captures it)
        p, m = config.p, config.m
        q = [0] + [m[k - 1] - p[k - 1] - m[k] for k in range(1, K)]
        cum = int(sum(p[:K - 1]))
        life = max([m[0] + 1] + [p[k] + m[k + 1] + 1 for k in range(K - 1)] + [q[k] + 1 for k in range(1, K)]
                   + [cum + m[K - 1] + 1])
        self.ring = life + 1
        self.horizon = cum + max(m) + max(p) + max(q) + 1
        h = C.c_void_p()
        L.check(lib.dsp_create(C.byref(cfg), C.byref(h)))
        self.h = h
        for k, blk in enumerate(model.blocks):
            src = np.ascontiguousarray(blk.params, dtype=np.float64)
            L.check(lib.dsp_set_params(h, k, src.ctypes.data_as(C.c_void_p), src.size, 0))
        steps = np.array([d[0] for d in schedule.decays], dtype=np.int64)
        facs = np.array([d[1] for d in schedule.decays], dtype=np.float64)
        L.check(lib.dsp_set_optimizer(h, RULES[rule], beta, s, weight_decay, schedule.base,
                                      steps.ctypes.data_as(C.POINTER(C.c_int64)),
                                      facs.ctypes.data_as(C.POINTER(C.c_double)), len(steps)))
        if rule == "adam":  # extension: the oracle's fixed Adam hyper-parameters
            from .optim import OptimizerState

            ad = OptimizerState(rule="adam")
            L.check(lib.dsp_set_adam(h, ad.beta1, ad.beta2, ad.eps))

    def __del__(self):
        h = getattr(self, "h", None)
        if h is not None and h.value:
            self.lib.dsp_destroy(h)
            self.h = None

    def run_batches(self, x: np.ndarray, labels: np.ndarray) -> None:
        """len(x) DSP steps on host batches x [n, B, C*H*W] (float32) and labels [n, B] (int64)."""
        x = np.ascontiguousarray(x, dtype=np.float32).reshape(len(x), self.B, -1)
        labels = np.ascontiguousarray(labels, dtype=np.int64).reshape(len(x), self.B)
        D = int(np.prod(self.model.blocks[0].in_shape))
        if x.shape[2] != D:
            from .blocks import ShapeError

            raise ShapeError(f"batch width {x.shape[2]} does not match the model input {self.model.blocks[0].in_shape}")
        L.check(self.lib.dsp_run(self.h, len(x), x.ctypes.data_as(C.POINTER(C.c_float)),
                                 labels.ctypes.data_as(C.POINTER(C.c_int64))))

    def run(self, n_steps: int, data_stream) -> None:
        """n_steps steps drawing (x, labels) batches from an iterator, like TrainEngine.run."""
        for _ in range(n_steps):
            x, lab = next(data_stream)
            self.run_batches(np.asarray(x)[None], np.asarray(lab)[None])

    @property
    def steps_done(self) -> int:
        return int(self.lib.dsp_steps_done(self.h))

    @property
    def log(self) -> TrainLog:
        n = C.c_size_t()
        L.check(self.lib.dsp_read_log(self.h, None, 0, C.byref(n)))
        recs = (L.LogRecordC * max(n.value, 1))()
        L.check(self.lib.dsp_read_log(self.h, recs, n.value, C.byref(n)))
        out = []
        for r in recs[: n.value]:
            out.append(LogRecord(step=int(r.step), block=int(r.block), batch_index=int(r.batch_index),
                                 grad_norm=float(r.grad_norm), loss=float(r.loss) if r.has_loss else None))
        return TrainLog(out)

    def params(self, k: int) -> np.ndarray:
        n = int(self.lib.dsp_param_count(self.h, k))
        out = np.empty(n, dtype=np.float64)
        L.check(self.lib.dsp_get_params(self.h, k, out.ctypes.data_as(C.POINTER(C.c_double)), n))
        return out

    def realized_staleness(self) -> list:
        """Per block, the constant lag (step - cum_p[k]) - batch_index (pipeline.py:682-694)."""
        cum = np.concatenate([[0], np.cumsum(self.config.p)])
        lags = {}
        for r in self.log.records:
            if r.batch_index >= 0:
                lags.setdefault(r.block, set()).add(r.step - int(cum[r.block]) - r.batch_index)
        out = []
        for k in range(self.config.k):
            lag = lags.get(k, {self.config.m[k]})
            if len(lag) != 1:
                raise AssertionError(f"block {k}: non-constant staleness {sorted(lag)}")
            out.append(lag.pop())
        return out
