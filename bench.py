#!/usr/bin/env python
"""bench.py -- DSP training throughput on B200 (BASELINE.json metric).

Headline workload (the largest BASELINE config that fits one GPU, configs[4]): ResNet-50,
synthetic ImageNet-shaped 224x224x3 batches of 256, DSP with K=4 blocks (K=8 at 8 GPUs), queue
config p_k=1, m_k=2(K-1-k), SUM momentum beta=0.9 s=1, lr 0.1, weight decay 5e-4,
bf16 storage / fp32 accumulate on tcgen05 tensor cores.  One "step" = one DSP iteration of every
block (fresh forward, recompute, backward, update) = one batch through the pipeline.  The same
line carries the metric's other parts: the K=1 plain-BP baseline on the same model and batch
(``k1_bp``), the per-conv tensor-pipe fraction of peak (``conv_tensor_pipe``) and configs[1]
(ResNet-56, K=4, B=128) as a second workload (``resnet56``).

  python bench.py [--gpus N --steps K --warmup W]       # this repo's B200 engine
  python bench.py --impl reference [...]                  # the CPU oracle (reference algorithm)
  python bench.py --model resnet56                        # configs[1] as the headline instead

--gpus N without torchrun re-launches itself under torch.distributed.run (one rank per GPU).
Prints ONE JSON line on rank 0. See DESIGN.md §5 for every field.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "training samples/sec (device-timed) at K=1/2/4/8 B200 vs BP; conv tensor-pipe % of peak"
UNIT = "samples/s"
L2_BYTES = 126 * 1024 * 1024
DEPTH = 56
CLASSES = 10
IN_SHAPE = (3, 32, 32)

# --model: BASELINE.json configs this bench can run (configs[4], ResNet-50, is the default bench line).
# configs[2] asks for Adam, which the reference rejects (optim.py:70-71): it runs this package's
# rule="adam" extension, checked against the oracle restatement only (tests/test_optim_gpu.py).
MODELS = {
    "resnet56": dict(cfg=1, depth=56, classes=10, in_shape=(3, 32, 32), batch=128,
                     desc="ResNet-56 DSP K={K}, synthetic CIFAR-10-shaped 32x32x3, batch {B}"),
    "resnet110": dict(cfg=2, depth=110, classes=10, in_shape=(3, 32, 32), batch=128, k=8,
                      opt=dict(rule="adam", beta=0.0, s=1.0, lr=1e-3),
                      desc="ResNet-110 DSP K={K}, synthetic CIFAR-10-shaped 32x32x3, batch {B}, Adam"),
    "resnet164": dict(cfg=3, depth=164, classes=100, in_shape=(3, 32, 32), batch=256,
                      desc="ResNet-164 (bottleneck) DSP K={K}, synthetic CIFAR-100-shaped 32x32x3, batch {B}"),
    "resnet50": dict(cfg=4, depth=50, classes=1000, in_shape=(3, 224, 224), batch=256,
                     desc="ResNet-50 DSP K={K}, synthetic ImageNet-shaped 224x224x3, batch {B}, bf16 tensor-core convs"),
}


def select_model(args):
    """Point the module-level workload constants at --model (default: configs[4], ResNet-50)."""
    global DEPTH, CLASSES, IN_SHAPE
    m = MODELS[args.model]
    DEPTH, CLASSES, IN_SHAPE = m["depth"], m["classes"], m["in_shape"]
    if not args.batch:
        args.batch = m["batch"]


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--batch", type=int, default=0, help="default: the config's batch (128 / 256)")
    ap.add_argument("--model", default="resnet50", choices=sorted(MODELS))
    ap.add_argument("--k", type=int, default=0, help="DSP blocks (default 4, or 8 when --gpus 8)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cuts", default="", help="block boundaries (layer indices), default FLOP-balanced")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-extras", action="store_true",
                    help="skip k1_bp / k_sweep_1gpu / conv_tensor_pipe / the resnet56 line")
    ap.add_argument("--precision", default="bf16", choices=["bf16", "fp32"])
    return ap.parse_args()


SUM_OPT = dict(rule="sum", beta=0.9, s=1.0, lr=0.1)


def opt_of(args) -> dict:
    """Optimizer of the --model config: SUM momentum, or Adam for configs[2]."""
    return MODELS[args.model].get("opt", SUM_OPT)


def opt_desc(args) -> str:
    o = opt_of(args)
    if o["rule"] == "adam":
        return f"Adam b1=0.9 b2=0.999 eps=1e-8 (extension), lr {o['lr']}, wd 5e-4"
    return f"SUM momentum beta={o['beta']} s={o['s']}, lr {o['lr']}, wd 5e-4"


def blocks_for(args) -> int:
    if args.k:
        return args.k
    return MODELS[args.model].get("k", 8 if args.gpus >= 8 else 4)


def workload(args):
    import paper_1909_02625_b200 as P

    K = blocks_for(args)
    if args.model == "resnet50":
        layers = P.resnet50_layers(CLASSES, IN_SHAPE)
    elif args.model == "resnet164":
        layers = P.resnet_cifar_bottleneck_layers(DEPTH, CLASSES)
    else:
        layers = P.resnet_cifar_layers(DEPTH, CLASSES)
    if getattr(args, "cuts", ""):
        bounds = [int(v) for v in args.cuts.split(",")]
    else:
        bounds = P.flop_balanced_boundaries(layers, K) if K > 1 else []
    cfg = P.default_queue_config(K)
    return layers, bounds, cfg


def config_dict_for(model: str, K: int, batch: int, world: int, opt: str = "") -> dict:
    m = MODELS[model]
    return {"workload": m["desc"].format(K=K, B=batch), "baseline_config": m["cfg"],
            "model": model if model == "resnet50" else f"{model}-cifar", "global_batch": batch, "k_blocks": K,
            "queues": "p_k=1, m_k=2(K-1-k)",
            "optimizer": opt or f"SUM momentum beta={SUM_OPT['beta']} s={SUM_OPT['s']}, lr {SUM_OPT['lr']}, wd 5e-4",
            "parallelism": f"dsp-pipeline k{K} over {world} gpu(s)",
            "l2": "L2 flushed (256 MiB write) between timed steps; step working set > L2"}


def config_dict(args, K, world):
    d = config_dict_for(args.model, K, args.batch, world, opt_desc(args))
    d["cuts"] = ([int(c) for c in args.cuts.split(",")] if args.cuts
                 else "FLOP-balanced residual-unit cuts (SURVEY 8)")
    return d


# ------------------------------------------------------------------ clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()
            self.thread.join(timeout=1)
        return False

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            for name, val in zip(names, r[4:8]):
                if val.strip().lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.rows)}


class NvmlClockSampler:
    """SM clocks + clock-event reasons sampled in-process through NVML every 5 ms while the
    timed region runs (the nvidia-smi sampler's ~1 s start-up outlasts a 50 ms timed region,
    leaving it without samples); falls back to ClockSampler when NVML is absent."""

    PERIOD_S = 0.005

    def __init__(self, index: int):
        self.index = index
        self.rows = []  # (sm_mhz, max_mhz, reasons bitmask)
        self.fallback = None
        self._stop = threading.Event()

    def __enter__(self):
        try:
            import pynvml as N

            N.nvmlInit()
            self.N = N
            self.h = None
            try:  # the CUDA device by UUID (NVML indices ignore CUDA_VISIBLE_DEVICES)
                import torch

                uuid = str(torch.cuda.get_device_properties(self.index).uuid)
                self.h = N.nvmlDeviceGetHandleByUUID(uuid if uuid.startswith("GPU-") else "GPU-" + uuid)
            except Exception:
                self.h = N.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = N.nvmlDeviceGetMaxClockInfo(self.h, N.NVML_CLOCK_SM)
            self._sample()  # one sample at the region start
            self.thread = threading.Thread(target=self._loop, daemon=True)
            self.thread.start()
        except Exception:
            self.N = None
            self.fallback = ClockSampler(self.index).__enter__()
        return self

    def _sample(self):
        N = self.N
        self.rows.append((N.nvmlDeviceGetClockInfo(self.h, N.NVML_CLOCK_SM), self.max_mhz,
                          N.nvmlDeviceGetCurrentClocksEventReasons(self.h)))

    def _loop(self):
        while not self._stop.wait(self.PERIOD_S):
            try:
                self._sample()
            except Exception:
                return

    def __exit__(self, *exc):
        if self.fallback is not None:
            return self.fallback.__exit__(*exc)
        self._stop.set()
        self.thread.join(timeout=1)
        return False

    def summary(self):
        if self.fallback is not None:
            return self.fallback.summary()
        N = self.N
        bits = {"hw_slowdown": N.nvmlClocksEventReasonHwSlowdown,
                "hw_thermal_slowdown": N.nvmlClocksEventReasonHwThermalSlowdown,
                "sw_thermal_slowdown": N.nvmlClocksEventReasonSwThermalSlowdown,
                "sw_power_cap": N.nvmlClocksEventReasonSwPowerCap}
        reasons = sorted({name for _, _, r in self.rows for name, b in bits.items() if r & b})
        return {"sm_mhz": statistics.median(r[0] for r in self.rows), "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(self.rows), "source": "nvml, 5 ms period over the timed region"}


# ------------------------------------------------------------------ CPU oracle (reference algorithm)
def cpu_oracle_steps(args, steps: int, warmup: int, batch: int):
    """Time the float64 CPU restatement of the reference DSP step (oracle/)."""
    import oracle.dsp_ref as R

    layers, bounds, cfg = workload(args)
    olayers = [R.LayerSpec(s.kind, s.in_dim, s.out_dim, s.bias, tuple(s.in_shape), s.out_c, s.mid_c, s.stride,
                           s.ksize) for s in layers]
    om = R.build_model(olayers, bounds)
    R.init_params(om, 0)
    pool = R.synthetic_batches(4, batch, IN_SHAPE, CLASSES, seed=0)
    eng = R.Engine(om, R.validate_config(cfg.p, cfg.m), R.cycle(pool), R.LrSchedule(opt_of(args)["lr"]),
                   rule=opt_of(args)["rule"], beta=opt_of(args)["beta"], weight_decay=5e-4)
    eng.run(warmup)
    t0 = time.perf_counter()
    r0 = os.times()
    eng.run(steps)
    dt = time.perf_counter() - t0
    r1 = os.times()
    cpu_s = (r1.user - r0.user) + (r1.system - r0.system)
    return batch * steps / dt, dt, cpu_s


def threads_used() -> int:
    try:
        from threadpoolctl import threadpool_info

        n = [i.get("num_threads", 1) for i in threadpool_info() if i.get("user_api") == "blas"]
        return int(max(n)) if n else 1
    except Exception:
        return os.cpu_count() or 1


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    K = blocks_for(args)
    big = IN_SHAPE[1] > 32
    sub = min(args.batch, 2 if big else 32)
    steps = max(1, args.steps)
    warm = max(1, min(args.warmup, 1 if big else 3))
    # bound the run to a few minutes: ~2.7 s per ResNet-56 K=4 step at batch 32 on 8 cores
    budget_s = 150.0
    est = sub * {"resnet56": 0.085, "resnet110": 0.17, "resnet164": 0.17, "resnet50": 3.0}.get(args.model, 0.1)
    if (steps + warm) * est > budget_s:
        steps = max(1, int(budget_s / est) - warm)
    v, dt, cpu_s = cpu_oracle_steps(args, steps, warm, sub)
    cores = threads_used()
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus, "steps": steps,
            "warmup": warm, "ms_per_step": 1000.0 * dt / steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {**config_dict(args, K, 1), "global_batch": sub, "workload_global_batch": args.batch,
                       "sample": f"each timed step runs the DSP step on a {sub}-sample sub-batch of the workload's "
                                 f"{args.batch}; samples/s counts the {sub} samples"},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "port",
                             "sample": f"oracle/dsp_ref.py float64 DSP step (reference algorithm, CPU restatement), "
                                       f"ResNet-{DEPTH} K={K}, {steps} timed steps of a {sub}-sample sub-batch "
                                       f"after {warm} warmup; cpu/wall={cpu_s / dt:.2f}"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ B200 arm
def ncu_traffic(model: str = "resnet56"):
    """DRAM bytes (read + write) per launch of the roofline kernel from the committed
    ncu --set full capture (profiles/ncu_roofline[_resnet50].json), or None."""
    name = "ncu_roofline_resnet50.json" if model == "resnet50" else "ncu_roofline.json"
    try:
        with open(os.path.join(ROOT, "profiles", name)) as f:
            d = json.load(f)
        return int(d["dram_bytes_read"]) + int(d["dram_bytes_write"])
    except Exception:
        return None


def roofline_spec(model: str, batch: int) -> dict:
    """The dominant conv of the model's step and how its roofline is read:
    CIFAR stage-1 3x3 convs are HBM/latency-bound (bytes), ResNet-50's stage-3 3x3 is
    tensor-bound (FLOPs)."""
    if model == "resnet50":
        H, C_, K = 14, 256, 256
        return dict(nimg=batch, H=H, C=C_, K=K, bound="tensor", M=batch * H * H, Kd=9 * C_,
                    kernel=f"igemm_kernel<bf16,FPROP,256> im2col (ResNet-50 stage-3 conv3x3 256->256 + BN stats, B={batch})")
    H, C_, K = 32, 16, 16
    return dict(nimg=batch, H=H, C=C_, K=K, bound="hbm", M=batch * H * H, Kd=9 * C_,
                kernel=f"igemm_kernel<bf16,FPROP,16> halo (stage-1 conv3x3 16->16 + BN stats, B={batch})")


def kernel_roofline(torch, peaks, batch, live_us, spec=None):
    """achieved = algorithmic bytes / the dominant kernel's average launch duration measured
    live in the timed steps (event pairs around each launch on its block stream, concurrent
    with the other blocks). Also timed alone on rotating buffers larger than L2 ("isolated")."""
    import ctypes as C

    from paper_1909_02625_b200 import _lib as L

    lib = L.load()
    st = torch.cuda.current_stream()
    spec = spec or roofline_spec("resnet56", batch)
    nimg, H, W, Cc, K = spec["nimg"], spec["H"], spec["H"], spec["C"], spec["K"]
    M = nimg * H * W
    nbuf = max(2, int(2 * L2_BYTES // (M * Cc * 2)) + 1)
    xs = [torch.randn(M * Cc, device="cuda").bfloat16() for _ in range(nbuf)]
    ys = [torch.empty(M * K, device="cuda", dtype=torch.bfloat16) for _ in range(nbuf)]
    w = torch.randn(K * 9 * Cc, device="cuda").bfloat16()
    tiles = (M + 127) // 128
    stats = torch.empty(tiles * 2 * K, device="cuda")
    g = L.ConvGeom(nimg, H, W, Cc, H, W, K, 3, 3, 1, 1)

    def launch(i):
        a = L.IgemmArgs()
        a.geom = g
        a.M, a.N, a.Kd = M, K, 9 * Cc
        a.A, a.B, a.D = xs[i].data_ptr(), w.data_ptr(), ys[i].data_ptr()
        a.ldd = K
        a.stats = stats.data_ptr()
        L.check(lib.dsp_igemm(L.DSP_IGEMM_FPROP, L.DSP_DTYPE_BF16, C.byref(a), 1, C.c_void_p(st.cuda_stream)))

    for i in range(nbuf):
        launch(i)
    torch.cuda.synchronize()
    reps = 4 * nbuf
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for i in range(reps):
        launch(i % nbuf)
    e1.record(st)
    e1.synchronize()
    t_iso = e0.elapsed_time(e1) / 1000.0 / reps
    algo = M * Cc * 2 + M * K * 2 + K * 9 * Cc * 2 + tiles * 2 * K * 4
    t = (sum(live_us) / len(live_us) / 1e6) if live_us else t_iso
    timing = ((f"live: mean of {len(live_us)} launches in timed steps of the same workload (event pairs on "
               "the block stream, concurrent with the other blocks; a probe pass after the value steps)")
              if live_us else "isolated (probe found no launch)")
    if spec["bound"] == "tensor":
        flops = 2.0 * M * K * 9 * Cc
        peak_key = "bf16_tflops_sustained" if ("bf16_tflops_sustained" in peaks and live_us) else "bf16_tflops"
        peak = peaks.get(peak_key, peaks.get("bf16_tflops", 2250.0))
        achieved = flops / t / 1e12
        return {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
                "traffic": ncu_traffic("resnet50"), "algorithmic_bytes_per_launch": algo, "kernel": spec["kernel"],
                "algorithmic_flops_per_launch": flops,
                "launch_us": t * 1e6, "timing": timing, "isolated_launch_us": t_iso * 1e6,
                "isolated_achieved": flops / t_iso / 1e12,
                "isolated_frac": flops / t_iso / 1e12 / peaks.get("bf16_tflops", 2250.0),
                "peak_source": f"MEASURED_PEAKS.json {peak_key}" if peak_key in peaks else "fallback 2250 TFLOP/s"}
    peak_key = "hbm_gbs_sustained" if ("hbm_gbs_sustained" in peaks and live_us) else "hbm_gbs"
    peak = peaks.get(peak_key, peaks.get("hbm_gbs", 6650.0))
    achieved = algo / t / 1e9
    return {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
            "traffic": ncu_traffic() if spec["M"] == 128 * 32 * 32 else None, "kernel": spec["kernel"],
            "algorithmic_bytes_per_launch": algo, "launch_us": t * 1e6,
            "timing": timing,
            "isolated_launch_us": t_iso * 1e6, "isolated_achieved": algo / t_iso / 1e9,
            "isolated_frac": algo / t_iso / 1e9 / peaks.get("hbm_gbs", 6650.0),
            "peak_source": f"MEASURED_PEAKS.json {peak_key}" if peak_key in peaks else "fallback 6650 GB/s"}


def workload_of(model: str, K: int, cuts: str = ""):
    """(layers, boundaries, queue config) of a BASELINE model at K blocks (FLOP-balanced cuts)."""
    import paper_1909_02625_b200 as P

    m = MODELS[model]
    if model == "resnet50":
        layers = P.resnet50_layers(m["classes"], m["in_shape"])
    elif model == "resnet164":
        layers = P.resnet_cifar_bottleneck_layers(m["depth"], m["classes"])
    else:
        layers = P.resnet_cifar_layers(m["depth"], m["classes"])
    bounds = [int(v) for v in cuts.split(",")] if cuts else (P.flop_balanced_boundaries(layers, K) if K > 1 else [])
    return layers, bounds, P.default_queue_config(K)


def measure(model: str, K: int, batch: int, steps: int, warmup: int, dev, world: int, cuts: str = "",
            probe=None, e2e: bool = True, clock: bool = False, precision: str = "bf16", opt=None):
    """Device-timed DSP steps of one workload through TrainEngine(backend="b200") on a device-resident
    synthetic pool (L2 flushed between steps, CUDA events on the engine stream, max over ranks), then
    optionally the live roofline probe pass and the end-to-end pass with host buffers."""
    import ctypes as C

    import torch
    import torch.distributed as dist

    import paper_1909_02625_b200 as P
    from paper_1909_02625_b200 import _lib as L
    from paper_1909_02625_b200.data import cycle, device_synthetic_batches, synthetic_batches

    lib = L.load()
    m = MODELS[model]
    in_shape, classes = m["in_shape"], m["classes"]
    layers, bounds, cfg = workload_of(model, K, cuts)
    o = opt or SUM_OPT
    npool = 16 if in_shape[1] <= 32 else 4  # ImageNet-shaped batches: 154 MB each on the host
    model_ = P.build_model(layers, bounds)
    P.init_params(model_, 0)
    stream = torch.cuda.current_stream(dev)
    # device-resident pool generated on the GPU (csrc/synth.cu): bitwise the packed host pool
    dev_pool = device_synthetic_batches(npool, batch, in_shape, classes, seed=0, device=dev, stream=stream,
                                        precision=precision)
    eng = P.TrainEngine(model_, cfg, cycle([(b, b.labels) for b in dev_pool]), P.LrSchedule(o["lr"]), rule=o["rule"],
                        beta=o["beta"], s=o["s"], weight_decay=5e-4, device=dev, precision=precision)
    flush = torch.empty(2 * L2_BYTES, dtype=torch.uint8, device=dev)

    def barrier():
        if world > 1:
            dist.barrier()

    # warm up through the zero-prefill horizon and one capture of every step-graph phase
    warm = max(3, warmup, eng._graph_horizon() + getattr(eng.rt, "R", 0) + 1)
    for _ in range(warm):
        eng.run(1)
    torch.cuda.synchronize()
    barrier()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    launches0 = eng.rt.kernels_executed()
    with NvmlClockSampler(dev.index) if clock else _Null() as clk:
        for i in range(steps):
            flush.zero_()  # evict L2 between timed steps (outside the timed window)
            starts[i].record(stream)
            eng.run(1)
            ends[i].record(stream)
        torch.cuda.synchronize()
    launches = eng.rt.kernels_executed() - launches0
    out = {"warm": warm, "launches": int(launches), "clocks": clk.summary() if clock else None}

    # ---- roofline kernel, live: the same steps again with event pairs around every launch of the
    # roofline conv on its block stream (re-captured into each phase graph). A separate pass so
    # the probe's event nodes never touch the timed steps above.
    live_us = []
    if probe is not None and world == 1:
        probe_pairs = 64
        probe_ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * probe_pairs)]
        for ev in probe_ev:
            ev.record(stream)  # materialise the handles
        torch.cuda.synchronize()
        handles = (C.c_void_p * (2 * probe_pairs))(*[C.c_void_p(ev.cuda_event) for ev in probe_ev])
        lib.dsp_probe_arm(L.DSP_IGEMM_FPROP | (probe["Kd"] << 8), probe["K"], probe["M"], handles, probe_pairs)
        for g in eng.rt.graphs.values():
            lib.dsp_graph_destroy(g[3])
        eng.rt.graphs.clear()
        probed = 0
        for i in range(getattr(eng.rt, "R", 0) + 1 + steps):
            flush.zero_()
            lib.dsp_probe_reset()
            eng.run(1)
            probed = max(probed, lib.dsp_probe_reset())
            if i > getattr(eng.rt, "R", 0):  # every phase captured: timed probe steps
                torch.cuda.synchronize()
                live_us += [probe_ev[2 * j].elapsed_time(probe_ev[2 * j + 1]) * 1000.0 for j in range(probed)]
        lib.dsp_probe_arm(0, 0, 0, None, 0)
        torch.cuda.synchronize()
    out["live_us"] = live_us
    barrier()
    step_ms = [s_.elapsed_time(e_) for s_, e_ in zip(starts, ends)]
    t = torch.tensor([float(sum(step_ms))], device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t.item())
    out["ms_per_step"] = total_ms / steps
    out["step_ms_median"] = statistics.median(step_ms)
    out["value"] = batch * steps / (total_ms / 1000.0)
    out["loss_finite"] = True
    log = eng.log  # raises NonFiniteError if a step went non-finite (tensor.py:34-37)
    if (K - 1) in eng.local:
        out["loss_finite"] = bool(all(np.isfinite([lv for _, lv in log.losses()])))
    del eng, model_, dev_pool
    torch.cuda.empty_cache()

    # ---- end to end through the public API with HOST buffers. One GPU: the engine-level
    # C-ABI (dsp_run via NativeEngine) -- every step copies its batch host->device (pinned)
    # and its loss / grad-norm row device->host inside the timed region. N GPUs: the
    # Python-orchestrated TrainEngine on host batches with a per-step loss read.
    out["e2e"] = None
    if e2e:
        host_pool = synthetic_batches(npool, batch, in_shape, classes, seed=0)
        model2 = P.build_model(layers, bounds)
        P.init_params(model2, 0)
        if world == 1:
            from paper_1909_02625_b200.native import NativeEngine

            eng2 = NativeEngine(model2, cfg, batch, P.LrSchedule(o["lr"]), rule=o["rule"], beta=o["beta"],
                                s=o["s"], weight_decay=5e-4, device=dev.index, precision=precision)
            xs = np.stack([np.asarray(x, dtype=np.float32) for x, _ in host_pool])
            ls = np.stack([np.asarray(lab, dtype=np.int64) for _, lab in host_pool])
            del host_pool
            warm2 = max(warm, eng2.horizon + eng2.ring + 1)  # every graph phase captured before timing
            sel = np.arange(warm2 + steps) % len(xs)
            xw, lw = xs[sel[:warm2]], ls[sel[:warm2]]
            xt, lt = np.ascontiguousarray(xs[sel[warm2:]]), np.ascontiguousarray(ls[sel[warm2:]])
            eng2.run_batches(xw, lw)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            eng2.run_batches(xt, lt)  # returns after the last step (and its D2H row) completed
            el = time.perf_counter() - t0
            h2d = int(xt[0].nbytes + lt[0].nbytes)
            d2h = 4 * 2 * K
            how = ("host wall clock around dsp_run (engine C-ABI): per step pinned H2D of the fp32 batch + labels "
                   "and async D2H of the step's loss/grad-norm row; graphs replayed natively")
        else:
            eng2 = P.TrainEngine(model2, cfg, cycle(host_pool), P.LrSchedule(o["lr"]), rule=o["rule"],
                                 beta=o["beta"], s=o["s"], weight_decay=5e-4, device=dev, precision=precision)
            for _ in range(warm):
                eng2.run(1)
                eng2.last_loss()
            torch.cuda.synchronize()
            barrier()
            t0 = time.perf_counter()
            for _ in range(steps):
                eng2.run(1)
                eng2.last_loss()  # device->host read of the step's result
            torch.cuda.synchronize()
            el = time.perf_counter() - t0
            tt = torch.tensor([el], device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            el = float(tt.item())
            h2d = batch * int(np.prod(in_shape)) * 4 + batch * 8 if 0 in eng2.local else 0
            d2h = 4 if (K - 1) in eng2.local else 0
            how = "host wall clock incl. pinned H2D + per-step loss D2H (Python engine, one rank per GPU)"
        out["e2e"] = {"value": batch * steps / el, "unit": UNIT, "h2d_bytes_per_step": h2d,
                      "d2h_bytes_per_step": d2h, "timing": how}
        del eng2, model2
        torch.cuda.empty_cache()
    return out


class _Null:
    def __enter__(self):
        return self

    def __exit__(self, *exc):
        return False


# shapes of the per-conv tensor-pipe summary: ResNet-50's 3x3 stage convs (the tensor-bound ones)
TC_SHAPES = [("s1.3x3", 56, 64, 64), ("s2.3x3", 28, 128, 128), ("s3.3x3", 14, 256, 256), ("s4.3x3", 7, 512, 512)]


def conv_tensor_pipe(torch, peaks, batch: int):
    """Per-conv fraction of the bf16 tensor peak: FLOP/s of isolated event-timed launches through
    dsp_igemm (FPROP with the fused BN statistics + finalize, DGRAD, WGRAD with split-K) on
    buffers rotated past L2, divided by MEASURED_PEAKS bf16_tflops.  The ncu counter view of the
    same kernels (sm__pipe_tensor_cycles_active) is committed under profiles/."""
    import ctypes as C

    from paper_1909_02625_b200 import _lib as L

    lib = L.load()
    st = torch.cuda.current_stream()
    peak = peaks.get("bf16_tflops", 2250.0)
    out = {}
    for name, H, Cc, K in TC_SHAPES:
        M = batch * H * H
        Kd = 9 * Cc
        nbuf = max(2, int(2 * L2_BYTES // (M * Cc * 2)) + 1)
        xs = [torch.randn(M * Cc, device="cuda").bfloat16() for _ in range(nbuf)]
        dys = [torch.randn(M * K, device="cuda").bfloat16() for _ in range(nbuf)]
        outs = [torch.empty(M * max(K, Cc), device="cuda", dtype=torch.bfloat16) for _ in range(nbuf)]
        w = (torch.randn(K * Kd, device="cuda") * 0.05).bfloat16()
        w_t = w.view(K, 9, Cc).permute(2, 1, 0).contiguous()
        gamma, beta = torch.ones(K, device="cuda"), torch.zeros(K, device="cuda")
        stats = torch.empty(L.IGEMM_MAX_CTAS * 3 * K, device="cuda")
        stat_out = torch.empty(4 * K, device="cuda")
        sem = torch.zeros(L.IGEMM_SEM_INTS, dtype=torch.int32, device="cuda")
        g = L.ConvGeom(batch, H, H, Cc, H, H, K, 3, 3, 1, 1)
        # WGRAD split-K as the block executor sizes it (block.cu wgrad_splits: ~148 CTAs)
        nkb = (M + 63) // 64
        mt, nt = (Kd + 127) // 128, (K + 255) // 256
        splits = max(1, min(148 // max(1, mt * nt), nkb))
        kbps = (nkb + splits - 1) // splits
        splits = (nkb + kbps - 1) // kbps
        part = torch.empty(splits * Kd * K, device="cuda")

        def launch(mode, i):
            a = L.IgemmArgs()
            a.geom = g
            if mode == L.DSP_IGEMM_FPROP:
                a.M, a.N, a.Kd = M, K, Kd
                a.A, a.B, a.D, a.ldd = xs[i].data_ptr(), w.data_ptr(), outs[i].data_ptr(), K
                a.stats, a.stat_out, a.gamma, a.beta, a.sem = (stats.data_ptr(), stat_out.data_ptr(), gamma.data_ptr(),
                                                               beta.data_ptr(), sem.data_ptr())
                a.n_valid = K
            elif mode == L.DSP_IGEMM_DGRAD:
                a.M, a.N, a.Kd = M, Cc, 9 * K
                a.A, a.B, a.D, a.ldd = dys[i].data_ptr(), w.data_ptr(), outs[i].data_ptr(), Cc
                a.B_t = w_t.data_ptr()
                a.n_valid = Cc
            else:
                a.M, a.N, a.Kd = Kd, K, M
                a.A, a.B, a.D = xs[i].data_ptr(), dys[i].data_ptr(), part.data_ptr()
                a.kb_per_split = kbps
            L.check(lib.dsp_igemm(mode, L.DSP_DTYPE_BF16, C.byref(a), splits if mode == L.DSP_IGEMM_WGRAD else 1,
                                  C.c_void_p(st.cuda_stream)))

        row = {}
        for mname, mode in (("fprop", L.DSP_IGEMM_FPROP), ("dgrad", L.DSP_IGEMM_DGRAD), ("wgrad", L.DSP_IGEMM_WGRAD)):
            for i in range(nbuf):
                launch(mode, i)
            torch.cuda.synchronize()
            reps = max(4 * nbuf, 12)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            for i in range(reps):
                launch(mode, i % nbuf)
            e1.record(st)
            e1.synchronize()
            us = e0.elapsed_time(e1) * 1000.0 / reps
            tflops = 2.0 * M * K * Kd / (us * 1e-6) / 1e12
            row[mname] = {"us": round(us, 2), "tflops": round(tflops, 1), "frac": round(tflops / peak, 4)}
        out[name] = row
        del xs, dys, outs, part
        torch.cuda.empty_cache()
    fr = [r[m]["frac"] for r in out.values() for m in r]
    return {"convs": out, "mean_frac": round(float(np.mean(fr)), 4), "peak_tflops": peak,
            "peak_source": "MEASURED_PEAKS.json bf16_tflops (burst)",
            "timing": f"isolated dsp_igemm launches, CUDA events, buffers rotated past L2, B={batch}",
            "ncu": "profiles/r02_conv_tensor_pipe.md"}


def relaunch_distributed(args) -> int:
    """--gpus N without a torchrun environment: re-exec this script under torch.distributed.run."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def run_b200(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    dev = torch.device("cuda", torch.cuda.current_device())
    K = blocks_for(args)
    peaks = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            peaks = json.load(f)
    except Exception:
        pass
    spec = roofline_spec(args.model, args.batch)
    main_run = measure(args.model, K, args.batch, args.steps, args.warmup, dev, world, cuts=args.cuts,
                       probe=spec, e2e=not args.no_e2e, clock=True, precision=args.precision, opt=opt_of(args))
    extras = {}
    if not args.no_extras:
        # the metric's "vs BP": K = 1 (p = (0,), m = (0,)) is plain backprop, bitwise
        # (tests/test_pipeline.py:152-168), on the same model and batch, one rank
        if world == 1:
            bp = measure(args.model, 1, args.batch, args.steps, args.warmup, dev, 1, e2e=False,
                         precision=args.precision, opt=opt_of(args))
            extras["k1_bp"] = {"value": bp["value"], "unit": UNIT, "ms_per_step": bp["ms_per_step"],
                               "dsp_over_bp": main_run["value"] / bp["value"],
                               "config": "same model / batch / optimizer, K=1 (one block, plain BP)"}
            extras["conv_tensor_pipe"] = conv_tensor_pipe(torch, peaks, MODELS["resnet50"]["batch"])
            # the metric's K = 2 / 8 with all K blocks on this ONE GPU (the K-GPU figures come from the
            # driver's --gpus N runs): what the schedule costs per sample as K grows, same model and batch
            sweep = {}
            for kk in (2, 8):
                if kk == K:
                    continue
                try:
                    r = measure(args.model, kk, args.batch, args.steps, args.warmup, dev, 1, e2e=False,
                                precision=args.precision, opt=opt_of(args))
                    sweep[str(kk)] = {"value": r["value"], "unit": UNIT, "ms_per_step": r["ms_per_step"]}
                except Exception as exc:  # an extra must never sink the bench line
                    sweep[str(kk)] = {"value": None, "error": repr(exc)[:200]}
            sweep["note"] = ("DSP with K blocks, all on one GPU (p_k=1, m_k=2(K-1-k), FLOP-balanced cuts); "
                             "K=1 is k1_bp, K=%d the main value" % K)
            extras["k_sweep_1gpu"] = sweep
        if args.model != "resnet56":
            r56 = measure("resnet56", 8 if world >= 8 else 4, MODELS["resnet56"]["batch"], args.steps, args.warmup, dev,
                          world, e2e=not args.no_e2e, precision=args.precision)
            extras["resnet56"] = {"value": r56["value"], "unit": UNIT, "ms_per_step": r56["ms_per_step"],
                                  "e2e": r56["e2e"], "config": config_dict_for("resnet56", 8 if world >= 8 else 4,
                                                                              MODELS["resnet56"]["batch"], world)}
    roof = kernel_roofline(torch, peaks, args.batch, main_run["live_us"], spec) if rank == 0 else None
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            sub = 32 if IN_SHAPE[1] <= 32 else 2
            v, dt, cpu_s = cpu_oracle_steps(args, 3 if sub > 2 else 1, 1, sub)
            cpu = {"value": v, "unit": UNIT, "cores": threads_used(), "kind": "port",
                   "sample": f"oracle/dsp_ref.py float64 DSP step (CPU restatement of the reference), {args.model} "
                             f"K={K}, {3 if sub > 2 else 1} timed step(s) of a {sub}-sample sub-batch after 1 warmup "
                             f"({dt:.1f} s)"}
        except Exception as exc:  # the baseline must never sink the bench line
            cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "port", "sample": f"failed: {exc!r}"}
    if rank == 0:
        line = {"metric": METRIC, "value": main_run["value"], "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": main_run["warm"], "ms_per_step": main_run["ms_per_step"], "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": args.precision, "data": "synthetic",
                "config": config_dict(args, K, world), "e2e": main_run["e2e"], "gpu_launches": main_run["launches"],
                "roofline": roof, "cpu_baseline": cpu, "clocks": main_run["clocks"],
                "step_ms_median": main_run["step_ms_median"], "loss_finite": main_run["loss_finite"], **extras}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    select_model(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch_distributed(args)
    if args.impl == "reference":
        return run_reference(args)
    return run_b200(args)


if __name__ == "__main__":
    sys.exit(main())
