"""Tensor-pipe throughput of the implicit-GEMM conv kernels on the tensor-bound shapes
(BASELINE configs[4]: ResNet-50, ImageNet-shaped, batch 256, bf16), beside cuDNN.

Every launch goes through the C-ABI `dsp_igemm` (FPROP / DGRAD / WGRAD, the same entry the
block executor uses). FLOPs are algorithmic: 2*M*N*Kd of the implicit GEMM. Peak = the measured
dense bf16 figure in MEASURED_PEAKS.json (burst). Prints one JSON object per (shape, mode) and a
summary line; `--json out.json` also writes them to a file.

    python tools/conv_tc.py [--batch 256] [--reps 20] [--json gpurun_out/conv_tc.json]
    python tools/conv_tc.py --shapes cifar --batch 128      # ResNet-56 stage convs
"""

from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

# name, H(=W) of the input, C_in, C_out, kernel, stride
R50 = [
    ("s1.3x3", 56, 64, 64, 3, 1),
    ("s1.1x1up", 56, 64, 256, 1, 1),
    ("s1.1x1down", 56, 256, 64, 1, 1),
    ("s2.3x3", 28, 128, 128, 3, 1),
    ("s2.1x1up", 28, 128, 512, 1, 1),
    ("s2.1x1down", 28, 512, 128, 1, 1),
    ("s3.3x3", 14, 256, 256, 3, 1),
    ("s3.1x1up", 14, 256, 1024, 1, 1),
    ("s3.1x1down", 14, 1024, 256, 1, 1),
    ("s4.3x3", 7, 512, 512, 3, 1),
    ("s4.1x1up", 7, 512, 2048, 1, 1),
    ("s4.1x1down", 7, 2048, 512, 1, 1),
]

# ResNet-56 / ResNet-110 (BASELINE configs[1], [2]: CIFAR-shaped, batch 128) 3x3 stage convs;
# c1.3x3 FPROP is bench.py's roofline kernel (stage-1 halo tiles + fused BN statistics)
CIFAR = [
    ("c1.3x3", 32, 16, 16, 3, 1),
    ("c2.3x3", 16, 32, 32, 3, 1),
    ("c3.3x3", 8, 64, 64, 3, 1),
]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=256)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--json", default="")
    ap.add_argument("--only", default="")
    ap.add_argument("--no-cudnn", action="store_true")
    ap.add_argument("--shapes", default="r50", choices=["r50", "cifar"])
    ap.add_argument("--fprop-stats", default="finalize", choices=["finalize", "partials", "none"],
                    help="FPROP epilogue: BN partials + fused finalize (the step's form), partials only, or none")
    ap.add_argument("--fin-dbg", type=int, default=0,
                    help="diagnostic: ticket debug bits (1 = skip the pre-ticket fence, 2 = skip the atomic, 4 = skip the winner's acquire fence); "
                         "results are not valid with these set")
    args = ap.parse_args()

    import torch
    import torch.nn.functional as F

    from paper_1909_02625_b200 import _lib as L

    lib = L.load()
    peaks = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            peaks = json.load(f)
    except Exception:
        pass
    peak = peaks.get("bf16_tflops", 2250.0)
    torch.cuda.set_device(0)
    st = torch.cuda.current_stream()
    torch.backends.cudnn.benchmark = True
    rows = []
    for name, H, Cc, K, R, stride in (CIFAR if args.shapes == "cifar" else R50):
        if args.only and args.only not in name:
            continue
        nimg = args.batch
        pad = R // 2
        P = (H + 2 * pad - R) // stride + 1
        g = L.ConvGeom(nimg, H, H, Cc, P, P, K, R, R, stride, pad)
        x = torch.randn(nimg, H, H, Cc, device="cuda").bfloat16()
        w = (torch.randn(K, R, R, Cc, device="cuda") / (R * R * Cc) ** 0.5).bfloat16()
        w_t = w.permute(3, 1, 2, 0).contiguous()
        dy = torch.randn(nimg, P, P, K, device="cuda").bfloat16()
        y = torch.empty(nimg, P, P, K, device="cuda", dtype=torch.bfloat16)
        dx = torch.empty(nimg, H, H, Cc, device="cuda", dtype=torch.bfloat16)
        Mf = nimg * P * P
        flops = 2.0 * Mf * K * R * R * Cc
        stats = torch.empty(L.IGEMM_MAX_CTAS * 2 * K, device="cuda")
        stat_out = torch.empty(4 * K, device="cuda")
        gamma = torch.ones(K, device="cuda")
        beta = torch.zeros(K, device="cuda")
        sem = torch.zeros(L.IGEMM_SEM_INTS, dtype=torch.int32, device="cuda")  # one ticket per n-tile
        # WGRAD split-K as the block executor sizes it (block.cu wgrad_splits, 148-CTA target)
        Mw, nkb = R * R * Cc, (Mf + 63) // 64
        mt, nt = (Mw + 127) // 128, (K + 255) // 256
        splits = min(max(1, 148 // (mt * nt)), nkb)
        kbs = (nkb + splits - 1) // splits
        splits = (nkb + kbs - 1) // kbs
        part = torch.empty(splits * Mw * K, device="cuda")

        def args_for(mode):
            a = L.IgemmArgs()
            a.geom = g
            if mode == L.DSP_IGEMM_FPROP:
                a.M, a.N, a.Kd = Mf, K, R * R * Cc
                a.A, a.B, a.D, a.ldd = x.data_ptr(), w.data_ptr(), y.data_ptr(), K
                a.stats, a.stat_out, a.gamma, a.beta, a.sem = (stats.data_ptr(), stat_out.data_ptr(),
                                                               gamma.data_ptr(), beta.data_ptr(), sem.data_ptr())
                a.n_valid = K
                a.out_f32 = args.fin_dbg << 8
                if args.fprop_stats != "finalize":
                    a.sem, a.stat_out = None, None
                if args.fprop_stats == "none":
                    a.stats = None
            elif mode == L.DSP_IGEMM_DGRAD:
                a.M, a.N, a.Kd = nimg * H * H, Cc, R * R * K
                a.A, a.B, a.D, a.ldd = dy.data_ptr(), w.data_ptr(), dx.data_ptr(), Cc
                a.B_t = w_t.data_ptr()
            else:
                a.M, a.N, a.Kd = Mw, K, Mf
                a.A, a.B, a.D = x.data_ptr(), dy.data_ptr(), part.data_ptr()
                a.kb_per_split = kbs
            return a

        def timed(fn):
            for _ in range(3):
                fn()
            torch.cuda.synchronize()
            evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.reps)]
            for e0, e1 in evs:
                e0.record(st)
                fn()
                e1.record(st)
            torch.cuda.synchronize()
            ts = sorted(e0.elapsed_time(e1) for e0, e1 in evs)
            return ts[len(ts) // 2] / 1e3

        xc = x.permute(0, 3, 1, 2)  # NHWC memory = channels_last NCHW view
        wc = w.permute(0, 3, 1, 2)
        dyc = dy.permute(0, 3, 1, 2)
        cudnn = {
            "fprop": lambda: F.conv2d(xc, wc, stride=stride, padding=pad),
            "dgrad": lambda: torch.ops.aten.convolution_backward(dyc, xc, wc, None, [stride] * 2, [pad] * 2, [1, 1],
                                                                 False, [0, 0], 1, [True, False, False]),
            "wgrad": lambda: torch.ops.aten.convolution_backward(dyc, xc, wc, None, [stride] * 2, [pad] * 2, [1, 1],
                                                                 False, [0, 0], 1, [False, True, False]),
        }
        for mode, mname in ((L.DSP_IGEMM_FPROP, "fprop"), (L.DSP_IGEMM_DGRAD, "dgrad"), (L.DSP_IGEMM_WGRAD, "wgrad")):
            a = args_for(mode)
            sp = splits if mode == L.DSP_IGEMM_WGRAD else 1
            sv = C.c_void_p(st.cuda_stream)
            t = timed(lambda: L.check(lib.dsp_igemm(mode, L.DSP_DTYPE_BF16, C.byref(a), sp, sv)))
            row = {"shape": name, "mode": mname, "M": a.M, "N": a.N, "Kd": a.Kd, "gflop": flops / 1e9,
                   "us": t * 1e6, "tflops": flops / t / 1e12, "frac": flops / t / 1e12 / peak,
                   # bf16 operand + result bytes (X, W|dY, Y|dX|fp32 split-K partials): the HBM-bound view
                   "gbs": (2 * (x.numel() + w.numel() + dy.numel()) + (4 * part.numel()
                           if mode == L.DSP_IGEMM_WGRAD else 0)) / t / 1e9}
            if not args.no_cudnn:
                tc = timed(cudnn[mname])
                row["cudnn_us"] = tc * 1e6
                row["cudnn_tflops"] = flops / tc / 1e12
            rows.append(row)
            print(json.dumps({k: (round(v, 3) if isinstance(v, float) else v) for k, v in row.items()}), flush=True)
    tot = sum(r["gflop"] for r in rows)
    summ = {"summary": ("cifar" if args.shapes == "cifar" else "resnet50") + " convs", "batch": args.batch,
            "peak_tflops": peak, "fprop_stats": args.fprop_stats,
            "tflops_all": tot / sum(r["us"] for r in rows) * 1e3,
            "frac_all": tot / sum(r["us"] for r in rows) * 1e3 / peak}
    if not args.no_cudnn:
        summ["cudnn_tflops_all"] = tot / sum(r["cudnn_us"] for r in rows) * 1e3
    print(json.dumps(summ))
    if args.json:
        with open(args.json, "w") as f:
            json.dump({"rows": rows, "summary": summ}, f, indent=1)


if __name__ == "__main__":
    main()
