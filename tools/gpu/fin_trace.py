"""Diagnostic: globaltimer timeline of the fused BN finalize tail of one FPROP launch.

Needs a library built with -DIG_TRACE_BUILD (tools/gpu/fin_trace.sh builds one under /tmp and
puts it first on sys.path). Per CTA: ctat[1] start, ctat[2] epilogue done (ticket taken next),
ctat[4] finalize done, ctat[3] TMEM dealloc (end); trace[186..188]: the finalizing CTA's ticket
won / first window loaded / finalize written; trace[192 + 8192 + 4b ..]: CTA b's ticket internals
(release fence done, atomic returned, acquire fence done). Prints one JSON line per shape.
"""

import ctypes as C
import json
import sys

import torch

from paper_1909_02625_b200 import _lib as L

SHAPES = [("c1.3x3", 128, 32, 16, 16), ("c2.3x3", 128, 16, 32, 32), ("c3.3x3", 128, 8, 64, 64),
          ("s3.3x3", 256, 14, 256, 256)]


def main():
    lib = L.load()
    torch.cuda.set_device(0)
    st = torch.cuda.current_stream()
    for name, nimg, H, Cc, K in SHAPES:
        g = L.ConvGeom(nimg, H, H, Cc, H, H, K, 3, 3, 1, 1)
        x = torch.randn(nimg, H, H, Cc, device="cuda").bfloat16()
        w = (torch.randn(K, 3, 3, Cc, device="cuda") / (9 * Cc) ** 0.5).bfloat16()
        y = torch.empty(nimg, H, H, K, device="cuda", dtype=torch.bfloat16)
        stats = torch.empty(L.IGEMM_MAX_CTAS * 2 * K, device="cuda")
        stat_out = torch.empty(4 * K, device="cuda")
        gamma, beta = torch.ones(K, device="cuda"), torch.zeros(K, device="cuda")
        sem = torch.zeros(L.IGEMM_SEM_INTS, dtype=torch.int32, device="cuda")
        trace = torch.zeros(192 + 12 * 1024, dtype=torch.int64, device="cuda")
        a = L.IgemmArgs()
        a.geom = g
        a.M, a.N, a.Kd = nimg * H * H, K, 9 * Cc
        a.A, a.B, a.D, a.ldd = x.data_ptr(), w.data_ptr(), y.data_ptr(), K
        a.stats, a.stat_out, a.gamma, a.beta, a.sem = (stats.data_ptr(), stat_out.data_ptr(), gamma.data_ptr(),
                                                       beta.data_ptr(), sem.data_ptr())
        a.n_valid = K
        a.trace = trace.data_ptr()
        res = []
        for rep in range(6):
            trace.zero_()
            torch.cuda.synchronize()
            L.check(lib.dsp_igemm(L.DSP_IGEMM_FPROP, L.DSP_DTYPE_BF16, C.byref(a), 1, C.c_void_p(st.cuda_stream)))
            torch.cuda.synchronize()
            t = trace.cpu().tolist()
            ct = [t[192 + 8 * b: 200 + 8 * b] for b in range(1024) if t[192 + 8 * b + 1] != 0]
            t0 = min(c[1] for c in ct)
            tk = [t[192 + 8 * 1024 + 4 * b: 196 + 8 * 1024 + 4 * b] for b in range(1024) if t[192 + 8 * b + 1] != 0]
            r = {"ctas": len(ct), "last_start_us": (max(c[1] for c in ct) - t0) / 1e3,
                 "work_done_max_us": (max(c[2] for c in ct) - t0) / 1e3,
                 "work_done_median_us": (sorted(c[2] for c in ct)[len(ct) // 2] - t0) / 1e3,
                 "ticket_us": (t[186] - t0) / 1e3 if t[186] else None,
                 "first_window_us": (t[187] - t0) / 1e3 if t[187] else None,
                 "finalized_us": (t[188] - t0) / 1e3 if t[188] else None,
                 "end_max_us": (max(c[3] for c in ct) - t0) / 1e3,
                 # ticket internals (all CTAs): release fence done / atomic returned; winner's acquire fence
                 "rel_fence_max_us": (max(k[0] for k in tk) - t0) / 1e3,
                 "atom_ret_median_us": (sorted(k[1] for k in tk)[len(tk) // 2] - t0) / 1e3,
                 "atom_ret_max_us": (max(k[1] for k in tk) - t0) / 1e3,
                 "acq_fence_us": (max(k[2] for k in tk) - t0) / 1e3 if max(k[2] for k in tk) else None}
            res.append(r)
        print(json.dumps({"shape": name, "runs": res[2:]}), flush=True)


if __name__ == "__main__":
    sys.exit(main())
