"""Summarise the per-conv ncu counters of tools/gpu/evidence_r02.sh (conv_tc.py --reps 1 under ncu)
into a markdown table: device time, tensor-pipe % (elapsed / active cycles), DRAM bytes.

usage: python tools/ncu_conv_summary.py <ncu.csv> <conv_tc.json> > profiles/r02_conv_tensor_pipe.md
The conv_tc json gives the launch order (shape x {fprop, dgrad, wgrad}) and the algorithmic GFLOP.
"""
import json
import statistics
import sys

from launch_table import load


def main():
    L = load(sys.argv[1])
    rows = json.load(open(sys.argv[2]))["rows"]
    ids = sorted(L)
    per = len(ids) // len(rows)
    print("| conv | mode | GFLOP | ncu us | TFLOP/s | tensor pipe % elapsed | % active | DRAM MB |")
    print("|---|---|---:|---:|---:|---:|---:|---:|")
    tot_f, tot_t = 0.0, 0.0
    for i, r in enumerate(rows):
        es = [L[k] for k in ids[i * per:(i + 1) * per]]
        med = lambda m: statistics.median(e.get(m, 0.0) for e in es)
        us = med("gpu__time_duration.sum") / 1e3
        el = med("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed")
        ac = med("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active")
        mb = (med("dram__bytes_read.sum") + med("dram__bytes_write.sum")) / 1e6
        tot_f += r["gflop"]
        tot_t += us
        print(f"| {r['shape']} | {r['mode']} | {r['gflop']:.1f} | {us:.1f} | {r['gflop'] / us * 1e3:.0f} |"
              f" {el:.1f} | {ac:.1f} | {mb:.0f} |")
    print(f"\nsum: {tot_f:.0f} GFLOP in {tot_t:.0f} us (ncu, serialised, cold L2) = {tot_f / tot_t * 1e3:.0f} TFLOP/s")


if __name__ == "__main__":
    main()
