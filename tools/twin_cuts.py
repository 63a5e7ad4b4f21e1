"""Twin-aware cut search (calibrate.twin_balanced_cuts) for a bench workload: the per-GPU DSP
step of every block timed whole (fresh forward on a forward twin beside recompute + backward,
then the update), starting from the FLOP-balanced cuts.

    python tools/twin_cuts.py [--model resnet56] [--k 4]
"""

import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="resnet56")
    ap.add_argument("--k", type=int, default=0)
    ap.add_argument("--reps", type=int, default=10)
    args = ap.parse_args()
    args.gpus, args.cuts, args.batch = 1, "", 0
    import bench
    from paper_1909_02625_b200 import calibrate as CAL

    bench.select_model(args)
    layers, bounds, _ = bench.workload(args)
    K = len(bounds) + 1
    base = [CAL.block_step_cost(layers, lo, hi, args.batch, hi == len(layers), reps=args.reps)
            for lo, hi in zip([0] + bounds, bounds + [len(layers)])]
    cuts, costs = CAL.twin_balanced_cuts(layers, K, args.batch, start=bounds, reps=args.reps,
                                         log=lambda m: print(m, flush=True))
    out = {"model": args.model, "k": K, "batch": args.batch,
           "flop_cuts": bounds, "flop_block_us": [round(c * 1e6, 1) for c in base],
           "twin_cuts": cuts, "twin_block_us": [round(c * 1e6, 1) for c in costs],
           "k_gpu_samples_per_s_flop_cuts": args.batch / max(base),
           "k_gpu_samples_per_s_twin_cuts": args.batch / max(costs)}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
