"""Per-GPU DSP step latency of each block when every block owns a GPU (K GPUs).

On K GPUs block k's device runs, per step: the fresh forward (pipeline.py:564), the
recompute forward + backward (pipeline.py:566-582) and the update (591-596). Serially that is
f_k + b_k; with a forward twin (dsp_block_share_weights) the fresh forward runs on its own
stream beside the recompute + backward, so the step approaches max(f_k, b_k) + update.
This times both as CUDA-graph replays of the real block kernels on ONE GPU, one block at a
time (what that block's GPU would do), for the bench workloads.

    python tools/block_step_latency.py [--model resnet56] [--k 4]
"""

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="resnet56")
    ap.add_argument("--k", type=int, default=0)
    ap.add_argument("--reps", type=int, default=20)
    args = ap.parse_args()
    args.gpus, args.cuts, args.batch = 1, "", 0
    import bench
    import paper_1909_02625_b200 as P
    from paper_1909_02625_b200.calibrate import _graph_time
    from paper_1909_02625_b200.runtime import DeviceBlock, torch_mod

    bench.select_model(args)
    layers, bounds, cfg = bench.workload(args)
    model = P.build_model(layers, bounds)
    P.init_params(model, 0)
    torch = torch_mod()
    dev = torch.device("cuda:0")
    B = args.batch
    rows = []
    for k, blk in enumerate(model.blocks):
        last = k == model.k - 1
        db = DeviceBlock(blk, B, is_last=last, device=dev)
        tw = None if last else db.make_twin()
        x = torch.randn(db.in_elems, device=dev).bfloat16()
        x2 = torch.randn(db.in_elems, device=dev).bfloat16()
        up = None if last else torch.randn(db.out_elems, device=dev).bfloat16() * 1e-3
        y = None if last else torch.empty(db.out_elems, dtype=torch.bfloat16, device=dev)
        gin = torch.empty(db.in_elems, dtype=torch.bfloat16, device=dev) if k > 0 else None
        labels = torch.zeros(B, dtype=torch.int64, device=dev)
        loss = torch.zeros(1, device=dev)
        gsq = torch.zeros(1, device=dev)
        ys = db.params.clone()
        fs = torch.cuda.Stream(dev)

        def step(st, twin):
            if not last:
                if twin:
                    fs.wait_stream(st)
                    tw.forward(x, y, record=False, stream=fs)
                else:
                    db.forward(x, y, record=False, stream=st)
            db.forward(x2, None, record=True, stream=st)
            if last:
                db.loss(labels, loss, stream=st)
            db.backward(up, gin, stream=st)
            if twin and not last:
                st.wait_stream(fs)
            db.update(1, ys, 1e-9, 1e-9, 0.9, 0.0, True, gsq, stream=st)

        serial = _graph_time(torch, lambda st: step(st, False), args.reps)
        twin = serial if last else _graph_time(torch, lambda st: step(st, True), args.reps)
        rows.append({"block": k, "serial_us": serial * 1e6, "twin_us": twin * 1e6})
        print(json.dumps(rows[-1]), flush=True)
    s = max(r["serial_us"] for r in rows)
    t = max(r["twin_us"] for r in rows)
    print(json.dumps({"model": args.model, "k": model.k, "batch": B, "max_serial_us": s, "max_twin_us": t,
                      "k_gpu_samples_per_s_serial": B / s * 1e6, "k_gpu_samples_per_s_twin": B / t * 1e6,
                      "note": "per-GPU step of the slowest block = the K-GPU DSP step interval (simulate.py:160-217) "
                              "excluding the exchange"}))


if __name__ == "__main__":
    main()
