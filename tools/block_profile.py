"""Run one block's recorded forward + backward (+ update) a few times through the block
executor, for ncu: realistic launch arguments for a single kernel of the DSP step.

    python tools/block_profile.py --block r50s1 [--reps 3] [--precision bf16]
    ncu --set full -k regex:igemm -s 20 -c 1 -o gpurun_out/prof python tools/block_profile.py --block r50s1
"""

from __future__ import annotations

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_1909_02625_b200 as P  # noqa: E402

BLOCKS = {
    # ResNet-50 stage-1 unit with identity shortcut (56x56, 256 -> 64 -> 256), B=256
    "r50s1": (lambda: [P.bottleneck((256, 56, 56), 64, 256, 1)], 256),
    # ResNet-50 stage-1 first unit (projection shortcut) after the stem + max pool
    "r50s1proj": (lambda: [P.bottleneck((64, 56, 56), 64, 256, 1)], 256),
    "r50s3": (lambda: [P.bottleneck((1024, 14, 14), 256, 1024, 1)], 256),
    "r50stem": (lambda: [P.conv_bn_relu((3, 224, 224), 64, ksize=7, stride=2), P.maxpool((64, 112, 112))], 256),
    "c1basic": (lambda: [P.basic_unit((16, 32, 32), 16, 1)], 128),
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--block", default="r50s1", choices=sorted(BLOCKS))
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--precision", default="bf16", choices=["bf16", "fp32"])
    ap.add_argument("--r50-block", type=int, default=-1,
                    help="instead of --block: block k of ResNet-50 cut into K=4 FLOP-balanced blocks (B=256)")
    ap.add_argument("--r56-block", type=int, default=-1,
                    help="instead of --block: block k of ResNet-56 cut into K=4 FLOP-balanced blocks (B=128)")
    args = ap.parse_args()
    import torch

    from paper_1909_02625_b200 import _lib as L
    from paper_1909_02625_b200.runtime import DeviceBlock

    if args.r56_block >= 0:
        full = P.resnet_cifar_layers(56, 10)
        cuts = [0] + P.flop_balanced_boundaries(full, 4) + [len(full)]
        layers, B = full[cuts[args.r56_block]:cuts[args.r56_block + 1]], 128
        last = args.r56_block == 3
        args.r50_block = -1
    elif args.r50_block >= 0:
        full = P.resnet50_layers()
        cuts = [0] + P.flop_balanced_boundaries(full, 4) + [len(full)]
        layers, B = full[cuts[args.r50_block]:cuts[args.r50_block + 1]], 256
        last = args.r50_block == 3
    else:
        layers, B = BLOCKS[args.block]
        layers = layers()
        last = False
    model = P.build_model(layers, [])
    P.init_params(model, 0)
    dt = L.storage_dtype(args.precision)
    st = torch.cuda.current_stream()
    db = DeviceBlock(model.blocks[0], B, is_last=last, stream=st, dtype=dt)
    tdt = L.torch_storage(dt)
    x = torch.randn(db.in_elems, device="cuda").to(tdt)
    y = torch.empty(db.out_elems, device="cuda", dtype=tdt)
    up = (torch.randn(db.out_elems, device="cuda") * 1e-2).to(tdt)
    gin = torch.empty(db.in_elems, device="cuda", dtype=tdt)
    ys = db.params.clone()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    labels = torch.zeros(B, dtype=torch.int64, device="cuda")
    loss = torch.zeros(1, device="cuda")
    first = args.r50_block == 0 or args.r56_block == 0
    for r in range(args.reps):
        if r == args.reps - 1:
            ev[0].record(st)
        if not last:
            db.forward(x, y, record=False)
        db.forward(x, None, record=True)
        if last:
            db.loss(labels, loss)
        db.backward(None if last else up, None if first else gin)  # block 0 has no dX (engine.cu:202)
        db.update(L.DSP_RULE_SUM, ys, 1e-3, 1e-3, 0.9, 5e-4, True, None)
        if r == args.reps - 1:
            ev[1].record(st)
    torch.cuda.synchronize()
    name = (f"resnet50 block {args.r50_block}" if args.r50_block >= 0 else
            f"resnet56 block {args.r56_block}" if args.r56_block >= 0 else args.block)
    print(f"{name}: one fwd + recompute + bwd + update {ev[0].elapsed_time(ev[1]) * 1000:.1f} us "
          f"({model.blocks[0].param_count} params)")


if __name__ == "__main__":
    main()
