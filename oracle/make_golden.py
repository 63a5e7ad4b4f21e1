"""Generate tests/golden/*.npz from the UNMODIFIED reference (`stalepipe`).

Run in the build container (needs /root/reference):
    python oracle/make_golden.py
The fixtures pin the oracle (oracle/dsp_ref.py) and, through it, the CUDA path:
  * mlp_*.npz   -- the reference TrainEngine on its own MLP kinds (serial backend):
                   per-(step, block) log (batch index, loss, grad norm), checksum,
                   final params. The oracle must reproduce these bitwise.
  * cnn_k2.npz  -- the reference TrainEngine (unmodified) driving the oracle's
                   float64 CNN layer math (stalepipe.pipeline.block_forward /
                   block_backward patched): pins the FIFO schedule,
                   warmup and optimizer plumbing for the CNN kinds.
  * kats.npz    -- optimizer / rng / data known answers from the reference.
  * c1_resnet20_k2.npz, c2_resnet56_k4.npz -- BASELINE configs[0] (ResNet-20 w16, K=2, B=32)
                   and configs[1] (ResNet-56, K=4, B=128), SUM 0.9, through the unmodified
                   reference TrainEngine + oracle CNN math, 24 steps: the trajectories the
                   GPU parity tests compare the device against.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
OUT = os.path.join(ROOT, "tests", "golden")
REF = "/root/reference/pkg/src"


def _ref():
    sys.dont_write_bytecode = True
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import stalepipe as sp

    return sp


def _log_arrays(log):
    recs = log.sorted()
    return {
        "step": np.array([r.step for r in recs]),
        "block": np.array([r.block for r in recs]),
        "batch_index": np.array([r.batch_index for r in recs]),
        "loss": np.array([np.nan if r.loss is None else r.loss for r in recs]),
        "grad_norm": np.array([r.grad_norm for r in recs]),
    }


MLP_CASES = {
    # name: (layers, boundaries, p, m, batch, steps, rule, beta, s, wd, warmup, lr, decays)
    "mlp_k3_sum": ([("dense", 12, 16), ("relu",), ("dense", 16, 12), ("relu",), ("dense", 12, 4)], [2, 4],
                   (1, 1, 0), (4, 2, 0), 16, 60, "sum", 0.9, 1.0, 0.0, "faithful_zero_updates", 0.05, ()),
    "mlp_k3_p2": ([("dense", 12, 16), ("relu",), ("dense", 16, 12), ("relu",), ("dense", 12, 4)], [2, 4],
                  (2, 2, 0), (6, 3, 0), 16, 40, "sum", 0.9, 0.7, 1e-3, "discard_warmup_updates", 0.05, ((20, 0.5),)),
    "mlp_k1_sgd": ([("dense", 12, 16), ("relu",), ("dense", 16, 12), ("relu",), ("dense", 12, 4)], [],
                   (0,), (0,), 16, 30, "sgd", 0.0, 1.0, 0.0, "faithful_zero_updates", 0.05, ()),
    "mlp_k2_tanh": ([("dense", 12, 8), ("tanh",), ("dense", 8, 4)], [2], (1, 0), (3, 1), 8, 25, "sgd", 0.0,
                    1.0, 0.0, "faithful_zero_updates", 0.05, ()),
}


def _mk_layers(sp, spec):
    out = []
    for t in spec:
        if t[0] == "dense":
            out.append(sp.dense(t[1], t[2]))
        elif t[0] == "relu":
            out.append(sp.relu())
        else:
            out.append(sp.tanh())
    return out


def gen_mlp(sp):
    from stalepipe.data import epoch_stream
    from stalepipe.pipeline import TrainEngine, validate_config

    ds = sp.gen_teacher_dataset(sp.TeacherSpec(dims=(12, 8, 4), n=400, seed=3))
    for name, (lay, bnd, p, m, B, steps, rule, beta, s, wd, warm, lr, dec) in MLP_CASES.items():
        model = sp.build_model(_mk_layers(sp, lay), bnd)
        sp.init_params(model, 11)
        init = model.flat_params().copy()
        eng = TrainEngine(model, validate_config(p, m, warmup=warm), epoch_stream(ds, B, 5),
                          sp.LrSchedule(lr, dec), rule=rule, beta=beta, s=s, weight_decay=wd)
        eng.run(steps)
        arrs = _log_arrays(eng.log)
        np.savez_compressed(os.path.join(OUT, f"{name}.npz"), init=init, final=model.flat_params(),
                            checksum=np.array(eng.log.checksum()), staleness=np.array(eng.realized_staleness()),
                            **arrs)
        print(name, eng.log.checksum()[:16])


def gen_cnn(sp):
    """Reference engine + oracle CNN math (flattened (B, C*H*W) packets)."""
    import stalepipe.pipeline as spp

    sys.path.insert(0, ROOT)
    import oracle.dsp_ref as R

    shape = (3, 8, 8)
    olayers = [R.conv_bn_relu(shape, 8), R.basic_unit((8, 8, 8), 8, 1), R.basic_unit((8, 8, 8), 16, 2),
               R.avgpool((16, 4, 4)), R.dense(16, 10)]
    om = R.build_model(olayers, [2])
    R.init_params(om, 0)
    init = om.flat_params().copy()

    class Shim:  # duck-typed model the reference engine drives (uses .k, .block_input_dims, .blocks[k].params)
        def __init__(self, m):
            self.m = m
            self.blocks = m.blocks
            self.k = m.k
            self.block_input_dims = m.block_input_dims

    orig_f, orig_b = spp.block_forward, spp.block_backward
    spp.block_forward = R.block_forward
    spp.block_backward = R.block_backward
    try:
        pool = R.synthetic_batches(5, 8, shape, 10, seed=1)
        eng = spp.TrainEngine(Shim(om), spp.validate_config((1, 0), (2, 0)), R.cycle(pool),
                              sp.LrSchedule(0.05, ((6, 0.5),)), rule="sum", beta=0.9, weight_decay=5e-4)
        eng.run(12)
    finally:
        spp.block_forward, spp.block_backward = orig_f, orig_b
    arrs = _log_arrays(eng.log)
    np.savez_compressed(os.path.join(OUT, "cnn_k2.npz"), init=init, final=om.flat_params(),
                        checksum=np.array(eng.log.checksum()), staleness=np.array(eng.realized_staleness()), **arrs)
    print("cnn_k2", eng.log.checksum()[:16])


# BASELINE configs[0]: ResNet-20 (width 16) split into K=2 DSP blocks, synthetic 32x32x3
# CIFAR-shaped data, batch 32, SUM momentum (beta 0.9), default queues p=(1,0), m=(2,0).
# configs[1]: ResNet-56, K=4 (p=(1,1,1,0), m=(6,4,2,0)), batch 128.  Both run past the CUDA-graph
# capture horizon of either engine (Python 9 / native 12 steps at K=4) into graph replays.
# Final parameters are stored every `stride`-th element (fixture size), plus full norms.
CONFIGS = {
    "c1_resnet20_k2": dict(depth=20, width=16, classes=10, batch=32, steps=24, pool=8, data_seed=7, init_seed=0,
                           p=(1, 0), m=(2, 0), boundaries=[5], lr=0.05, decays=((12, 0.5),), wd=5e-4, beta=0.9,
                           s=1.0, stride=4),
    "c2_resnet56_k4": dict(depth=56, width=16, classes=10, batch=128, steps=24, pool=8, data_seed=11, init_seed=0,
                           p=(1, 1, 1, 0), m=(6, 4, 2, 0), boundaries=[7, 13, 19], lr=0.05, decays=((12, 0.5),),
                           wd=5e-4, beta=0.9, s=1.0, stride=16),
}


def resnet_cifar_oracle_layers(R, depth, width, classes, in_shape=(3, 32, 32)):
    """ResNet-(6n+2): stem conv-BN-ReLU, 3 stages of n basic units (stride 2 + 1x1 projection at
    stages 2, 3), global average pool, dense head -- the product's resnet_cifar_layers."""
    n = (depth - 2) // 6
    L = [R.conv_bn_relu(in_shape, width)]
    shape = (width,) + tuple(in_shape[1:])
    for stage in range(3):
        c = width << stage
        for u in range(n):
            stride = 2 if (stage > 0 and u == 0) else 1
            L.append(R.basic_unit(shape, c, stride))
            shape = (c, (shape[1] - 1) // stride + 1, (shape[2] - 1) // stride + 1)
    L.append(R.avgpool(shape))
    L.append(R.dense(shape[0], classes))
    return L


def divergence(records, params, g):
    """(loss, grad norm, params) divergence of a run from a config golden: max over steps of
    |dL| / max(1, |L|), max over (step, block) of |dg| / max(g, 1e-3), max over blocks of the
    relative L2 error of the final parameters (every g["stride"]-th element).  records: sorted
    by (step, block), with .loss (None off the last block) and .grad_norm."""
    le = ge = 0.0
    for r, wl, wg in zip(records, g["loss"], g["grad_norm"]):
        if r.loss is not None:
            le = max(le, abs(r.loss - wl) / max(1.0, abs(wl)))
        ge = max(ge, abs(r.grad_norm - wg) / max(wg, 1e-3))
    st = int(g["stride"])
    pe = 0.0
    for k, p in enumerate(params):
        want = g[f"final_{k}"]
        pe = max(pe, float(np.linalg.norm(np.asarray(p, dtype=np.float64)[::st] - want) / np.linalg.norm(want)))
    return np.array([le, ge, pe])


def _oracle_model(R, c):
    om = R.build_model(resnet_cifar_oracle_layers(R, c["depth"], c["width"], c["classes"]), c["boundaries"])
    R.init_params(om, c["init_seed"])
    return om


def _pool(R, c):
    return R.synthetic_batches(c["pool"], c["batch"], (3, 32, 32), c["classes"], seed=c["data_seed"])


def gen_config(sp, name):
    """One BASELINE config through the UNMODIFIED reference TrainEngine driving the oracle's
    float64 CNN math (block_forward / block_backward patched, as gen_cnn): the trajectory the GPU
    tests (tests/test_configs_gpu.py) compare the device against, in both precisions.

    The trajectory is chaotic (BatchNorm over a small batch, ReLU-mask flips, faithful zero-packet
    updates): any rounding moves it.  So the fixture also records each precision's NOISE FLOOR --
    the divergence from the float64 golden of the oracle's own engine run with the device's
    arithmetic emulated: "f32" = every stored tensor rounded to float32 and float32 conv GEMMs
    (the device's fp32 mode), "bf16" = bf16 rounding at the device's storage points (bf16 mode)."""
    import stalepipe.pipeline as spp

    sys.path.insert(0, ROOT)
    import oracle.dsp_ref as R

    c = CONFIGS[name]
    om = _oracle_model(R, c)
    init = om.flat_params().copy()

    class Shim:
        def __init__(self, m):
            self.blocks, self.k, self.block_input_dims = m.blocks, m.k, m.block_input_dims

    orig_f, orig_b = spp.block_forward, spp.block_backward
    spp.block_forward, spp.block_backward = R.block_forward, R.block_backward
    try:
        eng = spp.TrainEngine(Shim(om), spp.validate_config(c["p"], c["m"]), R.cycle(_pool(R, c)),
                              sp.LrSchedule(c["lr"], c["decays"]), rule="sum", beta=c["beta"], s=c["s"],
                              weight_decay=c["wd"])
        eng.run(c["steps"])
    finally:
        spp.block_forward, spp.block_backward = orig_f, orig_b
    arrs = _log_arrays(eng.log)
    st = c["stride"]
    finals = {f"final_{k}": b.params[::st].copy() for k, b in enumerate(om.blocks)}
    norms = np.array([np.linalg.norm(b.params) for b in om.blocks])
    gold = dict(init_norm=np.linalg.norm(init), final_norms=norms, stride=np.array(st),
                boundaries=np.array(c["boundaries"]), checksum=np.array(eng.log.checksum()),
                staleness=np.array(eng.realized_staleness()), **finals, **arrs)
    for mode, acc in (("f32", "f32"), ("bf16", "f64")):
        with R.storage(mode, acc=acc):
            fm = _oracle_model(R, c)
            fe = R.Engine(fm, R.validate_config(c["p"], c["m"]), R.cycle(_pool(R, c)),
                          R.LrSchedule(c["lr"], c["decays"]), rule="sum", beta=c["beta"], s=c["s"],
                          weight_decay=c["wd"])
            fe.run(c["steps"])
        recs = sorted(fe.records, key=lambda r: (r.step, r.block))
        gold[f"floor_{mode}"] = divergence(recs, [b.params for b in fm.blocks], gold)
        print(name, "floor", mode, gold[f"floor_{mode}"])
    np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **gold)
    print(name, eng.log.checksum()[:16])


def gen_kats(sp):
    from stalepipe.optim import OptimizerState, lr_at, sgd_step, sum_step
    from stalepipe.rng import SeededRng, derive_seed

    rng = SeededRng(5)
    x0 = rng.normal(64)
    xs = x0.copy()
    st = OptimizerState.for_params("sum", xs, beta=0.9, s=0.7)
    gs = [rng.normal(64) for _ in range(20)]
    for g in gs:
        xs = sum_step(st, xs, g, 0.03)
    xg = x0.copy()
    for g in gs:
        xg = sgd_step(xg, g, 0.03)
    ds = sp.gen_teacher_dataset(sp.TeacherSpec(dims=(16, 32, 4), n=2000, seed=42))
    r7 = SeededRng(7)
    np.savez_compressed(os.path.join(OUT, "kats.npz"), x0=x0, grads=np.stack(gs), sum_final=xs, sum_ys=st.ys,
                        sgd_final=xg, lr=np.array([lr_at(sp.LrSchedule(0.01, ((150, 0.1), (225, 0.1))), n)
                                                   for n in range(300)]),
                        rng_u=r7.uniform(17), rng_n=r7.normal(9), rng_perm=r7.permutation(23),
                        derive=np.array([derive_seed(0, 1), derive_seed(123, 4)], dtype=np.uint64),
                        teacher_hist=np.bincount(ds.labels, minlength=4), teacher_first=ds.labels[:16])


def main():
    os.makedirs(OUT, exist_ok=True)
    sp = _ref()
    gen_mlp(sp)
    gen_cnn(sp)
    gen_kats(sp)
    for name in CONFIGS:
        gen_config(sp, name)


if __name__ == "__main__":
    main()
