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


if __name__ == "__main__":
    main()
