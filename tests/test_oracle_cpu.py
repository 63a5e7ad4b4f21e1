"""Pin the CPU oracle against fixtures produced by the unmodified reference.

tests/golden/*.npz were written by oracle/make_golden.py from `stalepipe`
itself. The oracle must reproduce them bitwise: same FIFO schedule, same
float64 losses / grad norms (TrainLog checksum) and the same final params.
When the reference checkout is present the same runs are also re-executed live.
"""

import os

import numpy as np
import pytest

import oracle.dsp_ref as R
from paper_1909_02625_b200.data import TeacherSpec, epoch_stream, gen_teacher_dataset

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _gold(name):
    return np.load(os.path.join(GOLD, name + ".npz"))


MLP = {
    "mlp_k3_sum": ([R.dense(12, 16), R.relu(), R.dense(16, 12), R.relu(), R.dense(12, 4)], [2, 4], (1, 1, 0),
                   (4, 2, 0), 16, 60, "sum", 0.9, 1.0, 0.0, "faithful_zero_updates", 0.05, ()),
    "mlp_k3_p2": ([R.dense(12, 16), R.relu(), R.dense(16, 12), R.relu(), R.dense(12, 4)], [2, 4], (2, 2, 0),
                  (6, 3, 0), 16, 40, "sum", 0.9, 0.7, 1e-3, "discard_warmup_updates", 0.05, ((20, 0.5),)),
    "mlp_k1_sgd": ([R.dense(12, 16), R.relu(), R.dense(16, 12), R.relu(), R.dense(12, 4)], [], (0,), (0,), 16, 30,
                   "sgd", 0.0, 1.0, 0.0, "faithful_zero_updates", 0.05, ()),
    "mlp_k2_tanh": ([R.dense(12, 8), R.tanh(), R.dense(8, 4)], [2], (1, 0), (3, 1), 8, 25, "sgd", 0.0, 1.0, 0.0,
                    "faithful_zero_updates", 0.05, ()),
}


@pytest.mark.parametrize("name", sorted(MLP))
def test_oracle_reproduces_reference_mlp_bitwise(name):
    lay, bnd, p, m, B, steps, rule, beta, s, wd, warm, lr, dec = MLP[name]
    g = _gold(name)
    model = R.build_model(lay, bnd)
    R.init_params(model, 11)
    assert np.array_equal(model.flat_params(), g["init"]), "init_params differs from the reference"
    ds = gen_teacher_dataset(TeacherSpec((12, 8, 4), 400, 3))
    eng = R.Engine(model, R.validate_config(p, m, warmup=warm), epoch_stream(ds, B, 5), R.LrSchedule(lr, dec),
                   rule=rule, beta=beta, s=s, weight_decay=wd)
    eng.run(steps)
    recs = sorted(eng.records, key=lambda r: (r.step, r.block))
    assert [r.batch_index for r in recs] == list(g["batch_index"])
    assert eng.checksum() == str(g["checksum"])
    assert np.array_equal(model.flat_params(), g["final"])
    assert eng.realized_staleness() == list(g["staleness"])


def test_oracle_cnn_matches_reference_engine_driven_run():
    """cnn_k2.npz = reference TrainEngine driving the oracle CNN math; the oracle's
    own engine must give the identical trajectory (schedule, warmup, optimizer)."""
    g = _gold("cnn_k2")
    shape = (3, 8, 8)
    lay = [R.conv_bn_relu(shape, 8), R.basic_unit((8, 8, 8), 8, 1), R.basic_unit((8, 8, 8), 16, 2),
           R.avgpool((16, 4, 4)), R.dense(16, 10)]
    om = R.build_model(lay, [2])
    R.init_params(om, 0)
    assert np.array_equal(om.flat_params(), g["init"])
    pool = R.synthetic_batches(5, 8, shape, 10, seed=1)
    eng = R.Engine(om, R.validate_config((1, 0), (2, 0)), R.cycle(pool), R.LrSchedule(0.05, ((6, 0.5),)),
                   rule="sum", beta=0.9, weight_decay=5e-4)
    eng.run(12)
    assert eng.checksum() == str(g["checksum"])
    assert np.array_equal(om.flat_params(), g["final"])


def test_oracle_engine_reproduces_baseline_config0_golden():
    """c1_resnet20_k2.npz = BASELINE configs[0] (ResNet-20 w16, K=2, B=32, SUM 0.9, 24 steps)
    through the reference TrainEngine driving the oracle CNN math; the oracle's own engine gives
    the identical schedule and checksum, and the product's layer builder / cuts / init give the
    same model (so the GPU tests of tests/test_configs_gpu.py compare like with like)."""
    from oracle.make_golden import CONFIGS, resnet_cifar_oracle_layers

    import paper_1909_02625_b200 as P

    g = _gold("c1_resnet20_k2")
    c = CONFIGS["c1_resnet20_k2"]
    lay = resnet_cifar_oracle_layers(R, c["depth"], c["width"], c["classes"])
    play = P.resnet_cifar_layers(c["depth"], c["classes"], width=c["width"])
    assert [(s.kind, tuple(s.in_shape), s.out_c, s.stride) for s in lay] == \
        [(s.kind, tuple(s.in_shape), s.out_c, s.stride) for s in play]
    assert P.flop_balanced_boundaries(play, 2) == c["boundaries"] == list(g["boundaries"])
    om = R.build_model(lay, c["boundaries"])
    R.init_params(om, c["init_seed"])
    pm = P.build_model(play, c["boundaries"])
    P.init_params(pm, c["init_seed"])
    assert np.array_equal(om.flat_params(), pm.flat_params())
    assert np.linalg.norm(om.flat_params()) == float(g["init_norm"])
    pool = R.synthetic_batches(c["pool"], c["batch"], (3, 32, 32), c["classes"], seed=c["data_seed"])
    eng = R.Engine(om, R.validate_config(c["p"], c["m"]), R.cycle(pool), R.LrSchedule(c["lr"], c["decays"]),
                   rule="sum", beta=c["beta"], s=c["s"], weight_decay=c["wd"])
    eng.run(c["steps"])
    assert eng.checksum() == str(g["checksum"])
    st = int(g["stride"])
    for k, b in enumerate(om.blocks):
        assert np.array_equal(b.params[::st], g[f"final_{k}"])
    assert eng.realized_staleness() == list(g["staleness"])


def test_optimizer_and_rng_kats():
    k = _gold("kats")
    xs = k["x0"].copy()
    st = R.OptimizerState.for_params("sum", xs, beta=0.9, s=0.7)
    for gr in k["grads"]:
        xs = R.sum_step(st, xs, gr, 0.03)
    assert np.array_equal(xs, k["sum_final"]) and np.array_equal(st.ys, k["sum_ys"])
    xg = k["x0"].copy()
    for gr in k["grads"]:
        xg = R.sgd_step(xg, gr, 0.03)
    assert np.array_equal(xg, k["sgd_final"])
    sched = R.LrSchedule(0.01, ((150, 0.1), (225, 0.1)))
    assert np.array_equal([R.lr_at(sched, n) for n in range(300)], k["lr"])
    r7 = R.SeededRng(7)
    assert np.array_equal(r7.uniform(17), k["rng_u"])
    assert np.array_equal(r7.normal(9), k["rng_n"])
    assert np.array_equal(r7.permutation(23), k["rng_perm"])
    assert [R.derive_seed(0, 1), R.derive_seed(123, 4)] == [int(v) for v in k["derive"]]


def test_reference_hand_values():
    """Known answers from the reference's own tests (test_optim.py:10-37, test_pipeline.py:35-76)."""
    assert R.sgd_step(np.array([1.0]), np.array([0.5]), 0.1)[0] == 1.0 - 0.1 * 0.5
    st = R.OptimizerState.for_params("sum", np.array([1.0]), beta=0.9, s=1.0)
    assert abs(R.sum_step(st, np.array([1.0]), np.array([0.5]), 0.1)[0] - 0.905) < 1e-15
    x = np.array([1.0])
    for _ in range(10):
        x = R.sgd_step(x, x, 0.1)
    assert abs(x[0] - 0.9**10) < 1e-15
    for p, m, q in [((1, 1, 0), (4, 2, 0), (0, 1, 1)), ((2, 2, 0), (6, 3, 0), (0, 1, 1)),
                    ((3, 3, 0), (10, 5, 0), (0, 2, 2))]:
        assert R.validate_config(p, m).q == q
    with pytest.raises(R.ConfigError) as e:
        R.validate_config((1, 1, 0), (2, 2, 0))
    assert e.value.constraint == "q_positive" and e.value.index == 1 and "2-1-2 = -1" in str(e.value)
    loss, grad = R.softmax_xent(np.array([[0.0, 0.0]]), np.array([0]))
    assert abs(loss - np.log(2)) < 1e-12 and np.allclose(grad, [[-0.5, 0.5]])


def test_teacher_dataset_golden_histogram():
    """test_data.py:32-36 golden class histogram for TeacherSpec((16,32,4),2000,42)."""
    k = _gold("kats")
    ds = gen_teacher_dataset(TeacherSpec((16, 32, 4), 2000, 42))
    assert list(np.bincount(ds.labels, minlength=4)) == [430, 468, 620, 482] == list(k["teacher_hist"])
    assert np.array_equal(ds.labels[:16], k["teacher_first"])


def test_warmup_tags_dsp_1_0_3_1():
    """test_pipeline.py:170-180: block tags [-3,-2,-1,0] and [-2,-1,0,1]."""
    ds = gen_teacher_dataset(TeacherSpec((12, 8, 4), 400, 3))
    model = R.build_model([R.dense(12, 8), R.relu(), R.dense(8, 4)], [2])
    R.init_params(model, 2)
    eng = R.Engine(model, R.validate_config((1, 0), (3, 1)), epoch_stream(ds, 8, 5), R.LrSchedule(0.05))
    eng.run(4)
    tags = {(r.block, r.step): r.batch_index for r in eng.records}
    assert [tags[(0, n)] for n in range(4)] == [-3, -2, -1, 0]
    assert [tags[(1, n)] for n in range(4)] == [-2, -1, 0, 1]


def test_survey_appendix_a_tables():
    """Stale tags per block over steps 0..9 (dumped from the reference)."""
    cases = {((1, 1, 0), (4, 2, 0)): [(-4, 5), (-3, 6), (-2, 7)],
             ((1, 1, 1, 0), (6, 4, 2, 0)): [(-6, 3), (-5, 4), (-4, 5), (-3, 6)],
             ((2, 2, 0), (6, 3, 0)): [(-6, 3), (-5, 4), (-4, 5)]}
    for (p, m), spans in cases.items():
        K = len(p)
        layers = []
        for k in range(K):
            layers += [R.dense(4, 4), R.relu()] if k < K - 1 else [R.dense(4, 3)]
        bounds = [2 * (k + 1) for k in range(K - 1)]
        model = R.build_model(layers, bounds)
        R.init_params(model, 0)
        pool = R.synthetic_batches(2, 2, (4, 1, 1), 3, seed=0)
        eng = R.Engine(model, R.validate_config(p, m), R.cycle(pool), R.LrSchedule(0.01))
        eng.run(10)
        for k, (a, b) in enumerate(spans):
            assert [r.batch_index for r in eng.records if r.block == k] == list(range(a, b + 1))


@pytest.mark.reference
def test_live_reference_cnn_driven(stalepipe):
    """Re-run the reference engine live with the oracle CNN math and compare to the fixture."""
    import stalepipe.pipeline as spp

    g = _gold("cnn_k2")
    shape = (3, 8, 8)
    lay = [R.conv_bn_relu(shape, 8), R.basic_unit((8, 8, 8), 8, 1), R.basic_unit((8, 8, 8), 16, 2),
           R.avgpool((16, 4, 4)), R.dense(16, 10)]
    om = R.build_model(lay, [2])
    R.init_params(om, 0)
    orig = spp.block_forward, spp.block_backward
    spp.block_forward, spp.block_backward = R.block_forward, R.block_backward
    try:
        eng = spp.TrainEngine(om, spp.validate_config((1, 0), (2, 0)),
                              R.cycle(R.synthetic_batches(5, 8, shape, 10, seed=1)),
                              stalepipe.LrSchedule(0.05, ((6, 0.5),)), rule="sum", beta=0.9, weight_decay=5e-4)
        eng.run(12)
    finally:
        spp.block_forward, spp.block_backward = orig
    assert eng.log.checksum() == str(g["checksum"])


def test_theory_port_matches_reference(stalepipe):
    """theory.py (Lemma-1 bookkeeping over deviation rows) vs the reference's theory module."""
    import paper_1909_02625_b200.theory as T
    from paper_1909_02625_b200.deviation import DeviationRow
    import stalepipe.theory as RT

    rng = np.random.default_rng(3)
    rows = []
    for b in range(6):
        diffs = list(np.abs(rng.standard_normal(3)))
        if b == 2:
            diffs = [0.0, 0.0, 0.0]
        rows.append(DeviationRow(batch_index=5 * b, raw=list(np.abs(rng.standard_normal(3))), per_param=[0.0] * 3,
                                 raw_fwd=[0.0] * 3 if b == 2 else list(np.abs(rng.standard_normal(3))), diffs=diffs,
                                 upstream_norms=list(np.abs(rng.standard_normal(3))), steps=[b, b + 1, b + 2]))
    assert T.estimate_constants(rows) == RT.estimate_constants(rows)
    L, M = T.estimate_constants(rows)
    for LL, MM in ((L, M), (0.5 * L, M), (1.0, 1.0)):
        assert T.lemma1_report(rows, LL, MM) == RT.lemma1_report(rows, LL, MM)
    assert T.lemma_bound_rhs(2.0, 3.0, [1.0, 0.5, 0.25]) == RT.lemma_bound_rhs(2.0, 3.0, [1.0, 0.5, 0.25])
    assert T.lemma1_report(rows, L, M)["holds_fraction"] == 1.0


def test_des_restatement_matches_reference(stalepipe):
    """calibrate.simulate_dsp / simulate_bp vs the reference's simulate.py on the same costs."""
    import importlib

    from paper_1909_02625_b200 import calibrate as CAL

    S = importlib.import_module("stalepipe.simulate")
    import paper_1909_02625_b200 as P

    f, b = (1.0, 2.5, 0.7, 1.3), (2.0, 3.1, 1.9, 2.2)
    for p, m in (((1, 1, 1, 0), (6, 4, 2, 0)), ((2, 1, 1, 0), (7, 4, 2, 0))):
        cfg_ref = stalepipe.validate_config(p, m)
        ref, _ = S.simulate("dsp", S.CostModel(f, b, transfer_cost=0.05), 40, cfg_ref)
        mine = CAL.simulate_dsp(f, b, P.validate_config(p, m), 40, link=0.05)
        assert mine["makespan"] == ref.makespan and mine["steady_interval"] == ref.steady_interval
        strag = S.StragglerModel(prob=0.3, rho=0.5, seed=4)
        ref2, _ = S.simulate("dsp", S.CostModel(f, b), 40, cfg_ref, strag)
        mult = CAL.straggler_multipliers(4, 40, 0.3, 0.5, seed=4)
        assert CAL.simulate_dsp(f, b, P.validate_config(p, m), 40, mult=mult)["makespan"] == ref2.makespan
        ref3, _ = S.simulate("sync_bp", S.CostModel(f, b), 40, None, strag)
        assert CAL.simulate_bp(f, b, 40, mult=mult)["makespan"] == ref3.makespan
