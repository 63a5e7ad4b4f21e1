"""Gradient-deviation diagnostics on the device (deviation.py).

Ports the reference's TestDeviation (/root/reference/pkg/tests/test_pipeline.py:314-375) to
the B200 engine: zero staleness gives exactly zero deviation, the runtime gradient equals the
device stale_gradient operator bit for bit, grad_deviation of BP gradients is zero, deviations
collapse near convergence; plus the operators against the oracle on a CNN.
"""

import numpy as np
import pytest

import oracle.dsp_ref as R
import paper_1909_02625_b200 as P
from paper_1909_02625_b200.data import epoch_stream
from paper_1909_02625_b200.deviation import DeviceOperators
from paper_1909_02625_b200.runtime import pack_input, torch_mod
from tests.gpu_util import rel_err, small_resnet, twin_models

pytestmark = pytest.mark.gpu


def toy_dataset(seed=3, n=400, d=12, c=4):
    return P.gen_teacher_dataset(P.TeacherSpec(dims=(d, 8, c), n=n, seed=seed))


def toy_layers():
    return [P.dense(12, 16), P.relu(), P.dense(16, 12), P.relu(), P.dense(12, 4)]


def toy_model(seed=11, boundaries=(2, 4)):
    m = P.build_model(toy_layers(), list(boundaries))
    P.init_params(m, seed)
    return m


def test_zero_staleness_deviation_exactly_zero():
    model = P.build_model(toy_layers(), [])
    P.init_params(model, 6)
    eng = P.TrainEngine(model, P.validate_config((0,), (0,)), epoch_stream(toy_dataset(), 16, 5),
                        P.LrSchedule(0.05), deviation_every=3)
    eng.run(30)
    rows = eng.deviation_rows()
    assert len(rows) >= 9
    for row in rows:
        assert row.raw == [0.0]
        assert row.raw_fwd == [0.0]
        assert row.diffs == [0.0]
    devs = [r.grad_deviation for r in eng.log.records if r.grad_deviation is not None]
    assert len(devs) == len(rows) and all(d == 0.0 for d in devs)


def test_runtime_gradients_match_device_operator_bitwise():
    eng = P.TrainEngine(toy_model(11), P.validate_config((1, 1, 0), (4, 2, 0)),
                        epoch_stream(toy_dataset(), 16, 5), P.LrSchedule(0.05), deviation_every=5)
    captured = []
    original = eng.tracker._score

    def capture(sample):
        captured.append(sample)
        return original(sample)

    eng.tracker._score = capture
    eng.run(60)
    assert len(captured) >= 6
    ops = eng.tracker.ops
    for s in captured[:6]:
        fwd = [s.fwd[k] for k in range(3)]
        bwd = [s.bwd[k] for k in range(3)]
        grads = ops.stale_gradient(fwd, bwd, s.x, s.labels)
        for k in range(3):
            assert bool((grads[k] == s.grads[k]).all()), (s.batch_index, k)
    rows = eng.deviation_rows()
    assert all(r.raw[2] >= 0 for r in rows)
    assert any(max(r.diffs[:2]) > 0 for r in rows)  # stale blocks see moved parameters


def test_grad_deviation_op_zero_for_bp_grads():
    torch = torch_mod()
    model = toy_model(2)
    rng = P.SeededRng(15)
    x = rng.normal(4 * 12).reshape(4, 12)
    labels = (rng.uniform(4) * 4).astype(np.int64)
    ops = DeviceOperators(model, 4)
    dev = ops.blocks[0].device
    xd = pack_input(x, model.blocks[0].in_shape, dev, ops.stream)
    ld = torch.tensor(labels, device=dev)
    params = [torch.tensor(b.params, dtype=torch.float32, device=dev) for b in model.blocks]
    grads = ops.bp_gradient(params, xd, ld)
    rows = ops.grad_deviation(params, xd, ld, grads)
    assert all(r["raw"] == 0.0 for r in rows)


def test_deviation_shrinks_near_convergence():
    ds = P.gen_teacher_dataset(P.TeacherSpec(dims=(6, 4, 3), n=64, seed=9))
    layers = [P.dense(6, 16), P.relu(), P.dense(16, 8), P.relu(), P.dense(8, 3)]
    model = P.build_model(layers, [2, 4])
    P.init_params(model, 8)
    eng = P.TrainEngine(model, P.validate_config((1, 1, 0), (4, 2, 0)), epoch_stream(ds, 32, 5),
                        P.LrSchedule(0.1), rule="sum", beta=0.9, deviation_every=10)
    eng.run(800)
    rows = eng.deviation_rows()
    early = np.median([max(r.raw) for r in rows[1:8]])
    late = np.median([max(r.raw) for r in rows[-8:]])
    assert late < early / 10


def test_cnn_operators_match_oracle():
    """Device bp_gradient / stale_gradient on a 3-block CNN vs the oracle's operators
    (bf16-storage emulation) on the same snapshots."""
    torch = torch_mod()
    layers = small_resnet(in_shape=(3, 8, 8))
    bounds = [2, 4]
    pm, om = twin_models(layers, bounds, seed=4)
    B = 8
    x, lab = R.synthetic_batches(1, B, (3, 8, 8), 10, seed=7)[0]
    rng = np.random.default_rng(0)
    f32 = lambda p: p.astype(np.float32).astype(np.float64)  # noqa: E731  (device master precision)
    fwd = [f32(b.params) for b in pm.blocks]
    bwd = [f32(p + 0.01 * rng.standard_normal(p.size)) for p in fwd]
    ops = DeviceOperators(pm, B)
    dev = ops.blocks[0].device
    xd = pack_input(x, pm.blocks[0].in_shape, dev, ops.stream)
    ld = torch.tensor(lab, device=dev)
    to_dev = lambda ps: [torch.tensor(p, dtype=torch.float32, device=dev) for p in ps]  # noqa: E731
    g_bp = [g.double().cpu().numpy() for g in ops.bp_gradient(to_dev(bwd), xd, ld)]
    g_st = [g.double().cpu().numpy() for g in ops.stale_gradient(to_dev(fwd), to_dev(bwd), xd, ld)]
    with R.storage("bf16"):
        om.load_params(bwd)
        want_bp, _ = R.bp_gradient(om, R.cnn.bf16_round(x), lab)
        want_st, _ = R.stale_gradient(om, fwd, bwd, R.cnn.bf16_round(x), lab)
    for k in range(3):
        assert rel_err(g_bp[k], want_bp[k]) < 2e-2, ("bp", k, rel_err(g_bp[k], want_bp[k]))
        assert rel_err(g_st[k], want_st[k]) < 2e-2, ("stale", k, rel_err(g_st[k], want_st[k]))
