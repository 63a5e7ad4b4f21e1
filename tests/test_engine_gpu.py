"""End-to-end DSP train-step parity: B200 TrainEngine vs the oracle engine.

Same model init, same synthetic batches, same queue config and optimizer.
Checked against the oracle twice (see tests/test_block_gpu.py for the modes):
  * FIFO / staleness schedule: (step, block, batch_index) log bit-exact;
  * realized_staleness() == m;
  * per-step loss: |dL| <= LOSS_TOL[mode] * max(1, |L_ref|)
  * per-(step, block) grad norm: relative <= GN_TOL[mode]
  * final parameters per block: relative L2 error <= PARAM_TOL[mode].
"""

import numpy as np
import pytest

import oracle.dsp_ref as R
import paper_1909_02625_b200 as P
from tests.gpu_util import rel_err, small_resnet, twin_models

pytestmark = pytest.mark.gpu

LOSS_TOL = {"bf16": 1e-2, "f64": 5e-2}
GN_TOL = {"bf16": 3e-2, "f64": 2e-1}
PARAM_TOL = {"bf16": 2e-2, "f64": 1e-1}


def _run(layers, boundaries, p, m, B, steps, in_shape, classes, rule="sum", beta=0.9, lr=0.05,
         warmup="faithful_zero_updates", wd=0.0):
    pool = R.synthetic_batches(6, B, in_shape, classes, seed=1)
    sched = ((steps // 2, 0.5),)
    pm, _ = twin_models(layers, boundaries, seed=3)
    eng = P.TrainEngine(pm, P.validate_config(p, m, warmup=warmup), R.cycle(pool), P.LrSchedule(lr, sched),
                        rule=rule, beta=beta, weight_decay=wd)
    eng.run(steps)
    refs = {}
    for mode in ("bf16", "f64"):
        with R.storage(mode):
            _, om = twin_models(layers, boundaries, seed=3)
            ref = R.Engine(om, R.validate_config(p, m, warmup=warmup), R.cycle(pool), R.LrSchedule(lr, sched),
                           rule=rule, beta=beta, weight_decay=wd)
            ref.run(steps)
        refs[mode] = (ref, om)
    return eng, pm, refs


def _check(eng, pm, refs, m, scale=1.0):
    log = eng.log
    assert eng.realized_staleness() == list(m)
    for mode, (ref, om) in refs.items():
        got_idx = [(r.step, r.block, r.batch_index) for r in log.sorted()]
        want_idx = sorted((r.step, r.block, r.batch_index) for r in ref.records)
        assert got_idx == want_idx
        ref_loss = {r.step: r.loss for r in ref.records if r.loss is not None}
        for step, loss in log.losses():
            want = ref_loss[step]
            assert abs(loss - want) <= scale * LOSS_TOL[mode] * max(1.0, abs(want)), (mode, step, loss, want)
        ref_gn = {(r.step, r.block): r.grad_norm for r in ref.records}
        for r in log.records:
            want = ref_gn[(r.step, r.block)]
            assert abs(r.grad_norm - want) <= scale * GN_TOL[mode] * max(want, 1e-3), (mode, r.step, r.block, r.grad_norm,
                                                                             want)
        for bp, bo in zip(pm.blocks, om.blocks):
            assert rel_err(bp.params, bo.params) < scale * PARAM_TOL[mode], (mode, bp.index, rel_err(bp.params, bo.params))


def test_resnet_k2_sum():
    layers = small_resnet(in_shape=(3, 8, 8))
    eng, pm, refs = _run(layers, [2], (1, 0), (2, 0), 16, 12, (3, 8, 8), 10)
    _check(eng, pm, refs, (2, 0))


def test_resnet_k3_discard_warmup_sgd_wd():
    layers = small_resnet(in_shape=(3, 8, 8))
    eng, pm, refs = _run(layers, [2, 4], (1, 1, 0), (4, 2, 0), 8, 10, (3, 8, 8), 10, rule="sgd", beta=0.0,
                         warmup="discard_warmup_updates", wd=5e-4)
    _check(eng, pm, refs, (4, 2, 0))


def test_resnet_k4_default_queues():
    layers = small_resnet(in_shape=(3, 8, 8))
    cfg = P.default_queue_config(4)
    eng, pm, refs = _run(layers, [1, 2, 3], cfg.p, cfg.m, 8, 12, (3, 8, 8), 10)
    _check(eng, pm, refs, cfg.m)


def test_mlp_k3_reference_kinds():
    layers = [P.dense(12, 16), P.relu(), P.dense(16, 12), P.relu(), P.dense(12, 4)]
    eng, pm, refs = _run(layers, [2, 4], (1, 1, 0), (4, 2, 0), 16, 30, (12, 1, 1), 4)
    _check(eng, pm, refs, (4, 2, 0))


def test_k1_is_plain_bp():
    layers = small_resnet(in_shape=(3, 8, 8))
    eng, pm, refs = _run(layers, [], (0,), (0,), 16, 8, (3, 8, 8), 10, rule="sgd", beta=0.0)
    _check(eng, pm, refs, (0,))


def test_resume_equals_single_run():
    """run(a); run(b) == run(a+b): queue contents persist across calls (pipeline.py:443-449)."""
    layers = small_resnet(in_shape=(3, 8, 8))
    pool = R.synthetic_batches(4, 8, (3, 8, 8), 10, seed=4)
    finals = []
    for chunks in ((7,), (3, 4)):
        pm, _ = twin_models(layers, [2], seed=2)
        eng = P.TrainEngine(pm, P.validate_config((1, 0), (2, 0)), R.cycle(pool), P.LrSchedule(0.05), rule="sum",
                            beta=0.9)
        for c in chunks:
            eng.run(c)
        finals.append((pm.flat_params(), eng.log.checksum()))
    assert np.array_equal(finals[0][0], finals[1][0])
    assert finals[0][1] == finals[1][1]


def test_deterministic_across_runs():
    layers = small_resnet(in_shape=(3, 8, 8))
    pool = R.synthetic_batches(4, 8, (3, 8, 8), 10, seed=4)
    sums = []
    for _ in range(2):
        pm, _ = twin_models(layers, [1, 3], seed=2)
        eng = P.TrainEngine(pm, P.validate_config((1, 1, 0), (4, 2, 0)), R.cycle(pool), P.LrSchedule(0.05),
                            rule="sum", beta=0.9)
        eng.run(9)
        sums.append(eng.log.checksum())
    assert sums[0] == sums[1]


def test_eval_forward_matches_oracle():
    layers = small_resnet(in_shape=(3, 8, 8))
    pm, om = twin_models(layers, [2], seed=5)
    x, _ = R.synthetic_batches(1, 8, (3, 8, 8), 10, seed=2)[0]
    got = pm.forward(x)
    with R.storage("bf16"):
        want = om.forward(R.cnn.bf16_round(x))
    assert rel_err(got, want) < 1e-2


def test_tape_single_use():
    from paper_1909_02625_b200.runtime import DeviceBlock

    pm, _ = twin_models([P.dense(8, 8), P.relu(), P.dense(8, 4)], [], seed=1)
    db = DeviceBlock(pm.blocks[0], 4, is_last=True)
    with pytest.raises(P.DspError):
        db.backward(None, None)  # no recorded forward


def test_label_out_of_range_rejected():
    layers = [P.dense(12, 8), P.relu(), P.dense(8, 4)]
    pm, _ = twin_models(layers, [], seed=1)
    bad = [(np.zeros((4, 12)), np.array([0, 1, 2, 4]))]
    eng = P.TrainEngine(pm, P.validate_config((0,), (0,)), R.cycle(bad), P.LrSchedule(0.1))
    with pytest.raises(ValueError, match="label out of range"):
        eng.run(1)


def _divergence(records, losses, blocks, ref, oblocks):
    """(max loss err, max grad-norm err, max param err) of a run vs an oracle run."""
    rl = {r.step: r.loss for r in ref.records if r.loss is not None}
    le = max(abs(l - rl[s]) / max(1.0, abs(rl[s])) for s, l in losses)
    rg = {(r.step, r.block): r.grad_norm for r in ref.records}
    ge = max(abs(r.grad_norm - rg[(r.step, r.block)]) / max(rg[(r.step, r.block)], 1e-3) for r in records)
    pe = max(rel_err(a.params, b.params) for a, b in zip(blocks, oblocks))
    return np.array([le, ge, pe])


def test_resnet20_k8_default_queues_graph_replay():
    """K = 8 blocks (config 3 / 8-GPU shape) with the default queues; 22 steps run past the
    zero-prefill horizon (17) so CUDA-graph capture and replay are exercised.

    Over 20+ training steps bf16 trajectories diverge chaotically (BatchNorm over small batches,
    ReLU-mask flips), so the value bound is relative to the emulation's own noise floor, measured
    in the test: the bf16 emulation re-run with fp32 conv accumulation (an equally valid order).
    The device must stay within 3x of that floor (+0.5%); the schedule stays bit-exact."""
    layers = P.resnet_cifar_layers(20, 10, width=8)
    cfg = P.default_queue_config(8)
    bounds = P.flop_balanced_boundaries(layers, 8)
    B, steps, lr = 16, 22, 0.02
    eng, pm, refs = _run(layers, bounds, cfg.p, cfg.m, B, steps, (3, 32, 32), 10, lr=lr)
    assert eng.rt.graphs, "no step graph was captured"
    assert eng.realized_staleness() == list(cfg.m)
    ref, om = refs["bf16"]
    assert [(r.step, r.block, r.batch_index) for r in eng.log.sorted()] == \
        sorted((r.step, r.block, r.batch_index) for r in ref.records)
    pool = R.synthetic_batches(6, B, (3, 32, 32), 10, seed=1)
    with R.storage("bf16", acc="f32"):
        _, om32 = twin_models(layers, bounds, seed=3)
        ref32 = R.Engine(om32, R.validate_config(cfg.p, cfg.m), R.cycle(pool), R.LrSchedule(lr, ((steps // 2, 0.5),)),
                         rule="sum", beta=0.9)
        ref32.run(steps)
    floor = _divergence(ref32.records, [(r.step, r.loss) for r in ref32.records if r.loss is not None],
                        om32.blocks, ref, om.blocks)
    dev = _divergence(eng.log.records, eng.log.losses(), pm.blocks, ref, om.blocks)
    assert np.all(dev <= 3 * floor + 5e-3), ("device (loss, grad-norm, params) err", dev, "noise floor", floor)
    f64 = _divergence(eng.log.records, eng.log.losses(), pm.blocks, refs["f64"][0], refs["f64"][1].blocks)
    assert np.all(f64 <= [LOSS_TOL["f64"], GN_TOL["f64"], PARAM_TOL["f64"]]), f64


def test_resnet_k3_adam_extension():
    """rule="adam" (BASELINE configs[2]; an extension the reference rejects) vs the oracle's
    adam_step restatement, discard warmup + weight decay, lr decay mid-run.  Adam's normalised
    step turns the bf16 storage rounding into O(lr) parameter moves wherever g ~ 0, so the
    trajectory tolerances are 3x the SUM/SGD ones (the update kernel itself is pinned to 1e-5
    in tests/test_optim_gpu.py)."""
    layers = small_resnet(in_shape=(3, 8, 8))
    eng, pm, refs = _run(layers, [2, 4], (1, 1, 0), (4, 2, 0), 8, 12, (3, 8, 8), 10, rule="adam", beta=0.0,
                         lr=2e-3, warmup="discard_warmup_updates", wd=5e-4)
    _check(eng, pm, refs, (4, 2, 0), scale=3.0)
    for k in range(3):  # applied-update counter = steps whose stale tag is >= 0
        assert eng.rt.opt_state(k).n == sum(1 for r in eng.log.records if r.block == k and r.batch_index >= 0)


def test_forward_twin_is_bitwise_neutral(monkeypatch):
    """The fresh forward on a forward twin (own workspace + stream, dsp_block_share_weights)
    gives the same log and parameters, bit for bit, as the fresh forward on the block itself."""
    layers = small_resnet(in_shape=(3, 8, 8))
    cfg = P.default_queue_config(3)
    pool = R.synthetic_batches(6, 8, (3, 8, 8), 10, seed=1)
    runs = []
    for env in ("0", "1"):
        monkeypatch.setenv("DSP_B200_TWIN", env)
        pm, _ = twin_models(layers, [2, 4], seed=3)
        eng = P.TrainEngine(pm, cfg, R.cycle(pool), P.LrSchedule(0.05, ((8, 0.5),)), rule="sum", beta=0.9)
        assert bool(eng.rt.twins) == (env == "1")
        eng.run(16)
        runs.append((eng.log.checksum(), [b.params.copy() for b in pm.blocks]))
    assert runs[0][0] == runs[1][0]
    for a, b in zip(runs[0][1], runs[1][1]):
        assert np.array_equal(a, b)


def _nan_model(layers, boundaries, block, seed=1):
    pm, _ = twin_models(layers, boundaries, seed=seed)
    p = pm.blocks[block].params.copy()
    p[len(p) // 2] = np.nan
    pm.blocks[block].params = p
    return pm


@pytest.mark.parametrize("block", [0, 1])
def test_nonfinite_gradient_raises(block):
    """NonFiniteError (optim.py:53 / 89, tensor.py:101-111): a NaN parameter poisons the step; the
    device's sticky flag is raised at the next sync point (the log read)."""
    layers = small_resnet(in_shape=(3, 8, 8))
    pm = _nan_model(layers, [2], block)
    pool = R.synthetic_batches(3, 8, (3, 8, 8), 10, seed=1)
    eng = P.TrainEngine(pm, P.validate_config((1, 0), (2, 0)), R.cycle(pool), P.LrSchedule(0.05), rule="sum",
                        beta=0.9)
    eng.run(4)
    with pytest.raises(P.NonFiniteError, match="non-finite"):
        _ = eng.log


def test_nonfinite_native_engine_raises():
    layers = small_resnet(in_shape=(3, 8, 8))
    pm = _nan_model(layers, [2], 1)
    pool = R.synthetic_batches(3, 8, (3, 8, 8), 10, seed=1)
    eng = P.NativeEngine(pm, P.validate_config((1, 0), (2, 0)), 8, P.LrSchedule(0.05), rule="sum", beta=0.9)
    with pytest.raises(P.NonFiniteError, match="non-finite"):
        eng.run(4, R.cycle(pool))


def test_finite_run_does_not_raise():
    layers = small_resnet(in_shape=(3, 8, 8))
    pm, _ = twin_models(layers, [2], seed=1)
    pool = R.synthetic_batches(3, 8, (3, 8, 8), 10, seed=1)
    eng = P.TrainEngine(pm, P.validate_config((1, 0), (2, 0)), R.cycle(pool), P.LrSchedule(0.05), rule="sum",
                        beta=0.9)
    eng.run(6)
    eng.synchronize()
    assert all(np.isfinite(r.grad_norm) for r in eng.log.records)
