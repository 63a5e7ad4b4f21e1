"""Parity on the BASELINE configs themselves (not toy nets).

configs[0] (ResNet-20 w16, K=2, B=32) and configs[1] (ResNet-56, K=4, B=128), SUM momentum 0.9,
default queues, 24 steps -- past the CUDA-graph capture horizon of both engines, so captured and
replayed step graphs are covered.  The device runs through the Python drop-in
(``TrainEngine(backend="b200")``) and through the engine C-ABI (``NativeEngine`` -> ``dsp_run``),
in both precisions, against the goldens ``oracle/make_golden.py`` produced by driving the
UNMODIFIED reference ``TrainEngine`` with the oracle's float64 CNN math
(/root/reference/pkg/src/stalepipe/pipeline.py:538-606).

Two kinds of evidence:

* trajectories -- the FIFO schedule and realized staleness are exact.  Values: these 24-step
  trajectories are chaotic (BatchNorm over small batches, ReLU-mask flips, faithful zero-packet
  updates), so ANY rounding moves them: the oracle's own engine run with float32 arithmetic ends
  5-10% away from its float64 run (the golden's ``floor_f32``; ``floor_bf16`` for bf16 storage).
  Bounds: tight absolute bounds on the first steps, before the chaos has amplified the rounding
  (EARLY), and the whole run within FLOOR_X times the floor of the same arithmetic;
* teacher-forced operators -- at the device's trained state (after the 24 steps) the loss and the
  chained BP gradient of every block, computed by the device kernels and by the float64 oracle
  from the SAME parameters and batch (pipeline.py:256-267): no trajectory chaos is involved, only
  the ReLU-mask sensitivity of one backward pass, bounded against the oracle run with the same
  arithmetic emulated.
"""

import numpy as np
import pytest

import oracle.dsp_ref as R
import paper_1909_02625_b200 as P
from oracle.make_golden import CONFIGS, divergence, resnet_cifar_oracle_layers
from paper_1909_02625_b200.data import cycle, synthetic_batches
from tests.gpu_util import rel_err

pytestmark = pytest.mark.gpu

GOLDEN = "tests/golden/{}.npz"
FLOOR = {"fp32": "floor_f32", "bf16": "floor_bf16"}
# steps 0..EARLY_STEPS-1: (loss, grad norm) relative bounds against the float64 golden
EARLY_STEPS = 3
EARLY = {"fp32": (1e-5, 5e-4), "bf16": (1e-2, 3e-2)}
FLOOR_X, FLOOR_ABS = 3.0, 1e-2
# teacher-forced BP gradient per block: relative L2 error within OP_X x the emulated-arithmetic floor
# (+ OP_ABS); loss relative error
OP_X = 4.0
OP_ABS = {"fp32": 1e-3, "bf16": 2e-2}
OP_LOSS = {"fp32": 1e-6, "bf16": 5e-3}


def _setup(name):
    c = CONFIGS[name]
    layers = P.resnet_cifar_layers(c["depth"], c["classes"], width=c["width"])
    assert P.flop_balanced_boundaries(layers, len(c["p"])) == c["boundaries"]
    model = P.build_model(layers, c["boundaries"])
    P.init_params(model, c["init_seed"])
    g = np.load(GOLDEN.format(name))
    assert np.isclose(np.linalg.norm(model.flat_params()), float(g["init_norm"]), rtol=0, atol=1e-9)
    pool = synthetic_batches(c["pool"], c["batch"], (3, 32, 32), c["classes"], seed=c["data_seed"])
    return c, model, g, pool


def _check_trajectory(tag, records, params, g, precision):
    idx = [(r.step, r.block, r.batch_index) for r in records]
    assert idx == list(zip(g["step"].tolist(), g["block"].tolist(), g["batch_index"].tolist())), \
        "FIFO / staleness schedule differs from the reference"
    early = [r for r in records if r.step < EARLY_STEPS]
    pos = {(r.step, r.block): i for i, r in enumerate(records)}
    le = max((abs(r.loss - g["loss"][pos[(r.step, r.block)]]) / max(1.0, abs(g["loss"][pos[(r.step, r.block)]]))
              for r in early if r.loss is not None), default=0.0)
    ge = max(abs(r.grad_norm - g["grad_norm"][pos[(r.step, r.block)]]) / max(g["grad_norm"][pos[(r.step, r.block)]],
                                                                           1e-3) for r in early)
    div = divergence(records, params, g)
    floor = g[FLOOR[precision]]
    print(f"\n{tag}: early loss {le:.1e} gn {ge:.1e} | 24 steps (loss, gn, params) {np.array2string(div, precision=2)}"
          f" floor {np.array2string(floor, precision=2)}")
    assert le <= EARLY[precision][0] and ge <= EARLY[precision][1], (le, ge, EARLY[precision])
    assert np.all(div <= FLOOR_X * floor + FLOOR_ABS), (div, floor)
    assert np.all(np.isfinite(div))


@pytest.mark.parametrize("precision", ["fp32", "bf16"])
@pytest.mark.parametrize("name", sorted(CONFIGS))
def test_trajectory_python_engine(name, precision):
    c, model, g, pool = _setup(name)
    cfg = P.validate_config(c["p"], c["m"])
    eng = P.TrainEngine(model, cfg, cycle(pool), P.LrSchedule(c["lr"], c["decays"]), rule="sum", beta=c["beta"],
                        s=c["s"], weight_decay=c["wd"], precision=precision)
    eng.run(c["steps"])
    assert eng.rt.graphs, "no step graph was captured"
    assert eng.realized_staleness() == list(g["staleness"])
    _check_trajectory(f"{name} python {precision}", eng.log.sorted(), [b.params for b in model.blocks], g, precision)


@pytest.mark.parametrize("precision", ["fp32", "bf16"])
@pytest.mark.parametrize("name", sorted(CONFIGS))
def test_trajectory_native_engine(name, precision):
    c, model, g, pool = _setup(name)
    cfg = P.validate_config(c["p"], c["m"])
    eng = P.NativeEngine(model, cfg, c["batch"], P.LrSchedule(c["lr"], c["decays"]), rule="sum", beta=c["beta"],
                         s=c["s"], weight_decay=c["wd"], precision=precision)
    xs = np.stack([np.asarray(pool[i % len(pool)][0], dtype=np.float32) for i in range(c["steps"])])
    ls = np.stack([np.asarray(pool[i % len(pool)][1]) for i in range(c["steps"])])
    eng.run_batches(xs, ls)
    assert eng.steps_done == c["steps"] and c["steps"] > eng.horizon + eng.ring  # graph replays happened
    assert eng.realized_staleness() == list(g["staleness"])
    _check_trajectory(f"{name} native {precision}", eng.log.sorted(),
                      [eng.params(k) for k in range(len(c["p"]))], g, precision)


def _oracle_bp(c, params, x, lab, mode="f64", acc="f64"):
    with R.storage(mode, acc=acc):
        om = R.build_model(resnet_cifar_oracle_layers(R, c["depth"], c["width"], c["classes"]), c["boundaries"])
        for b, p in zip(om.blocks, params):
            b.params = np.asarray(p, dtype=np.float32).astype(np.float64)
        return R.bp_gradient(om, x, lab)


@pytest.mark.parametrize("precision", ["fp32", "bf16"])
@pytest.mark.parametrize("name", sorted(CONFIGS))
def test_bp_gradient_at_trained_state(name, precision):
    """Teacher-forced: after the 24 DSP steps, the device's chained BP gradient of every block vs the
    float64 oracle's from the same parameters on the same batch.  A trained state has many
    pre-activations within rounding of 0 (each ReLU-mask flip moves a whole upstream term), so the
    same computation in the oracle with the device's arithmetic emulated (``floor``) is measured
    beside it: the device must stay within OP_X x that floor (+ OP_ABS)."""
    import torch

    from paper_1909_02625_b200.deviation import DeviceOperators
    from paper_1909_02625_b200.runtime import pack_input

    c, model, g, pool = _setup(name)
    cfg = P.validate_config(c["p"], c["m"])
    eng = P.TrainEngine(model, cfg, cycle(pool), P.LrSchedule(c["lr"], c["decays"]), rule="sum", beta=c["beta"],
                        s=c["s"], weight_decay=c["wd"], precision=precision)
    eng.run(c["steps"])
    params = [b.params.copy() for b in model.blocks]  # the trained state (host float64 of the fp32 masters)
    x, lab = pool[3]
    ops = DeviceOperators(model, c["batch"], device=eng.rt.device, stream=eng.rt.stream, dtype=eng.rt.dtype_code)
    dev = eng.rt.device
    xd = pack_input(np.asarray(x), (3, 32, 32), dev, eng.rt.stream, dtype=eng.rt.dtype_code)
    ld = torch.from_numpy(np.asarray(lab, dtype=np.int64)).to(dev)
    got = ops.bp_gradient([torch.from_numpy(p.astype(np.float32)).to(dev) for p in params], xd, ld)
    eng.rt.stream.synchronize()
    loss_dev = float(ops.loss.item())
    want, loss_ref = _oracle_bp(c, params, x, lab)
    emu, _ = _oracle_bp(c, params, x, lab, *(("f32", "f32") if precision == "fp32" else ("bf16", "f64")))
    errs = np.array([rel_err(gd.double().cpu().numpy(), w) for gd, w in zip(got, want)])
    floor = np.array([rel_err(e, w) for e, w in zip(emu, want)])
    lerr = abs(loss_dev - loss_ref) / max(1.0, abs(loss_ref))
    print(f"\n{name} BP operator {precision}: per-block grad rel err {np.array2string(errs, precision=2)}"
          f" floor {np.array2string(floor, precision=2)} loss {lerr:.1e}")
    assert np.all(errs <= OP_X * floor + OP_ABS[precision]), (errs, floor)
    assert lerr <= OP_LOSS[precision], lerr


@pytest.mark.parametrize("precision", ["bf16", "fp32"])
def test_resnet50_config4_early_steps_vs_oracle(precision):
    """configs[4]'s network (ResNet-50, K=4 FLOP-balanced cuts, default queues, SUM momentum) on a
    2-sample batch for 5 steps, device (bf16 / fp32) vs the float64 oracle engine: the FIFO /
    staleness schedule exact, the loss and gradient norms within 3x the emulated floor + EARLY (every
    ResNet-50 kernel path in play: space-to-depth stem fused with the max pool, im2col / 2-D TMA
    operands, TMA-stored slabs, parity-split stride-2 DGRAD, projection units, 1000-way head)."""
    from tests.gpu_util import twin_models

    layers = P.resnet50_layers()
    bounds = P.flop_balanced_boundaries(layers, 4)
    cfg = P.default_queue_config(4)
    B, steps = 2, 5
    pool = R.synthetic_batches(3, B, (3, 224, 224), 1000, seed=5)
    pm, _ = twin_models(layers, bounds, seed=0)
    eng = P.TrainEngine(pm, cfg, cycle(pool), P.LrSchedule(0.05), rule="sum", beta=0.9, weight_decay=5e-4,
                        precision=precision)
    eng.run(steps)
    def oracle_run(mode):
        _, om2 = twin_models(layers, bounds, seed=0)
        with R.storage(mode):
            ref = R.Engine(om2, R.validate_config(cfg.p, cfg.m), R.cycle(pool), R.LrSchedule(0.05), rule="sum",
                           beta=0.9, weight_decay=5e-4)
            ref.run(steps)
        return sorted(ref.records, key=lambda r: (r.step, r.block))

    got = eng.log.sorted()
    want, emu = oracle_run("f64"), oracle_run("bf16" if precision == "bf16" else "f32")
    assert [(r.step, r.block, r.batch_index) for r in got] == [(r.step, r.block, r.batch_index) for r in want]
    # K=4, p_k=1: the head first sees a real activation at step cum_p[3] = 3 and every block's first
    # real (non-zero-packet) gradient arrives at step cum_p[k] + m_k = 6, so through step 4 the
    # parameters move only by the zero-packet weight decay -- no trajectory chaos yet. Every record
    # is held to FLOOR_X x the same record's error of the oracle with bf16 storage emulated (+ the
    # EARLY bounds as the absolute slack); steps 3-4 check the full 4-block forward's loss.
    le, ge = EARLY[precision]
    assert any(r.loss is not None and r.step >= 3 for r in got)
    last = [(rg, rw, re) for rg, rw, re in zip(got, want, emu) if rw.loss is not None][-1]
    print(f"\nresnet50 {precision} step {last[0].step}: loss dev {last[0].loss:.4f} f64 {last[1].loss:.4f} emu {last[2].loss:.4f}; "
          f"head grad norm dev {last[0].grad_norm:.3f} f64 {last[1].grad_norm:.3f} emu {last[2].grad_norm:.3f}")
    for rg, rw, re in zip(got, want, emu):
        if rw.loss is not None:
            fl = abs(re.loss - rw.loss)
            assert abs(rg.loss - rw.loss) <= FLOOR_X * fl + le * max(1.0, abs(rw.loss)), (rg.step, rg.loss, rw.loss, fl)
        fg = abs(re.grad_norm - rw.grad_norm)
        assert abs(rg.grad_norm - rw.grad_norm) <= FLOOR_X * fg + ge * max(rw.grad_norm, 1e-3), (
            rg.step, rg.block, rg.grad_norm, rw.grad_norm, re.grad_norm)
