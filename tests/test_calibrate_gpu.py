"""DES calibration from measured block costs and device straggler injection."""

import numpy as np
import pytest

import oracle.dsp_ref as R
import paper_1909_02625_b200 as P
from paper_1909_02625_b200 import calibrate as CAL
from paper_1909_02625_b200.runtime import torch_mod
from tests.gpu_util import small_resnet, twin_models

pytestmark = pytest.mark.gpu


def test_measured_costs_drive_the_des():
    layers = P.resnet_cifar_layers(20, 10, width=8)
    model = P.build_model(layers, P.flop_balanced_boundaries(layers, 3))
    P.init_params(model, 0)
    f, b = CAL.measure_block_costs(model, 16, reps=3)
    assert len(f) == 3 and all(v > 0 for v in f + b)
    sim = CAL.simulate_dsp(f, b, P.default_queue_config(3), 60)
    # steady pipeline interval = the slowest block's per-step cost (simulate.py, test_simulate.py:43-46)
    assert sim["steady_interval"] == pytest.approx(max(fi + bi for fi, bi in zip(f, b)), rel=1e-9)
    assert CAL.simulate_bp(f, b, 60)["steady_interval"] == pytest.approx(sum(f) + sum(b), rel=1e-9)
    cuts = CAL.measured_cuts(layers, 3, 16, reps=2)
    assert len(cuts) == 2 and 0 < cuts[0] < cuts[1] < len(layers)


def test_twin_balanced_cuts_never_worse_than_start():
    layers = P.resnet_cifar_layers(20, 10, width=8)
    start = [1, 2]  # deliberately unbalanced: a 1-layer block 0
    c0 = max(CAL.block_step_cost(layers, lo, hi, 16, hi == len(layers), reps=3)
             for lo, hi in zip([0] + start, start + [len(layers)]))
    cuts, costs = CAL.twin_balanced_cuts(layers, 3, 16, start=start, reps=3)
    assert len(cuts) == 2 and 0 < cuts[0] < cuts[1] < len(layers)
    assert len(costs) == 3 and all(c > 0 for c in costs)
    assert max(costs) <= c0 * 1.05


def test_device_straggler_changes_timing_not_values():
    torch = torch_mod()
    layers = small_resnet(in_shape=(3, 8, 8))
    cfg = P.default_queue_config(3)
    pool = R.synthetic_batches(4, 8, (3, 8, 8), 10, seed=1)
    out = []
    for strag in (None, P.DeviceStraggler(prob=0.5, delay_s=1e-3, seed=3)):
        pm, _ = twin_models(layers, [2, 4], seed=2)
        eng = P.TrainEngine(pm, cfg, R.cycle(pool), P.LrSchedule(0.05), rule="sum", beta=0.9, straggler=strag)
        eng.rt.use_graphs = False  # both runs eager: compare like with like
        eng.run(4)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        eng.run(12)
        e1.record()
        e1.synchronize()
        out.append((eng.log.checksum(), e0.elapsed_time(e1), [b.params.copy() for b in pm.blocks]))
    assert out[0][0] == out[1][0]
    for a, b in zip(out[0][2], out[1][2]):
        assert np.array_equal(a, b)
    hits = sum(P.DeviceStraggler(prob=0.5, delay_s=1e-3, seed=3).hits(k, n, ph)
               for k in range(3) for n in range(4, 16) for ph in (0, 1))
    assert hits > 0 and out[1][1] > out[0][1]  # the injected device delays show up in GPU time
