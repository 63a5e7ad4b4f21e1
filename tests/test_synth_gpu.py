"""On-device synthetic data supply (csrc/synth.cu) vs the host pipeline.

device_synthetic_batches must store exactly what to_device_batches(synthetic_batches(...))
stores -- the counter-based splitmix64 stream, Box-Muller pairs, batch counter bases (including
an odd B*D, where normal() consumes a padding draw) and the derived label stream.
"""

import numpy as np
import pytest

import oracle.dsp_ref as R
import paper_1909_02625_b200 as P
from paper_1909_02625_b200.data import (cycle, device_synthetic_batches, synthetic_batches,
                                        to_device_batches)
from tests.gpu_util import small_resnet, twin_models

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("B,shape,classes,seed", [(16, (3, 32, 32), 10, 0), (5, (3, 1, 1), 4, 7),
                                                  (4, (12, 1, 1), 4, 3), (3, (3, 8, 8), 100, 2**63 + 5)])
def test_device_batches_equal_host_pipeline(B, shape, classes, seed):
    host = to_device_batches(synthetic_batches(4, B, shape, classes, seed=seed), shape)
    dev = device_synthetic_batches(4, B, shape, classes, seed=seed)
    for h, d in zip(host, dev):
        assert np.array_equal(h.labels.cpu().numpy(), d.labels.cpu().numpy())
        hv = h.act.view(dtype=__import__("torch").int16).cpu().numpy()
        dv = d.act.view(dtype=__import__("torch").int16).cpu().numpy()
        assert np.array_equal(hv, dv), int((hv != dv).sum())


def test_engine_on_device_data_equals_host_data():
    layers = small_resnet(in_shape=(3, 8, 8))
    cfg = P.default_queue_config(2)
    logs = []
    for pool in (to_device_batches(synthetic_batches(3, 8, (3, 8, 8), 10, seed=1), (3, 8, 8)),
                 device_synthetic_batches(3, 8, (3, 8, 8), 10, seed=1)):
        pm, _ = twin_models(layers, [2], seed=3)
        eng = P.TrainEngine(pm, cfg, cycle([(b, b.labels) for b in pool]), P.LrSchedule(0.05), rule="sum", beta=0.9)
        eng.run(12)
        logs.append(eng.log.checksum())
    assert logs[0] == logs[1]


def test_device_batches_equal_the_oracle_pool():
    """The device-generated pool (csrc/synth.cu) holds the oracle's synthetic_batches --
    x ~ SeededRng(seed).normal, labels floor(uniform * C) -- bit for bit after storage rounding."""
    import torch

    from paper_1909_02625_b200.runtime import unpack_output

    shape = (3, 8, 8)
    dev = device_synthetic_batches(4, 8, shape, 10, seed=5)
    ref = R.synthetic_batches(4, 8, shape, 10, seed=5)
    st = torch.cuda.current_stream()
    for db, (x, lab) in zip(dev, ref):
        got = unpack_output(db.act, 8, shape, st)
        assert np.array_equal(got, R.cnn.bf16_round(x))
        assert np.array_equal(db.labels.cpu().numpy(), lab)
