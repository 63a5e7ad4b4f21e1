"""Host-side pieces of the product package vs the oracle and the reference's known answers."""

import numpy as np
import pytest

import oracle.dsp_ref as R
import paper_1909_02625_b200 as P
from paper_1909_02625_b200.data import synthetic_batches
from tests.gpu_util import to_oracle_layers


class TestValidateConfig:
    @pytest.mark.parametrize("p,m,q", [((1, 1, 0), (4, 2, 0), (0, 1, 1)), ((2, 2, 0), (6, 3, 0), (0, 1, 1)),
                                       ((3, 3, 0), (10, 5, 0), (0, 2, 2))])
    def test_reference_configs(self, p, m, q):
        assert P.validate_config(p, m).q == q

    @pytest.mark.parametrize("p,m,kw,constraint,index", [
        ((1, 1, 0), (2, 2, 0), {}, "q_positive", 1),
        ((1, 1, 1), (4, 2, 0), {}, "p_last_zero", 2),
        ((0, 1, 0), (4, 2, 0), {}, "p_positive", 0),
        ((1, 1, 0), (4, 0, 0), {"warmup": "discard_warmup_updates"}, "m_positive", 1),
        ((1, 0), (2, -1), {}, "m_last_nonneg", 1),
        ((1, 0), (2,), {}, "length", 0),
        ((1, 0), (2, 0), {"warmup": "bogus"}, "warmup", 0),
    ])
    def test_rejections_match_oracle(self, p, m, kw, constraint, index):
        with pytest.raises(P.ConfigError) as e:
            P.validate_config(p, m, **kw)
        assert (e.value.constraint, e.value.index) == (constraint, index)
        with pytest.raises(R.ConfigError) as e2:
            R.validate_config(p, m, **kw)
        assert str(e.value) == str(e2.value)

    def test_message_and_k1(self):
        with pytest.raises(P.ConfigError, match="2-1-2 = -1"):
            P.validate_config((1, 1, 0), (2, 2, 0))
        assert P.validate_config((0,), (0,)).q == (0,)
        assert P.staleness_of(P.validate_config((2, 2, 0), (6, 3, 0))) == P.StalenessProfile((6, 3, 0), 6)

    @pytest.mark.parametrize("k", range(1, 9))
    def test_default_queue_config_valid(self, k):
        cfg = P.default_queue_config(k)
        assert cfg.m == tuple(2 * (k - 1 - i) for i in range(k))
        assert cfg.q == tuple([0] + [1] * (k - 1))


LAYER_LISTS = {
    "mlp": ([P.dense(12, 16), P.relu(), P.dense(16, 12), P.tanh(), P.dense(12, 4)], [2]),
    "resnet20": (P.resnet_cifar_layers(20), None),
    "resnet56": (P.resnet_cifar_layers(56), None),
    "resnet164": (P.resnet_cifar_bottleneck_layers(164), None),
}


@pytest.mark.parametrize("name", sorted(LAYER_LISTS))
def test_model_layout_and_init_match_oracle(name):
    layers, bounds = LAYER_LISTS[name]
    if bounds is None:
        bounds = P.flop_balanced_boundaries(layers, 4)
    pm = P.build_model(layers, bounds)
    om = R.build_model(to_oracle_layers(layers), bounds)
    assert pm.block_input_dims == om.block_input_dims
    assert [b.param_count for b in pm.blocks] == [b.param_count for b in om.blocks]
    for s in layers:
        assert s.param_count == to_oracle_layers([s])[0].param_count
    if name != "resnet164":  # (init of 1.7M params is covered by the smaller lists)
        P.init_params(pm, 5)
        R.init_params(om, 5)
        for bp, bo in zip(pm.blocks, om.blocks):
            assert np.array_equal(bp.params, bo.params)


def test_init_independent_of_boundaries():
    layers = P.resnet_cifar_layers(20)
    a = P.build_model(layers, [3])
    b = P.build_model(layers, [2, 5, 8])
    P.init_params(a, 1)
    P.init_params(b, 1)
    assert np.array_equal(a.flat_params(), b.flat_params())


def test_resnet_flops_match_survey():
    """Forward FLOP/sample from SURVEY.md §8d: R20 81.6M, R56 251.5M, R110 506.3M, R164 495.3M, R50 8174M."""
    def f(layers):
        return sum(s.flops() for s in layers) / 1e6
    assert abs(f(P.resnet_cifar_layers(20)) - 81.6) < 1.0
    assert abs(f(P.resnet_cifar_layers(56)) - 251.5) < 2.0
    assert abs(f(P.resnet_cifar_layers(110)) - 506.3) < 4.0
    assert abs(f(P.resnet_cifar_bottleneck_layers(164, 100)) - 495.3) < 5.0
    assert abs(f(P.resnet50_layers()) / 8174 - 1.0) < 0.01


@pytest.mark.parametrize("depth,k,limit", [(56, 4, 1.15), (110, 8, 1.15), (56, 2, 1.1)])
def test_flop_balanced_cuts(depth, k, limit):
    layers = P.resnet_cifar_layers(depth)
    cuts = P.flop_balanced_boundaries(layers, k)
    assert len(cuts) == k - 1 and cuts == sorted(set(cuts))
    pre = np.cumsum([0.0] + [s.flops() for s in layers])
    edges = [0, *cuts, len(layers)]
    cost = [(pre[b] - pre[a]) * (3.0 if j == k - 1 else 4.0) for j, (a, b) in enumerate(zip(edges[:-1], edges[1:]))]
    assert max(cost) / np.mean(cost) < limit


def test_suggest_boundaries_param_balanced():
    layers = [P.dense(12, 16), P.relu(), P.dense(16, 12), P.relu(), P.dense(12, 4)]
    assert P.suggest_boundaries(layers, 3) == [1, 3]
    with pytest.raises(ValueError):
        P.suggest_boundaries(layers, 9)


def test_lr_schedule_and_rng():
    k = np.load("tests/golden/kats.npz")
    sched = P.LrSchedule(0.01, ((150, 0.1), (225, 0.1)))
    assert np.array_equal([P.lr_at(sched, n) for n in range(300)], k["lr"])
    with pytest.raises(ValueError):
        P.lr_at(sched, -1)
    with pytest.raises(ValueError):
        P.LrSchedule(0.0)
    r = P.SeededRng(7)
    assert np.array_equal(r.uniform(17), k["rng_u"])
    assert np.array_equal(r.normal(9), k["rng_n"])
    assert np.array_equal(r.permutation(23), k["rng_perm"])


def test_synthetic_batches_match_oracle():
    a = synthetic_batches(3, 5, (3, 4, 4), 10, seed=9)
    b = R.synthetic_batches(3, 5, (3, 4, 4), 10, seed=9)
    for (xa, la), (xb, lb) in zip(a, b):
        assert np.array_equal(xa, xb) and np.array_equal(la, lb)


def test_trainlog_checksum_format_matches_reference():
    recs = [P.LogRecord(0, 0, -2, 1.5), P.LogRecord(0, 1, -1, 0.25, loss=2.3), P.LogRecord(1, 0, -1, 0.0)]
    orecs = [R.Record(r.step, r.block, r.batch_index, r.grad_norm, r.loss) for r in recs]
    assert P.TrainLog(recs).checksum() == R.log_checksum(orecs)


def test_optimizer_state_validation():
    with pytest.raises(ValueError):
        P.OptimizerState(rule="rmsprop")
    # "adam" is this package's extension (BASELINE configs[2]); the reference rejects it
    ad = P.OptimizerState.for_params("adam", np.ones(3))
    assert np.array_equal(ad.m1, np.zeros(3)) and np.array_equal(ad.m2, np.zeros(3)) and ad.n == 0
    with pytest.raises(ValueError):
        P.OptimizerState(rule="sum", beta=1.0)
    with pytest.raises(ValueError):
        P.OptimizerState(rule="sum", s=-0.5)
    st = P.OptimizerState.for_params("sum", np.ones(3), beta=0.9)
    assert np.array_equal(st.ys, np.ones(3))


def test_layer_desc_program():
    m = P.build_model(P.resnet_cifar_layers(20), [4])
    d = m.blocks[1].layer_descs()
    assert d[0].kind == 11 and (d[0].in_c, d[0].in_h) == (16, 32) or d[0].in_c in (16, 32)
    assert d[len(d) - 1].kind == 0 and d[len(d) - 1].out_c == 10
    assert sum(x.param_count for x in d) == m.blocks[1].param_count
