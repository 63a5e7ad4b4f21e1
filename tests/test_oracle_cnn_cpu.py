"""Independent check of the oracle's CNN layer math against torch float64 autograd.

The reference has no CNN kinds, so the oracle's conv / BN /
residual / pooling restatement is pinned here against torch.nn.functional in
float64 (training-mode BN, biased variance, eps 1e-5), forward and backward.
"""

import numpy as np
import pytest
import torch
import torch.nn.functional as F

import oracle.dsp_ref as R
from oracle import cnn


def _conv_bn(x, w, g, b, stride, pad, relu):
    y = F.conv2d(x, w.permute(0, 3, 1, 2), stride=stride, padding=pad)
    z = F.batch_norm(y, None, None, g, b, training=True, eps=cnn.BN_EPS)
    return F.relu(z) if relu else z


def _torch_layer(spec, vec, x):
    prm = {}
    off = 0
    for name, co, k, ci, st, pad in cnn.conv_list(spec):
        nw = co * k * k * ci
        prm[name] = (vec[off:off + nw].view(co, k, k, ci), vec[off + nw:off + nw + co],
                     vec[off + nw + co:off + nw + 2 * co], st, pad)
        off += nw + 2 * co
    if spec.kind == "conv_bn_relu":
        w, g, b, st, pad = prm["c"]
        return _conv_bn(x, w, g, b, st, pad, True)
    if spec.kind == "avgpool":
        return x.mean(dim=(2, 3))
    if spec.kind == "maxpool":
        return F.max_pool2d(x, 3, 2, 1)
    names = ["c1", "c2"] if spec.kind == "basic_unit" else ["c1", "c2", "c3"]
    h = x
    for i, n in enumerate(names):
        w, g, b, st, pad = prm[n]
        h = _conv_bn(h, w, g, b, st, pad, i < len(names) - 1)
    sc = x
    if "sc" in prm:
        w, g, b, st, pad = prm["sc"]
        sc = _conv_bn(x, w, g, b, st, pad, False)
    return F.relu(h + sc)


SPECS = [
    R.conv_bn_relu((3, 9, 9), 8),
    R.conv_bn_relu((3, 12, 12), 8, ksize=7, stride=2),
    R.basic_unit((8, 8, 8), 8, 1),
    R.basic_unit((8, 8, 8), 16, 2),
    R.basic_unit((8, 7, 7), 12, 1),
    R.bottleneck((16, 8, 8), 4, 16, 1),
    R.bottleneck((16, 8, 8), 8, 32, 2),
    R.avgpool((8, 5, 5)),
    R.maxpool((8, 9, 9)),
]


@pytest.mark.parametrize("spec", SPECS, ids=lambda s: f"{s.kind}-{s.in_shape}-{s.stride}")
def test_cnn_layer_vs_torch_autograd(spec):
    rng = np.random.default_rng(0)
    B = 3
    vec = rng.standard_normal(spec.param_count) * 0.3
    x = rng.standard_normal((B, int(np.prod(spec.in_shape))))
    out, ent = cnn.layer_forward(spec, vec, x)
    u = rng.standard_normal(out.shape)
    g, dx = cnn.layer_backward(spec, vec, ent, u)

    tv = torch.tensor(vec, requires_grad=True)
    tx = torch.tensor(x.reshape(B, *spec.in_shape), requires_grad=True)
    ty = _torch_layer(spec, tv, tx)
    np.testing.assert_allclose(out, ty.detach().reshape(B, -1).numpy(), rtol=1e-10, atol=1e-10)
    ty.backward(torch.tensor(u).reshape(ty.shape))
    if spec.param_count:
        np.testing.assert_allclose(g, tv.grad.numpy(), rtol=1e-8, atol=1e-9)
    np.testing.assert_allclose(dx, tx.grad.reshape(B, -1).numpy(), rtol=1e-8, atol=1e-9)


def test_zero_packet_bn_is_finite():
    """Warmup packets are all-zero (pipeline.py:524-528): zero-variance BN stays finite."""
    spec = R.basic_unit((8, 4, 4), 8, 1)
    vec = np.random.default_rng(1).standard_normal(spec.param_count)
    out, ent = cnn.layer_forward(spec, vec, np.zeros((2, 128)))
    g, dx = cnn.layer_backward(spec, vec, ent, np.ones_like(out))
    assert np.isfinite(out).all() and np.isfinite(g).all() and np.isfinite(dx).all()


def test_bf16_round_is_round_to_nearest_even():
    vals = np.array([1.0, 1.00390625, 1.005859375, -3.14159, 65504.0, 1e-30])
    want = torch.tensor(vals, dtype=torch.float32).bfloat16().double().numpy()
    np.testing.assert_array_equal(cnn.bf16_round(vals), want)
