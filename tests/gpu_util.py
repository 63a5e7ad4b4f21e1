"""Helpers shared by the GPU parity tests (CUDA path vs the fp64 oracle)."""

from __future__ import annotations

import numpy as np

import oracle.dsp_ref as R
import paper_1909_02625_b200 as P


def to_oracle_layers(layers):
    """Product LayerSpecs -> oracle LayerSpecs (same kinds, same fields)."""
    out = []
    for s in layers:
        out.append(R.LayerSpec(s.kind, s.in_dim, s.out_dim, s.bias, tuple(s.in_shape), s.out_c, s.mid_c, s.stride,
                               s.ksize))
    return out


def twin_models(layers, boundaries, seed=0):
    """The same initial model on both sides (init is checked equal in test_oracle_cpu)."""
    pm = P.build_model(layers, boundaries)
    P.init_params(pm, seed)
    om = R.build_model(to_oracle_layers(layers), boundaries)
    R.init_params(om, seed)
    for bp, bo in zip(pm.blocks, om.blocks):
        assert np.array_equal(bp.params, bo.params)
    return pm, om


def rel_err(a, b) -> float:
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-12))


def small_resnet(num_classes=10, width=8, in_shape=(3, 8, 8)):
    """stem + one basic unit per stage (projection at stages 2, 3) + head."""
    L = [P.conv_bn_relu(in_shape, width)]
    sh = L[-1].out_shape
    L.append(P.basic_unit(sh, width, 1))
    sh = L[-1].out_shape
    L.append(P.basic_unit(sh, 2 * width, 2))
    sh = L[-1].out_shape
    L.append(P.basic_unit(sh, 4 * width, 2))
    sh = L[-1].out_shape
    L.append(P.avgpool(sh))
    L.append(P.dense(4 * width, num_classes))
    return L
