"""The C-ABI library loads without a GPU and exports exactly what include/dsp_b200.h declares.

Only host-side entry points are called here (block planning does no CUDA
work); every compute entry point is exercised by the -m gpu tests.
"""

import ctypes as C
import os
import re

import pytest

import paper_1909_02625_b200 as P
from paper_1909_02625_b200 import _lib as L

HEADER = os.path.join(os.path.dirname(os.path.dirname(__file__)), "include", "dsp_b200.h")


@pytest.fixture(scope="module")
def lib():
    if not L.LIB_PATH.exists():
        from paper_1909_02625_b200 import _build

        _build.build()
    return L.load()


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(dsp_[a-z0-9_]+)\s*\(", src)))


def test_header_and_binding_agree():
    assert declared_functions() == sorted(L.exported_symbols())


def test_library_exports_every_declared_symbol(lib):
    for name in declared_functions():
        assert hasattr(lib, name), name
    assert lib.dsp_abi_version() == 2
    assert lib.dsp_launch_count() >= 0


def _plan(layers, bounds, batch, k):
    m = P.build_model(layers, bounds)
    blk = m.blocks[k]
    descs = blk.layer_descs()
    h = C.c_void_p()
    rc = L.load().dsp_block_create(descs, len(descs), batch, L.DSP_DTYPE_BF16, int(k == m.k - 1), C.byref(h))
    return m, blk, h, rc


def test_block_planning_host_only(lib):
    layers = P.resnet_cifar_layers(20)
    bounds = P.flop_balanced_boundaries(layers, 2)
    for k in range(2):
        m, blk, h, rc = _plan(layers, bounds, 32, k)
        L.check(rc)
        try:
            assert lib.dsp_block_param_count(h) == blk.param_count
            c, hh, ww = blk.in_shape
            assert lib.dsp_block_in_elems(h) == 32 * hh * ww * ((c + 7) // 8 * 8)
            assert lib.dsp_block_workspace_bytes(h) > 0
        finally:
            lib.dsp_block_destroy(h)


def test_block_planning_rejects_bad_programs(lib):
    # last block must end with a dense (logits) layer
    m, blk, h, rc = _plan([P.conv_bn_relu((3, 8, 8), 8)], [], 4, 0)
    assert rc == 1 and b"dense" in lib.dsp_last_error()
    # a shape mismatch between consecutive layers
    bad = P.build_model([P.dense(4, 6), P.dense(6, 3)], [])
    descs = bad.blocks[0].layer_descs()
    descs[1].in_c = 5
    h = C.c_void_p()
    assert lib.dsp_block_create(descs, 2, 4, L.DSP_DTYPE_BF16, 1, C.byref(h)) == 1
    # fp32 storage (3xTF32) plans; an unknown storage dtype is rejected
    descs = P.build_model([P.dense(4, 3)], []).blocks[0].layer_descs()
    assert lib.dsp_block_create(descs, 1, 4, L.DSP_DTYPE_F32, 1, C.byref(h)) == 0
    lib.dsp_block_destroy(h)
    assert lib.dsp_block_create(descs, 1, 4, 7, 1, C.byref(h)) == 1 and b"dtype" in lib.dsp_last_error()


def test_engine_without_gpu_fails_loudly():
    import torch

    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    m = P.build_model([P.dense(4, 3)], [])
    P.init_params(m, 0)
    batches = iter([(torch.zeros(2, 4).numpy(), torch.zeros(2, dtype=torch.int64).numpy())] * 3)
    with pytest.raises(P.B200Unavailable):
        P.TrainEngine(m, P.validate_config((0,), (0,)), batches, P.LrSchedule(0.1))


def test_engine_create_validates_queue_config_on_host(lib):
    """dsp_create checks Eq.(5) (pipeline.py:85-128) before touching the device."""
    layers = [P.dense(12, 8), P.relu(), P.dense(8, 4)]
    m = P.build_model(layers, [2])
    descs = [blk.layer_descs() for blk in m.blocks]
    flat = (L.LayerDesc * sum(len(d) for d in descs))(*[e for d in descs for e in d])
    cases = [((1, 1), (1, 0), "p_last_zero"), ((0, 0), (1, 0), "p_positive"), ((1, 0), (0, 0), "m_positive"),
             ((1, 0), (1, -1), "m_last_nonneg"), ((1, 0), (1, 1), "q_positive")]
    for p, mm, name in cases:
        cfg = L.EngineConfig()
        cfg.K = 2
        for k in range(2):
            cfg.p[k], cfg.m[k] = p[k], mm[k]
            cfg.n_layers[k] = len(descs[k])
        cfg.batch, cfg.dtype, cfg.in_c, cfg.in_h, cfg.in_w, cfg.num_classes = 4, L.DSP_DTYPE_BF16, 12, 1, 1, 4
        cfg.layers = C.cast(flat, C.POINTER(L.LayerDesc))
        h = C.c_void_p()
        assert lib.dsp_create(C.byref(cfg), C.byref(h)) == L.DSP_E_INVALID
        assert name in lib.dsp_last_error().decode()
        assert not h.value
