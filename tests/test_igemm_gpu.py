"""tcgen05 implicit-GEMM conv kernels vs a torch fp32 reference of the same op.

Inputs are rounded to the storage dtype first, so the only difference left is
fp32-accumulation order (bf16 / tf32 multiply products are exact in fp32 for
bf16, rounded for tf32).
"""

import ctypes as C

import pytest
import torch
import torch.nn.functional as F

from paper_1909_02625_b200 import _lib as L

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True, scope="module")
def _lib_loaded():
    L.load(require_symbols=False)

CASES = [
    # nimg, H, W, C, K, R, stride, pad
    (2, 8, 8, 16, 16, 3, 1, 1),
    (4, 32, 32, 16, 16, 3, 1, 1),
    (3, 16, 16, 16, 32, 3, 2, 1),
    (3, 16, 16, 16, 32, 1, 2, 0),
    (2, 8, 8, 64, 64, 3, 1, 1),
    (5, 7, 7, 24, 40, 3, 1, 1),
    (2, 9, 11, 8, 8, 3, 2, 1),
    (37, 1, 1, 72, 136, 1, 1, 0),       # dense layer as 1x1 conv, ragged M
    (2, 8, 8, 256, 272, 1, 1, 0),       # multiple N tiles
    (1, 4, 4, 8, 520, 3, 1, 1),         # > 2 N tiles
    # FPROP halo tiles (one A stage per 128-pixel tile, resident weights)
    (2, 16, 16, 32, 32, 3, 1, 1),       # C=32: SWIZZLE_64B rows, hb=8
    (2, 32, 32, 16, 32, 3, 1, 1),       # N=32 tile
    (1, 16, 16, 64, 64, 3, 1, 1),       # C=64: SWIZZLE_128B rows
    (2, 16, 16, 16, 16, 5, 1, 2),       # 5x5: 4 halo rows
    (2, 16, 16, 32, 64, 1, 1, 0),       # 1x1: a single box per tile
    # im2col-mode TMA (output width does not divide 128: tiles cross rows and images)
    (2, 14, 14, 64, 128, 3, 1, 1),
    (3, 7, 7, 128, 256, 3, 1, 1),       # BN=256, ragged last tile
    (2, 28, 28, 64, 128, 3, 2, 1),      # stride 2
    (2, 12, 12, 128, 64, 1, 2, 0),      # 1x1 stride-2 projection
    (1, 20, 20, 64, 320, 1, 1, 0),      # two n-tiles of 256
    (2, 14, 14, 128, 256, 1, 1, 0),     # 1x1 stride 1: A as a plain 2-D [pixels][C] TMA map
    (3, 7, 7, 64, 64, 1, 1, 0),         # ... ragged M
    (2, 20, 20, 8, 64, 7, 2, 3),        # ResNet-50 stem shape: 8-channel im2col boxes, Kd = 392
    (2, 14, 14, 16, 32, 3, 1, 1),       # 16 / 32-channel im2col boxes (SW32 / SW64)
    (2, 14, 14, 256, 128, 3, 2, 1),     # stride-2 DGRAD split by output parity (BN=256)
    (1, 14, 14, 512, 256, 1, 2, 0),     # 1x1 stride-2 projection: 3 parities without taps
]


def _geom(nimg, H, W, C_, K, R, stride, pad):
    P = (H + 2 * pad - R) // stride + 1
    Q = (W + 2 * pad - R) // stride + 1
    return L.ConvGeom(nimg, H, W, C_, P, Q, K, R, R, stride, pad), P, Q


def _run(mode, dtype, g, M, N, Kd, A, B, D, splits=1, kb=1, stats=None, residual=None, bias=None, ldd=None,
         out_f32=0, stat_out=None, gamma=None, beta=None, sem=None, n_valid=0, B_t=None):
    a = L.IgemmArgs()
    a.geom = g
    a.M, a.N, a.Kd = M, N, Kd
    a.A, a.B, a.D = A.data_ptr(), B.data_ptr(), D.data_ptr()
    a.ldd = ldd if ldd is not None else N
    a.out_f32 = out_f32
    a.residual = residual.data_ptr() if residual is not None else None
    a.bias = bias.data_ptr() if bias is not None else None
    a.stats = stats.data_ptr() if stats is not None else None
    a.kb_per_split = kb
    a.n_valid = n_valid
    for name, t in (("stat_out", stat_out), ("gamma", gamma), ("beta", beta), ("sem", sem), ("B_t", B_t)):
        setattr(a, name, t.data_ptr() if t is not None else None)
    L.check(L.load().dsp_igemm(mode, dtype, C.byref(a), splits, C.c_void_p(torch.cuda.current_stream().cuda_stream)))


def _tol(dtype):
    # fp32 storage runs 3xTF32 (fp32-faithful); the torch reference is run without TF32
    return (2e-2, 2e-2) if dtype == torch.bfloat16 else (1e-4, 1e-4)


@pytest.fixture(autouse=True)
def _exact_fp32_reference():
    prev = (torch.backends.cudnn.allow_tf32, torch.backends.cuda.matmul.allow_tf32)
    torch.backends.cudnn.allow_tf32 = False
    torch.backends.cuda.matmul.allow_tf32 = False
    yield
    torch.backends.cudnn.allow_tf32, torch.backends.cuda.matmul.allow_tf32 = prev


def _setup(case, dt):
    torch.manual_seed(0)
    nimg, H, W, Cc, K, R, stride, pad = case
    g, P, Q = _geom(*case)
    dcode = L.DSP_DTYPE_BF16 if dt == torch.bfloat16 else L.DSP_DTYPE_F32
    dev = "cuda"
    x = torch.randn(nimg, H, W, Cc, device=dev).to(dt)
    w = (torch.randn(K, R, R, Cc, device=dev) / (R * R * Cc) ** 0.5).to(dt)
    dy = torch.randn(nimg, P, Q, K, device=dev).to(dt)
    return g, P, Q, dcode, x, w, dy


DTYPES = [torch.bfloat16, torch.float32]


@pytest.mark.parametrize("dt", DTYPES)
@pytest.mark.parametrize("case", CASES)
def test_fprop(case, dt):
    nimg, H, W, Cc, K, R, stride, pad = case
    g, P, Q, dcode, x, w, dy = _setup(case, dt)
    rtol, atol = _tol(dt)
    M = nimg * P * Q
    y = torch.empty(nimg, P, Q, K, device="cuda", dtype=dt)
    ntiles = (M + 127) // 128
    stats = torch.full((L.IGEMM_MAX_CTAS, 2, K), float("nan"), device="cuda")
    stat_out = torch.full((4, K), float("nan"), device="cuda")
    gamma = torch.rand(K, device="cuda") + 0.5
    beta = torch.randn(K, device="cuda")
    sem = torch.zeros(L.IGEMM_SEM_INTS, dtype=torch.int32, device="cuda")  # one ticket per n-tile
    nvalid = K - 8 if K > 8 else K
    _run(L.DSP_IGEMM_FPROP, dcode, g, M, K, R * R * Cc, x, w, y, stats=stats, stat_out=stat_out, gamma=gamma,
         beta=beta, sem=sem, n_valid=nvalid)
    ref = F.conv2d(x.float().permute(0, 3, 1, 2), w.float().permute(0, 3, 1, 2), stride=stride,
                   padding=pad).permute(0, 2, 3, 1)
    ref[..., nvalid:] = 0.0
    torch.testing.assert_close(y.float(), ref, rtol=rtol, atol=atol)
    yv = y.float().reshape(-1, K)
    bn = next(b for b in (16, 32, 64, 128, 256) if K <= b or b == 256)
    if bn == 256 and R * R * Cc <= 128:
        bn = 128  # short-K launches use 128-wide tiles (igemm.cu launch_mode)
    nt = (K + bn - 1) // bn
    ctas = min(296 if bn <= 128 else 148, (M + 127) // 128 * nt) // nt * nt
    # CTA c holds the partial sums of n-tile c % nt only (single-level finalize: <= 16 CTAs per
    # n-tile; larger grids overwrite group leaders' rows with their group sums)
    if ctas // nt <= 16:
        owner = (torch.arange(ctas, device="cuda")[:, None] % nt) == (torch.arange(K, device="cuda")[None, :] // bn)
        part = torch.where(owner[:, None, :], stats[:ctas], torch.zeros_like(stats[:ctas]))
        torch.testing.assert_close(part[:, 0].sum(0), yv.sum(0), rtol=1e-3, atol=1e-2)
        torch.testing.assert_close(part[:, 1].sum(0), (yv * yv).sum(0), rtol=1e-3, atol=1e-2)
    # fused BatchNorm finalize (last CTA): mean / invstd / scale / shift, pad columns zero
    mean = yv.double().mean(0)
    var = yv.double().var(0, unbiased=False)
    inv = 1.0 / torch.sqrt(var + 1e-5)
    want = torch.stack([mean, inv, gamma.double() * inv, beta.double() - mean * gamma.double() * inv]).float()
    want[:, nvalid:] = 0.0
    torch.testing.assert_close(stat_out, want, rtol=2e-3, atol=2e-3)
    assert int(sem.abs().sum().item()) == 0


@pytest.mark.parametrize("dt", DTYPES)
@pytest.mark.parametrize("transposed", [False, True])
@pytest.mark.parametrize("case", CASES)
def test_dgrad(case, dt, transposed):
    """transposed: also pass the per-tap transposed weights B_t [C][R][S][K] -- stride-1 'same'
    convs with K in {16, 32, 64} then take the halo path (TMA dY boxes + resident weights)."""
    nimg, H, W, Cc, K, R, stride, pad = case
    g, P, Q, dcode, x, w, dy = _setup(case, dt)
    rtol, atol = _tol(dt)
    dx = torch.empty(nimg, H, W, Cc, device="cuda", dtype=dt)
    res = torch.randn(nimg, H, W, Cc, device="cuda").to(dt)
    w_t = w.permute(3, 1, 2, 0).contiguous() if transposed else None
    _run(L.DSP_IGEMM_DGRAD, dcode, g, nimg * H * W, Cc, R * R * K, dy, w, dx, residual=res, B_t=w_t)
    refdx = torch.nn.grad.conv2d_input((nimg, Cc, H, W), w.float().permute(0, 3, 1, 2),
                                       dy.float().permute(0, 3, 1, 2), stride=stride,
                                       padding=pad).permute(0, 2, 3, 1)
    torch.testing.assert_close(dx.float(), refdx + res.float(), rtol=rtol, atol=atol * 4)


@pytest.mark.parametrize("dt", DTYPES)
@pytest.mark.parametrize("case", CASES)
def test_wgrad(case, dt):
    nimg, H, W, Cc, K, R, stride, pad = case
    g, P, Q, dcode, x, w, dy = _setup(case, dt)
    Mw = R * R * Cc
    Kpix = nimg * P * Q
    ks = 64 if dt == torch.bfloat16 else 32
    nkb = (Kpix + ks - 1) // ks
    splits = min(nkb, 7)
    kb = (nkb + splits - 1) // splits
    splits = (nkb + kb - 1) // kb
    part = torch.full((splits, Mw, K), float("nan"), device="cuda")
    _run(L.DSP_IGEMM_WGRAD, dcode, g, Mw, K, Kpix, x, dy, part, splits=splits, kb=kb)
    dw = part.sum(0).reshape(R, R, Cc, K).permute(3, 0, 1, 2)  # [K][R][S][C]
    refdw = torch.nn.grad.conv2d_weight(x.float().permute(0, 3, 1, 2), (K, Cc, R, R),
                                        dy.float().permute(0, 3, 1, 2), stride=stride,
                                        padding=pad).permute(0, 2, 3, 1)
    scale = refdw.abs().max().item() + 1e-6
    assert (dw - refdw).abs().max().item() / scale < (2e-2 if dt == torch.bfloat16 else 1e-5)


def test_fprop_bias_fp32_out():
    torch.manual_seed(1)
    B, D, O = 50, 40, 24
    g, _, _ = _geom(B, 1, 1, D, O, 1, 1, 0)
    x = torch.randn(B, D, device="cuda").bfloat16()
    w = torch.randn(O, D, device="cuda").bfloat16()
    bias = torch.randn(O, device="cuda")
    y = torch.empty(B, O, device="cuda")
    _run(L.DSP_IGEMM_FPROP, L.DSP_DTYPE_BF16, g, B, O, D, x, w, y, bias=bias, out_f32=1)
    torch.testing.assert_close(y, x.float() @ w.float().t() + bias, rtol=1e-3, atol=1e-3)
