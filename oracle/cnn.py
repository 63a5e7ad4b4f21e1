"""Float64 CNN layer kinds for the oracle -- TEST INFRASTRUCTURE ONLY.

The reference is MLP-only (blocks.py:21-33; "Convolutional blocks"
out of scope). These kinds follow blocks.py conventions -- a layer owns a
contiguous slice of its block's flat parameter vector, activations cross block
boundaries as 2-D (B, C*H*W) float64 packets in (C,H,W) order
(pipeline.py:494, 524-528), and backward returns a flat gradient laid out like
the parameters (blocks.py:126-127).

Parameter layout per kind (shared with the product):
  conv weight  [C_out][k][k][C_in]  (then BN gamma[C_out], beta[C_out])
  conv_bn_relu : W, gamma, beta
  basic_unit   : W1,g1,b1, W2,g2,b2 [, Wsc,gsc,bsc if stride!=1 or C_in!=C_out]
  bottleneck   : W1(1x1),g1,b1, W2(3x3, stride),g2,b2, W3(1x1),g3,b3 [, Wsc,gsc,bsc]
BatchNorm: training-mode batch statistics (biased variance, eps=1e-5) in every
forward (fresh and recompute alike), no running statistics.
Convolutions use im2col + BLAS GEMM in float64 (not the reference's
ascending-k loop: there is no reference CNN path to be bitwise with).
"""

from __future__ import annotations

import numpy as np

BN_EPS = 1e-5


# ------------------------------------------------------------ shapes / params
def conv_out(h: int, k: int, stride: int, pad: int) -> int:
    return (h + 2 * pad - k) // stride + 1


def has_projection(s) -> bool:
    c = s.in_shape[0]
    return s.stride != 1 or c != s.out_c


def out_shape(s) -> tuple:
    c, h, w = s.in_shape
    if s.kind == "conv_bn_relu":
        p = s.ksize // 2
        return (s.out_c, conv_out(h, s.ksize, s.stride, p), conv_out(w, s.ksize, s.stride, p))
    if s.kind in ("basic_unit", "bottleneck"):
        return (s.out_c, conv_out(h, 3, s.stride, 1), conv_out(w, 3, s.stride, 1))
    if s.kind == "avgpool":
        return (c,)
    if s.kind == "maxpool":
        return (c, conv_out(h, 3, 2, 1), conv_out(w, 3, 2, 1))
    raise ValueError(s.kind)


def conv_list(s):
    """[(name, c_out, k, c_in, stride, pad)] in parameter order."""
    c = s.in_shape[0]
    if s.kind == "conv_bn_relu":
        return [("c", s.out_c, s.ksize, c, s.stride, s.ksize // 2)]
    if s.kind == "basic_unit":
        lst = [("c1", s.out_c, 3, c, s.stride, 1), ("c2", s.out_c, 3, s.out_c, 1, 1)]
    elif s.kind == "bottleneck":
        lst = [("c1", s.mid_c, 1, c, 1, 0), ("c2", s.mid_c, 3, s.mid_c, s.stride, 1),
               ("c3", s.out_c, 1, s.mid_c, 1, 0)]
    else:
        return []
    if has_projection(s):
        lst.append(("sc", s.out_c, 1, c, s.stride, 0))
    return lst


def param_count(s) -> int:
    return sum(co * k * k * ci + 2 * co for _, co, k, ci, _, _ in conv_list(s))


def split_params(s, vec: np.ndarray) -> dict:
    """name -> (W[co][k][k][ci], gamma, beta) views into the flat slice."""
    out = {}
    off = 0
    for name, co, k, ci, _, _ in conv_list(s):
        nw = co * k * k * ci
        w = vec[off:off + nw].reshape(co, k, k, ci)
        off += nw
        g = vec[off:off + co]
        off += co
        b = vec[off:off + co]
        off += co
        out[name] = (w, g, b)
    return out


def init_layer(s, vec: np.ndarray, rng) -> None:
    """He-uniform conv weights (limit sqrt(6/fan_in)), BN gamma=1, beta=0, drawn
    conv by conv from the model-wide stream (as blocks.py:278-302 does for dense)."""
    for name, (w, g, b) in split_params(s, vec).items():
        fan_in = w.shape[1] * w.shape[2] * w.shape[3]
        lim = np.sqrt(6.0 / fan_in)
        w[:] = rng.uniform(w.size, -lim, lim).reshape(w.shape)
        g[:] = 1.0
        b[:] = 0.0


# ------------------------------------------------------------ primitives (NCHW)
def _im2col(x: np.ndarray, k: int, stride: int, pad: int):
    B, C, H, W = x.shape
    P, Q = conv_out(H, k, stride, pad), conv_out(W, k, stride, pad)
    xp = np.pad(x, ((0, 0), (0, 0), (pad, pad), (pad, pad)))
    sb, sc, sh, sw = xp.strides
    cols = np.lib.stride_tricks.as_strided(
        xp, shape=(B, P, Q, k, k, C), strides=(sb, sh * stride, sw * stride, sh, sw, sc))
    return cols.reshape(B * P * Q, k * k * C), P, Q


def conv_fwd(x, w, stride, pad):
    """y[b,co,p,q] = sum_{r,s,ci} x[b,ci,p*st+r-pad,q*st+s-pad] w[co,r,s,ci]."""
    co, k = w.shape[0], w.shape[1]
    cols, P, Q = _im2col(x, k, stride, pad)
    y = _mm(cols, w.reshape(co, -1).T)
    return y.reshape(x.shape[0], P, Q, co).transpose(0, 3, 1, 2), cols


def conv_bwd(dy, cols, x_shape, w, stride, pad):
    B, C, H, W = x_shape
    co, k = w.shape[0], w.shape[1]
    dyf = dy.transpose(0, 2, 3, 1).reshape(-1, co)
    dw = _mm(dyf.T, cols).reshape(w.shape)
    dcols = _mm(dyf, w.reshape(co, -1)).reshape(B, dy.shape[2], dy.shape[3], k, k, C)
    dxp = np.zeros((B, H + 2 * pad, W + 2 * pad, C))  # NHWC scatter: contiguous inner dim
    P, Q = dy.shape[2], dy.shape[3]
    for r in range(k):
        for s_ in range(k):
            dxp[:, r:r + stride * P:stride, s_:s_ + stride * Q:stride, :] += dcols[:, :, :, r, s_, :]
    dx = dxp[:, pad:pad + H, pad:pad + W, :].transpose(0, 3, 1, 2)
    return dx, dw


def bn_fwd(y, gamma, beta):
    mean = y.mean(axis=(0, 2, 3))
    var = y.var(axis=(0, 2, 3))
    inv = 1.0 / np.sqrt(var + BN_EPS)
    xhat = (y - mean[None, :, None, None]) * inv[None, :, None, None]
    return gamma[None, :, None, None] * xhat + beta[None, :, None, None], (xhat, inv)


def bn_bwd(g, cache, gamma):
    xhat, inv = cache
    M = g.shape[0] * g.shape[2] * g.shape[3]
    dbeta = g.sum(axis=(0, 2, 3))
    dgamma = (g * xhat).sum(axis=(0, 2, 3))
    dy = (gamma * inv / M)[None, :, None, None] * (M * g - dbeta[None, :, None, None]
                                                   - xhat * dgamma[None, :, None, None])
    return dy, dgamma, dbeta


# ------------------------------------------------------------ storage emulation
# "f64": pure float64 (the reference's precision).  "f32": round every stored tensor to float32
# (the device's fp32 parity mode; with acc="f32" also the conv GEMMs).  "bf16": round every tensor
# the device stores in bf16 at exactly the device's storage points (conv
# outputs, BN/ReLU outputs, unit outputs, activation gradients, the bf16
# weight shadow) so that ReLU masks match the device; sums stay float64.
STORAGE = {"mode": "f64", "acc": "f64"}


def _mm(a, b):
    """Matrix product in the accumulation precision: float64, or float32 ("acc": "f32") to
    measure how far an equally valid accumulation order moves the bf16 emulation from itself
    (the noise floor the parity tolerances must sit above)."""
    if STORAGE["acc"] == "f32":
        return (a.astype(np.float32) @ b.astype(np.float32)).astype(np.float64)
    return a @ b


def bf16_round(x):
    f = np.ascontiguousarray(x, dtype=np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000).astype(np.uint32)
    return r.view(np.float32).astype(np.float64)


def f32_round(x):
    return np.asarray(x, dtype=np.float32).astype(np.float64)


def q(x):
    mode = STORAGE["mode"]
    if mode == "bf16":
        return bf16_round(x)
    if mode == "f32":
        return f32_round(x)
    return x


# ------------------------------------------------------------ layer fwd / bwd
def _conv_bn(x, prm, name, spec, relu, store=True):
    _, co, k, ci, st, pad = spec
    w, g, b = prm[name]
    y, cols = conv_fwd(x, q(w), st, pad)
    y = q(y)
    z, cache = bn_fwd(y, g, b)
    if relu:
        z = np.maximum(z, 0.0)
    if store:
        z = q(z)
    return z, {"x_shape": x.shape, "cols": cols, "bn": cache, "z": z}


def layer_forward(s, vec, h2d):
    """2-D packet in, 2-D packet out; returns (out, tape entry)."""
    B = h2d.shape[0]
    x = h2d.reshape(B, *s.in_shape)
    if s.kind == "avgpool":
        out = q(x.mean(axis=(2, 3)))
        return out, {"shape": x.shape}
    if s.kind == "maxpool":
        c, h, w = s.in_shape
        xp = np.pad(x, ((0, 0), (0, 0), (1, 1), (1, 1)), constant_values=-np.inf)
        P, Q = conv_out(h, 3, 2, 1), conv_out(w, 3, 2, 1)
        win = np.stack([xp[:, :, r:r + 2 * P:2, t:t + 2 * Q:2] for r in range(3) for t in range(3)], 0)
        arg = win.argmax(axis=0)  # first max in (r, s) order
        out = np.take_along_axis(win, arg[None], 0)[0]
        return out.reshape(B, -1), {"arg": arg, "shape": x.shape, "PQ": (P, Q)}
    prm = split_params(s, vec)
    specs = {c[0]: c for c in conv_list(s)}
    if s.kind == "conv_bn_relu":
        z, e = _conv_bn(x, prm, "c", specs["c"], True)
        return z.reshape(B, -1), {"c": e}
    ent = {}
    z1, ent["c1"] = _conv_bn(x, prm, "c1", specs["c1"], True)
    if s.kind == "basic_unit":
        top, ent["c2"] = _conv_bn(z1, prm, "c2", specs["c2"], False, store=False)
    else:
        z2, ent["c2"] = _conv_bn(z1, prm, "c2", specs["c2"], True)
        top, ent["c3"] = _conv_bn(z2, prm, "c3", specs["c3"], False, store=False)
    if "sc" in specs:
        sc, ent["sc"] = _conv_bn(x, prm, "sc", specs["sc"], False, store=False)
    else:
        sc = x
    out = q(np.maximum(top + sc, 0.0))
    ent["out"] = out
    return out.reshape(B, -1), ent


def _bn_back(g, e, prm, name):
    w, gam, _ = prm[name]
    dy, dgam, dbet = bn_bwd(g, e["bn"], gam)
    return q(dy), dgam, dbet


def _conv_back(dy, e, prm, name, spec, residual=None, want_dx=True):
    _, co, k, ci, st, pad = spec
    w = prm[name][0]
    dx, dw = conv_bwd(dy, e["cols"], e["x_shape"], q(w), st, pad)
    if residual is not None:
        dx = dx + residual
    return q(dx), dw


def _pack_grads(s, grads: dict) -> np.ndarray:
    parts = []
    for name, *_ in conv_list(s):
        dw, dg, db = grads[name]
        parts += [dw.reshape(-1), dg, db]
    return np.concatenate(parts)


def layer_backward(s, vec, ent, u2d):
    B = u2d.shape[0]
    if s.kind == "avgpool":
        shp = ent["shape"]
        dx = np.broadcast_to(u2d[:, :, None, None] / (shp[2] * shp[3]), shp)
        return np.zeros(0), q(dx.reshape(B, -1).copy())
    if s.kind == "maxpool":
        shp = ent["shape"]
        P, Q = ent["PQ"]
        u = u2d.reshape(B, shp[1], P, Q)
        dxp = np.zeros((B, shp[1], shp[2] + 2, shp[3] + 2))
        for idx in range(9):
            r, t = divmod(idx, 3)
            dxp[:, :, r:r + 2 * P:2, t:t + 2 * Q:2] += u * (ent["arg"] == idx)
        return np.zeros(0), q(dxp[:, :, 1:-1, 1:-1].reshape(B, -1))
    prm = split_params(s, vec)
    specs = {c[0]: c for c in conv_list(s)}
    oc, oh, ow = out_shape(s)
    u = u2d.reshape(B, oc, oh, ow)
    grads = {}
    if s.kind == "conv_bn_relu":
        e = ent["c"]
        dy, dg, db = _bn_back(u * (e["z"] > 0.0), e, prm, "c")
        dx, dw = _conv_back(dy, e, prm, "c", specs["c"])
        grads["c"] = (dw, dg, db)
        return _pack_grads(s, grads), dx.reshape(B, -1)
    g = u * (ent["out"] > 0.0)
    main = ["c1", "c2"] if s.kind == "basic_unit" else ["c1", "c2", "c3"]
    top = main[-1]
    dy, dg, db = _bn_back(g, ent[top], prm, top)
    if "sc" in specs:
        dysc, dgs, dbs = _bn_back(g, ent["sc"], prm, "sc")
    for i in range(len(main) - 1, -1, -1):
        name = main[i]
        if i == 0:
            break
        dz, dw = _conv_back(dy, ent[name], prm, name, specs[name])
        grads[name] = (dw, dg, db)
        below = main[i - 1]
        dy, dg, db = _bn_back(dz * (ent[below]["z"] > 0.0), ent[below], prm, below)
    if "sc" in specs:
        dxs, dws = _conv_back(dysc, ent["sc"], prm, "sc", specs["sc"])
        grads["sc"] = (dws, dgs, dbs)
        res = dxs
    else:
        res = g
    dx, dw = _conv_back(dy, ent["c1"], prm, "c1", specs["c1"], residual=res)
    grads["c1"] = (dw, dg, db)
    return _pack_grads(s, grads), dx.reshape(B, -1)


def layer_flops(s) -> float:
    """Forward MACs*2 per sample (conv/dense only)."""
    if s.kind in ("avgpool", "maxpool"):
        return 0.0
    c, h, w = s.in_shape
    total = 0.0
    cur = {"x": (h, w)}
    for name, co, k, ci, st, pad in conv_list(s):
        if name in ("c1", "sc", "c"):
            ih, iw = h, w
        else:
            ih, iw = cur["prev"]
        P, Q = conv_out(ih, k, st, pad), conv_out(iw, k, st, pad)
        if name != "sc":
            cur["prev"] = (P, Q)
        total += 2.0 * P * Q * co * k * k * ci
    return total
