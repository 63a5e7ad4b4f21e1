// Block executor: plans one DSP block (a consecutive run of layers,
// blocks.py:65-93) over a single caller-provided device workspace and
// sequences the sm_100a kernels for block_forward (blocks.py:96-118),
// softmax_xent (tensor.py:86-111), block_backward (blocks.py:121-154) and the
// optimizer step (pipeline.py:591-596, optim.py:48-109).
//
// Memory plan (all offsets into one workspace, 256-byte aligned):
//   per layer   : output activation (storage dtype, NHWC, channels padded to 8)
//   per conv    : pre-BN conv output y, BN stats [4][Cp], BN-backward coef [3][Cp]
//   per unit    : intermediate ReLU outputs z1 (and z2 for bottlenecks)
//   shared      : 4 unit-backward scratch tensors, 2 layer-gradient ping-pong
//                 tensors, BN / split-K / update partial-sum scratch, packed
//                 storage-dtype weight shadow + its pack table.
// The fresh forward and the recompute write the same buffers (the fresh pass's
// block output goes straight to the caller's out-ring slot), so one block holds
// exactly one tape, like the reference's single-use ForwardTape (blocks.py:54-62).
#include "common.cuh"
#include "kernels.cuh"
#include <cstdlib>
#include "abi_internal.h"

#include <algorithm>
#include <cstring>
#include <vector>

namespace dsp {

namespace {

inline int pad8(int c) { return (c + 7) / 8 * 8; }
inline size_t align256(size_t x) { return (x + 255) / 256 * 256; }

struct ConvP {
  dsp_conv_geom_t g;
  int ci_real = 0, co_real = 0;
  // space-to-depth stem (s2d_r > 0): a stride-2 R x R conv on <= 4 channels runs as the stride-1
  // ((R+1)/2)^2-tap conv over the 2x2 space-to-depth input (4x the channels, 16-channel TMA boxes
  // instead of 8, (R+1)^2 / R^2 of the padded MACs); g describes that conv, these the original
  int s2d_r = 0, s2d_ci = 0, s2d_h = 0, s2d_w = 0, s2d_cpx = 0, s2d_pad = 0;
  size_t s2d_buf = 0;  // the s2d input (forward, WGRAD) / its gradient (DGRAD) in the workspace
  int64_t w_off = 0, gamma_off = 0, beta_off = 0;  // floats, into block params
  int64_t wpack = 0;                               // elements, into packed weights
  int64_t wpack_t = -1;                            // transposed pack [Cin_p][R][S][Cout_p] (stride-1 convs)
  size_t y = 0, stat = 0, coef = 0;                // workspace byte offsets
  int64_t M() const { return (int64_t)g.nimg * g.P * g.Q; }
  int64_t Min() const { return (int64_t)g.nimg * g.H * g.W; }
};

struct LayerP {
  dsp_layer_desc_t d{};
  int in_cp = 0, out_cp = 0;
  int in_h = 1, in_w = 1, out_h = 1, out_w = 1;
  int in_real = 0, out_real = 0;  // real channels / dense widths
  int64_t in_rows = 0, out_rows = 0;  // B*H*W
  std::vector<ConvP> convs;
  bool proj = false;
  size_t out = 0, z1 = 0, z2 = 0, arg = 0;
  size_t mbits = 0;  // residual units (bf16): ReLU mask bits of `out`, one byte per 8 channels (0 = none)
  // dense
  ConvP dense;  // 1x1 conv view of the dense layer
  int64_t b_off = -1;
  bool logits = false;
  int64_t in_elems() const { return in_rows * in_cp; }
  int64_t out_elems() const { return out_rows * out_cp; }
};

}  // namespace
}  // namespace dsp

struct dsp_block {
  int B = 0, dtype = 0, is_last = 0, esz = 2;
  std::vector<dsp::LayerP> L;
  size_t ws_bytes = 0;
  size_t S[4] = {0, 0, 0, 0};
  size_t G[2] = {0, 0};
  size_t fpart = 0, bpart = 0, bpart2 = 0, wpart = 0, upart = 0, sem = 0, usem = 0, nf = 0, lsem = 0, rowloss = 0;
  size_t packed = 0, ptable = 0, utable = 0;
  std::vector<dsp::PackEntry> packs;
  std::vector<dsp::UpdTile> utiles;  // fused update + repack tile table (elementwise.cu update_pack)
  int pack_max = 0;
  size_t dlogits = 0;
  int classes = 0, classes_pad = 0;
  int64_t param_count = 0;
  uint8_t* ws = nullptr;
  float* params = nullptr;
  float* grads = nullptr;
  bool tape_valid = false;
  const void* rec_x = nullptr;
  // forward twin (dsp_block_share_weights): reads the primary block's packed weight shadow
  // instead of its own, so a fresh forward runs on its own workspace beside the primary's
  // recompute + backward
  const uint8_t* wsrc = nullptr;
  // side stream for the weight gradients of residual units: WGRAD (+ split-K reduce) of a conv
  // runs beside the DGRAD that reads the same dY, forked / joined with events (graph-capturable)
  cudaStream_t side = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  bool side_busy = false;
  ~dsp_block() {
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (ev_join) cudaEventDestroy(ev_join);
    if (side) cudaStreamDestroy(side);
  }
};

namespace dsp {
namespace {

struct Planner {
  size_t off = 0;
  size_t take(size_t bytes) {
    size_t o = off;
    off = align256(off + std::max<size_t>(bytes, 1));
    return o;
  }
};

void make_conv(ConvP& c, int B, int H, int W, int ci, int co, int k, int stride, int pad) {
  c.g.nimg = B;
  c.g.H = H;
  c.g.W = W;
  c.g.C = pad8(ci);
  c.g.R = c.g.S = k;
  c.g.stride = stride;
  c.g.pad = pad;
  c.g.P = (H + 2 * pad - k) / stride + 1;
  c.g.Q = (W + 2 * pad - k) / stride + 1;
  c.g.K = pad8(co);
  c.ci_real = ci;
  c.co_real = co;
}

int wgrad_splits(const ConvP& c, int* kb_per_split, int dtype) {
  const int ks = dtype == DSP_DTYPE_BF16 ? 64 : 32;
  const int64_t kd = c.M();
  const int nkb = (int)((kd + ks - 1) / ks);
  const int mw = c.g.R * c.g.S * c.g.C;
  const int mt = (mw + 127) / 128;
  const int nt = (c.g.K + 255) / 256;
  // split-K target of one CTA per SM: the K blocks' streams share the GPU, and fewer
  // splits mean fewer partials to reduce (measured: 148 -> +4% over 296, 74 too few)
  static const int target = getenv("DSP_B200_WGRAD_CTAS") ? atoi(getenv("DSP_B200_WGRAD_CTAS")) : 148;
  int splits = std::max(1, target / std::max(1, mt * nt));
  splits = std::min(splits, nkb);
  int kb = (nkb + splits - 1) / splits;
  splits = (nkb + kb - 1) / kb;
  *kb_per_split = kb;
  return splits;
}

template <typename P>
inline P* at(dsp_block* b, size_t off) {
  return reinterpret_cast<P*>(b->ws + off);
}

// packed storage-dtype weights this block's convs read (its own, or a forward twin's primary's)
inline const uint8_t* packed_base(const dsp_block* b) { return b->wsrc ? b->wsrc : b->ws + b->packed; }

// Tile table of the fused update + repack (kernels.cuh UpdTile): every weight tensor in 32 x 32
// tiles carrying its shadow destinations (conv: [co][tap][ci] same orientation + the per-tap
// transposed DGRAD copy [ci][tap][co]; dense W[in][out]: its [out][in] shadow, transposed),
// then every remaining parameter (BatchNorm gamma / beta, biases) in flat runs of <= 1024.
// Each parameter is covered exactly once (checked).
int build_update_tiles(dsp_block* b) {
  std::vector<char> cov((size_t)std::max<int64_t>(b->param_count, 1), 0);
  auto mark = [&](int64_t i) {
    if (i < 0 || i >= b->param_count || cov[(size_t)i]) return false;
    cov[(size_t)i] = 1;
    return true;
  };
  for (const PackEntry& e : b->packs) {
    if (e.dense_src == 2) continue;  // folded into its conv's tiles below
    if (e.dense_src == 0 && e.s2d_r > 0) {  // space-to-depth stem: per original tap (r, s) = (2a+i, 2b+j)
      int64_t dst_t = -1;
      for (const PackEntry& t : b->packs)
        if (t.dense_src == 2 && t.src_off == e.src_off) dst_t = t.dst_off;
      const int R = e.s2d_r, rs2 = (R + 1) / 2;
      for (int tap = 0; tap < R * R; ++tap) {
        const int r = tap / R, sx = tap % R;
        const int tp = (r / 2) * rs2 + sx / 2, sub = (r & 1) * 2 + (sx & 1);
        for (int co0 = 0; co0 < e.co; co0 += 32)
          for (int ci0 = 0; ci0 < e.ci; ci0 += 32) {
            UpdTile u{};
            u.rows = std::min(32, e.co - co0);
            u.cols = std::min(32, e.ci - ci0);
            u.src = e.src_off + ((int64_t)co0 * R * R + tap) * e.ci + ci0;
            u.src_rs = R * R * e.ci;
            u.dst_a = e.dst_off + ((int64_t)co0 * e.rs + tp) * e.cip + sub * e.ci + ci0;
            u.dst_a_rs = e.rs * e.cip;
            u.dst_b = dst_t < 0 ? -1 : dst_t + ((int64_t)(sub * e.ci + ci0) * e.rs + tp) * e.cop + co0;
            u.dst_b_cs = e.rs * e.cop;
            for (int rr = 0; rr < u.rows; ++rr)
              for (int cc = 0; cc < u.cols; ++cc)
                if (!mark(u.src + (int64_t)rr * u.src_rs + cc)) return set_error(DSP_E_INVALID, "update tiles overlap");
            b->utiles.push_back(u);
          }
      }
    } else if (e.dense_src == 0) {
      int64_t dst_t = -1;
      for (const PackEntry& t : b->packs)
        if (t.dense_src == 2 && t.src_off == e.src_off) dst_t = t.dst_off;
      for (int tap = 0; tap < e.rs; ++tap)
        for (int co0 = 0; co0 < e.co; co0 += 32)
          for (int ci0 = 0; ci0 < e.ci; ci0 += 32) {
            UpdTile u{};
            u.rows = std::min(32, e.co - co0);
            u.cols = std::min(32, e.ci - ci0);
            u.src = e.src_off + ((int64_t)co0 * e.rs + tap) * e.ci + ci0;
            u.src_rs = e.rs * e.ci;
            u.dst_a = e.dst_off + ((int64_t)co0 * e.rs + tap) * e.cip + ci0;
            u.dst_a_rs = e.rs * e.cip;
            u.dst_b = dst_t < 0 ? -1 : dst_t + ((int64_t)ci0 * e.rs + tap) * e.cop + co0;
            u.dst_b_cs = e.rs * e.cop;
            for (int r = 0; r < u.rows; ++r)
              for (int c = 0; c < u.cols; ++c)
                if (!mark(u.src + (int64_t)r * u.src_rs + c)) return set_error(DSP_E_INVALID, "update tiles overlap");
            b->utiles.push_back(u);
          }
    } else {  // dense W[in = ci][out = co] -> shadow [co][cip]
      for (int i0 = 0; i0 < e.ci; i0 += 32)
        for (int o0 = 0; o0 < e.co; o0 += 32) {
          UpdTile u{};
          u.rows = std::min(32, e.ci - i0);
          u.cols = std::min(32, e.co - o0);
          u.src = e.src_off + (int64_t)i0 * e.co + o0;
          u.src_rs = e.co;
          u.dst_a = -1;
          u.dst_b = e.dst_off + (int64_t)o0 * e.cip + i0;
          u.dst_b_cs = e.cip;
          for (int r = 0; r < u.rows; ++r)
            for (int c = 0; c < u.cols; ++c)
              if (!mark(u.src + (int64_t)r * u.src_rs + c)) return set_error(DSP_E_INVALID, "update tiles overlap");
          b->utiles.push_back(u);
        }
    }
  }
  for (int64_t i = 0; i < b->param_count;) {
    if (cov[(size_t)i]) {
      ++i;
      continue;
    }
    int64_t j = i;
    while (j < b->param_count && !cov[(size_t)j] && j - i < 1024) cov[(size_t)j++] = 1;
    UpdTile u{};
    u.src = i;
    u.cols = (int)(j - i);
    u.dst_a = u.dst_b = -1;
    b->utiles.push_back(u);
    i = j;
  }
  return DSP_OK;
}

// ------------------------------------------------------------------ kernels per conv
int conv_fprop(dsp_block* b, const ConvP& c, const void* x, cudaStream_t st) {
  dsp_igemm_args_t a{};
  a.geom = c.g;
  a.M = (int)c.M();
  a.N = c.g.K;
  a.Kd = c.g.R * c.g.S * c.g.C;
  a.A = x;
  a.B = packed_base(b) + (size_t)c.wpack * b->esz;
  a.D = b->ws + c.y;
  a.ldd = c.g.K;
  a.stats = at<float>(b, b->fpart);
  a.n_valid = c.co_real;
  // BatchNorm statistics: per-CTA partials in the epilogue, finalized by the last CTA
  a.stat_out = at<float>(b, c.stat);
  a.gamma = b->params + c.gamma_off;
  a.beta = b->params + c.beta_off;
  a.sem = at<int32_t>(b, b->sem);
  DSP_CUDA(igemm_launch(DSP_IGEMM_FPROP, b->dtype, a, 1, st));
  return DSP_OK;
}

int conv_wgrad(dsp_block* b, const ConvP& c, const void* x, const void* dy, cudaStream_t st) {
  dsp_igemm_args_t a{};
  a.geom = c.g;
  a.M = c.g.R * c.g.S * c.g.C;
  a.N = c.g.K;
  a.Kd = (int)c.M();
  a.A = x;
  a.B = dy;
  a.D = b->ws + b->wpart;
  int kb = 1;
  const int splits = wgrad_splits(c, &kb, b->dtype);
  a.kb_per_split = kb;
  DSP_CUDA(igemm_launch(DSP_IGEMM_WGRAD, b->dtype, a, splits, st));
  DSP_CUDA(wgrad_reduce(at<float>(b, b->wpart), splits, a.M, a.N, c.g.R * c.g.S, c.g.C, c.s2d_r ? c.s2d_ci : c.ci_real,
                        c.co_real, c.s2d_r ? 2 : 0, b->grads + c.w_off, st, c.s2d_r));
  return DSP_OK;
}

// WGRAD of conv c on the block's side stream, ordered after everything already on st.
int conv_wgrad_side(dsp_block* b, const ConvP& c, const void* x, const void* dy, cudaStream_t st) {
  static const bool off = getenv("DSP_B200_NO_WGRAD_SIDE") != nullptr;
  if (off || b->side == nullptr) return conv_wgrad(b, c, x, dy, st);
  DSP_CUDA(cudaEventRecord(b->ev_fork, st));
  DSP_CUDA(cudaStreamWaitEvent(b->side, b->ev_fork, 0));
  DSP_TRY(conv_wgrad(b, c, x, dy, b->side));
  DSP_CUDA(cudaEventRecord(b->ev_join, b->side));
  b->side_busy = true;
  return DSP_OK;
}
// st waits for every side-stream WGRAD issued so far (before their dY / x buffers are reused).
int side_join(dsp_block* b, cudaStream_t st) {
  if (b->side_busy) {
    DSP_CUDA(cudaStreamWaitEvent(st, b->ev_join, 0));
    b->side_busy = false;
  }
  return DSP_OK;
}

// The BatchNorm below a DGRAD output whose backward statistics the DGRAD epilogue computes.
struct BnbFuse {
  const void* mask;  // ReLU mask tensor (the BN's stored output); nullptr: from y (mask_of)
  const ConvP* c1;   // the BN's conv (its y / stat / coef / gamma, beta grads)
  const ConvP* c2;   // optional second BN sharing g (projection shortcut)
  const uint8_t* bits = nullptr;  // the mask as bits (a residual unit's output), read instead
};

void set_bnb_target(dsp_block* b, const ConvP& c, dsp_bnb_target_t& t) {
  t.y = b->ws + c.y;
  t.stat = at<float>(b, c.stat);
  t.gamma = b->params + c.gamma_off;
  t.dgamma = b->grads + c.gamma_off;
  t.dbeta = b->grads + c.beta_off;
  t.coef = at<float>(b, c.coef);
}

int conv_dgrad(dsp_block* b, const ConvP& c, const void* dy, void* dx, const void* residual, cudaStream_t st,
               const BnbFuse* fuse = nullptr) {
  dsp_igemm_args_t a{};
  a.geom = c.g;
  a.M = (int)c.Min();
  a.N = c.g.C;
  a.Kd = c.g.R * c.g.S * c.g.K;
  a.A = dy;
  a.B = packed_base(b) + (size_t)c.wpack * b->esz;
  a.D = dx;
  a.ldd = c.g.C;
  a.residual = residual;
  a.n_valid = c.ci_real;
  if (c.wpack_t >= 0) a.B_t = packed_base(b) + (size_t)c.wpack_t * b->esz;
  if (fuse != nullptr) {
    a.stats = at<float>(b, b->fpart);
    a.sem = at<int32_t>(b, b->sem);
    a.bnb_mask = fuse->bits ? nullptr : fuse->mask;
    a.bnb_mask_bits = fuse->bits;
    a.bnb_count = fuse->c2 ? 2 : 1;
    a.bnb_c_real = fuse->c1->co_real;
    set_bnb_target(b, *fuse->c1, a.bnb[0]);
    if (fuse->c2) set_bnb_target(b, *fuse->c2, a.bnb[1]);
  }
  DSP_CUDA(igemm_launch(DSP_IGEMM_DGRAD, b->dtype, a, 1, st));
  return DSP_OK;
}

// Which BN-backward statistics ride on a DGRAD epilogue (DSP_B200_BNB_FUSE bit mask, A/B knob):
// bit 0 = a unit's inner BNs (on the conv above's DGRAD), bit 1 = the top BN(s) of the layer below
// (on this layer's input DGRAD). Unfused, bn_bwd_stats reads the DGRAD output back.
int bnb_fuse_mask() {
  static const int m = getenv("DSP_B200_BNB_FUSE") ? atoi(getenv("DSP_B200_BNB_FUSE")) : 3;
  return m;
}

// The ReLU mask of a BN whose output is exactly relu(bn(y)) (stem, intra-unit BNs; not a unit's top
// BN, which adds the shortcut first): mask_of returns nullptr and the backward kernels recompute
// the mask from y and the forward's scale / shift instead of reading the stored output -- one
// tensor read fewer per BN backward pass. DSP_B200_MASK_FROM_Y=0 reads the stored output (A/B).
const void* mask_of(const void* stored) {
  static const bool off = getenv("DSP_B200_MASK_FROM_Y") && getenv("DSP_B200_MASK_FROM_Y")[0] == '0';
  return off ? stored : nullptr;
}

// Second pass of the BN backward once its statistics (coef, dgamma, dbeta) exist.
// mask == nullptr: recompute the mask from y (mask_of).
// mbits (optional): the mask as bits (a residual unit's output, LayerP.mbits) -- read instead of `mask`.
int bn_backward_apply(dsp_block* b, const void* gsrc, const void* mask, const ConvP& c1, void* dy1, const ConvP* c2,
                      void* dy2, void* g_out, cudaStream_t st, const uint8_t* mbits = nullptr) {
  DSP_CUDA(bn_bwd_apply(b->dtype, gsrc, mbits ? nullptr : mask, b->ws + c1.y, at<float>(b, c1.stat),
                        at<float>(b, c1.coef), dy1, c2 ? b->ws + c2->y : nullptr, c2 ? at<float>(b, c2->stat) : nullptr,
                        c2 ? at<float>(b, c2->coef) : nullptr, c2 ? dy2 : nullptr, g_out, c1.M(), c1.g.K, st,
                        (mask == nullptr && mbits == nullptr) ? 1 : 0, mbits));
  return DSP_OK;
}

// BN backward for one conv: dy = BNback(g = gsrc*(mask>0)), grads into params layout.
int bn_backward_pair(dsp_block* b, const void* gsrc, const void* mask, const ConvP& c1, void* dy1, const ConvP* c2,
                     void* dy2, void* g_out, cudaStream_t st, const uint8_t* mbits = nullptr) {
  const int64_t M = c1.M();
  const int Cp = c1.g.K;
  int* sem = at<int32_t>(b, b->sem);
  const void* mk = mbits ? nullptr : mask;
  DSP_CUDA(bn_bwd_stats(b->dtype, gsrc, mk, b->ws + c1.y, at<float>(b, c1.stat), at<float>(b, b->bpart), M, Cp,
                        c1.co_real, b->params + c1.gamma_off, b->grads + c1.gamma_off, b->grads + c1.beta_off,
                        at<float>(b, c1.coef), sem, st, (mask == nullptr && mbits == nullptr) ? 1 : 0, mbits));
  if (c2) {
    DSP_CUDA(bn_bwd_stats(b->dtype, gsrc, mk, b->ws + c2->y, at<float>(b, c2->stat), at<float>(b, b->bpart2), M, Cp,
                          c2->co_real, b->params + c2->gamma_off, b->grads + c2->gamma_off, b->grads + c2->beta_off,
                          at<float>(b, c2->coef), sem, st, 0, mbits));
  }
  return bn_backward_apply(b, gsrc, mask, c1, dy1, c2, dy2, g_out, st, mbits);
}

// ------------------------------------------------------------------ layer forward / backward
// The stem's BN-apply + ReLU can ride on the max pool right after it (bf16, mask from y): the
// stem's activation is then never materialised (DSP_B200_NO_POOL_FUSE=1 keeps both launches).
bool stem_pool_fused(const dsp_block* b, const LayerP& l, const LayerP* next) {
  static const bool off = getenv("DSP_B200_NO_POOL_FUSE") != nullptr;
  return !off && next != nullptr && b->dtype == DSP_DTYPE_BF16 && l.d.kind == DSP_LAYER_CONV_BN_RELU &&
         next->d.kind == DSP_LAYER_MAXPOOL && mask_of(b->ws + l.out) == nullptr && (l.convs[0].g.K % 8) == 0 &&
         256 % (l.convs[0].g.K / 8) == 0;
}

// tape = false (a fresh forward): what only the recorded pass's backward reads -- max-pool argmax
// taps, residual units' ReLU mask bits -- is not written
int layer_forward(dsp_block* b, LayerP& l, const void* x, void* out, cudaStream_t st, bool skip_apply = false,
                  const LayerP* fused_stem = nullptr, bool tape = true) {
  const int dt = b->dtype;
  switch (l.d.kind) {
    case DSP_LAYER_DENSE: {
      dsp_igemm_args_t a{};
      a.geom = l.dense.g;
      a.M = b->B;
      a.N = l.out_cp;
      a.Kd = l.in_cp;
      a.A = x;
      a.B = packed_base(b) + (size_t)l.dense.wpack * b->esz;
      a.D = out;
      a.ldd = l.out_cp;
      a.out_f32 = l.logits ? 1 : 0;
      a.bias = l.b_off >= 0 ? b->params + l.b_off : nullptr;
      a.n_valid = l.out_real;
      DSP_CUDA(igemm_launch(DSP_IGEMM_FPROP, dt, a, 1, st));
      return DSP_OK;
    }
    case DSP_LAYER_RELU:
    case DSP_LAYER_TANH:
      DSP_CUDA(act_forward(dt, l.d.kind == DSP_LAYER_TANH, x, out, l.in_elems(), st));
      return DSP_OK;
    case DSP_LAYER_AVGPOOL:
      DSP_CUDA(avgpool_forward(dt, x, out, b->B, l.in_h * l.in_w, l.in_cp, st));
      return DSP_OK;
    case DSP_LAYER_MAXPOOL:
      if (fused_stem != nullptr) {
        const ConvP& c = fused_stem->convs[0];
        DSP_CUDA(maxpool_bnrelu_forward(dt, b->ws + c.y, at<float>(b, c.stat), out,
                                        tape ? at<uint8_t>(b, l.arg) : nullptr, b->B, l.in_h, l.in_w, l.out_h,
                                        l.out_w, l.in_cp, st));
        return DSP_OK;
      }
      DSP_CUDA(maxpool_forward(dt, x, out, tape ? at<uint8_t>(b, l.arg) : nullptr, b->B, l.in_h, l.in_w, l.out_h,
                               l.out_w, l.in_cp, st));
      return DSP_OK;
    case DSP_LAYER_CONV_BN_RELU: {
      const ConvP& c = l.convs[0];
      if (c.s2d_r) {
        DSP_CUDA(s2d_pack(dt, x, b->ws + c.s2d_buf, b->B, c.s2d_h, c.s2d_w, c.s2d_ci, c.s2d_cpx, c.g.H, c.g.W, c.g.C,
                          c.s2d_pad, st));
        x = b->ws + c.s2d_buf;
      }
      DSP_TRY(conv_fprop(b, c, x, st));
      if (!skip_apply)
        DSP_CUDA(bn_apply(dt, b->ws + c.y, at<float>(b, c.stat), nullptr, nullptr, nullptr, out, c.M(), c.g.K, 1, st));
      return DSP_OK;
    }
    case DSP_LAYER_BASIC_UNIT:
    case DSP_LAYER_BOTTLENECK: {
      const bool bott = l.d.kind == DSP_LAYER_BOTTLENECK;
      const int nmain = bott ? 3 : 2;
      const void* cur = x;
      for (int i = 0; i < nmain - 1; ++i) {
        const ConvP& c = l.convs[i];
        DSP_TRY(conv_fprop(b, c, cur, st));
        void* z = b->ws + (i == 0 ? l.z1 : l.z2);
        DSP_CUDA(bn_apply(dt, b->ws + c.y, at<float>(b, c.stat), nullptr, nullptr, nullptr, z, c.M(), c.g.K, 1, st));
        cur = z;
      }
      const ConvP& cl = l.convs[nmain - 1];
      DSP_TRY(conv_fprop(b, cl, cur, st));
      uint8_t* mb = (l.mbits && tape) ? at<uint8_t>(b, l.mbits) : nullptr;
      if (l.proj) {
        const ConvP& cs = l.convs[nmain];
        DSP_TRY(conv_fprop(b, cs, x, st));
        DSP_CUDA(bn_apply(dt, b->ws + cl.y, at<float>(b, cl.stat), nullptr, b->ws + cs.y, at<float>(b, cs.stat), out,
                          cl.M(), cl.g.K, 1, st, mb));
      } else {
        DSP_CUDA(bn_apply(dt, b->ws + cl.y, at<float>(b, cl.stat), x, nullptr, nullptr, out, cl.M(), cl.g.K, 1, st, mb));
      }
      return DSP_OK;
    }
  }
  return set_error(DSP_E_INVALID, "unknown layer kind %d", l.d.kind);
}

// u: gradient w.r.t. the layer output; x: the layer input; dx may be null.
// below: the top BatchNorm(s) of the layer under this one, whose backward statistics the
// final DGRAD (producing dx = that layer's upstream) accumulates; top_done: this layer's top
// BN statistics were produced that way by the layer above (only the apply pass is left).
// pool_u / pool (the fused stem + max pool, stem_pool_fused): the stem's BN backward re-gathers its
// upstream from the pool's upstream pool_u and argmax taps instead of reading a stored gradient
int layer_backward(dsp_block* b, LayerP& l, const void* x, const void* u, void* dx, cudaStream_t st,
                   const BnbFuse* below = nullptr, bool top_done = false, const void* pool_u = nullptr,
                   const LayerP* pool = nullptr) {
  const int dt = b->dtype;
  switch (l.d.kind) {
    case DSP_LAYER_DENSE: {
      if (l.b_off >= 0) {  // bias gradient = column sums of u
        DSP_CUDA(bn_bwd_stats(dt, u, nullptr, nullptr, nullptr, at<float>(b, b->bpart), b->B, l.out_cp, l.out_real,
                              nullptr, nullptr, b->grads + l.b_off, nullptr, at<int32_t>(b, b->sem), st));
      }
      const ConvP& c = l.dense;
      dsp_igemm_args_t a{};
      a.geom = c.g;
      a.M = l.in_cp;
      a.N = l.out_cp;
      a.Kd = b->B;
      a.A = x;
      a.B = u;
      a.D = b->ws + b->wpart;
      int kb = 1;
      const int splits = wgrad_splits(c, &kb, dt);
      a.kb_per_split = kb;
      DSP_CUDA(igemm_launch(DSP_IGEMM_WGRAD, dt, a, splits, st));
      DSP_CUDA(wgrad_reduce(at<float>(b, b->wpart), splits, a.M, a.N, 1, l.in_cp, l.in_real, l.out_real, 1,
                            b->grads + c.w_off, st));
      if (dx) DSP_TRY(conv_dgrad(b, c, u, dx, nullptr, st));
      return DSP_OK;
    }
    case DSP_LAYER_RELU:
    case DSP_LAYER_TANH:
      if (dx) DSP_CUDA(act_backward(dt, l.d.kind == DSP_LAYER_TANH, x, u, dx, l.in_elems(), st));
      return DSP_OK;
    case DSP_LAYER_AVGPOOL:
      if (dx) DSP_CUDA(avgpool_backward(dt, u, dx, b->B, l.in_h * l.in_w, l.in_cp, st));
      return DSP_OK;
    case DSP_LAYER_MAXPOOL:
      if (dx)
        DSP_CUDA(maxpool_backward(dt, u, at<uint8_t>(b, l.arg), dx, b->B, l.in_h, l.in_w, l.out_h, l.out_w, l.in_cp,
                                  st));
      return DSP_OK;
    case DSP_LAYER_CONV_BN_RELU: {
      const ConvP& c = l.convs[0];
      void* dy = b->ws + b->S[0];
      if (pool != nullptr) {
        DSP_CUDA(pool_bn_backward(dt, pool_u, at<uint8_t>(b, pool->arg), b->ws + c.y, at<float>(b, c.stat),
                                  at<float>(b, b->bpart), c.co_real, b->params + c.gamma_off, b->grads + c.gamma_off,
                                  b->grads + c.beta_off, at<float>(b, c.coef), dy, b->B, pool->in_h, pool->in_w,
                                  pool->out_h, pool->out_w, c.g.K, st));
      } else if (top_done)
        DSP_TRY(bn_backward_apply(b, u, mask_of(b->ws + l.out), c, dy, nullptr, nullptr, nullptr, st));
      else
        DSP_TRY(bn_backward_pair(b, u, mask_of(b->ws + l.out), c, dy, nullptr, nullptr, nullptr, st));
      if (c.s2d_r) {  // WGRAD on the recorded s2d input; DGRAD into its gradient, then back to x's layout
        DSP_TRY(conv_wgrad(b, c, b->ws + c.s2d_buf, dy, st));
        if (dx) {
          DSP_TRY(conv_dgrad(b, c, dy, b->ws + c.s2d_buf, nullptr, st));
          DSP_CUDA(s2d_unpack(dt, b->ws + c.s2d_buf, dx, b->B, c.s2d_h, c.s2d_w, c.s2d_ci, c.s2d_cpx, c.g.H, c.g.W,
                              c.g.C, c.s2d_pad, st));
        }
        return DSP_OK;
      }
      DSP_TRY(conv_wgrad(b, c, x, dy, st));
      if (dx) DSP_TRY(conv_dgrad(b, c, dy, dx, nullptr, st, below));
      return DSP_OK;
    }
    case DSP_LAYER_BASIC_UNIT:
    case DSP_LAYER_BOTTLENECK: {
      const bool bott = l.d.kind == DSP_LAYER_BOTTLENECK;
      const int nmain = bott ? 3 : 2;
      void* S0 = b->ws + b->S[0];
      void* S1 = b->ws + b->S[1];
      void* S2 = b->ws + b->S[2];
      void* S3 = b->ws + b->S[3];
      const ConvP& cl = l.convs[nmain - 1];
      const ConvP* cs = l.proj ? &l.convs[nmain] : nullptr;
      // top BN(s): g = u * (out > 0); dy_last -> S0, dy_sc -> S1 (proj) or g -> S1 (identity)
      const uint8_t* mb = l.mbits ? at<uint8_t>(b, l.mbits) : nullptr;
      if (top_done)
        DSP_TRY(bn_backward_apply(b, u, b->ws + l.out, cl, S0, cs, cs ? S1 : nullptr, cs ? nullptr : S1, st, mb));
      else
        DSP_TRY(bn_backward_pair(b, u, b->ws + l.out, cl, S0, cs, cs ? S1 : nullptr, cs ? nullptr : S1, st, mb));
      // walk the main path down
      for (int i = nmain - 1; i >= 0; --i) {
        const ConvP& c = l.convs[i];
        const void* cin = i == 0 ? x : b->ws + (i == 1 ? l.z1 : l.z2);
        DSP_TRY(conv_wgrad_side(b, c, cin, S0, st));
        if (i == 0) break;
        // dz_{i}, with the BN-backward statistics of conv i-1 accumulated in the epilogue
        const ConvP& cb = l.convs[i - 1];
        const void* zmask = b->ws + (i == 1 ? l.z1 : l.z2);
        const BnbFuse fuse{mask_of(zmask), &cb, nullptr};
        const bool fused = (bnb_fuse_mask() & 1) != 0;
        DSP_TRY(conv_dgrad(b, c, S0, S2, nullptr, st, fused ? &fuse : nullptr));
        DSP_TRY(side_join(b, st));  // the WGRAD reading S0 is done before S0 is overwritten
        if (fused)
          DSP_TRY(bn_backward_apply(b, S2, mask_of(zmask), cb, S0, nullptr, nullptr, nullptr, st));
        else
          DSP_TRY(bn_backward_pair(b, S2, mask_of(zmask), cb, S0, nullptr, nullptr, nullptr, st));
      }
      const void* res = S1;
      if (cs) {
        DSP_TRY(conv_wgrad_side(b, *cs, x, S1, st));
        if (dx) DSP_TRY(conv_dgrad(b, *cs, S1, S3, nullptr, st));
        res = S3;
      }
      if (dx) DSP_TRY(conv_dgrad(b, l.convs[0], S0, dx, res, st, below));
      DSP_TRY(side_join(b, st));
      return DSP_OK;
    }
  }
  return set_error(DSP_E_INVALID, "unknown layer kind %d", l.d.kind);
}

}  // namespace
}  // namespace dsp

using namespace dsp;

// ==================================================================== C ABI
extern "C" int dsp_block_create(const dsp_layer_desc_t* layers, int n_layers, int batch, int dtype, int is_last,
                                dsp_block_t** out) {
  if (!layers || n_layers <= 0 || batch <= 0 || !out) return set_error(DSP_E_INVALID, "dsp_block_create: bad args");
  if (dtype != DSP_DTYPE_BF16 && dtype != DSP_DTYPE_F32)
    return set_error(DSP_E_INVALID, "dsp_block_create: dtype %d is neither DSP_DTYPE_BF16 nor DSP_DTYPE_F32", dtype);
  dsp_block* b = new dsp_block();
  b->B = batch;
  b->dtype = dtype;
  b->is_last = is_last;
  b->esz = dtype == DSP_DTYPE_F32 ? 4 : 2;
  Planner pl;
  const int B = batch;
  // running shape (real channels, h, w)
  int cur_c = 0, cur_h = 1, cur_w = 1;
  {
    const dsp_layer_desc_t& d0 = layers[0];
    cur_c = d0.in_c;
    cur_h = d0.kind == DSP_LAYER_DENSE ? 1 : std::max(1, d0.in_h);
    cur_w = d0.kind == DSP_LAYER_DENSE ? 1 : std::max(1, d0.in_w);
    if (d0.kind == DSP_LAYER_RELU || d0.kind == DSP_LAYER_TANH) {
      delete b;
      return set_error(DSP_E_INVALID, "a block cannot start with an activation (its width is unknown)");
    }
  }
  int64_t max_act = 0, max_fpart = 0, max_bpart = 0, max_wpart = 0;
  int64_t pack_elems = 0;
  std::vector<ConvP*> all_convs;
  b->L.resize(n_layers);
  for (int i = 0; i < n_layers; ++i) {
    LayerP& l = b->L[i];
    l.d = layers[i];
    const dsp_layer_desc_t& d = l.d;
    const int kind = d.kind;
    b->param_count = std::max<int64_t>(b->param_count, d.param_offset + d.param_count);
    if (kind == DSP_LAYER_DENSE) {
      if (cur_h * cur_w != 1 || d.in_c != cur_c) {
        const int flat = cur_c * cur_h * cur_w;
        delete b;
        return set_error(DSP_E_INVALID, "layer %d: dense(%d,%d) does not accept width %d", i, d.in_c, d.out_c, flat);
      }
      l.in_real = d.in_c;
      l.out_real = d.out_c;
      l.in_cp = pad8(d.in_c);
      l.out_cp = pad8(d.out_c);
      l.in_rows = l.out_rows = B;
      make_conv(l.dense, B, 1, 1, d.in_c, d.out_c, 1, 1, 0);
      l.dense.w_off = d.param_offset;
      l.b_off = d.bias ? d.param_offset + (int64_t)d.in_c * d.out_c : -1;
      l.dense.wpack = pack_elems;
      pack_elems += (int64_t)l.dense.g.K * l.dense.g.C;
      b->packs.push_back({l.dense.w_off, l.dense.wpack, d.out_c, d.in_c, 1, l.dense.g.K, l.dense.g.C, 1, 0, 0});
      l.logits = is_last && i == n_layers - 1;
      cur_c = d.out_c;
      int kb = 1;
      const int sp = wgrad_splits(l.dense, &kb, dtype);
      max_wpart = std::max<int64_t>(max_wpart, (int64_t)sp * l.in_cp * l.out_cp);
      max_bpart = std::max<int64_t>(max_bpart, (int64_t)bn_bwd_chunks(B, l.out_cp) * 2 * l.out_cp);
    } else if (kind == DSP_LAYER_RELU || kind == DSP_LAYER_TANH) {
      l.in_real = l.out_real = cur_c;
      l.in_cp = l.out_cp = pad8(cur_c);
      l.in_h = l.out_h = cur_h;
      l.in_w = l.out_w = cur_w;
      l.in_rows = l.out_rows = (int64_t)B * cur_h * cur_w;
    } else {
      if (d.in_c != cur_c || d.in_h != cur_h || d.in_w != cur_w) {
        delete b;
        return set_error(DSP_E_INVALID, "layer %d: expects input (%d,%d,%d), got (%d,%d,%d)", i, d.in_c, d.in_h,
                         d.in_w, cur_c, cur_h, cur_w);
      }
      l.in_real = d.in_c;
      l.in_cp = pad8(d.in_c);
      l.in_h = d.in_h;
      l.in_w = d.in_w;
      l.in_rows = (int64_t)B * d.in_h * d.in_w;
      int64_t off = d.param_offset;
      auto add_conv = [&](int H, int W, int ci, int co, int k, int stride, int pad) {
        ConvP c;
        make_conv(c, B, H, W, ci, co, k, stride, pad);
        c.w_off = off;
        off += (int64_t)co * k * k * ci;
        c.gamma_off = off;
        off += co;
        c.beta_off = off;
        off += co;
        c.wpack = pack_elems;
        pack_elems += (int64_t)c.g.K * k * k * c.g.C;
        if (stride == 1 || stride == 2) {  // DGRAD's K-major weights (TMA / halo tiles, parity-split stride 2)
          c.wpack_t = pack_elems;
          pack_elems += (int64_t)c.g.K * k * k * c.g.C;
        }
        l.convs.push_back(c);
        return l.convs.back().g;
      };
      if (kind == DSP_LAYER_CONV_BN_RELU) {
        const int k = d.ksize > 0 ? d.ksize : 3;
        const int pad = k / 2;
        static const bool no_s2d = getenv("DSP_B200_NO_S2D") != nullptr;
        const bool s2d = !no_s2d && d.stride == 2 && k >= 5 && (k & 1) && d.in_c <= 4 && (d.in_h + 2 * pad) % 2 == 0 &&
                         (d.in_w + 2 * pad) % 2 == 0;
        if (s2d) {
          const int rs2 = (k + 1) / 2, hs = (d.in_h + 2 * pad) / 2, ws = (d.in_w + 2 * pad) / 2;
          ConvP c;
          make_conv(c, B, hs, ws, 4 * d.in_c, d.out_c, rs2, 1, 0);
          c.s2d_r = k;
          c.s2d_ci = d.in_c;
          c.s2d_h = d.in_h;
          c.s2d_w = d.in_w;
          c.s2d_cpx = pad8(d.in_c);
          c.s2d_pad = pad;
          c.w_off = off;
          off += (int64_t)d.out_c * k * k * d.in_c;
          c.gamma_off = off;
          off += d.out_c;
          c.beta_off = off;
          off += d.out_c;
          c.wpack = pack_elems;
          pack_elems += (int64_t)c.g.K * rs2 * rs2 * c.g.C;
          c.wpack_t = pack_elems;
          pack_elems += (int64_t)c.g.K * rs2 * rs2 * c.g.C;
          l.convs.push_back(c);
          l.out_h = c.g.P;
          l.out_w = c.g.Q;
        } else {
          auto g = add_conv(d.in_h, d.in_w, d.in_c, d.out_c, k, d.stride, pad);
          l.out_h = g.P;
          l.out_w = g.Q;
        }
        l.out_real = d.out_c;
      } else if (kind == DSP_LAYER_BASIC_UNIT) {
        auto g1 = add_conv(d.in_h, d.in_w, d.in_c, d.out_c, 3, d.stride, 1);
        add_conv(g1.P, g1.Q, d.out_c, d.out_c, 3, 1, 1);
        l.proj = d.stride != 1 || d.in_c != d.out_c;
        if (l.proj) add_conv(d.in_h, d.in_w, d.in_c, d.out_c, 1, d.stride, 0);
        l.out_h = g1.P;
        l.out_w = g1.Q;
        l.out_real = d.out_c;
      } else if (kind == DSP_LAYER_BOTTLENECK) {
        add_conv(d.in_h, d.in_w, d.in_c, d.mid_c, 1, 1, 0);
        auto g2 = add_conv(d.in_h, d.in_w, d.mid_c, d.mid_c, 3, d.stride, 1);
        add_conv(g2.P, g2.Q, d.mid_c, d.out_c, 1, 1, 0);
        l.proj = d.stride != 1 || d.in_c != d.out_c;
        if (l.proj) add_conv(d.in_h, d.in_w, d.in_c, d.out_c, 1, d.stride, 0);
        l.out_h = g2.P;
        l.out_w = g2.Q;
        l.out_real = d.out_c;
      } else if (kind == DSP_LAYER_AVGPOOL) {
        l.out_h = l.out_w = 1;
        l.out_real = d.in_c;
      } else if (kind == DSP_LAYER_MAXPOOL) {
        l.out_h = (d.in_h + 2 - 3) / 2 + 1;
        l.out_w = (d.in_w + 2 - 3) / 2 + 1;
        l.out_real = d.in_c;
      } else {
        delete b;
        return set_error(DSP_E_INVALID, "layer %d: unknown kind %d", i, kind);
      }
      if (off != d.param_offset + d.param_count) {
        delete b;
        return set_error(DSP_E_INVALID, "layer %d: param_count %lld does not match the layout (%lld)", i,
                         (long long)d.param_count, (long long)(off - d.param_offset));
      }
      l.out_cp = pad8(l.out_real);
      l.out_rows = (int64_t)B * l.out_h * l.out_w;
      cur_c = l.out_real;
      cur_h = l.out_h;
      cur_w = l.out_w;
    }
    max_act = std::max(max_act, std::max(l.in_elems(), l.out_elems()));
  }
  // second pass: per-layer buffers (after all convs exist so vectors are stable)
  for (int i = 0; i < n_layers; ++i) {
    LayerP& l = b->L[i];
    l.out = pl.take((size_t)l.out_elems() * (l.logits ? 4 : b->esz));
    if (l.d.kind == DSP_LAYER_MAXPOOL) l.arg = pl.take((size_t)l.out_elems());  // argmax tap bytes
    for (size_t ci = 0; ci < l.convs.size(); ++ci) {
      ConvP& c = l.convs[ci];
      c.y = pl.take((size_t)c.M() * c.g.K * b->esz);
      c.stat = pl.take((size_t)4 * c.g.K * 4);
      c.coef = pl.take((size_t)3 * c.g.K * 4);
      max_act = std::max(max_act, std::max(c.M() * c.g.K, c.Min() * c.g.C));
      max_fpart = std::max<int64_t>(max_fpart, (int64_t)DSP_IGEMM_MAX_CTAS * 3 * std::max(c.g.K, c.g.C));
      max_bpart = std::max<int64_t>(max_bpart, (int64_t)bn_bwd_chunks(c.M(), c.g.K) * 2 * c.g.K);
      int kb = 1;
      const int sp = wgrad_splits(c, &kb, dtype);
      max_wpart = std::max<int64_t>(max_wpart, (int64_t)sp * c.g.R * c.g.S * c.g.C * c.g.K);
      const int pci = c.s2d_r ? c.s2d_ci : c.ci_real;  // the parameter tensor's input channels
      b->packs.push_back({c.w_off, c.wpack, c.co_real, pci, c.g.R * c.g.S, c.g.K, c.g.C, 0, c.s2d_r, 0});
      if (c.wpack_t >= 0)
        b->packs.push_back({c.w_off, c.wpack_t, c.co_real, pci, c.g.R * c.g.S, c.g.K, c.g.C, 2, c.s2d_r, 0});
      if (c.s2d_r) c.s2d_buf = pl.take((size_t)c.Min() * c.g.C * b->esz);
    }
    if (l.d.kind == DSP_LAYER_BASIC_UNIT || l.d.kind == DSP_LAYER_BOTTLENECK) {
      static const bool no_bits = getenv("DSP_B200_MASK_BITS") && getenv("DSP_B200_MASK_BITS")[0] == '0';
      if (dtype == DSP_DTYPE_BF16 && !no_bits) l.mbits = pl.take((size_t)l.out_elems() / 8);
      l.z1 = pl.take((size_t)l.convs[0].M() * l.convs[0].g.K * b->esz);
      if (l.d.kind == DSP_LAYER_BOTTLENECK) l.z2 = pl.take((size_t)l.convs[1].M() * l.convs[1].g.K * b->esz);
    }
  }
  const LayerP& last = b->L.back();
  if (is_last) {
    if (!last.logits) {
      delete b;
      return set_error(DSP_E_INVALID, "the last block must end with a dense layer (logits)");
    }
    b->classes = last.out_real;
    b->classes_pad = last.out_cp;
    b->dlogits = pl.take((size_t)B * last.out_cp * b->esz);
  }
  for (int s = 0; s < 4; ++s) b->S[s] = pl.take((size_t)max_act * b->esz);
  for (int s = 0; s < 2; ++s) b->G[s] = pl.take((size_t)max_act * b->esz);
  b->fpart = pl.take((size_t)std::max<int64_t>(max_fpart, 1) * 4);
  b->sem = pl.take(4096);  // DSP_IGEMM_SEM_INTS tickets, zeroed at bind; the fused-finalize kernels leave them zero
  b->bpart = pl.take((size_t)std::max<int64_t>(max_bpart, 1) * 4);
  b->bpart2 = pl.take((size_t)std::max<int64_t>(max_bpart, 1) * 4);
  b->wpart = pl.take((size_t)std::max<int64_t>(max_wpart, 1) * 4);
  if (build_update_tiles(b) != DSP_OK) {
    delete b;
    return DSP_E_INVALID;
  }
  b->upart = pl.take((size_t)std::max(update_grid(std::max<int64_t>(b->param_count, 1)),
                                      update_pack_grid((int)b->utiles.size())) * 8);
  b->usem = pl.take(256);  // update grad-norm ticket (zeroed at bind, left zero)
  b->nf = pl.take(256);    // sticky non-finite flags (dsp_block_nonfinite)
  b->lsem = pl.take(256);  // softmax_xent ticket
  b->rowloss = pl.take((size_t)B * 4);
  b->packed = pl.take((size_t)std::max<int64_t>(pack_elems, 1) * b->esz);
  b->ptable = pl.take(sizeof(PackEntry) * std::max<size_t>(b->packs.size(), 1));
  b->utable = pl.take(sizeof(UpdTile) * std::max<size_t>(b->utiles.size(), 1));
  for (auto& p : b->packs) b->pack_max = std::max(b->pack_max, p.cop * p.rs * p.cip);
  b->ws_bytes = pl.off;
  *out = b;
  return DSP_OK;
}

extern "C" void dsp_block_destroy(dsp_block_t* blk) { delete blk; }
extern "C" int64_t dsp_block_workspace_bytes(const dsp_block_t* b) { return b ? (int64_t)b->ws_bytes : -1; }
extern "C" int64_t dsp_block_in_elems(const dsp_block_t* b) { return b ? b->L.front().in_elems() : -1; }
extern "C" int64_t dsp_block_out_elems(const dsp_block_t* b) { return b ? b->L.back().out_elems() : -1; }
extern "C" int64_t dsp_block_param_count(const dsp_block_t* b) { return b ? b->param_count : -1; }

extern "C" int dsp_block_pack(dsp_block_t* b, void* stream) {
  if (!b || !b->ws) return set_error(DSP_E_STATE, "dsp_block_pack: block not bound");
  if (b->wsrc) return DSP_OK;  // forward twin: the primary's pack is the one read
  DSP_CUDA(pack_weights(b->dtype, b->params, b->ws + b->packed, at<PackEntry>(b, b->ptable), (int)b->packs.size(),
                        b->pack_max, (cudaStream_t)stream));
  return DSP_OK;
}

extern "C" int dsp_block_bind(dsp_block_t* b, void* workspace, float* params, float* grads, void* stream) {
  if (!b || !workspace || (b->param_count > 0 && (!params || !grads)))
    return set_error(DSP_E_INVALID, "dsp_block_bind: null pointer");
  b->ws = static_cast<uint8_t*>(workspace);
  b->params = params;
  b->grads = grads;
  b->tape_valid = false;
  cudaStream_t st = (cudaStream_t)stream;
  if (b->side == nullptr) {  // created here, never during a graph capture
    DSP_CUDA(cudaStreamCreateWithFlags(&b->side, cudaStreamNonBlocking));
    DSP_CUDA(cudaEventCreateWithFlags(&b->ev_fork, cudaEventDisableTiming));
    DSP_CUDA(cudaEventCreateWithFlags(&b->ev_join, cudaEventDisableTiming));
  }
  // pad channels of every activation must read as zero; zero the whole workspace once
  DSP_CUDA(cudaMemsetAsync(b->ws, 0, b->ws_bytes, st));
  if (!b->packs.empty())
    DSP_CUDA(cudaMemcpyAsync(b->ws + b->ptable, b->packs.data(), sizeof(PackEntry) * b->packs.size(),
                             cudaMemcpyHostToDevice, st));
  if (!b->utiles.empty())
    DSP_CUDA(cudaMemcpyAsync(b->ws + b->utable, b->utiles.data(), sizeof(UpdTile) * b->utiles.size(),
                             cudaMemcpyHostToDevice, st));
  DSP_CUDA(cudaStreamSynchronize(st));  // the table sources are host vectors
  return dsp_block_pack(b, stream);
}

extern "C" int dsp_block_forward(dsp_block_t* b, const void* x, void* y, int record, void* stream) {
  if (!b || !b->ws) return set_error(DSP_E_STATE, "dsp_block_forward: block not bound");
  if (!x) return set_error(DSP_E_INVALID, "dsp_block_forward: null input");
  cudaStream_t st = (cudaStream_t)stream;
  const int n = (int)b->L.size();
  const void* cur = x;
  b->tape_valid = false;
  for (int i = 0; i < n; ++i) {
    LayerP& l = b->L[i];
    void* out = b->ws + l.out;
    if (i == n - 1 && !record && !b->is_last) {
      if (!y) return set_error(DSP_E_INVALID, "dsp_block_forward: fresh forward needs an output buffer");
      out = y;
    }
    const bool fuse_next = stem_pool_fused(b, l, i + 1 < n ? &b->L[i + 1] : nullptr);
    const bool fused_here = i > 0 && stem_pool_fused(b, b->L[i - 1], &l);
    DSP_TRY(layer_forward(b, l, cur, out, st, fuse_next, fused_here ? &b->L[i - 1] : nullptr, record != 0));
    cur = out;
  }
  if (b->is_last && y) {
    const LayerP& l = b->L.back();
    DSP_CUDA(cudaMemcpyAsync(y, b->ws + l.out, (size_t)b->B * l.out_cp * sizeof(float), cudaMemcpyDeviceToDevice, st));
  }
  if (record) {
    b->tape_valid = true;
    b->rec_x = x;
  }
  return DSP_OK;
}

extern "C" int dsp_block_loss(dsp_block_t* b, const int64_t* labels, float* loss, void* stream) {
  if (!b || !b->ws) return set_error(DSP_E_STATE, "dsp_block_loss: block not bound");
  if (!b->is_last) return set_error(DSP_E_STATE, "dsp_block_loss: only the last block owns the loss");
  if (!b->tape_valid) return set_error(DSP_E_STATE, "dsp_block_loss: no recorded forward");
  if (!labels || !loss) return set_error(DSP_E_INVALID, "dsp_block_loss: null pointer");
  const LayerP& l = b->L.back();
  DSP_CUDA(softmax_xent(b->dtype, at<float>(b, l.out), l.out_cp, b->B, b->classes, labels, b->ws + b->dlogits, loss,
                        at<float>(b, b->rowloss), at<int>(b, b->lsem), at<int>(b, b->nf), (cudaStream_t)stream));
  return DSP_OK;
}

extern "C" int dsp_block_backward(dsp_block_t* b, const void* upstream, void* grad_in, void* stream) {
  if (!b || !b->ws) return set_error(DSP_E_STATE, "dsp_block_backward: block not bound");
  if (!b->tape_valid) return set_error(DSP_E_STATE, "forward tape already consumed or never recorded");
  b->tape_valid = false;
  cudaStream_t st = (cudaStream_t)stream;
  const void* u = b->is_last ? (const void*)(b->ws + b->dlogits) : upstream;
  if (!u) return set_error(DSP_E_INVALID, "dsp_block_backward: null upstream");
  const int n = (int)b->L.size();
  DSP_CUDA(cudaMemsetAsync(b->grads, 0, sizeof(float) * b->param_count, st));
  auto has_top_bn = [](const LayerP& l) {
    return l.d.kind == DSP_LAYER_CONV_BN_RELU || l.d.kind == DSP_LAYER_BASIC_UNIT ||
           l.d.kind == DSP_LAYER_BOTTLENECK;
  };
  bool top_done = false;
  const void* pool_u = nullptr;  // upstream of a max pool whose stem below is fused with it
  for (int i = n - 1; i >= 0; --i) {
    LayerP& l = b->L[i];
    // fused stem + max pool: the pool's backward is folded into the stem's BN backward
    if (l.d.kind == DSP_LAYER_MAXPOOL && i > 0 && stem_pool_fused(b, b->L[i - 1], &l)) {
      pool_u = u;
      top_done = false;
      continue;
    }
    if (pool_u != nullptr) {
      const void* x0 = i == 0 ? b->rec_x : (const void*)(b->ws + b->L[i - 1].out);
      void* dx0 = i == 0 ? grad_in : (void*)(b->ws + b->G[i & 1]);
      DSP_TRY(layer_backward(b, l, x0, nullptr, dx0, st, nullptr, false, pool_u, &b->L[i + 1]));
      pool_u = nullptr;
      top_done = false;
      u = dx0;
      continue;
    }
    const void* x = i == 0 ? b->rec_x : (const void*)(b->ws + b->L[i - 1].out);
    void* dx = i == 0 ? grad_in : (void*)(b->ws + b->G[i & 1]);
    // the layer below's top BN statistics ride on this layer's final DGRAD (g = dx * (x > 0))
    BnbFuse fz{};
    const BnbFuse* below = nullptr;
    const bool s2d = l.d.kind == DSP_LAYER_CONV_BN_RELU && l.convs[0].s2d_r;  // its dx is unpacked after DGRAD
    if (i > 0 && dx != nullptr && !s2d && has_top_bn(l) && has_top_bn(b->L[i - 1]) && (bnb_fuse_mask() & 2)) {
      const LayerP& lb = b->L[i - 1];
      const int nmain = lb.d.kind == DSP_LAYER_BOTTLENECK ? 3 : lb.d.kind == DSP_LAYER_BASIC_UNIT ? 2 : 1;
      // a stem below (relu(bn(y)), no shortcut): its mask comes from y too
      fz = BnbFuse{lb.d.kind == DSP_LAYER_CONV_BN_RELU ? mask_of(x) : x, &lb.convs[nmain - 1],
                   lb.proj ? &lb.convs[nmain] : nullptr, lb.mbits ? at<uint8_t>(b, lb.mbits) : nullptr};
      below = &fz;
    }
    DSP_TRY(layer_backward(b, l, x, u, dx, st, below, top_done));
    top_done = below != nullptr;
    u = dx;
  }
  return DSP_OK;
}

extern "C" int dsp_block_update(dsp_block_t* b, int rule, float* ys, double lr, double slr, double beta, double wd,
                                int apply, float* grad_sq_out, void* stream) {
  if (!b || !b->ws) return set_error(DSP_E_STATE, "dsp_block_update: block not bound");
  if (rule != DSP_RULE_SGD && rule != DSP_RULE_SUM) return set_error(DSP_E_INVALID, "dsp_block_update: bad rule");
  if (rule == DSP_RULE_SUM && !ys) return set_error(DSP_E_INVALID, "dsp_block_update: SUM needs ys");
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t n = b->param_count;
  if (n == 0) {
    if (grad_sq_out) DSP_CUDA(cudaMemsetAsync(grad_sq_out, 0, sizeof(float), st));
    return DSP_OK;
  }
  // one launch: update + weight-shadow repack + grad norm (or, for a discarded warmup update,
  // pipeline.py:594, the grad norm alone)
  DSP_CUDA(update_pack(b->dtype, rule, apply, at<UpdTile>(b, b->utable), (int)b->utiles.size(), b->params, b->grads,
                       ys, b->ws + b->packed, (float)lr, (float)slr, (float)beta, (float)wd, at<float>(b, b->upart),
                       at<int>(b, b->usem), grad_sq_out, at<int>(b, b->nf), st));
  return DSP_OK;
}

extern "C" int dsp_block_update_adam(dsp_block_t* b, void* state, double lr, double b1, double b2, double eps,
                                     double wd, int apply, float* grad_sq_out, void* stream) {
  if (!b || !b->ws) return set_error(DSP_E_STATE, "dsp_block_update_adam: block not bound");
  if (!state) return set_error(DSP_E_INVALID, "dsp_block_update_adam: null state");
  if (!(b1 >= 0.0 && b1 < 1.0) || !(b2 >= 0.0 && b2 < 1.0) || !(eps > 0.0))
    return set_error(DSP_E_INVALID, "dsp_block_update_adam: bad hyper-parameters");
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t n = b->param_count;
  if (n == 0) {
    if (grad_sq_out) DSP_CUDA(cudaMemsetAsync(grad_sq_out, 0, sizeof(float), st));
    return DSP_OK;
  }
  float* part = at<float>(b, b->upart);
  float* m = static_cast<float*>(state);
  if (apply) {
    int64_t* t = reinterpret_cast<int64_t*>(m + 2 * n);
    DSP_CUDA(update_adam<float>(n, b->params, b->grads, m, m + n, t, 0.0, 0.0, lr, b1, b2, eps, wd, part, st));
  } else {
    DSP_CUDA(sumsq_f32(n, b->grads, part, st));  // grad norm only (discarded warmup update)
  }
  if (grad_sq_out) DSP_CUDA(sum_partials_f32(part, update_grid(n), grad_sq_out, st));
  if (apply) DSP_TRY(dsp_block_pack(b, stream));
  return DSP_OK;
}

extern "C" int dsp_block_share_weights(dsp_block_t* twin, const dsp_block_t* primary) {
  if (!twin || !primary || !twin->ws || !primary->ws)
    return set_error(DSP_E_STATE, "dsp_block_share_weights: both blocks must be bound");
  if (twin == primary) return set_error(DSP_E_INVALID, "dsp_block_share_weights: a block cannot twin itself");
  bool same = twin->B == primary->B && twin->dtype == primary->dtype && twin->param_count == primary->param_count &&
              twin->packs.size() == primary->packs.size() && twin->params == primary->params;
  for (size_t i = 0; same && i < twin->packs.size(); ++i)
    same = memcmp(&twin->packs[i], &primary->packs[i], sizeof(PackEntry)) == 0;
  if (!same)
    return set_error(DSP_E_INVALID,
                     "dsp_block_share_weights: twin must be planned from the same program and bound to the "
                     "primary's params");
  twin->wsrc = primary->ws + primary->packed;
  return DSP_OK;
}

extern "C" int dsp_block_nonfinite(dsp_block_t* b, int clear, int* flags_out, void* stream) {
  if (!b || !b->ws) return set_error(DSP_E_STATE, "dsp_block_nonfinite: block not bound");
  if (!flags_out) return set_error(DSP_E_INVALID, "dsp_block_nonfinite: null output");
  cudaStream_t st = (cudaStream_t)stream;
  int v = 0;
  DSP_CUDA(cudaMemcpyAsync(&v, b->ws + b->nf, sizeof(int), cudaMemcpyDeviceToHost, st));
  DSP_CUDA(cudaStreamSynchronize(st));
  if (clear && v) DSP_CUDA(cudaMemsetAsync(b->ws + b->nf, 0, sizeof(int), st));
  *flags_out = v;
  return DSP_OK;
}
