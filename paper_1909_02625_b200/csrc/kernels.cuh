// Launch wrappers for the non-GEMM kernels of the DSP block step (elementwise.cu).
// All activation tensors are NHWC with the channel dimension padded to a
// multiple of 8 ("Cp"); pad channels always hold exact zeros.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include "../../include/dsp_b200.h"

namespace dsp {

// Counts every kernel launch issued by this library (dsp_launch_count()).
void note_launch();

cudaError_t igemm_launch(int mode, int dtype, const dsp_igemm_args_t& a, int splits, cudaStream_t st);
int probe_arm(int mode, int n, int64_t m, void* const* events, int n_pairs);
int probe_reset();

// BatchNorm forward: reduce igemm partials [tiles][2][Cp] -> per-channel
// stat[0]=mean, stat[1]=invstd, stat[2]=scale(gamma*invstd), stat[3]=shift(beta-mean*scale)
// (each [Cp]). gamma/beta point into the fp32 params (c_real entries).
cudaError_t bn_finalize(const float* part, int tiles, int Cp, int c_real, int64_t count, const float* gamma,
                        const float* beta, float* stat, cudaStream_t st);

// out = act(y*scale + shift  [+ res]  [+ y2*scale2 + shift2]); act = relu if relu.
// mbits (optional, bf16): one byte per 8 channels of every row, bit i = stored out > 0 -- the ReLU
// mask the backward reads instead of the 16-byte output vector.
cudaError_t bn_apply(int dtype, const void* y, const float* stat, const void* res, const void* y2,
                     const float* stat2, void* out, int64_t M, int Cp, int relu, cudaStream_t st,
                     uint8_t* mbits = nullptr);

// BatchNorm backward, reduction half: g = gsrc * (mask > 0 if mask);
// xhat = (y - mean) * invstd (if y != null, else 0).  Writes per-chunk
// partial (sum g, sum g*xhat) [chunks][2][Cp]; returns the chunk count.
int bn_bwd_chunks(int64_t M, int Cp);
// relu_y (mask == nullptr): the ReLU mask is recomputed from y as relu(y*scale + shift) > 0 with the
// forward's scale / shift (stat rows 2, 3) -- for BNs whose output is exactly relu(bn(y)) (no
// residual), so the backward never reads the stored BN output.
cudaError_t bn_bwd_reduce(int dtype, const void* gsrc, const void* mask, const void* y, const float* stat,
                          float* part, int64_t M, int Cp, cudaStream_t st, int relu_y = 0,
                          const uint8_t* mbits = nullptr);
// Reduction + finalize in one launch: the last CTA to finish (atomic ticket on
// *sem, which must be 0 and is left 0) sums the partials in fixed order and
// writes dgamma/dbeta/coef exactly like bn_bwd_finalize.
cudaError_t bn_bwd_stats(int dtype, const void* gsrc, const void* mask, const void* y, const float* stat, float* part,
                         int64_t M, int Cp, int c_real, const float* gamma, float* dgamma, float* dbeta, float* coef,
                         int* sem, cudaStream_t st, int relu_y = 0, const uint8_t* mbits = nullptr);
// Finalize: sum partials -> dgamma/dbeta into the flat grad (if non-null) and
// coefficients coef[0]=gamma*invstd, coef[1]=sum(g)/M, coef[2]=sum(g*xhat)/M.
// With gamma == null (bias gradient) only dbeta = sum(g) is produced.
cudaError_t bn_bwd_finalize(const float* part, int chunks, int Cp, int c_real, int64_t count, const float* gamma,
                            const float* stat, float* dgamma, float* dbeta, float* coef, cudaStream_t st);
// Apply: dy = coef0*(g - coef1 - xhat*coef2); optional second BN (y_b, stat_b, coef_b -> dy_b)
// sharing g; optional g_out = g.
cudaError_t bn_bwd_apply(int dtype, const void* gsrc, const void* mask, const void* y, const float* stat,
                         const float* coef, void* dy, const void* y_b, const float* stat_b, const float* coef_b,
                         void* dy_b, void* g_out, int64_t M, int Cp, cudaStream_t st, int relu_y = 0,
                         const uint8_t* mbits = nullptr);

// Dense activations (tensor.py:59-83): out = relu/tanh(x); dx = u * act'(x).
cudaError_t act_forward(int dtype, int tanh_kind, const void* x, void* out, int64_t n, cudaStream_t st);
cudaError_t act_backward(int dtype, int tanh_kind, const void* x, const void* u, void* dx, int64_t n, cudaStream_t st);

// Global average pool NHWC [B][HW][Cp] -> [B][Cp] and its backward.
cudaError_t avgpool_forward(int dtype, const void* x, void* out, int B, int HW, int Cp, cudaStream_t st);
cudaError_t avgpool_backward(int dtype, const void* u, void* dx, int B, int HW, int Cp, cudaStream_t st);

// 3x3 stride-2 pad-1 max pool and backward (argmax of the first max in (r,s) order).
// arg: the argmax tap (0..8) of every output element, one byte each.
// the stem's BN-apply + ReLU fused into the pool (bf16; y / stat = the stem conv's output and BN stats)
cudaError_t maxpool_bnrelu_forward(int dtype, const void* y, const float* stat, void* out, uint8_t* arg, int B, int H,
                                   int W, int P, int Q, int Cp, cudaStream_t st);
// the stem's BN backward fused with the max-pool backward (bf16, stem mask from y): reduce + finalize
// + apply, the pool's input gradient re-gathered from u / arg instead of stored
cudaError_t pool_bn_backward(int dtype, const void* u, const uint8_t* arg, const void* y, const float* stat, float* part,
                             int c_real, const float* gamma, float* dgamma, float* dbeta, float* coef, void* dy, int B,
                             int H, int W, int P, int Q, int Cp, cudaStream_t st);
cudaError_t maxpool_forward(int dtype, const void* x, void* out, uint8_t* arg, int B, int H, int W, int P, int Q,
                            int Cp, cudaStream_t st);
cudaError_t maxpool_backward(int dtype, const void* u, const uint8_t* arg, void* dx, int B, int H, int W, int P,
                             int Q, int Cp, cudaStream_t st);

// Space-to-depth of a stride-2 stem's input (R x R kernel, padding pad): x [B][H][W][cpx] (c real
// channels) -> s [B][Hs][Ws][cps], s(n, hs, ws, (i*2 + j)*c + k) = x(n, 2hs+i-pad, 2ws+j-pad, k) (0 off
// the image / past 4c channels); and the gradient's way back (dx from ds, pad channels 0).
cudaError_t s2d_pack(int dtype, const void* x, void* s, int B, int H, int W, int c, int cpx, int Hs, int Ws, int cps,
                     int pad, cudaStream_t st);
cudaError_t s2d_unpack(int dtype, const void* ds, void* dx, int B, int H, int W, int c, int cpx, int Hs, int Ws, int cps,
                       int pad, cudaStream_t st);

// softmax_xent (tensor.py:86-111) on fp32 logits [B][ld] (C real classes):
// dlogits (storage dtype, pads zero) and the mean loss into *loss (device).
// One warp per row; row_loss: B floats of scratch; sem: a device int, 0 on entry (left 0), the
// last CTA sums the row losses in order. nf (optional): sticky flags, bit 0 set when the loss is
// not finite (tensor.py:101-111).
cudaError_t softmax_xent(int dtype, const float* logits, int ld, int B, int C, const int64_t* labels,
                         void* dlogits, float* loss, float* row_loss, int* sem, int* nf, cudaStream_t st);

// Split-K WGRAD partials [splits][Mw][N] -> flat fp32 weight gradient.
//  conv  (dense_layout=0): grad[(co*RS + tap)*ci_real + ci] for Mw = RS*Cp rows (tap*Cp + ci)
//  dense (dense_layout=1): grad[i*out_real + o]   (reference W[in][out] layout)
// dense_layout 2: the space-to-depth stem (RS = its (R'+1)/2 squared taps, Cp its padded 4*ci_real channels,
// s2d_r = the original kernel size R'): grad[(co*R' + 2a+i)*R' + 2b+j][c] for s2d (tap (a,b), channel
// (i*2+j)*ci_real + c).
cudaError_t wgrad_reduce(const float* part, int splits, int Mw, int N, int RS, int Cp, int ci_real, int co_real,
                         int dense_layout, float* grad, cudaStream_t st, int s2d_r = 0);

// Weight shadow packing: fp32 params -> storage dtype [cop][RS][cip] (zero pads).
// dense_src=1: source is the reference W[in=ci][out=co] layout (transposed on the fly).
struct PackEntry {
  int64_t src_off;   // into params (floats)
  int64_t dst_off;   // into the packed buffer (elements)
  int32_t co, ci, rs, cop, cip, dense_src;  // dense_src: 0 conv [cop][rs][cip], 1 dense, 2 conv transposed
                                             //   per tap [cip][rs][cop] (DGRAD K-major weights)
  // space-to-depth stem (s2d_r = the original kernel size R, 0 otherwise): the packed tensor is the
  // ((R+1)/2)^2-tap, 4*ci-channel kernel of the stride-1 conv over the 2x2 space-to-depth input;
  // s2d tap (a, b), channel ((i*2 + j)*ci + c) holds W[co][2a+i][2b+j][c] (0 past R or ci)
  int32_t s2d_r, pad_;
};
cudaError_t pack_weights(int dtype, const float* params, void* packed, const PackEntry* entries_dev, int n_entries,
                         int max_elems, cudaStream_t st);

// Fused per-block optimizer step + weight-shadow repack (one launch per block update): a
// tile table covers the block's flat parameter vector exactly once. Matrix tiles are <= 32 x 32
// sub-matrices of one weight tensor (conv W[co][tap][ci] at one tap, dense W[in][out]) whose
// updated values also go to the storage-dtype shadow, in the same orientation (dst_a, row
// stride dst_a_rs) and/or transposed (element (r, c) -> dst_b + c * dst_b_cs + r); flat tiles
// (BatchNorm gamma / beta, biases) are <= 1024 consecutive parameters.
struct UpdTile {
  int64_t src;       // first parameter (flat index)
  int64_t dst_a;     // same-orientation shadow destination (elements into the packed buffer), -1: none
  int64_t dst_b;     // transposed shadow destination, -1: none
  int32_t rows;      // matrix tile rows (0: flat tile)
  int32_t cols;      // matrix tile columns, or the flat tile's length
  int32_t src_rs;    // parameter row stride
  int32_t dst_a_rs;  // same-orientation row stride
  int32_t dst_b_cs;  // transposed column stride
  int32_t pad_;
};
int update_pack_grid(int n_tiles);
// apply = 0: only the grad-norm (a discarded warmup update, pipeline.py:594).  part: >=
// update_pack_grid(n_tiles) floats; sem: a device int, 0 on entry (left 0); grad_sq_out: sum of
// grad^2 (pre-WD, pipeline.py:602), written by the last CTA in fixed order; nf: sticky flags, bit 1
// set when an applied update meets a non-finite gradient (optim.py:53, 89).
cudaError_t update_pack(int dtype, int rule, int apply, const UpdTile* tiles_dev, int n_tiles, float* x,
                        const float* grad, float* ys, void* packed, float lr, float slr, float beta, float wd,
                        float* part, int* sem, float* grad_sq_out, int* nf, cudaStream_t st);

// Optimizer step over a flat vector (optim.py:48-109, pipeline.py:591-596).
int update_grid(int64_t n);
cudaError_t update_f32(int rule, int64_t n, float* x, const float* grad, float* ys, float lr, float slr, float beta,
                       float wd, float* part, cudaStream_t st);
cudaError_t update_f64(int rule, int64_t n, double* x, const double* grad, double* ys, double* y, double lr,
                       double slr, double beta, double wd, double* part, cudaStream_t st);
// Bias-corrected Adam (extension, BASELINE configs[2]); tstep: device step counter (bumped by
// a follow-up launch) or nullptr with host bias corrections bc1/bc2.
template <typename T>
cudaError_t update_adam(int64_t n, T* x, const T* grad, T* m, T* v, const int64_t* tstep, double bc1, double bc2,
                        double lr, double b1, double b2, double eps, double wd, T* part, cudaStream_t st);
// Per-CTA partial sums of v^2 (grid = update_grid(n)).
cudaError_t sumsq_f32(int64_t n, const float* v, float* part, cudaStream_t st);
// Sum per-CTA partials in fixed order into *out.
cudaError_t sum_partials_f32(const float* part, int n, float* out, cudaStream_t st);
cudaError_t sum_partials_f64(const double* part, int n, double* out, cudaStream_t st);

// NCHW-flattened fp32 [B][C*H*W] <-> padded NHWC storage dtype.
cudaError_t pack_input(const float* x, void* out, int B, int C, int H, int W, int Cp, int dtype, int nchw,
                       cudaStream_t st);
cudaError_t unpack_output(const void* in, float* out, int B, int C, int H, int W, int Cp, int dtype, int nchw,
                          cudaStream_t st);

}  // namespace dsp
