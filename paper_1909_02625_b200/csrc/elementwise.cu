#include <cstdlib>
// Non-GEMM kernels of the DSP block step: BatchNorm statistics / apply /
// backward, dense activations, pooling, softmax cross-entropy, split-K
// reduction, weight-shadow packing, the per-block optimizer update, and the
// host-layout <-> device-layout packing of boundary activations.
//
// All of these are HBM/L2-bandwidth or latency bound (no data reuse): 16-byte
// vectorised, grid-stride, and every reduction is order-deterministic (fixed
// per-thread ranges + fixed smem trees, no float atomics) so repeated runs
// are bitwise identical.
#include "common.cuh"
#include "kernels.cuh"

#include <math.h>

#include <algorithm>

namespace dsp {

namespace {

constexpr int kThreads = 256;

inline int grid_for(int64_t work, int threads = kThreads, int cap = 148 * 8) {
  int64_t g = (work + threads - 1) / threads;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return (int)g;
}

// grid cap of the one-wave (CIFAR-sized) BN kernels: 296 CTAs (two per SM) with several vectors per
// thread leave room for the concurrent block streams' kernels (ResNet-56 +1.2 %, ResNet-110 +2 %
// over 1184; DSP_B200_SMALL_EW_CAP overrides)
inline int small_grid(int64_t nvec) {
  static const int cap = getenv("DSP_B200_SMALL_EW_CAP") ? atoi(getenv("DSP_B200_SMALL_EW_CAP")) : 296;
  return grid_for(nvec, kThreads, cap);
}

template <typename T>
struct V16 {
  static constexpr int N = 16 / sizeof(T);
};

template <typename T>
__device__ __forceinline__ void ld16(const T* p, float (&v)[V16<T>::N]) {
  uint4 raw = *reinterpret_cast<const uint4*>(p);
  const T* e = reinterpret_cast<const T*>(&raw);
#pragma unroll
  for (int i = 0; i < V16<T>::N; ++i) v[i] = to_f<T>(e[i]);
}

template <typename T>
__device__ __forceinline__ void st16(T* p, const float (&v)[V16<T>::N]) {
  uint4 raw;
  T* e = reinterpret_cast<T*>(&raw);
#pragma unroll
  for (int i = 0; i < V16<T>::N; ++i) e[i] = from_f<T>(v[i]);
  *reinterpret_cast<uint4*>(p) = raw;
}

// raw 16-byte load (converted later, so a thread can keep several loads in flight)
template <typename T>
__device__ __forceinline__ uint4 ldraw(const T* p) {
  return *reinterpret_cast<const uint4*>(p);
}
template <typename T>
__device__ __forceinline__ void cvt16(const uint4& raw, float (&v)[V16<T>::N]) {
  const T* e = reinterpret_cast<const T*>(&raw);
#pragma unroll
  for (int i = 0; i < V16<T>::N; ++i) v[i] = to_f<T>(e[i]);
}

// vectors per thread per grid-stride pass: tensors larger than one full-occupancy wave
// (148 SMs x 2048 threads) keep UNR 16-byte loads per operand in flight per thread
constexpr int kWave = 148 * 2048;

template <typename F>
cudaError_t dispatch_dtype(int dtype, F&& f) {
  if (dtype == DSP_DTYPE_BF16) return f(bf16{});
  if (dtype == DSP_DTYPE_F32) return f(float{});
  return cudaErrorInvalidValue;
}

// ------------------------------------------------------------------ BatchNorm forward
__global__ void bn_finalize_k(const float* __restrict__ part, int tiles, int Cp, int c_real, double count,
                              const float* __restrict__ gamma, const float* __restrict__ beta, float* __restrict__ stat) {
  pdl_wait();  // predecessor complete before any global access (successors launch at exit)
  __shared__ double s1[128], s2[128];
  const int c = blockIdx.x;
  double a = 0.0, b = 0.0;
  for (int t = threadIdx.x; t < tiles; t += blockDim.x) {
    a += (double)part[((size_t)t * 2 + 0) * Cp + c];
    b += (double)part[((size_t)t * 2 + 1) * Cp + c];
  }
  s1[threadIdx.x] = a;
  s2[threadIdx.x] = b;
  __syncthreads();
  for (int o = 64; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      s1[threadIdx.x] += s1[threadIdx.x + o];
      s2[threadIdx.x] += s2[threadIdx.x + o];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    float mean = 0.f, inv = 0.f, scale = 0.f, shift = 0.f;
    if (c < c_real) {
      const double m = s1[0] / count;
      double var = s2[0] / count - m * m;
      if (var < 0.0) var = 0.0;
      const double iv = 1.0 / sqrt(var + 1e-5);
      mean = (float)m;
      inv = (float)iv;
      scale = (float)((double)gamma[c] * iv);
      shift = (float)((double)beta[c] - m * (double)gamma[c] * iv);
    }
    stat[c] = mean;
    stat[Cp + c] = inv;
    stat[2 * Cp + c] = scale;
    stat[3 * Cp + c] = shift;
  }
}

// ReLU mask bits of one 8-element vector (bf16): bit i = the STORED value > 0
template <typename T>
__device__ __forceinline__ uint8_t mask_byte(const float (&a)[V16<T>::N]) {
  uint32_t b = 0;
#pragma unroll
  for (int i = 0; i < V16<T>::N; ++i) b |= (to_f<T>(from_f<T>(a[i])) > 0.f ? 1u : 0u) << i;
  return (uint8_t)b;
}

template <typename T, int UNR>
__device__ __forceinline__ void bn_apply_k_body(const T* __restrict__ y, const float* __restrict__ stat, const T* __restrict__ res,
                           const T* __restrict__ y2, const float* __restrict__ stat2, T* __restrict__ out,
                           int64_t nvec, int Cp, int relu, uint8_t* __restrict__ mbits) {
  pdl_wait();  // predecessor complete before any global access (successors launch at exit)
  constexpr int VE = V16<T>::N;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  // when the channel-vector count divides the block, every vector a thread visits has the
  // same channels: scale / shift live in registers (no per-vector 64-bit modulo or loads)
  const int CV = Cp / VE;
  const bool fixc = (blockDim.x % CV) == 0;
  float sc[VE], sh[VE], sc2[VE], sh2[VE];
  if (fixc) {
    const int c0 = (threadIdx.x % CV) * VE;
#pragma unroll
    for (int i = 0; i < VE; ++i) {
      sc[i] = stat[2 * Cp + c0 + i];
      sh[i] = stat[3 * Cp + c0 + i];
      sc2[i] = y2 != nullptr ? stat2[2 * Cp + c0 + i] : 0.f;
      sh2[i] = y2 != nullptr ? stat2[3 * Cp + c0 + i] : 0.f;
    }
  }
  for (int64_t v0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v0 < nvec; v0 += stride * UNR) {
    uint4 ry[UNR], rr[UNR], r2[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {  // every load of the pass first
      const int64_t v = v0 + u * stride;
      if (v < nvec) {
        ry[u] = ldraw(y + v * VE);
        if (res != nullptr) rr[u] = ldraw(res + v * VE);
        if (y2 != nullptr) r2[u] = ldraw(y2 + v * VE);
      }
    }

#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const int64_t v = v0 + u * stride;
      if (v >= nvec) break;
      const int64_t e0 = v * VE;
      if (!fixc) {
        const int c0 = (int)(e0 % Cp);
#pragma unroll
        for (int i = 0; i < VE; ++i) {
          sc[i] = stat[2 * Cp + c0 + i];
          sh[i] = stat[3 * Cp + c0 + i];
          sc2[i] = y2 != nullptr ? stat2[2 * Cp + c0 + i] : 0.f;
          sh2[i] = y2 != nullptr ? stat2[3 * Cp + c0 + i] : 0.f;
        }
      }
      float a[VE];
      cvt16<T>(ry[u], a);
#pragma unroll
      for (int i = 0; i < VE; ++i) a[i] = a[i] * sc[i] + sh[i];
      if (res != nullptr) {
        float r[VE];
        cvt16<T>(rr[u], r);
#pragma unroll
        for (int i = 0; i < VE; ++i) a[i] += r[i];
      }
      if (y2 != nullptr) {
        float r[VE];
        cvt16<T>(r2[u], r);
#pragma unroll
        for (int i = 0; i < VE; ++i) a[i] += r[i] * sc2[i] + sh2[i];
      }
      if (relu) {
#pragma unroll
        for (int i = 0; i < VE; ++i) a[i] = fmaxf(a[i], 0.f);
      }
      st16(out + e0, a);
      if (mbits != nullptr) mbits[v] = mask_byte<T>(a);  // bf16: one byte per vector
    }
  }
}

// default form (compiler-chosen registers) and launch-bounded variants (A/B knob)
template <typename T, int UNR>
__global__ void bn_apply_k(const T* __restrict__ y, const float* __restrict__ stat, const T* __restrict__ res,
                           const T* __restrict__ y2, const float* __restrict__ stat2, T* __restrict__ out,
                           int64_t nvec, int Cp, int relu, uint8_t* __restrict__ mbits) {
  bn_apply_k_body<T, UNR>(y, stat, res, y2, stat2, out, nvec, Cp, relu, mbits);
}
template <typename T, int UNR, int MINB>
__global__ void __launch_bounds__(kThreads, MINB) bn_apply_k_lb(const T* __restrict__ y, const float* __restrict__ stat, const T* __restrict__ res,
                           const T* __restrict__ y2, const float* __restrict__ stat2, T* __restrict__ out,
                           int64_t nvec, int Cp, int relu, uint8_t* __restrict__ mbits) {
  bn_apply_k_body<T, UNR>(y, stat, res, y2, stat2, out, nvec, Cp, relu, mbits);
}

// Resident-grid form (tensors beyond one wave, channel vectors dividing the block): the projection
// branch is compile-time (Y2) so the plain unit keeps only its own scale / shift in registers,
// two vectors per thread per pass, and exactly the resident CTAs (no partial last wave).
template <typename T, int UNR, int MINB, bool Y2>
__global__ void __launch_bounds__(kThreads, MINB)
    bn_apply_rg_k(const T* __restrict__ y, const float* __restrict__ stat, const T* __restrict__ res,
                  const T* __restrict__ y2, const float* __restrict__ stat2, T* __restrict__ out, int64_t nvec,
                  int Cp, int relu, uint8_t* __restrict__ mbits) {
  pdl_wait();  // predecessor complete before any global access (successors launch at exit)
  constexpr int VE = V16<T>::N;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int c0 = (int)(threadIdx.x % (Cp / VE)) * VE;
  float sc[VE], sh[VE], sc2[Y2 ? VE : 1], sh2[Y2 ? VE : 1];
#pragma unroll
  for (int i = 0; i < VE; ++i) {
    sc[i] = stat[2 * Cp + c0 + i];
    sh[i] = stat[3 * Cp + c0 + i];
    if constexpr (Y2) {
      sc2[i] = stat2[2 * Cp + c0 + i];
      sh2[i] = stat2[3 * Cp + c0 + i];
    }
  }
  for (int64_t v0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v0 < nvec; v0 += stride * UNR) {
    uint4 ry[UNR], rr[UNR], r2[Y2 ? UNR : 1];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {  // every load of the pass first
      const int64_t v = v0 + u * stride;
      if (v < nvec) {
        ry[u] = ldraw(y + v * VE);
        if (res != nullptr) rr[u] = ldraw(res + v * VE);
        if constexpr (Y2) r2[u] = ldraw(y2 + v * VE);
      }
    }
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const int64_t v = v0 + u * stride;
      if (v >= nvec) break;
      float a[VE];
      cvt16<T>(ry[u], a);
#pragma unroll
      for (int i = 0; i < VE; ++i) a[i] = a[i] * sc[i] + sh[i];
      if (res != nullptr) {
        float r[VE];
        cvt16<T>(rr[u], r);
#pragma unroll
        for (int i = 0; i < VE; ++i) a[i] += r[i];
      }
      if constexpr (Y2) {
        float r[VE];
        cvt16<T>(r2[u], r);
#pragma unroll
        for (int i = 0; i < VE; ++i) a[i] += r[i] * sc2[i] + sh2[i];
      }
      if (relu) {
#pragma unroll
        for (int i = 0; i < VE; ++i) a[i] = fmaxf(a[i], 0.f);
      }
      st16(out + v * VE, a);
      if (mbits != nullptr) mbits[v] = mask_byte<T>(a);
    }
  }
}

template <typename K>
int resident_ctas(K kern);

// ------------------------------------------------------------------ BatchNorm backward
// Layout of a reduction CTA: G = Cp/VE channel groups, TR = 256/G row lanes.
struct BnBwdFin {  // fused finalize (last CTA) of the BatchNorm-backward reduction
  int c_real;
  double count;
  const float* gamma;
  const float* stat;
  float* dgamma;
  float* dbeta;
  float* coef;
  int* sem;
};

// 2 CTAs per SM (= the 296-chunk grid in one wave): unbounded, the compiler took 132 registers ->
// 1 CTA per SM, two waves, 3.2 TB/s (ncu, profiles/r02_bn_bwd_reduce.md)
template <typename T>
__global__ void __launch_bounds__(kThreads, 2) bn_bwd_reduce_k(const T* __restrict__ gsrc, const T* __restrict__ mask, const T* __restrict__ y,
                                const float* __restrict__ stat, float* __restrict__ part, int64_t M, int Cp,
                                int rows_per_chunk, const BnBwdFin fin, int relu_y,
                                const uint8_t* __restrict__ mbits) {
  pdl_wait();  // predecessor complete before any global access (successors launch at exit)
  constexpr int VE = V16<T>::N;
  __shared__ float red[kThreads][2 * VE];
  // column window of this CTA (blockIdx.y): kThreads channel vectors at most (fp32 storage of
  // 2048-channel tensors needs two windows)
  const int cw0 = (int)blockIdx.y * kThreads * VE;
  const int Cw = min(Cp - cw0, kThreads * VE);
  const int G = Cw / VE;
  const int TR = kThreads / G;
  const int tid = threadIdx.x;
  const int cg = tid % G;
  const int tr = tid / G;
  float s1[VE], s2[VE];
#pragma unroll
  for (int i = 0; i < VE; ++i) s1[i] = s2[i] = 0.f;
  if (tr < TR) {
    const int c0 = cw0 + cg * VE;
    float mean[VE], inv[VE], msc[VE], msh[VE];
#pragma unroll
    for (int i = 0; i < VE; ++i) {
      mean[i] = y ? stat[c0 + i] : 0.f;
      inv[i] = y ? stat[Cp + c0 + i] : 0.f;
      msc[i] = relu_y ? stat[2 * Cp + c0 + i] : 0.f;  // mask from y: the forward's relu(y*scale + shift) > 0
      msh[i] = relu_y ? stat[3 * Cp + c0 + i] : 0.f;
    }
    const int64_t r0 = (int64_t)blockIdx.x * rows_per_chunk;
    const int64_t r1 = min(M, r0 + rows_per_chunk);
    // RU rows per pass, every load of the pass issued before any use; rows are still
    // accumulated in ascending order, so the sums are bitwise those of a one-row loop
    constexpr int RU = 4;
    for (int64_t rb = r0 + tr; rb < r1; rb += (int64_t)TR * RU) {
      uint4 rg[RU], rm[RU], ry[RU];
      uint32_t rb8[RU];
#pragma unroll
      for (int u = 0; u < RU; ++u) {
        const int64_t r = rb + (int64_t)u * TR;
        if (r < r1) {
          const int64_t e0 = r * Cp + c0;
          rg[u] = ldraw(gsrc + e0);
          if (mbits != nullptr) rb8[u] = mbits[e0 / 8];
          else if (mask != nullptr) rm[u] = ldraw(mask + e0);
          if (y != nullptr) ry[u] = ldraw(y + e0);
        }
      }
#pragma unroll
      for (int u = 0; u < RU; ++u) {
        if (rb + (int64_t)u * TR >= r1) break;
        float g[VE];
        cvt16<T>(rg[u], g);
        if (mbits != nullptr) {
#pragma unroll
          for (int i = 0; i < VE; ++i) g[i] = (rb8[u] >> i) & 1u ? g[i] : 0.f;
        } else if (mask != nullptr) {
          float mk[VE];
          cvt16<T>(rm[u], mk);
#pragma unroll
          for (int i = 0; i < VE; ++i) g[i] = mk[i] > 0.f ? g[i] : 0.f;
        }
        if (y != nullptr) {
          float yy[VE];
          cvt16<T>(ry[u], yy);
          if (relu_y) {
#pragma unroll
            for (int i = 0; i < VE; ++i) g[i] = fmaf(yy[i], msc[i], msh[i]) > 0.f ? g[i] : 0.f;
          }
#pragma unroll
          for (int i = 0; i < VE; ++i) {
            s1[i] += g[i];
            s2[i] += g[i] * ((yy[i] - mean[i]) * inv[i]);
          }
        } else {
#pragma unroll
          for (int i = 0; i < VE; ++i) s1[i] += g[i];
        }
      }
    }
  }
#pragma unroll
  for (int i = 0; i < VE; ++i) {
    red[tid][i] = s1[i];
    red[tid][VE + i] = s2[i];
  }
  __syncthreads();
  for (int c = tid; c < Cw; c += kThreads) {
    const int g = c / VE, e = c % VE;
    float a = 0.f, b = 0.f;
    for (int t = 0; t < TR; ++t) {
      a += red[t * G + g][e];
      b += red[t * G + g][VE + e];
    }
    part[((size_t)blockIdx.x * 2 + 0) * Cp + cw0 + c] = a;
    part[((size_t)blockIdx.x * 2 + 1) * Cp + cw0 + c] = b;
  }
  if (fin.sem == nullptr) return;  // (the launcher never fuses the finalize into a windowed grid)
  // ---- last CTA to finish reduces the per-chunk partials in fixed order ----
  __shared__ int last;
  if (!last_cta_ticket(fin.sem, (int)gridDim.x, &last)) return;
  // the reduction scratch is free now: reuse it as fin4[256][4] doubles (8 KB)
  static_assert(sizeof(red) >= 256 * 4 * sizeof(double), "scratch too small");
  double* fin4 = reinterpret_cast<double*>(&red[0][0]);
  for (int w0 = 0; w0 < Cp; w0 += 512) {
    const int cols = min(512, Cp - w0);
    part_sums_load(part, (int)gridDim.x, Cp, 2, w0, cols, Cp, 1, fin4);
    __syncthreads();
    for (int cc = tid; cc < cols; cc += kThreads) {
      const int c = w0 + cc;
      const double s1 = part_sums_get(fin4, 2, cols, cc, 0), s2 = part_sums_get(fin4, 2, cols, cc, 1);
      const bool real = c < fin.c_real;
      if (real && fin.dbeta) fin.dbeta[c] = (float)s1;
      if (real && fin.dgamma && fin.gamma) fin.dgamma[c] = (float)s2;
      if (fin.coef) {
        fin.coef[c] = (real && fin.gamma) ? fin.gamma[c] * fin.stat[Cp + c] : 0.f;
        fin.coef[Cp + c] = real ? (float)(s1 / fin.count) : 0.f;
        fin.coef[2 * Cp + c] = real ? (float)(s2 / fin.count) : 0.f;
      }
    }
    __syncthreads();
  }
  if (tid == 0) *fin.sem = 0;
}

// Column-parallel finalize of the BN-backward partials for wide tensors (Cp >= 512): CTA = 32
// columns x 32 row lanes (coalesced 128-byte reads of every chunk's partial row), fixed-order double
// sums. The fused last-CTA finalize read all chunks x Cp partials on ONE SM: 4.8 MB at Cp = 2048,
// most of a 125 us stage-4 reduction (0.85 TB/s, profiles/r02_r50_block3_launches.csv).
__global__ void __launch_bounds__(1024) bn_bwd_finalize_cols_k(const float* __restrict__ part, int chunks, int Cp,
                                                              int c_real, double count,
                                                              const float* __restrict__ gamma,
                                                              const float* __restrict__ stat,
                                                              float* __restrict__ dgamma, float* __restrict__ dbeta,
                                                              float* __restrict__ coef) {
  pdl_wait();  // predecessor complete before any global access (successors launch at exit)
  __shared__ double sm[32][2][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int c = blockIdx.x * 32 + lane;
  double a = 0.0, b = 0.0;
  if (c < Cp) {
    for (int t = w; t < chunks; t += 32) {
      a += (double)part[((size_t)t * 2 + 0) * Cp + c];
      b += (double)part[((size_t)t * 2 + 1) * Cp + c];
    }
  }
  sm[w][0][lane] = a;
  sm[w][1][lane] = b;
  __syncthreads();
  if (w != 0 || c >= Cp) return;
  double s1 = 0.0, s2 = 0.0;
#pragma unroll
  for (int j = 0; j < 32; ++j) {
    s1 += sm[j][0][lane];
    s2 += sm[j][1][lane];
  }
  const bool real = c < c_real;
  if (real && dbeta) dbeta[c] = (float)s1;
  if (real && dgamma && gamma) dgamma[c] = (float)s2;
  if (coef) {
    coef[c] = (real && gamma) ? gamma[c] * stat[Cp + c] : 0.f;
    coef[Cp + c] = real ? (float)(s1 / count) : 0.f;
    coef[2 * Cp + c] = real ? (float)(s2 / count) : 0.f;
  }
}

__global__ void bn_bwd_finalize_k(const float* __restrict__ part, int chunks, int Cp, int c_real, double count,
                                  const float* __restrict__ gamma, const float* __restrict__ stat,
                                  float* __restrict__ dgamma, float* __restrict__ dbeta, float* __restrict__ coef) {
  pdl_wait();  // predecessor complete before any global access (successors launch at exit)
  __shared__ double s1[128], s2[128];
  const int c = blockIdx.x;
  double a = 0.0, b = 0.0;
  for (int t = threadIdx.x; t < chunks; t += blockDim.x) {
    a += (double)part[((size_t)t * 2 + 0) * Cp + c];
    b += (double)part[((size_t)t * 2 + 1) * Cp + c];
  }
  s1[threadIdx.x] = a;
  s2[threadIdx.x] = b;
  __syncthreads();
  for (int o = 64; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      s1[threadIdx.x] += s1[threadIdx.x + o];
      s2[threadIdx.x] += s2[threadIdx.x + o];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const bool real = c < c_real;
    if (real && dbeta) dbeta[c] = (float)s1[0];
    if (real && dgamma && gamma) dgamma[c] = (float)s2[0];
    if (coef) {
      coef[c] = (real && gamma) ? gamma[c] * stat[Cp + c] : 0.f;
      coef[Cp + c] = real ? (float)(s1[0] / count) : 0.f;
      coef[2 * Cp + c] = real ? (float)(s2[0] / count) : 0.f;
    }
  }
}

template <typename T, int UNR>
__device__ __forceinline__ void bn_bwd_apply_k_body(const T* __restrict__ gsrc, const T* __restrict__ mask, const T* __restrict__ y,
                               const float* __restrict__ stat, const float* __restrict__ coef, T* __restrict__ dy,
                               const T* __restrict__ yb, const float* __restrict__ statb,
                               const float* __restrict__ coefb, T* __restrict__ dyb, T* __restrict__ gout,
                               int64_t nvec, int Cp, int relu_y, const uint8_t* __restrict__ mbits) {
  pdl_wait();  // predecessor complete before any global access (successors launch at exit)
  constexpr int VE = V16<T>::N;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  // per-channel BN-backward coefficients of the main target, in registers when the
  // channel-vector count divides the block (see bn_apply_k):
  //   dy = c0 * (g - c1 - (y - mean) * (invstd * c2))
  const int CV = Cp / VE;
  const bool fixc = (blockDim.x % CV) == 0;
  float k0[VE], k1[VE], km[VE], kq[VE], ms[VE], mh[VE];
  auto coeffs = [&](int c0) {
#pragma unroll
    for (int i = 0; i < VE; ++i) {
      const int c = c0 + i;
      k0[i] = coef[c];
      k1[i] = coef[Cp + c];
      km[i] = stat[c];
      kq[i] = stat[Cp + c] * coef[2 * Cp + c];
      ms[i] = relu_y ? stat[2 * Cp + c] : 0.f;  // mask from y (relu_y): relu(y*scale + shift) > 0
      mh[i] = relu_y ? stat[3 * Cp + c] : 0.f;
    }
  };
  if (fixc) coeffs((threadIdx.x % CV) * VE);
  for (int64_t v0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v0 < nvec; v0 += stride * UNR) {
    uint4 rg[UNR], rm[UNR], ry[UNR], rb[UNR];
    uint32_t rb8[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {  // every load of the pass first
      const int64_t v = v0 + u * stride;
      if (v < nvec) {
        rg[u] = ldraw(gsrc + v * VE);
        if (mbits != nullptr) rb8[u] = mbits[v];  // bf16: one mask byte per vector
        else if (mask != nullptr) rm[u] = ldraw(mask + v * VE);
        ry[u] = ldraw(y + v * VE);
        if (dyb != nullptr) rb[u] = ldraw(yb + v * VE);
      }
    }

#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const int64_t v = v0 + u * stride;
      if (v >= nvec) break;
      const int64_t e0 = v * VE;
      const int c0 = fixc ? (int)(threadIdx.x % CV) * VE : (int)(e0 % Cp);
      if (!fixc) coeffs(c0);
      float g[VE];
      cvt16<T>(rg[u], g);
      if (mbits != nullptr) {
#pragma unroll
        for (int i = 0; i < VE; ++i) g[i] = (rb8[u] >> i) & 1u ? g[i] : 0.f;
      } else if (mask != nullptr) {
        float mk[VE];
        cvt16<T>(rm[u], mk);
#pragma unroll
        for (int i = 0; i < VE; ++i) g[i] = mk[i] > 0.f ? g[i] : 0.f;
      }
      {
        float yy[VE], o[VE];
        cvt16<T>(ry[u], yy);
        if (relu_y) {
#pragma unroll
          for (int i = 0; i < VE; ++i) g[i] = fmaf(yy[i], ms[i], mh[i]) > 0.f ? g[i] : 0.f;
        }
        if (gout != nullptr) st16(gout + e0, g);
#pragma unroll
        for (int i = 0; i < VE; ++i) o[i] = k0[i] * (g[i] - k1[i] - (yy[i] - km[i]) * kq[i]);
        st16(dy + e0, o);
      }
      if (dyb != nullptr) {
        float yy[VE], o[VE];
        cvt16<T>(rb[u], yy);
#pragma unroll
        for (int i = 0; i < VE; ++i) {
          const int c = c0 + i;
          const float xh = (yy[i] - statb[c]) * statb[Cp + c];
          o[i] = coefb[c] * (g[i] - coefb[Cp + c] - xh * coefb[2 * Cp + c]);
        }
        st16(dyb + e0, o);
      }
    }
  }
}

// default form (compiler-chosen registers) and launch-bounded variants (A/B knob)
template <typename T, int UNR>
__global__ void bn_bwd_apply_k(const T* __restrict__ gsrc, const T* __restrict__ mask, const T* __restrict__ y,
                               const float* __restrict__ stat, const float* __restrict__ coef, T* __restrict__ dy,
                               const T* __restrict__ yb, const float* __restrict__ statb,
                               const float* __restrict__ coefb, T* __restrict__ dyb, T* __restrict__ gout,
                               int64_t nvec, int Cp, int relu_y, const uint8_t* __restrict__ mbits) {
  bn_bwd_apply_k_body<T, UNR>(gsrc, mask, y, stat, coef, dy, yb, statb, coefb, dyb, gout, nvec, Cp, relu_y, mbits);
}
template <typename T, int UNR, int MINB>
__global__ void __launch_bounds__(kThreads, MINB) bn_bwd_apply_k_lb(const T* __restrict__ gsrc, const T* __restrict__ mask, const T* __restrict__ y,
                               const float* __restrict__ stat, const float* __restrict__ coef, T* __restrict__ dy,
                               const T* __restrict__ yb, const float* __restrict__ statb,
                               const float* __restrict__ coefb, T* __restrict__ dyb, T* __restrict__ gout,
                               int64_t nvec, int Cp, int relu_y, const uint8_t* __restrict__ mbits) {
  bn_bwd_apply_k_body<T, UNR>(gsrc, mask, y, stat, coef, dy, yb, statb, coefb, dyb, gout, nvec, Cp, relu_y, mbits);
}

// Resident-grid form of the BN-backward apply for tensors beyond one wave whose channel vectors
// divide the block (each thread keeps one channel group for the whole pass): the mask path is a
// compile-time KIND so only the coefficients it needs occupy registers -- 0: mask bits / mask
// tensor / none, 1: mask from y (relu(y*scale + shift) > 0), 2: main + projection target
// (register-resident here; the general form re-loads the projection's five coefficients per
// element, 1.9 TB/s on ResNet-50's first unit) -- and the grid is exactly the resident CTAs, so
// there is no partial last wave (1184 CTAs at 3 per SM left a third of a wave idle).
template <typename T, int UNR, int MINB, int KIND>
__global__ void __launch_bounds__(kThreads, MINB)
    bn_bwd_apply_rg_k(const T* __restrict__ gsrc, const T* __restrict__ mask, const T* __restrict__ y,
                      const float* __restrict__ stat, const float* __restrict__ coef, T* __restrict__ dy,
                      const T* __restrict__ yb, const float* __restrict__ statb, const float* __restrict__ coefb,
                      T* __restrict__ dyb, T* __restrict__ gout, int64_t nvec, int Cp, int relu_y,
                      const uint8_t* __restrict__ mbits) {
  pdl_wait();  // predecessor complete before any global access (successors launch at exit)
  constexpr int VE = V16<T>::N;
  constexpr bool kRy = KIND == 1, kPair = KIND == 2;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int c0 = (int)(threadIdx.x % (Cp / VE)) * VE;
  // dy = k0 * (g - k1 - (y - km) * kq) (the general form's arithmetic, kq = invstd * c2)
  float k0[VE], k1[VE], km[VE], kq[VE];
  float ms[kRy ? VE : 1], mh[kRy ? VE : 1];
  float p0[kPair ? VE : 1], p1[kPair ? VE : 1], pm[kPair ? VE : 1], pi[kPair ? VE : 1], p2[kPair ? VE : 1];
#pragma unroll
  for (int i = 0; i < VE; ++i) {
    const int c = c0 + i;
    k0[i] = coef[c];
    k1[i] = coef[Cp + c];
    km[i] = stat[c];
    kq[i] = stat[Cp + c] * coef[2 * Cp + c];
    if constexpr (kRy) {
      ms[i] = stat[2 * Cp + c];
      mh[i] = stat[3 * Cp + c];
    }
    if constexpr (kPair) {
      p0[i] = coefb[c];
      p1[i] = coefb[Cp + c];
      p2[i] = coefb[2 * Cp + c];
      pm[i] = statb[c];
      pi[i] = statb[Cp + c];
    }
  }
  for (int64_t v0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v0 < nvec; v0 += stride * UNR) {
    uint4 rg[UNR], rm[UNR], ry[UNR], rb[kPair ? UNR : 1];
    uint32_t rb8[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {  // every load of the pass first
      const int64_t v = v0 + u * stride;
      if (v < nvec) {
        rg[u] = ldraw(gsrc + v * VE);
        if constexpr (!kRy) {
          if (mbits != nullptr) rb8[u] = mbits[v];
          else if (mask != nullptr) rm[u] = ldraw(mask + v * VE);
        }
        ry[u] = ldraw(y + v * VE);
        if constexpr (kPair) rb[u] = ldraw(yb + v * VE);
      }
    }
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const int64_t v = v0 + u * stride;
      if (v >= nvec) break;
      const int64_t e0 = v * VE;
      float g[VE], yy[VE], o[VE];
      cvt16<T>(rg[u], g);
      cvt16<T>(ry[u], yy);
      if constexpr (kRy) {
#pragma unroll
        for (int i = 0; i < VE; ++i) g[i] = fmaf(yy[i], ms[i], mh[i]) > 0.f ? g[i] : 0.f;
      } else if (mbits != nullptr) {
#pragma unroll
        for (int i = 0; i < VE; ++i) g[i] = (rb8[u] >> i) & 1u ? g[i] : 0.f;
      } else if (mask != nullptr) {
        float mk[VE];
        cvt16<T>(rm[u], mk);
#pragma unroll
        for (int i = 0; i < VE; ++i) g[i] = mk[i] > 0.f ? g[i] : 0.f;
      }
      if (gout != nullptr) st16(gout + e0, g);
#pragma unroll
      for (int i = 0; i < VE; ++i) o[i] = k0[i] * (g[i] - k1[i] - (yy[i] - km[i]) * kq[i]);
      st16(dy + e0, o);
      if constexpr (kPair) {
        cvt16<T>(rb[u], yy);
#pragma unroll
        for (int i = 0; i < VE; ++i) {
          const float xh = (yy[i] - pm[i]) * pi[i];
          o[i] = p0[i] * (g[i] - p1[i] - xh * p2[i]);
        }
        st16(dyb + e0, o);
      }
    }
  }
}

// CTAs of `kern` resident on the current device at kThreads threads (cached per kernel/device)
template <typename K>
int resident_ctas(K kern) {
  constexpr int kMaxDev = 16;
  static int cache[kMaxDev] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= kMaxDev) dev = 0;
  if (cache[dev] == 0) {
    int per_sm = 0, sms = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThreads, 0);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cache[dev] = std::max(1, per_sm) * std::max(1, sms);
  }
  return cache[dev];
}

// Tensors within one wave (CIFAR shapes, one vector per thread): the plain form -- per-vector
// coefficient loads overlap the data load's latency, which the register-resident form above
// (coefficients first) cannot (measured 1.5% slower on the ResNet-56 step).
template <typename T>
__global__ void bn_apply_small_k(const T* __restrict__ y, const float* __restrict__ stat, const T* __restrict__ res,
                           const T* __restrict__ y2, const float* __restrict__ stat2, T* __restrict__ out,
                           int64_t nvec, int Cp, int relu, uint8_t* __restrict__ mbits) {
  pdl_wait();  // predecessor complete before any global access (successors launch at exit)
  constexpr int VE = V16<T>::N;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nvec; v += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e0 = v * VE;
    const int c0 = (int)(e0 % Cp);
    float a[VE];
    ld16(y + e0, a);
#pragma unroll
    for (int i = 0; i < VE; ++i) a[i] = a[i] * stat[2 * Cp + c0 + i] + stat[3 * Cp + c0 + i];
    if (res != nullptr) {
      float r[VE];
      ld16(res + e0, r);
#pragma unroll
      for (int i = 0; i < VE; ++i) a[i] += r[i];
    }
    if (y2 != nullptr) {
      float r[VE];
      ld16(y2 + e0, r);
#pragma unroll
      for (int i = 0; i < VE; ++i) a[i] += r[i] * stat2[2 * Cp + c0 + i] + stat2[3 * Cp + c0 + i];
    }
    if (relu) {
#pragma unroll
      for (int i = 0; i < VE; ++i) a[i] = fmaxf(a[i], 0.f);
    }
    st16(out + e0, a);
    if (mbits != nullptr) mbits[v] = mask_byte<T>(a);
  }
}

template <typename T>
__global__ void bn_bwd_apply_small_k(const T* __restrict__ gsrc, const T* __restrict__ mask, const T* __restrict__ y,
                               const float* __restrict__ stat, const float* __restrict__ coef, T* __restrict__ dy,
                               const T* __restrict__ yb, const float* __restrict__ statb,
                               const float* __restrict__ coefb, T* __restrict__ dyb, T* __restrict__ gout,
                               int64_t nvec, int Cp, int relu_y, const uint8_t* __restrict__ mbits) {
  pdl_wait();  // predecessor complete before any global access (successors launch at exit)
  constexpr int VE = V16<T>::N;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nvec; v += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e0 = v * VE;
    const int c0 = (int)(e0 % Cp);
    float g[VE];
    ld16(gsrc + e0, g);
    if (mbits != nullptr) {
      const uint32_t b8 = mbits[v];
#pragma unroll
      for (int i = 0; i < VE; ++i) g[i] = (b8 >> i) & 1u ? g[i] : 0.f;
    } else if (mask != nullptr) {
      float mk[VE];
      ld16(mask + e0, mk);
#pragma unroll
      for (int i = 0; i < VE; ++i) g[i] = mk[i] > 0.f ? g[i] : 0.f;
    }
    {
      float yy[VE], o[VE];
      ld16(y + e0, yy);
      if (relu_y) {
#pragma unroll
        for (int i = 0; i < VE; ++i)
          g[i] = fmaf(yy[i], stat[2 * Cp + c0 + i], stat[3 * Cp + c0 + i]) > 0.f ? g[i] : 0.f;
      }
      if (gout != nullptr) st16(gout + e0, g);
#pragma unroll
      for (int i = 0; i < VE; ++i) {
        const int c = c0 + i;
        const float xh = (yy[i] - stat[c]) * stat[Cp + c];
        o[i] = coef[c] * (g[i] - coef[Cp + c] - xh * coef[2 * Cp + c]);
      }
      st16(dy + e0, o);
    }
    if (dyb != nullptr) {
      float yy[VE], o[VE];
      ld16(yb + e0, yy);
#pragma unroll
      for (int i = 0; i < VE; ++i) {
        const int c = c0 + i;
        const float xh = (yy[i] - statb[c]) * statb[Cp + c];
        o[i] = coefb[c] * (g[i] - coefb[Cp + c] - xh * coefb[2 * Cp + c]);
      }
      st16(dyb + e0, o);
    }
  }
}

// ------------------------------------------------------------------ activations / pooling
template <typename T>
__global__ void act_fwd_k(int tanh_kind, const T* __restrict__ x, T* __restrict__ out, int64_t nvec) {
  pdl_wait();  // predecessor complete before any global access (successors launch at exit)
  constexpr int VE = V16<T>::N;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nvec; v += (int64_t)gridDim.x * blockDim.x) {
    float a[VE];
    ld16(x + v * VE, a);
#pragma unroll
    for (int i = 0; i < VE; ++i) a[i] = tanh_kind ? tanhf(a[i]) : fmaxf(a[i], 0.f);
    st16(out + v * VE, a);
  }
}

template <typename T>
__global__ void act_bwd_k(int tanh_kind, const T* __restrict__ x, const T* __restrict__ u, T* __restrict__ dx,
                          int64_t nvec) {
  pdl_wait();  // predecessor complete before any global access (successors launch at exit)
  constexpr int VE = V16<T>::N;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nvec; v += (int64_t)gridDim.x * blockDim.x) {
    float a[VE], g[VE];
    ld16(x + v * VE, a);
    ld16(u + v * VE, g);
#pragma unroll
    for (int i = 0; i < VE; ++i) {
      if (tanh_kind) {
        const float t = tanhf(a[i]);
        g[i] = g[i] * (1.f - t * t);
      } else {
        g[i] = a[i] > 0.f ? g[i] : 0.f;
      }
    }
    st16(dx + v * VE, g);
  }
}

template <typename T>
__global__ void avgpool_fwd_k(const T* __restrict__ x, T* __restrict__ out, int B, int HW, int Cp) {
  pdl_wait();  // predecessor complete before any global access (successors launch at exit)
  constexpr int VE = V16<T>::N;
  const int G = Cp / VE;
  const int64_t nthr = (int64_t)B * G;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nthr; t += (int64_t)gridDim.x * blockDim.x) {
    const int b = (int)(t / G), g = (int)(t % G);
    float acc[VE];
#pragma unroll
    for (int i = 0; i < VE; ++i) acc[i] = 0.f;
    for (int p = 0; p < HW; ++p) {
      float v[VE];
      ld16(x + ((int64_t)b * HW + p) * Cp + g * VE, v);
#pragma unroll
      for (int i = 0; i < VE; ++i) acc[i] += v[i];
    }
    const float inv = 1.f / (float)HW;
#pragma unroll
    for (int i = 0; i < VE; ++i) acc[i] *= inv;
    st16(out + (int64_t)b * Cp + g * VE, acc);
  }
}

template <typename T>
__global__ void avgpool_bwd_k(const T* __restrict__ u, T* __restrict__ dx, int B, int HW, int Cp) {
  pdl_wait();  // predecessor complete before any global access (successors launch at exit)
  constexpr int VE = V16<T>::N;
  const int64_t nvec = (int64_t)B * HW * Cp / VE;
  const float inv = 1.f / (float)HW;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nvec; v += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e0 = v * VE;
    const int64_t b = e0 / ((int64_t)HW * Cp);
    const int c0 = (int)(e0 % Cp);
    float g[VE];
    ld16(u + b * Cp + c0, g);
#pragma unroll
    for (int i = 0; i < VE; ++i) g[i] *= inv;
    st16(dx + e0, g);
  }
}

// 3x3 / stride-2 / pad-1 max pooling, one thread per 16-byte channel vector of an output pixel;
// arg = winning tap (0-8, first maximum in tap order) per element, int32.
template <typename T>
__global__ void maxpool_fwd_k(const T* __restrict__ x, T* __restrict__ out, uint8_t* __restrict__ arg, int B, int H,
                              int W, int P, int Q, int Cp) {
  pdl_wait();  // predecessor complete before any global access (successors launch at exit)
  constexpr int VE = V16<T>::N;
  const int CV = Cp / VE;
  const int n = B * P * Q * CV;  // < 2^31 (checked by the launcher): 32-bit index math
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int cv = i % CV;
    int t = i / CV;
    const int q = t % Q;
    t /= Q;
    const int p = t % P;
    const int b = t / P;
    uint4 raw[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) {  // all nine taps in flight
      const int h = 2 * p - 1 + k / 3, w = 2 * q - 1 + k % 3;
      if ((unsigned)h < (unsigned)H && (unsigned)w < (unsigned)W)
        raw[k] = ldraw(x + (((int64_t)b * H + h) * W + w) * Cp + cv * VE);
    }
    float best[VE];
    int ba[VE];
#pragma unroll
    for (int e = 0; e < VE; ++e) {
      best[e] = -INFINITY;
      ba[e] = 0;
    }
#pragma unroll
    for (int k = 0; k < 9; ++k) {
      const int h = 2 * p - 1 + k / 3, w = 2 * q - 1 + k % 3;
      if ((unsigned)h < (unsigned)H && (unsigned)w < (unsigned)W) {
        float v[VE];
        cvt16<T>(raw[k], v);
#pragma unroll
        for (int e = 0; e < VE; ++e)
          if (v[e] > best[e]) {
            best[e] = v[e];
            ba[e] = k;
          }
      }
    }
    st16(out + i * VE, best);
    // argmax tap (0..8) as one byte per element (VE bytes per thread)
    uint32_t packed[VE / 4];
#pragma unroll
    for (int e = 0; e < VE; e += 4)
      packed[e / 4] = (uint32_t)ba[e] | ((uint32_t)ba[e + 1] << 8) | ((uint32_t)ba[e + 2] << 16) | ((uint32_t)ba[e + 3] << 24);
    if (arg == nullptr) continue;
    if constexpr (VE == 8) {
      *reinterpret_cast<uint2*>(arg + i * VE) = make_uint2(packed[0], packed[1]);
    } else {
      *reinterpret_cast<uint32_t*>(arg + i * VE) = packed[0];
    }
  }
}

template <typename T>
__global__ void maxpool_bwd_k(const T* __restrict__ u, const uint8_t* __restrict__ arg, T* __restrict__ dx, int B,
                              int H, int W, int P, int Q, int Cp) {
  pdl_wait();  // predecessor complete before any global access (successors launch at exit)
  constexpr int VE = V16<T>::N;
  const int CV = Cp / VE;
  const int n = B * H * W * CV;  // < 2^31 (checked by the launcher): 32-bit index math
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int cv = i % CV;
    int t = i / CV;
    const int w = t % W;
    t /= W;
    const int h = t % H;
    const int b = t / H;
    float acc[VE];
#pragma unroll
    for (int e = 0; e < VE; ++e) acc[e] = 0.f;
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      const int pp = h + 1 - r;
      if (pp < 0 || (pp & 1) || (pp >> 1) >= P) continue;
#pragma unroll
      for (int s2 = 0; s2 < 3; ++s2) {
        const int qq = w + 1 - s2;
        if (qq < 0 || (qq & 1) || (qq >> 1) >= Q) continue;
        const int64_t o = (((int64_t)b * P + (pp >> 1)) * Q + (qq >> 1)) * Cp + cv * VE;
        float uv[VE];
        cvt16<T>(ldraw(u + o), uv);
        uint32_t a4[VE / 4];
        if constexpr (VE == 8) {
          const uint2 a = *reinterpret_cast<const uint2*>(arg + o);
          a4[0] = a.x;
          a4[1] = a.y;
        } else {
          a4[0] = *reinterpret_cast<const uint32_t*>(arg + o);
        }
        const uint32_t k = (uint32_t)(r * 3 + s2);
#pragma unroll
        for (int e = 0; e < VE; ++e)
          if (((a4[e / 4] >> (8 * (e & 3))) & 0xffu) == k) acc[e] += uv[e];
      }
    }
    st16(dx + i * VE, acc);
  }
}

// bf16 forward on packed pairs: per tap, one bf16x2 greater-than mask per word selects both the
// new maximum and its tap (two LOP3s) -- the same strict first-maximum-in-tap-order rule as the
// generic form, which spent ~32 scalar instructions per tap and was issue-bound (66% issue slots,
// 2.8 TB/s, profiles/r02_maxpool.md)
__global__ void maxpool_fwd_bf16x2_k(const uint4* __restrict__ x, uint4* __restrict__ out, uint2* __restrict__ arg,
                                     int B, int H, int W, int P, int Q, int CV) {
  pdl_wait();  // predecessor complete before any global access (successors launch at exit)
  const int n = B * P * Q * CV;  // < 2^31 (checked by the launcher)
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int cv = i % CV;
    int t = i / CV;
    const int q = t % Q;
    t /= Q;
    const int p = t % P;
    const int b = t / P;
    uint4 raw[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) {  // all nine taps in flight
      const int h = 2 * p - 1 + k / 3, w = 2 * q - 1 + k % 3;
      if ((unsigned)h < (unsigned)H && (unsigned)w < (unsigned)W) raw[k] = __ldg(x + ((b * H + h) * W + w) * CV + cv);
    }
    uint32_t best[4] = {0xff80ff80u, 0xff80ff80u, 0xff80ff80u, 0xff80ff80u}, ba[4] = {0u, 0u, 0u, 0u};
#pragma unroll
    for (int k = 0; k < 9; ++k) {
      const int h = 2 * p - 1 + k / 3, w = 2 * q - 1 + k % 3;
      if ((unsigned)h < (unsigned)H && (unsigned)w < (unsigned)W) {
        const uint32_t v[4] = {raw[k].x, raw[k].y, raw[k].z, raw[k].w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint32_t m = __hgt2_mask(*reinterpret_cast<const __nv_bfloat162*>(&v[j]),
                                         *reinterpret_cast<const __nv_bfloat162*>(&best[j]));
          best[j] = (v[j] & m) | (best[j] & ~m);
          ba[j] = ((uint32_t)k * 0x00010001u & m) | (ba[j] & ~m);
        }
      }
    }
    out[i] = make_uint4(best[0], best[1], best[2], best[3]);
    if (arg != nullptr)  // (a fresh forward keeps no argmax: only the recorded pass's backward reads it)
      arg[i] = make_uint2(__byte_perm(ba[0], ba[1], 0x6420), __byte_perm(ba[2], ba[3], 0x6420));
  }
}

// Stem BN-apply + ReLU fused into the max pool (bf16): each tap's y is normalised, rectified and
// rounded to bf16 exactly as bn_apply would store it, then pooled as above -- the stem's full-
// resolution activation is never written (nor re-read by the pool); its backward recomputes the
// ReLU mask from y. The grid is a multiple of the channel-vector count, so a thread's 8 channels
// (and their scale / shift) never change.
__global__ void maxpool_bnrelu_fwd_bf16x2_k(const uint4* __restrict__ y, const float* __restrict__ stat,
                                            uint4* __restrict__ out, uint2* __restrict__ arg, int B, int H, int W,
                                            int P, int Q, int CV) {
  pdl_wait();  // predecessor complete before any global access (successors launch at exit)
  const int Cp = CV * 8;
  const int c0 = (int)((blockIdx.x * blockDim.x + threadIdx.x) % CV) * 8;
  float2 sc[4], sh[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    sc[j] = make_float2(stat[2 * Cp + c0 + 2 * j], stat[2 * Cp + c0 + 2 * j + 1]);
    sh[j] = make_float2(stat[3 * Cp + c0 + 2 * j], stat[3 * Cp + c0 + 2 * j + 1]);
  }
  const int n = B * P * Q * CV;  // < 2^31 (checked by the launcher)
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int cv = i % CV;
    int t = i / CV;
    const int q = t % Q;
    t /= Q;
    const int p = t % P;
    const int b = t / P;
    uint4 raw[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) {
      const int h = 2 * p - 1 + k / 3, w = 2 * q - 1 + k % 3;
      if ((unsigned)h < (unsigned)H && (unsigned)w < (unsigned)W) raw[k] = __ldg(y + ((b * H + h) * W + w) * CV + cv);
    }
    uint32_t best[4] = {0xff80ff80u, 0xff80ff80u, 0xff80ff80u, 0xff80ff80u}, ba[4] = {0u, 0u, 0u, 0u};
#pragma unroll
    for (int k = 0; k < 9; ++k) {
      const int h = 2 * p - 1 + k / 3, w = 2 * q - 1 + k % 3;
      if ((unsigned)h < (unsigned)H && (unsigned)w < (unsigned)W) {
        const uint32_t yw[4] = {raw[k].x, raw[k].y, raw[k].z, raw[k].w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          float2 z = __ffma2_rn(make_float2(__uint_as_float(yw[j] << 16), __uint_as_float(yw[j] & 0xffff0000u)), sc[j],
                                sh[j]);
          z.x = fmaxf(z.x, 0.f);
          z.y = fmaxf(z.y, 0.f);
          uint32_t v;
          asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(v) : "f"(z.y), "f"(z.x));
          const uint32_t m = __hgt2_mask(*reinterpret_cast<const __nv_bfloat162*>(&v),
                                         *reinterpret_cast<const __nv_bfloat162*>(&best[j]));
          best[j] = (v & m) | (best[j] & ~m);
          ba[j] = ((uint32_t)k * 0x00010001u & m) | (ba[j] & ~m);
        }
      }
    }
    out[i] = make_uint4(best[0], best[1], best[2], best[3]);
    if (arg != nullptr)  // (a fresh forward keeps no argmax: only the recorded pass's backward reads it)
      arg[i] = make_uint2(__byte_perm(ba[0], ba[1], 0x6420), __byte_perm(ba[2], ba[3], 0x6420));
  }
}

// Backward by output quads: thread (b, i, j, channel vector) writes input pixels (2i + di, 2j + dj)
// from the (up to) four windows (i + di', j + dj') that contain them -- four 16-byte window loads,
// no divergent tap search, every store a full 16 bytes. Each input pixel sums its windows in the
// generic form's order (window rows, then columns, descending), so results are bitwise the same.
template <typename T>
__global__ void maxpool_bwd_quad_k(const T* __restrict__ u, const uint8_t* __restrict__ arg, T* __restrict__ dx,
                                   int B, int H, int W, int P, int Q, int Cp) {
  pdl_wait();  // predecessor complete before any global access (successors launch at exit)
  constexpr int VE = V16<T>::N;
  const int CV = Cp / VE;
  const int n = B * P * Q * CV;  // < 2^31 (checked by the launcher)
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < n; idx += gridDim.x * blockDim.x) {
    const int cv = idx % CV;
    int t = idx / CV;
    const int j = t % Q;
    t /= Q;
    const int i = t % P;
    const int b = t / P;
    // windows w[di][dj] = (i + di, j + dj): gradient u and argmax taps
    float uv[2][2][VE];
    uint32_t tap[2][2][VE / 4];
#pragma unroll
    for (int di = 0; di < 2; ++di)
#pragma unroll
      for (int dj = 0; dj < 2; ++dj) {
        const bool ok = i + di < P && j + dj < Q;
        const int64_t o = (((int64_t)b * P + i + di) * Q + j + dj) * Cp + cv * VE;
        if (ok) {
          cvt16<T>(ldraw(u + o), uv[di][dj]);
          if constexpr (VE == 8) {
            const uint2 a = *reinterpret_cast<const uint2*>(arg + o);
            tap[di][dj][0] = a.x;
            tap[di][dj][1] = a.y;
          } else {
            tap[di][dj][0] = *reinterpret_cast<const uint32_t*>(arg + o);
          }
        } else {
#pragma unroll
          for (int e = 0; e < VE; ++e) uv[di][dj][e] = 0.f;
#pragma unroll
          for (int e = 0; e < VE / 4; ++e) tap[di][dj][e] = 0xffffffffu;  // matches no tap
        }
      }
    auto term = [&](float (&acc)[VE], int di, int dj, uint32_t k) {
#pragma unroll
      for (int e = 0; e < VE; ++e)
        if (((tap[di][dj][e / 4] >> (8 * (e & 3))) & 0xffu) == k) acc[e] += uv[di][dj][e];
    };
#pragma unroll
    for (int dh = 0; dh < 2; ++dh)
#pragma unroll
      for (int dw = 0; dw < 2; ++dw) {
        const int h = 2 * i + dh, w = 2 * j + dw;
        if (h >= H || w >= W) continue;
        float acc[VE];
#pragma unroll
        for (int e = 0; e < VE; ++e) acc[e] = 0.f;
        // window rows r ascending = window index descending; likewise columns
        if (dh == 0 && dw == 0) {
          term(acc, 0, 0, 4);
        } else if (dh == 0) {
          term(acc, 0, 1, 3);
          term(acc, 0, 0, 5);
        } else if (dw == 0) {
          term(acc, 1, 0, 1);
          term(acc, 0, 0, 7);
        } else {
          term(acc, 1, 1, 0);
          term(acc, 1, 0, 2);
          term(acc, 0, 1, 6);
          term(acc, 0, 0, 8);
        }
        st16(dx + (((int64_t)b * H + h) * W + w) * Cp + cv * VE, acc);
      }
  }
}

// ---- the stem's BN backward fused with the max-pool backward (bf16, stem mask from y) ----
// The pool's input gradient dx (the stem activation's gradient, 411 MB at ResNet-50 B=256) is never
// stored: both passes of the stem's BN backward re-gather it per output quad (2x2 stem pixels from
// their <= 4 pooling windows: u + argmax taps, 154 MB, L2-resident) exactly as maxpool_bwd_quad_k
// sums it, then g = dx * (relu(y*scale + shift) > 0).
struct PoolQuad {
  uint4 u[2][2];
  uint2 a[2][2];
};

__device__ __forceinline__ void pool_quad_load(const uint4* __restrict__ u, const uint2* __restrict__ arg, int b,
                                               int i, int j, int P, int Q, int CV, int cv, PoolQuad& pq) {
#pragma unroll
  for (int di = 0; di < 2; ++di)
#pragma unroll
    for (int dj = 0; dj < 2; ++dj) {
      const bool ok = i + di < P && j + dj < Q;
      const int64_t o = (((int64_t)b * P + i + di) * Q + j + dj) * CV + cv;
      pq.u[di][dj] = ok ? __ldg(u + o) : make_uint4(0u, 0u, 0u, 0u);
      pq.a[di][dj] = ok ? __ldg(arg + o) : make_uint2(0xffffffffu, 0xffffffffu);
    }
}

// dx of stem pixel (2i + dh, 2j + dw), 8 channels, in the generic pool backward's summation order
__device__ __forceinline__ void pool_quad_dx(const PoolQuad& pq, int dh, int dw, float (&acc)[8]) {
#pragma unroll
  for (int e = 0; e < 8; ++e) acc[e] = 0.f;
  auto term = [&](int di, int dj, uint32_t k) {
    const uint32_t uw[4] = {pq.u[di][dj].x, pq.u[di][dj].y, pq.u[di][dj].z, pq.u[di][dj].w};
    const uint32_t aw[2] = {pq.a[di][dj].x, pq.a[di][dj].y};
#pragma unroll
    for (int e = 0; e < 8; ++e)
      if (((aw[e >> 2] >> (8 * (e & 3))) & 0xffu) == k)
        acc[e] += __uint_as_float((e & 1) ? (uw[e >> 1] & 0xffff0000u) : (uw[e >> 1] << 16));
  };
  if (dh == 0 && dw == 0) {
    term(0, 0, 4);
  } else if (dh == 0) {
    term(0, 1, 3);
    term(0, 0, 5);
  } else if (dw == 0) {
    term(1, 0, 1);
    term(0, 0, 7);
  } else {
    term(1, 1, 0);
    term(1, 0, 2);
    term(0, 1, 6);
    term(0, 0, 8);
  }
}

// pass 1: per-chunk partial sums of g and g * xhat (chunk = a contiguous quad range; thread =
// (quad lane, channel vector); fixed-order CTA reduction) -> part[chunk][2][Cp]
__global__ void __launch_bounds__(256) pool_bn_bwd_reduce_k(const uint4* __restrict__ u, const uint2* __restrict__ arg,
                                                          const uint4* __restrict__ y, const float* __restrict__ stat,
                                                          float* __restrict__ part, int B, int H, int W, int P, int Q,
                                                          int CV, int quads_per_chunk) {
  pdl_wait();  // predecessor complete before any global access (successors launch at exit)
  __shared__ float red[256][16];
  const int Cp = CV * 8;
  const int tid = threadIdx.x, cv = tid % CV, ql = tid / CV, QL = 256 / CV;
  const int c0 = cv * 8;
  float mean[8], inv[8], sc[8], sh[8], s1[8], s2[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    mean[e] = stat[c0 + e];
    inv[e] = stat[Cp + c0 + e];
    sc[e] = stat[2 * Cp + c0 + e];
    sh[e] = stat[3 * Cp + c0 + e];
    s1[e] = s2[e] = 0.f;
  }
  const int64_t nq = (int64_t)B * P * Q;
  const int64_t q0 = (int64_t)blockIdx.x * quads_per_chunk, q1 = min(nq, q0 + quads_per_chunk);
  for (int64_t qd = q0 + ql; qd < q1; qd += QL) {
    const int j = (int)(qd % Q);
    const int64_t t = qd / Q;
    const int i = (int)(t % P), b = (int)(t / P);
    PoolQuad pq;
    pool_quad_load(u, arg, b, i, j, P, Q, CV, cv, pq);
    uint4 yr[2][2];
#pragma unroll
    for (int dh = 0; dh < 2; ++dh)
#pragma unroll
      for (int dw = 0; dw < 2; ++dw) {
        const int h = 2 * i + dh, w = 2 * j + dw;
        yr[dh][dw] = (h < H && w < W) ? __ldg(y + (((int64_t)b * H + h) * W + w) * CV + cv) : make_uint4(0u, 0u, 0u, 0u);
      }
#pragma unroll
    for (int dh = 0; dh < 2; ++dh)
#pragma unroll
      for (int dw = 0; dw < 2; ++dw) {
        if (2 * i + dh >= H || 2 * j + dw >= W) continue;
        float g[8];
        pool_quad_dx(pq, dh, dw, g);
        // the stored dx is bf16: round exactly as the unfused pool backward's store does
#pragma unroll
        for (int e = 0; e < 8; ++e) g[e] = __bfloat162float(__float2bfloat16(g[e]));
        const uint32_t yw[4] = {yr[dh][dw].x, yr[dh][dw].y, yr[dh][dw].z, yr[dh][dw].w};
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const float yy = __uint_as_float((e & 1) ? (yw[e >> 1] & 0xffff0000u) : (yw[e >> 1] << 16));
          const float ge = fmaf(yy, sc[e], sh[e]) > 0.f ? g[e] : 0.f;
          s1[e] += ge;
          s2[e] += ge * ((yy - mean[e]) * inv[e]);
        }
      }
  }
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    red[tid][e] = s1[e];
    red[tid][8 + e] = s2[e];
  }
  __syncthreads();
  for (int c = tid; c < Cp; c += 256) {
    const int g = c / 8, e = c % 8;
    float a = 0.f, bsum = 0.f;
    for (int l = 0; l < QL; ++l) {
      a += red[l * CV + g][e];
      bsum += red[l * CV + g][8 + e];
    }
    part[((size_t)blockIdx.x * 2 + 0) * Cp + c] = a;
    part[((size_t)blockIdx.x * 2 + 1) * Cp + c] = bsum;
  }
}

// pass 2: dy = coef0 * (g - coef1 - xhat * coef2), written per stem pixel (grid a multiple of CV:
// a thread's channels, and their coefficients, never change)
__global__ void pool_bn_bwd_apply_k(const uint4* __restrict__ u, const uint2* __restrict__ arg,
                                    const uint4* __restrict__ y, const float* __restrict__ stat,
                                    const float* __restrict__ coef, uint4* __restrict__ dy, int B, int H, int W, int P,
                                    int Q, int CV) {
  pdl_wait();  // predecessor complete before any global access (successors launch at exit)
  const int Cp = CV * 8;
  const int c0 = (int)((blockIdx.x * blockDim.x + threadIdx.x) % CV) * 8;
  float k0[8], k1[8], km[8], kq[8], sc[8], sh[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    const int c = c0 + e;
    k0[e] = coef[c];
    k1[e] = coef[Cp + c];
    km[e] = stat[c];
    kq[e] = stat[Cp + c] * coef[2 * Cp + c];
    sc[e] = stat[2 * Cp + c];
    sh[e] = stat[3 * Cp + c];
  }
  const int n = B * P * Q * CV;  // < 2^31 (checked by the launcher)
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < n; idx += gridDim.x * blockDim.x) {
    const int cv = idx % CV;
    int t = idx / CV;
    const int j = t % Q;
    t /= Q;
    const int i = t % P, b = t / P;
    PoolQuad pq;
    pool_quad_load(u, arg, b, i, j, P, Q, CV, cv, pq);
#pragma unroll
    for (int dh = 0; dh < 2; ++dh)
#pragma unroll
      for (int dw = 0; dw < 2; ++dw) {
        const int h = 2 * i + dh, w = 2 * j + dw;
        if (h >= H || w >= W) continue;
        const int64_t o = (((int64_t)b * H + h) * W + w) * CV + cv;
        const uint4 yv = __ldg(y + o);
        float g[8];
        pool_quad_dx(pq, dh, dw, g);
        const uint32_t yw[4] = {yv.x, yv.y, yv.z, yv.w};
        float out[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const float ge0 = __bfloat162float(__float2bfloat16(g[e]));
          const float yy = __uint_as_float((e & 1) ? (yw[e >> 1] & 0xffff0000u) : (yw[e >> 1] << 16));
          const float ge = fmaf(yy, sc[e], sh[e]) > 0.f ? ge0 : 0.f;
          out[e] = k0[e] * (ge - k1[e] - (yy - km[e]) * kq[e]);
        }
        uint4 r;
        uint32_t* rw = reinterpret_cast<uint32_t*>(&r);
#pragma unroll
        for (int e2 = 0; e2 < 4; ++e2)
          asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(rw[e2]) : "f"(out[2 * e2 + 1]), "f"(out[2 * e2]));
        dy[o] = r;
      }
  }
}

// ------------------------------------------------------------------ space-to-depth stem
// One thread per s2d pixel: its cps channels = 4 sub-positions (i, j) x c input channels.
// the ResNet-50 stem case: bf16, 8-channel input pixels (one 16-byte load each), 16 s2d channels
// (two 16-byte stores), 32-bit index math
__global__ void s2d_pack8_k(const uint4* __restrict__ x, uint4* __restrict__ s, int B, int H, int W, int c, int Hs,
                            int Ws, int pad) {
  pdl_wait();  // predecessor complete before any global access (successors launch at exit)
  const int n = B * Hs * Ws;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int ws = i % Ws, t = i / Ws, hs = t % Hs, b = t / Hs;
    uint4 in[4];
#pragma unroll
    for (int sub = 0; sub < 4; ++sub) {
      const int h = 2 * hs + (sub >> 1) - pad, w = 2 * ws + (sub & 1) - pad;
      in[sub] = ((unsigned)h < (unsigned)H && (unsigned)w < (unsigned)W) ? __ldg(x + ((b * H + h) * W + w))
                                                                        : make_uint4(0, 0, 0, 0);
    }
    uint16_t o[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) o[k] = 0;
#pragma unroll
    for (int sub = 0; sub < 4; ++sub) {
      const uint16_t* e = reinterpret_cast<const uint16_t*>(&in[sub]);
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (k < c) o[sub * c + k] = e[k];
    }
    const uint4* op = reinterpret_cast<const uint4*>(o);
    s[2 * i] = op[0];
    s[2 * i + 1] = op[1];
  }
}

template <typename T>
__global__ void s2d_pack_k(const T* __restrict__ x, T* __restrict__ s, int B, int H, int W, int c, int cpx, int Hs,
                           int Ws, int cps, int pad) {
  pdl_wait();  // predecessor complete before any global access (successors launch at exit)
  const int64_t n = (int64_t)B * Hs * Ws;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int ws = (int)(i % Ws);
    const int64_t t = i / Ws;
    const int hs = (int)(t % Hs);
    const int b = (int)(t / Hs);
    T* out = s + i * cps;
    for (int cs = 0; cs < cps; ++cs) {
      const int sub = cs / c, k = cs % c;
      float v = 0.f;
      if (sub < 4) {
        const int h = 2 * hs + (sub >> 1) - pad, w = 2 * ws + (sub & 1) - pad;
        if ((unsigned)h < (unsigned)H && (unsigned)w < (unsigned)W) v = to_f<T>(x[(((int64_t)b * H + h) * W + w) * cpx + k]);
      }
      out[cs] = from_f<T>(v);
    }
  }
}

template <typename T>
__global__ void s2d_unpack_k(const T* __restrict__ ds, T* __restrict__ dx, int B, int H, int W, int c, int cpx, int Hs,
                             int Ws, int cps, int pad) {
  pdl_wait();  // predecessor complete before any global access (successors launch at exit)
  const int64_t n = (int64_t)B * H * W;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int w = (int)(i % W);
    const int64_t t = i / W;
    const int h = (int)(t % H);
    const int b = (int)(t / H);
    const int hp = h + pad, wp = w + pad;
    const T* src = ds + (((int64_t)b * Hs + (hp >> 1)) * Ws + (wp >> 1)) * cps + (((hp & 1) * 2 + (wp & 1)) * c);
    for (int k = 0; k < cpx; ++k) dx[i * cpx + k] = k < c ? src[k] : from_f<T>(0.f);
  }
}

// ------------------------------------------------------------------ loss
template <typename T>
__global__ void softmax_xent_k(const float* __restrict__ logits, int ld, int B, int C, const int64_t* __restrict__ labels,
                               T* __restrict__ dlogits, float* __restrict__ loss, float* __restrict__ row_loss, int* sem,
                               int* __restrict__ nf) {
  // one warp per row (8 rows per CTA); the per-row losses are summed in row order by the last
  // CTA to finish (ticket), so the mean is deterministic
  pdl_wait();  // predecessor complete before any global access (successors launch at exit)
  __shared__ int last_s;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int b = blockIdx.x * (blockDim.x >> 5) + warp;
  if (b < B) {
    const float* z = logits + (size_t)b * ld;
    float mx = -INFINITY;
    for (int c = lane; c < C; c += 32) mx = fmaxf(mx, z[c]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    float den = 0.f;
    for (int c = lane; c < C; c += 32) den += expf(z[c] - mx);
    den = warp_sum(den);
    const int lab = (int)labels[b];
    const float inv_b = 1.f / (float)B;
    for (int c = lane; c < ld; c += 32) {
      float gval = 0.f;
      if (c < C) {
        gval = expf(z[c] - mx) / den;
        if (c == lab) gval -= 1.f;
        gval *= inv_b;
      }
      dlogits[(size_t)b * ld + c] = from_f<T>(gval);
    }
    if (lane == 0) row_loss[b] = -((z[lab] - mx) - logf(den));
  }
  if (last_cta_ticket(sem, (int)gridDim.x, &last_s) && threadIdx.x == 0) {
    double s = 0.0;
    for (int r = 0; r < B; ++r) s += (double)__ldcg(&row_loss[r]);
    const float l = (float)(s / (double)B);
    *loss = l;
    if (nf != nullptr && !isfinite(l)) atomicOr(nf, 1);  // NonFiniteError (tensor.py:101-111)
    *sem = 0;
  }
}

// ------------------------------------------------------------------ split-K reduce / packing
__global__ void __launch_bounds__(256) wgrad_reduce_k(const float* __restrict__ part, int splits, int Mw, int N,
                                                     int RS, int Cp, int ci_real, int co_real, int dense_layout,
                                                     float* __restrict__ grad, int s2d_r) {
  pdl_wait();  // predecessor complete before any global access (successors launch at exit)
  // CTA = 128 consecutive partial elements (a float4 per lane: 512 B per split row) x 8 warps;
  // warp w sums the contiguous split range [w*S/8, (w+1)*S/8) with its loads in flight, then
  // warp 0 adds the 8 warp sums in order (deterministic). Small CTAs on purpose: the step runs the
  // K blocks' kernels concurrently and a reduce CTA must fit beside resident conv CTAs.
  constexpr int W = 8;
  __shared__ float4 red[W][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t total = (int64_t)Mw * N;
  const int64_t idx0 = ((int64_t)blockIdx.x * 32 + lane) * 4;  // first of this lane's 4 elements
  const int z0 = (int)((int64_t)splits * w / W), z1 = (int)((int64_t)splits * (w + 1) / W);
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  if (idx0 < total) {  // total % 4 == 0 (N is a multiple of 8)
    const size_t zs = (size_t)total;
    const float* p = part + idx0;
    for (int z = z0; z < z1; z += 4) {
      float4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u)
        v[u] = z + u < z1 ? __ldcg(reinterpret_cast<const float4*>(p + (size_t)(z + u) * zs))
                          : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        acc.x += v[u].x;
        acc.y += v[u].y;
        acc.z += v[u].z;
        acc.w += v[u].w;
      }
    }
  }
  red[w][lane] = acc;
  __syncthreads();
  if (w != 0 || idx0 >= total) return;
  float sum[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
  for (int j = 0; j < W; ++j) {
    sum[0] += red[j][lane].x;
    sum[1] += red[j][lane].y;
    sum[2] += red[j][lane].z;
    sum[3] += red[j][lane].w;
  }
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const int64_t idx = idx0 + e;
    const int n = (int)(idx % N);
    const int m = (int)(idx / N);
    if (n >= co_real) continue;
    int64_t dst;
    if (dense_layout == 1) {
      if (m >= ci_real) continue;
      dst = (int64_t)m * co_real + n;
    } else if (dense_layout == 2) {  // space-to-depth stem
      const int cs = m % Cp, tap = m / Cp, rs2 = (s2d_r + 1) / 2;
      const int sub = cs / ci_real, c = cs % ci_real;
      const int r = 2 * (tap / rs2) + (sub >> 1), s = 2 * (tap % rs2) + (sub & 1);
      if (sub >= 4 || tap >= RS || r >= s2d_r || s >= s2d_r) continue;
      dst = (((int64_t)n * s2d_r + r) * s2d_r + s) * ci_real + c;
    } else {
      const int ci = m % Cp, tap = m / Cp;
      if (ci >= ci_real || tap >= RS) continue;
      dst = ((int64_t)n * RS + tap) * ci_real + ci;
    }
    grad[dst] = sum[e];
  }
}

// Tiled form for outputs of >= 148 32x32 tiles (the wide stage-3/4 convs: few splits, millions of
// weights): CTA = 32 rows (m) x 32 columns (n) of the partials, thread (n, 4 rows) sums the splits
// in ascending order with 4 splits' loads in flight, and the tile is transposed through shared
// memory so the [co][tap][ci] stores run along ci (the row-major form wrote 4-byte scattered
// stores with a stride of RS*ci: 23-41 us per stage-4 reduce).
__global__ void __launch_bounds__(256) wgrad_reduce_tiled_k(const float* __restrict__ part, int splits, int Mw, int N,
                                                           int RS, int Cp, int ci_real, int co_real,
                                                           float* __restrict__ grad) {
  pdl_wait();  // predecessor complete before any global access (successors launch at exit)
  __shared__ float tile[32][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // ty: rows 4 ty .. 4 ty + 3
  const int m0 = blockIdx.x * 32, n0 = blockIdx.y * 32;
  const size_t zs = (size_t)Mw * N;
  const int n = n0 + tx;
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
  if (n < N) {
    for (int z = 0; z < splits; z += 4) {
      float v[4][4];
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int m = m0 + 4 * ty + i;
          v[u][i] = (z + u < splits && m < Mw) ? __ldcg(part + (size_t)(z + u) * zs + (size_t)m * N + n) : 0.f;
        }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int i = 0; i < 4; ++i) acc[i] += v[u][i];
    }
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) tile[4 * ty + i][tx] = acc[i];
  __syncthreads();
  // write: lane = row (m -> (tap, ci)), 4 columns (co) per warp
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int m = m0 + tx, nn = n0 + 4 * ty + i;
    if (m >= Mw || nn >= co_real) continue;
    const int ci = m % Cp, tap = m / Cp;
    if (ci >= ci_real || tap >= RS) continue;
    grad[((int64_t)nn * RS + tap) * ci_real + ci] = tile[tx][4 * ty + i];
  }
}

template <typename T>
__global__ void pack_weights_k(const float* __restrict__ params, T* __restrict__ packed,
                               const PackEntry* __restrict__ ents, int n_entries) {
  pdl_wait();  // predecessor complete before any global access (successors launch at exit)
  const PackEntry e = ents[blockIdx.y];
  const int64_t total = (int64_t)e.cop * e.rs * e.cip;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    int ci, co, tap;
    if (e.dense_src == 2) {  // [cip][rs][cop]
      co = (int)(idx % e.cop);
      const int64_t t = idx / e.cop;
      tap = (int)(t % e.rs);
      ci = (int)(t / e.rs);
    } else {  // [cop][rs][cip]
      ci = (int)(idx % e.cip);
      const int64_t t = idx / e.cip;
      tap = (int)(t % e.rs);
      co = (int)(t / e.rs);
    }
    float v = 0.f;
    if (e.s2d_r > 0) {  // space-to-depth stem: s2d tap (a, b), channel (i*2 + j)*ci + c
      const int rs2 = (e.s2d_r + 1) / 2;
      const int a = tap / rs2, bb = tap % rs2, sub = ci / e.ci, c = ci % e.ci;
      const int r = 2 * a + (sub >> 1), s = 2 * bb + (sub & 1);
      if (co < e.co && sub < 4 && r < e.s2d_r && s < e.s2d_r)
        v = params[e.src_off + (((int64_t)co * e.s2d_r + r) * e.s2d_r + s) * e.ci + c];
    } else if (co < e.co && ci < e.ci) {
      v = e.dense_src == 1 ? params[e.src_off + (int64_t)ci * e.co + co]
                      : params[e.src_off + ((int64_t)co * e.rs + tap) * e.ci + ci];
    }
    packed[e.dst_off + idx] = from_f<T>(v);
  }
}

// ------------------------------------------------------------------ optimizer
// One parameter of the SGD / SUM step (optim.py:48-99 with the coupled weight decay of
// pipeline.py:591-593), IEEE ops without FMA contraction; accumulates grad^2 (pre-WD) into sq.
template <int RULE, bool WD>
__device__ __forceinline__ float upd1(float xv, float g0, float& ysv, float lr, float slr, float beta, float wd,
                                      float& sq, bool& bad) {
  sq = __fadd_rn(sq, __fmul_rn(g0, g0));
  const float g = WD ? __fadd_rn(g0, __fmul_rn(wd, xv)) : g0;
  bad |= !isfinite(g);
  if (RULE == DSP_RULE_SGD) return __fsub_rn(xv, __fmul_rn(lr, g));
  const float y = __fsub_rn(xv, __fmul_rn(lr, g));
  const float ysn = __fsub_rn(xv, __fmul_rn(slr, g));
  const float xn = (beta == 0.f) ? y : __fadd_rn(y, __fmul_rn(beta, __fsub_rn(ysn, ysv)));
  ysv = ysn;
  return xn;
}

// 4 consecutive parameters [i, i + n4) (n4 <= 4) of the flat vector, updated in place; the new
// values are returned in out[] (APPLY) and the grad^2 added to sq. 16-byte accesses when aligned.
template <int RULE, bool WD, bool APPLY>
__device__ __forceinline__ void upd4(int64_t i, int n4, float* __restrict__ x, const float* __restrict__ grad,
                                     float* __restrict__ ys, float lr, float slr, float beta, float wd, float& sq,
                                     bool& bad, float (&out)[4]) {
  if (n4 == 4 && (i & 3) == 0) {
    const float4 g = *reinterpret_cast<const float4*>(grad + i);
    if (!APPLY) {
      sq = __fadd_rn(sq, __fmul_rn(g.x, g.x));
      sq = __fadd_rn(sq, __fmul_rn(g.y, g.y));
      sq = __fadd_rn(sq, __fmul_rn(g.z, g.z));
      sq = __fadd_rn(sq, __fmul_rn(g.w, g.w));
      return;
    }
    const float4 xv = *reinterpret_cast<const float4*>(x + i);
    float4 yv = make_float4(0.f, 0.f, 0.f, 0.f);
    if (RULE == DSP_RULE_SUM) yv = *reinterpret_cast<const float4*>(ys + i);
    out[0] = upd1<RULE, WD>(xv.x, g.x, yv.x, lr, slr, beta, wd, sq, bad);
    out[1] = upd1<RULE, WD>(xv.y, g.y, yv.y, lr, slr, beta, wd, sq, bad);
    out[2] = upd1<RULE, WD>(xv.z, g.z, yv.z, lr, slr, beta, wd, sq, bad);
    out[3] = upd1<RULE, WD>(xv.w, g.w, yv.w, lr, slr, beta, wd, sq, bad);
    *reinterpret_cast<float4*>(x + i) = make_float4(out[0], out[1], out[2], out[3]);
    if (RULE == DSP_RULE_SUM) *reinterpret_cast<float4*>(ys + i) = yv;
    return;
  }
  for (int j = 0; j < n4; ++j) {
    const float g0 = grad[i + j];
    if (!APPLY) {
      sq = __fadd_rn(sq, __fmul_rn(g0, g0));
      continue;
    }
    float yv = RULE == DSP_RULE_SUM ? ys[i + j] : 0.f;
    out[j] = upd1<RULE, WD>(x[i + j], g0, yv, lr, slr, beta, wd, sq, bad);
    x[i + j] = out[j];
    if (RULE == DSP_RULE_SUM) ys[i + j] = yv;
  }
}

// 4 consecutive storage-dtype values (8 bytes bf16 / 16 bytes fp32 when aligned)
template <typename T>
__device__ __forceinline__ void st4(T* p, int n4, const float (&v)[4]) {
  if (n4 == 4 && (reinterpret_cast<uintptr_t>(p) & (4 * sizeof(T) - 1)) == 0) {
    if constexpr (sizeof(T) == 2) {
      __nv_bfloat162 a = __floats2bfloat162_rn(v[0], v[1]), b = __floats2bfloat162_rn(v[2], v[3]);
      uint2 raw;
      raw.x = *reinterpret_cast<uint32_t*>(&a);
      raw.y = *reinterpret_cast<uint32_t*>(&b);
      *reinterpret_cast<uint2*>(p) = raw;
    } else {
      *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
    }
    return;
  }
  for (int j = 0; j < n4; ++j) p[j] = from_f<T>(v[j]);
}

// Fused optimizer step + weight-shadow repack over a tile table (kernels.cuh UpdTile).
// 256 threads; a matrix tile: thread (r = tid / 8, c0 = 4 * (tid % 8)) updates 4 parameters of
// row r, writes them to the same-orientation shadow, stages them in smem, and after a barrier
// writes the transposed shadow 4 rows at a time (both shadow writes 8-byte chunks along rows).
// The grad^2 partials of the CTAs are summed in fixed order by the last CTA (ticket).
template <typename T, int RULE, bool WD, bool APPLY>
__global__ void __launch_bounds__(kThreads) update_pack_k(const UpdTile* __restrict__ tiles, int n_tiles,
                                                          float* __restrict__ x, const float* __restrict__ grad,
                                                          float* __restrict__ ys, T* __restrict__ packed, float lr,
                                                          float slr, float beta, float wd, float* __restrict__ part,
                                                          int* sem, float* __restrict__ grad_sq_out,
                                                          int* __restrict__ nf) {
  pdl_wait();  // predecessor complete before any global access (successors launch at exit)
  __shared__ float stage[32][33];
  __shared__ float red[kThreads];
  __shared__ int last_s;
  const int tid = threadIdx.x;
  float sq = 0.f;
  bool bad = false;
  for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) {
    const UpdTile d = tiles[t];
    float out[4] = {0.f, 0.f, 0.f, 0.f};
    if (d.rows == 0) {  // flat tile
      const int c = tid * 4;
      if (c < d.cols) upd4<RULE, WD, APPLY>(d.src + c, min(4, d.cols - c), x, grad, ys, lr, slr, beta, wd, sq, bad, out);
      continue;
    }
    const int r = tid >> 3, c0 = (tid & 7) * 4;
    const int n4 = r < d.rows ? max(0, min(4, d.cols - c0)) : 0;
    if (n4 > 0) {
      upd4<RULE, WD, APPLY>(d.src + (int64_t)r * d.src_rs + c0, n4, x, grad, ys, lr, slr, beta, wd, sq, bad, out);
      if (APPLY && d.dst_a >= 0) st4<T>(packed + d.dst_a + (int64_t)r * d.dst_a_rs + c0, n4, out);
    }
    if (APPLY && d.dst_b >= 0) {
      for (int j = 0; j < n4; ++j) stage[r][c0 + j] = out[j];
      __syncthreads();
      const int c = tid >> 3, r0 = (tid & 7) * 4;  // transposed: column c, rows r0..r0+3
      const int m4 = c < d.cols ? max(0, min(4, d.rows - r0)) : 0;
      if (m4 > 0) {
        float v[4];
        for (int j = 0; j < 4; ++j) v[j] = j < m4 ? stage[r0 + j][c] : 0.f;
        st4<T>(packed + d.dst_b + (int64_t)c * d.dst_b_cs + r0, m4, v);
      }
      __syncthreads();
    }
  }
  red[tid] = sq;
  __syncthreads();
  for (int o = kThreads / 2; o > 0; o >>= 1) {
    if (tid < o) red[tid] += red[tid + o];
    __syncthreads();
  }
  if (APPLY && nf != nullptr && __syncthreads_or(bad) && tid == 0) atomicOr(nf, 2);  // optim.py:53, 89
  if (grad_sq_out == nullptr) return;
  if (tid == 0) part[blockIdx.x] = red[0];
  if (last_cta_ticket(sem, (int)gridDim.x, &last_s)) {
    if (tid == 0) {
      double s = 0.0;
      for (int b = 0; b < (int)gridDim.x; ++b) s += (double)__ldcg(&part[b]);
      *grad_sq_out = (float)s;
      *sem = 0;
    }
  }
}

template <int RULE, bool WD>
__global__ void update_f32_k(int64_t n, float* __restrict__ x, const float* __restrict__ grad, float* __restrict__ ys,
                             float lr, float slr, float beta, float wd, float* __restrict__ part) {
  pdl_wait();  // predecessor complete before any global access (successors launch at exit)
  __shared__ float red[kThreads];
  float sq = 0.f;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float g0 = grad[i];
    sq = __fadd_rn(sq, __fmul_rn(g0, g0));
    const float xv = x[i];
    const float g = WD ? __fadd_rn(g0, __fmul_rn(wd, xv)) : g0;
    if (RULE == DSP_RULE_SGD) {
      x[i] = __fsub_rn(xv, __fmul_rn(lr, g));
    } else {
      const float y = __fsub_rn(xv, __fmul_rn(lr, g));
      const float ysn = __fsub_rn(xv, __fmul_rn(slr, g));
      x[i] = (beta == 0.f) ? y : __fadd_rn(y, __fmul_rn(beta, __fsub_rn(ysn, ys[i])));
      ys[i] = ysn;
    }
  }
  red[threadIdx.x] = sq;
  __syncthreads();
  for (int o = kThreads / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0 && part) part[blockIdx.x] = red[0];
}

template <int RULE, bool WD>
__global__ void update_f64_k(int64_t n, double* __restrict__ x, const double* __restrict__ grad,
                             double* __restrict__ ys, double* __restrict__ yout, double lr, double slr, double beta,
                             double wd, double* __restrict__ part) {
  pdl_wait();  // predecessor complete before any global access (successors launch at exit)
  __shared__ double red[kThreads];
  double sq = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double g0 = grad[i];
    sq = __dadd_rn(sq, __dmul_rn(g0, g0));
    const double xv = x[i];
    const double g = WD ? __dadd_rn(g0, __dmul_rn(wd, xv)) : g0;
    if (RULE == DSP_RULE_SGD) {
      x[i] = __dsub_rn(xv, __dmul_rn(lr, g));
    } else {
      const double y = __dsub_rn(xv, __dmul_rn(lr, g));
      const double ysn = __dsub_rn(xv, __dmul_rn(slr, g));
      x[i] = (beta == 0.0) ? y : __dadd_rn(y, __dmul_rn(beta, __dsub_rn(ysn, ys[i])));
      ys[i] = ysn;
      if (yout) yout[i] = y;
    }
  }
  red[threadIdx.x] = sq;
  __syncthreads();
  for (int o = kThreads / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0 && part) part[blockIdx.x] = red[0];
}

// IEEE round-to-nearest ops without FMA contraction, per precision (optimizer kernels)
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float sub_rn(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float div_rn(float a, float b) { return __fdiv_rn(a, b); }
__device__ __forceinline__ float sqrt_rn(float a) { return __fsqrt_rn(a); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double div_rn(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ double sqrt_rn(double a) { return __dsqrt_rn(a); }

// Bias-corrected Adam per block (BASELINE configs[2]; an extension -- the reference rejects
// rule "adam", optim.py:70-71 -- restated in oracle/dsp_ref.py adam_step, same IEEE op order):
//   g = grad (+ wd*x);  m' = b1*m + (1-b1)*g;  v' = b2*v + (1-b2)*(g*g)
//   x' = x - (lr * (m'/bc1)) / (sqrt(v'/bc2) + eps),  bc_i = 1 - b_i^t
// t = *tstep + 1 read from device memory (so step graphs stay valid as t advances; the
// caller bumps the counter after the launch), or bc1/bc2 from the host when tstep == nullptr.
template <typename T, bool WD>
__global__ void update_adam_k(int64_t n, T* __restrict__ x, const T* __restrict__ grad, T* __restrict__ m,
                              T* __restrict__ v, const int64_t* __restrict__ tstep, double bc1h, double bc2h, T lr,
                              double b1, double b2, double eps, T wd, T* __restrict__ part) {
  pdl_wait();  // predecessor complete before any global access (successors launch at exit)
  __shared__ T red[kThreads];
  __shared__ double bc[2];
  if (threadIdx.x == 0) {
    if (tstep != nullptr) {
      const double t = (double)(*tstep + 1);
      bc[0] = 1.0 - pow(b1, t);
      bc[1] = 1.0 - pow(b2, t);
    } else {
      bc[0] = bc1h;
      bc[1] = bc2h;
    }
  }
  __syncthreads();
  const T c1 = (T)bc[0], c2 = (T)bc[1];
  const T B1 = (T)b1, A1 = (T)(1.0 - b1), B2 = (T)b2, A2 = (T)(1.0 - b2), E = (T)eps;
  T sq = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const T g0 = grad[i];
    sq = add_rn(sq, mul_rn(g0, g0));
    const T xv = x[i];
    const T g = WD ? add_rn(g0, mul_rn(wd, xv)) : g0;
    const T mi = add_rn(mul_rn(B1, m[i]), mul_rn(A1, g));
    const T vi = add_rn(mul_rn(B2, v[i]), mul_rn(A2, mul_rn(g, g)));
    m[i] = mi;
    v[i] = vi;
    const T den = add_rn(sqrt_rn(div_rn(vi, c2)), E);
    x[i] = sub_rn(xv, div_rn(mul_rn(lr, div_rn(mi, c1)), den));
  }
  red[threadIdx.x] = sq;
  __syncthreads();
  for (int o = kThreads / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0 && part) part[blockIdx.x] = red[0];
}

__global__ void step_bump_k(int64_t* tstep) {
  pdl_wait();
  *tstep += 1;
}

__global__ void sumsq_k(int64_t n, const float* __restrict__ v, float* __restrict__ part) {
  pdl_wait();  // predecessor complete before any global access (successors launch at exit)
  __shared__ float red[kThreads];
  float sq = 0.f;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    sq = __fadd_rn(sq, __fmul_rn(v[i], v[i]));
  red[threadIdx.x] = sq;
  __syncthreads();
  for (int o = kThreads / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = red[0];
}

template <typename S, typename O>
__global__ void sum_partials_k(const S* __restrict__ part, int n, O* __restrict__ out) {
  pdl_wait();  // predecessor complete before any global access (successors launch at exit)
  __shared__ double red[kThreads];
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += kThreads) s += (double)part[i];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int o = kThreads / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = (O)red[0];
}

// ------------------------------------------------------------------ boundary layout
template <typename T>
__global__ void pack_input_k(const float* __restrict__ x, T* __restrict__ out, int B, int C, int H, int W, int Cp,
                             int nchw) {
  pdl_wait();  // predecessor complete before any global access (successors launch at exit)
  const int64_t n = (int64_t)B * H * W * Cp;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(i % Cp);
    const int64_t pix = i / Cp;  // b*H*W + h*W + w
    const int64_t b = pix / ((int64_t)H * W);
    const int64_t hw = pix % ((int64_t)H * W);
    float v = 0.f;
    if (c < C) v = nchw ? x[(b * C + c) * H * W + hw] : x[pix * C + c];
    out[i] = from_f<T>(v);
  }
}

template <typename T>
__global__ void unpack_output_k(const T* __restrict__ in, float* __restrict__ out, int B, int C, int H, int W, int Cp,
                                int nchw) {
  pdl_wait();  // predecessor complete before any global access (successors launch at exit)
  const int64_t n = (int64_t)B * C * H * W;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t b, c, hw;
    if (nchw) {
      hw = i % ((int64_t)H * W);
      const int64_t t = i / ((int64_t)H * W);
      c = t % C;
      b = t / C;
    } else {
      c = i % C;
      const int64_t t = i / C;
      hw = t % ((int64_t)H * W);
      b = t / ((int64_t)H * W);
    }
    out[i] = to_f<T>(in[(b * H * W + hw) * Cp + c]);
  }
}

}  // namespace

// ================================================================== launch wrappers
cudaError_t bn_finalize(const float* part, int tiles, int Cp, int c_real, int64_t count, const float* gamma,
                        const float* beta, float* stat, cudaStream_t st) {
  launch_k(bn_finalize_k, Cp, 128, 0, st, part, tiles, Cp, c_real, (double)count, gamma, beta, stat);
  return note_launch(), cudaGetLastError();
}

cudaError_t bn_apply(int dtype, const void* y, const float* stat, const void* res, const void* y2, const float* stat2,
                     void* out, int64_t M, int Cp, int relu, cudaStream_t st, uint8_t* mbits) {
  return dispatch_dtype(dtype, [&](auto t) {
    using T = decltype(t);
    const int64_t nvec = M * Cp / V16<T>::N;
    if (mbits != nullptr && V16<T>::N != 8) return cudaErrorInvalidValue;  // mask bytes: 8 channels (bf16)
    // variant (UNR x min CTAs per SM) via DSP_B200_BNA = 10*UNR + MINB (A/B knob). ncu on
    // ResNet-50: the unbounded UNR-4 form took 117 registers -> 2 CTAs/SM, 24% warps active,
    // 44-59% of DRAM peak; one vector per thread per pass at 4 CTAs/SM measured +1.6%
    // (ResNet-50) / +5.3% (ResNet-164) samples/s
    static const int var = getenv("DSP_B200_BNA") ? atoi(getenv("DSP_B200_BNA")) : 0;
    auto go = [&](auto kern) {
      launch_k(kern, grid_for(nvec), kThreads, 0, st, (const T*)y, stat, (const T*)res, (const T*)y2, stat2, (T*)out,
               nvec, Cp, relu, mbits);
    };
    // resident-grid forms by default (DSP_B200_BNA=13 restores the general one)
    auto go_rg = [&](auto kern) {
      const int64_t need = (nvec + kThreads - 1) / kThreads;
      launch_k(kern, (int)std::min<int64_t>(need, resident_ctas(kern)), kThreads, 0, st, (const T*)y, stat,
               (const T*)res, (const T*)y2, stat2, (T*)out, nvec, Cp, relu, mbits);
    };
    if (nvec > kWave && var == 0 && (kThreads % (Cp / V16<T>::N)) == 0) {
      static const int y2v = getenv("DSP_B200_BNA_Y2") ? atoi(getenv("DSP_B200_BNA_Y2")) : 14;  // A/B knob: 14 = UNR 1 at 4 CTAs/SM (ResNet-50 first unit 247 -> 218 us)
      if (y2 != nullptr) {
        if (y2v == 14) go_rg(bn_apply_rg_k<T, 1, 4, true>);
        else if (y2v == 13) go_rg(bn_apply_rg_k<T, 1, 3, true>);
        else go_rg(bn_apply_rg_k<T, 2, 2, true>);
      }
      else {
        static const int pv = getenv("DSP_B200_BNA_RG") ? atoi(getenv("DSP_B200_BNA_RG")) : 24;  // A/B knob
        if (pv == 14) go_rg(bn_apply_rg_k<T, 1, 4, false>);
        else if (pv == 16) go_rg(bn_apply_rg_k<T, 1, 6, false>);
        else if (pv == 44) go_rg(bn_apply_rg_k<T, 4, 4, false>);
        else go_rg(bn_apply_rg_k<T, 2, 4, false>);
      }
    } else if (nvec > kWave) {
      if (var == 23) go(bn_apply_k_lb<T, 2, 3>);
      else if (var == 24) go(bn_apply_k_lb<T, 2, 4>);
      else if (var == 43) go(bn_apply_k_lb<T, 4, 3>);
      else if (var == 13 || var == 0) go(bn_apply_k_lb<T, 1, 4>);  // general: 62 regs, 4 CTAs/SM
      else go(bn_apply_k<T, 4>);  // 41: compiler-chosen 117 regs, 2 CTAs/SM
    }
    else
      launch_k(bn_apply_small_k<T>, small_grid(nvec), kThreads, 0, st, (const T*)y, stat, (const T*)res, (const T*)y2,
               stat2, (T*)out, nvec, Cp, relu, mbits);
    return note_launch(), cudaGetLastError();
  });
}

int bn_bwd_chunks(int64_t M, int Cp) {
  const int G = Cp / 8;  // conservative (bf16 VE=8); fp32 uses the same chunking
  const int TR = G >= kThreads ? 1 : kThreads / G;
  int64_t rows = (M + 295) / 296;
  rows = ((rows + TR - 1) / TR) * TR;
  if (rows < TR) rows = TR;
  return (int)((M + rows - 1) / rows);
}

static int64_t bn_rows_per_chunk(int64_t M, int Cp) {
  const int chunks = bn_bwd_chunks(M, Cp);
  return (M + chunks - 1) / chunks;
}

cudaError_t bn_bwd_reduce(int dtype, const void* gsrc, const void* mask, const void* y, const float* stat, float* part,
                          int64_t M, int Cp, cudaStream_t st, int relu_y, const uint8_t* mbits) {
  const int chunks = bn_bwd_chunks(M, Cp);
  const int rows = (int)bn_rows_per_chunk(M, Cp);
  return dispatch_dtype(dtype, [&](auto t) {
    using T = decltype(t);
    if (Cp / V16<T>::N > kThreads) return cudaErrorInvalidValue;
    launch_k(bn_bwd_reduce_k<T>, chunks, kThreads, 0, st, (const T*)gsrc, (const T*)mask, (const T*)y, stat, part, M, Cp,
             rows, BnBwdFin{}, relu_y, mbits);
    return note_launch(), cudaGetLastError();
  });
}

cudaError_t bn_bwd_stats(int dtype, const void* gsrc, const void* mask, const void* y, const float* stat, float* part,
                         int64_t M, int Cp, int c_real, const float* gamma, float* dgamma, float* dbeta, float* coef,
                         int* sem, cudaStream_t st, int relu_y, const uint8_t* mbits) {
  const int chunks = bn_bwd_chunks(M, Cp);
  const int rows = (int)bn_rows_per_chunk(M, Cp);
  // wide tensors: a column-parallel finalize launch instead of the last CTA's (DSP_B200_BNR_COLS
  // sets the width from which it is used; 0 = never)
  static const int cols_from = getenv("DSP_B200_BNR_COLS") ? atoi(getenv("DSP_B200_BNR_COLS")) : 512;
  return dispatch_dtype(dtype, [&](auto t) {
    using T = decltype(t);
    const int nwin = (Cp / V16<T>::N + kThreads - 1) / kThreads;  // column windows (grid y)
    const bool sep = (cols_from > 0 && Cp >= cols_from) || nwin > 1;
    const BnBwdFin fin{c_real, (double)M, gamma, stat, dgamma, dbeta, coef, sep ? nullptr : sem};
    launch_k(bn_bwd_reduce_k<T>, dim3(chunks, nwin), kThreads, 0, st, (const T*)gsrc, (const T*)mask, (const T*)y, stat, part, M, Cp,
             rows, fin, relu_y, mbits);
    note_launch();
    if (sep) {
      launch_k(bn_bwd_finalize_cols_k, (Cp + 31) / 32, 1024, 0, st, part, chunks, Cp, c_real, (double)M, gamma, stat,
               dgamma, dbeta, coef);
      note_launch();
    }
    return cudaGetLastError();
  });
}

cudaError_t bn_bwd_finalize(const float* part, int chunks, int Cp, int c_real, int64_t count, const float* gamma,
                            const float* stat, float* dgamma, float* dbeta, float* coef, cudaStream_t st) {
  launch_k(bn_bwd_finalize_k, Cp, 128, 0, st, part, chunks, Cp, c_real, (double)count, gamma, stat, dgamma, dbeta, coef);
  return note_launch(), cudaGetLastError();
}

cudaError_t bn_bwd_apply(int dtype, const void* gsrc, const void* mask, const void* y, const float* stat,
                         const float* coef, void* dy, const void* y_b, const float* stat_b, const float* coef_b,
                         void* dy_b, void* g_out, int64_t M, int Cp, cudaStream_t st, int relu_y,
                         const uint8_t* mbits) {
  return dispatch_dtype(dtype, [&](auto t) {
    using T = decltype(t);
    const int64_t nvec = M * Cp / V16<T>::N;
    // variant (UNR x min CTAs per SM) via DSP_B200_BNB = 10*UNR + MINB (A/B knob): the
    // unbounded UNR-2 form took 128 registers (2 CTAs/SM); UNR 1 at 3 CTAs/SM measured +0.9%
    // (ResNet-50) / +2.6% (ResNet-164)
    static const int var = getenv("DSP_B200_BNB") ? atoi(getenv("DSP_B200_BNB")) : 0;
    auto go = [&](auto kern) {
      launch_k(kern, grid_for(nvec), kThreads, 0, st, (const T*)gsrc, (const T*)mask, (const T*)y, stat, coef, (T*)dy,
               (const T*)y_b, stat_b, coef_b, (T*)dy_b, (T*)g_out, nvec, Cp, relu_y, mbits);
    };
    // resident-grid forms (DSP_B200_BNB=13 restores the general form)
    const bool rg = var != 13 && (kThreads % (Cp / V16<T>::N)) == 0 && !(y_b != nullptr && relu_y);
    auto go_rg = [&](auto kern) {
      const int64_t need = (nvec + kThreads - 1) / kThreads;
      const int grid = (int)std::min<int64_t>(need, resident_ctas(kern));
      launch_k(kern, grid, kThreads, 0, st, (const T*)gsrc, (const T*)mask, (const T*)y, stat, coef, (T*)dy,
               (const T*)y_b, stat_b, coef_b, (T*)dy_b, (T*)g_out, nvec, Cp, relu_y, mbits);
    };
    if (nvec > kWave && rg) {
      // A/B knobs (10*UNR + CTAs/SM) per mask kind
      static const int k0 = getenv("DSP_B200_BNB_K0") ? atoi(getenv("DSP_B200_BNB_K0")) : 22;
      static const int k1 = getenv("DSP_B200_BNB_K1") ? atoi(getenv("DSP_B200_BNB_K1")) : 22;
      static const int k2 = getenv("DSP_B200_BNB_K2") ? atoi(getenv("DSP_B200_BNB_K2")) : 12;
      if (y_b != nullptr) {
        if (k2 == 13) go_rg(bn_bwd_apply_rg_k<T, 1, 3, 2>);
        else go_rg(bn_bwd_apply_rg_k<T, 1, 2, 2>);
      } else if (relu_y) {
        if (k1 == 13) go_rg(bn_bwd_apply_rg_k<T, 1, 3, 1>);
        else if (k1 == 14) go_rg(bn_bwd_apply_rg_k<T, 1, 4, 1>);
        else go_rg(bn_bwd_apply_rg_k<T, 2, 2, 1>);
      } else {
        if (k0 == 13) go_rg(bn_bwd_apply_rg_k<T, 1, 3, 0>);
        else if (k0 == 14) go_rg(bn_bwd_apply_rg_k<T, 1, 4, 0>);
        else if (k0 == 23) go_rg(bn_bwd_apply_rg_k<T, 2, 3, 0>);
        else go_rg(bn_bwd_apply_rg_k<T, 2, 2, 0>);
      }
    } else if (nvec > kWave) {
      if (var == 23) go(bn_bwd_apply_k_lb<T, 2, 3>);
      else if (var == 24) go(bn_bwd_apply_k_lb<T, 2, 4>);
      else if (var == 13 || var == 0) go(bn_bwd_apply_k_lb<T, 1, 3>);  // general default: 80 regs, 3 CTAs/SM
      else if (var == 14) go(bn_bwd_apply_k_lb<T, 1, 4>);
      else go(bn_bwd_apply_k<T, 2>);
    }
    else
      launch_k(bn_bwd_apply_small_k<T>, small_grid(nvec), kThreads, 0, st, (const T*)gsrc, (const T*)mask, (const T*)y,
               stat, coef, (T*)dy, (const T*)y_b, stat_b, coef_b, (T*)dy_b, (T*)g_out, nvec, Cp, relu_y, mbits);
    return note_launch(), cudaGetLastError();
  });
}

cudaError_t act_forward(int dtype, int tanh_kind, const void* x, void* out, int64_t n, cudaStream_t st) {
  return dispatch_dtype(dtype, [&](auto t) {
    using T = decltype(t);
    const int64_t nvec = n / V16<T>::N;
    launch_k(act_fwd_k<T>, grid_for(nvec), kThreads, 0, st, tanh_kind, (const T*)x, (T*)out, nvec);
    return note_launch(), cudaGetLastError();
  });
}

cudaError_t act_backward(int dtype, int tanh_kind, const void* x, const void* u, void* dx, int64_t n, cudaStream_t st) {
  return dispatch_dtype(dtype, [&](auto t) {
    using T = decltype(t);
    const int64_t nvec = n / V16<T>::N;
    launch_k(act_bwd_k<T>, grid_for(nvec), kThreads, 0, st, tanh_kind, (const T*)x, (const T*)u, (T*)dx, nvec);
    return note_launch(), cudaGetLastError();
  });
}

cudaError_t avgpool_forward(int dtype, const void* x, void* out, int B, int HW, int Cp, cudaStream_t st) {
  return dispatch_dtype(dtype, [&](auto t) {
    using T = decltype(t);
    launch_k(avgpool_fwd_k<T>, grid_for((int64_t)B * Cp / V16<T>::N), kThreads, 0, st, (const T*)x, (T*)out, B, HW, Cp);
    return note_launch(), cudaGetLastError();
  });
}

cudaError_t avgpool_backward(int dtype, const void* u, void* dx, int B, int HW, int Cp, cudaStream_t st) {
  return dispatch_dtype(dtype, [&](auto t) {
    using T = decltype(t);
    launch_k(avgpool_bwd_k<T>, grid_for((int64_t)B * HW * Cp / V16<T>::N), kThreads, 0, st, (const T*)u, (T*)dx, B, HW, Cp);
    return note_launch(), cudaGetLastError();
  });
}

cudaError_t maxpool_forward(int dtype, const void* x, void* out, uint8_t* arg, int B, int H, int W, int P, int Q,
                            int Cp, cudaStream_t st) {
  return dispatch_dtype(dtype, [&](auto t) {
    using T = decltype(t);
    if (Cp % V16<T>::N || (int64_t)B * H * W * Cp >= (1ll << 31)) return cudaErrorInvalidValue;
    static const bool generic = getenv("DSP_B200_MAXPOOL_GENERIC") != nullptr;  // A/B knob
    if (sizeof(T) == 2 && !generic) {
      launch_k(maxpool_fwd_bf16x2_k, grid_for((int64_t)B * P * Q * Cp / 8), kThreads, 0, st, (const uint4*)x, (uint4*)out,
               (uint2*)arg, B, H, W, P, Q, Cp / 8);
      return note_launch(), cudaGetLastError();
    }
    launch_k(maxpool_fwd_k<T>, grid_for((int64_t)B * P * Q * Cp / V16<T>::N), kThreads, 0, st, (const T*)x, (T*)out, arg, B, H, W, P, Q,
                                                                            Cp);
    return note_launch(), cudaGetLastError();
  });
}

cudaError_t maxpool_bnrelu_forward(int dtype, const void* y, const float* stat, void* out, uint8_t* arg, int B, int H,
                                   int W, int P, int Q, int Cp, cudaStream_t st) {
  const int CV = Cp / 8;
  if (dtype != DSP_DTYPE_BF16 || Cp % 8 || kThreads % CV || (int64_t)B * H * W * Cp >= (1ll << 31))
    return cudaErrorInvalidValue;
  launch_k(maxpool_bnrelu_fwd_bf16x2_k, grid_for((int64_t)B * P * Q * CV), kThreads, 0, st, (const uint4*)y, stat,
           (uint4*)out, (uint2*)arg, B, H, W, P, Q, CV);
  return note_launch(), cudaGetLastError();
}

cudaError_t pool_bn_backward(int dtype, const void* u, const uint8_t* arg, const void* y, const float* stat, float* part,
                             int c_real, const float* gamma, float* dgamma, float* dbeta, float* coef, void* dy, int B,
                             int H, int W, int P, int Q, int Cp, cudaStream_t st) {
  const int CV = Cp / 8;
  if (dtype != DSP_DTYPE_BF16 || Cp % 8 || 256 % CV || (int64_t)B * H * W * Cp >= (1ll << 31)) return cudaErrorInvalidValue;
  const int64_t nq = (int64_t)B * P * Q;
  const int chunks = (int)std::min<int64_t>(296, nq);
  const int qpc = (int)((nq + chunks - 1) / chunks);
  launch_k(pool_bn_bwd_reduce_k, chunks, 256, 0, st, (const uint4*)u, (const uint2*)arg, (const uint4*)y, stat, part, B, H,
           W, P, Q, CV, qpc);
  note_launch();
  launch_k(bn_bwd_finalize_cols_k, (Cp + 31) / 32, 1024, 0, st, (const float*)part, chunks, Cp, c_real,
           (double)B * H * W, gamma, stat, dgamma, dbeta, coef);
  note_launch();
  launch_k(pool_bn_bwd_apply_k, grid_for(nq * CV), kThreads, 0, st, (const uint4*)u, (const uint2*)arg, (const uint4*)y,
           stat, (const float*)coef, (uint4*)dy, B, H, W, P, Q, CV);
  return note_launch(), cudaGetLastError();
}

cudaError_t maxpool_backward(int dtype, const void* u, const uint8_t* arg, void* dx, int B, int H, int W, int P, int Q,
                             int Cp, cudaStream_t st) {
  return dispatch_dtype(dtype, [&](auto t) {
    using T = decltype(t);
    if (Cp % V16<T>::N || (int64_t)B * H * W * Cp >= (1ll << 31)) return cudaErrorInvalidValue;
    static const bool generic = getenv("DSP_B200_MAXPOOL_GENERIC") != nullptr;  // A/B knob
    // the quad form covers input rows / columns [0, 2P) x [0, 2Q): exactly H x W when 2P >= H, 2Q >= W
    if (!generic && 2 * P >= H && 2 * Q >= W) {
      launch_k(maxpool_bwd_quad_k<T>, grid_for((int64_t)B * P * Q * Cp / V16<T>::N), kThreads, 0, st, (const T*)u, arg,
               (T*)dx, B, H, W, P, Q, Cp);
      return note_launch(), cudaGetLastError();
    }
    launch_k(maxpool_bwd_k<T>, grid_for((int64_t)B * H * W * Cp / V16<T>::N), kThreads, 0, st, (const T*)u, arg, (T*)dx, B, H, W, P, Q,
                                                                            Cp);
    return note_launch(), cudaGetLastError();
  });
}

cudaError_t softmax_xent(int dtype, const float* logits, int ld, int B, int C, const int64_t* labels, void* dlogits,
                         float* loss, float* row_loss, int* sem, int* nf, cudaStream_t st) {
  return dispatch_dtype(dtype, [&](auto t) {
    using T = decltype(t);
    launch_k(softmax_xent_k<T>, (B + 7) / 8, 256, 0, st, logits, ld, B, C, labels, (T*)dlogits, loss, row_loss, sem, nf);
    return note_launch(), cudaGetLastError();
  });
}

cudaError_t wgrad_reduce(const float* part, int splits, int Mw, int N, int RS, int Cp, int ci_real, int co_real,
                         int dense_layout, float* grad, cudaStream_t st, int s2d_r) {
  const int64_t total = (int64_t)Mw * N;
  if (N % 4) return cudaErrorInvalidValue;
  const int64_t tiles = (int64_t)((Mw + 31) / 32) * ((N + 31) / 32);
  static const bool flat = getenv("DSP_B200_WGRAD_REDUCE_FLAT") != nullptr;  // A/B knob
  if (dense_layout == 0 && tiles >= 148 && !flat) {
    launch_k(wgrad_reduce_tiled_k, dim3((Mw + 31) / 32, (N + 31) / 32), 256, 0, st, part, splits, Mw, N, RS, Cp, ci_real,
             co_real, grad);
    return note_launch(), cudaGetLastError();
  }
  launch_k(wgrad_reduce_k, (unsigned)((total + 127) / 128), 256, 0, st, part, splits, Mw, N, RS, Cp, ci_real, co_real,
           dense_layout, grad, s2d_r);
  return note_launch(), cudaGetLastError();
}

cudaError_t pack_weights(int dtype, const float* params, void* packed, const PackEntry* entries_dev, int n_entries,
                         int max_elems, cudaStream_t st) {
  if (n_entries == 0) return cudaSuccess;
  return dispatch_dtype(dtype, [&](auto t) {
    using T = decltype(t);
    dim3 grid(grid_for(max_elems, kThreads, 256), n_entries);
    launch_k(pack_weights_k<T>, grid, kThreads, 0, st, params, (T*)packed, entries_dev, n_entries);
    return note_launch(), cudaGetLastError();
  });
}

cudaError_t s2d_pack(int dtype, const void* x, void* s, int B, int H, int W, int c, int cpx, int Hs, int Ws, int cps,
                     int pad, cudaStream_t st) {
  if (dtype == DSP_DTYPE_BF16 && cpx == 8 && cps == 16 && c <= 4 && (int64_t)B * H * W < (1ll << 31)) {
    launch_k(s2d_pack8_k, grid_for((int64_t)B * Hs * Ws), kThreads, 0, st, (const uint4*)x, (uint4*)s, B, H, W, c, Hs,
             Ws, pad);
    return note_launch(), cudaGetLastError();
  }
  return dispatch_dtype(dtype, [&](auto t) {
    using T = decltype(t);
    launch_k(s2d_pack_k<T>, grid_for((int64_t)B * Hs * Ws), kThreads, 0, st, (const T*)x, (T*)s, B, H, W, c, cpx, Hs, Ws,
             cps, pad);
    return note_launch(), cudaGetLastError();
  });
}

cudaError_t s2d_unpack(int dtype, const void* ds, void* dx, int B, int H, int W, int c, int cpx, int Hs, int Ws, int cps,
                       int pad, cudaStream_t st) {
  return dispatch_dtype(dtype, [&](auto t) {
    using T = decltype(t);
    launch_k(s2d_unpack_k<T>, grid_for((int64_t)B * H * W), kThreads, 0, st, (const T*)ds, (T*)dx, B, H, W, c, cpx, Hs,
             Ws, cps, pad);
    return note_launch(), cudaGetLastError();
  });
}

int update_grid(int64_t n) { return grid_for(n, kThreads, 148 * 4); }

int update_pack_grid(int n_tiles) { return std::max(1, std::min(n_tiles, 148 * 8)); }

cudaError_t update_pack(int dtype, int rule, int apply, const UpdTile* tiles, int n_tiles, float* x, const float* grad,
                        float* ys, void* packed, float lr, float slr, float beta, float wd, float* part, int* sem,
                        float* grad_sq_out, int* nf, cudaStream_t st) {
  if (n_tiles <= 0) return cudaSuccess;
  const int g = update_pack_grid(n_tiles);
  return dispatch_dtype(dtype, [&](auto t) {
    using T = decltype(t);
    T* pk = static_cast<T*>(packed);
    auto go = [&](auto kern) {
      launch_k(kern, g, kThreads, 0, st, tiles, n_tiles, x, grad, ys, pk, lr, slr, beta, wd, part, sem, grad_sq_out, nf);
    };
    const bool w = wd != 0.f;
    if (!apply) go(update_pack_k<T, DSP_RULE_SGD, false, false>);
    else if (rule == DSP_RULE_SGD) w ? go(update_pack_k<T, DSP_RULE_SGD, true, true>) : go(update_pack_k<T, DSP_RULE_SGD, false, true>);
    else w ? go(update_pack_k<T, DSP_RULE_SUM, true, true>) : go(update_pack_k<T, DSP_RULE_SUM, false, true>);
    return note_launch(), cudaGetLastError();
  });
}

cudaError_t update_f32(int rule, int64_t n, float* x, const float* grad, float* ys, float lr, float slr, float beta,
                       float wd, float* part, cudaStream_t st) {
  const int g = update_grid(n);
  const bool w = wd != 0.f;
  if (rule == DSP_RULE_SGD) {
    if (w) launch_k(update_f32_k<DSP_RULE_SGD, true>, g, kThreads, 0, st, n, x, grad, ys, lr, slr, beta, wd, part);
    else launch_k(update_f32_k<DSP_RULE_SGD, false>, g, kThreads, 0, st, n, x, grad, ys, lr, slr, beta, wd, part);
  } else {
    if (w) launch_k(update_f32_k<DSP_RULE_SUM, true>, g, kThreads, 0, st, n, x, grad, ys, lr, slr, beta, wd, part);
    else launch_k(update_f32_k<DSP_RULE_SUM, false>, g, kThreads, 0, st, n, x, grad, ys, lr, slr, beta, wd, part);
  }
  return note_launch(), cudaGetLastError();
}

template <typename T>
cudaError_t update_adam(int64_t n, T* x, const T* grad, T* m, T* v, const int64_t* tstep, double bc1, double bc2,
                        double lr, double b1, double b2, double eps, double wd, T* part, cudaStream_t st) {
  const int g = update_grid(n);
  if (wd != 0.0)
    launch_k(update_adam_k<T, true>, g, kThreads, 0, st, n, x, grad, m, v, tstep, bc1, bc2, (T)lr, b1, b2, eps,
             (T)wd, part);
  else
    launch_k(update_adam_k<T, false>, g, kThreads, 0, st, n, x, grad, m, v, tstep, bc1, bc2, (T)lr, b1, b2, eps,
             (T)wd, part);
  note_launch();
  if (tstep != nullptr) {
    // device-side step counter: bumped after every CTA of the update has read it
    launch_k(step_bump_k, 1, 1, 0, st, const_cast<int64_t*>(tstep));
    note_launch();
  }
  return cudaGetLastError();
}
template cudaError_t update_adam<float>(int64_t, float*, const float*, float*, float*, const int64_t*, double, double,
                                        double, double, double, double, double, float*, cudaStream_t);
template cudaError_t update_adam<double>(int64_t, double*, const double*, double*, double*, const int64_t*, double,
                                         double, double, double, double, double, double, double*, cudaStream_t);

cudaError_t update_f64(int rule, int64_t n, double* x, const double* grad, double* ys, double* y, double lr, double slr,
                       double beta, double wd, double* part, cudaStream_t st) {
  const int g = update_grid(n);
  const bool w = wd != 0.0;
  if (rule == DSP_RULE_SGD) {
    if (w) launch_k(update_f64_k<DSP_RULE_SGD, true>, g, kThreads, 0, st, n, x, grad, ys, y, lr, slr, beta, wd, part);
    else launch_k(update_f64_k<DSP_RULE_SGD, false>, g, kThreads, 0, st, n, x, grad, ys, y, lr, slr, beta, wd, part);
  } else {
    if (w) launch_k(update_f64_k<DSP_RULE_SUM, true>, g, kThreads, 0, st, n, x, grad, ys, y, lr, slr, beta, wd, part);
    else launch_k(update_f64_k<DSP_RULE_SUM, false>, g, kThreads, 0, st, n, x, grad, ys, y, lr, slr, beta, wd, part);
  }
  return note_launch(), cudaGetLastError();
}

cudaError_t sumsq_f32(int64_t n, const float* v, float* part, cudaStream_t st) {
  launch_k(sumsq_k, update_grid(n), kThreads, 0, st, n, v, part);
  return note_launch(), cudaGetLastError();
}

cudaError_t sum_partials_f32(const float* part, int n, float* out, cudaStream_t st) {
  launch_k(sum_partials_k<float, float>, 1, kThreads, 0, st, part, n, out);
  return note_launch(), cudaGetLastError();
}

cudaError_t sum_partials_f64(const double* part, int n, double* out, cudaStream_t st) {
  launch_k(sum_partials_k<double, double>, 1, kThreads, 0, st, part, n, out);
  return note_launch(), cudaGetLastError();
}

cudaError_t pack_input(const float* x, void* out, int B, int C, int H, int W, int Cp, int dtype, int nchw,
                       cudaStream_t st) {
  return dispatch_dtype(dtype, [&](auto t) {
    using T = decltype(t);
    launch_k(pack_input_k<T>, grid_for((int64_t)B * H * W * Cp), kThreads, 0, st, x, (T*)out, B, C, H, W, Cp, nchw);
    return note_launch(), cudaGetLastError();
  });
}

cudaError_t unpack_output(const void* in, float* out, int B, int C, int H, int W, int Cp, int dtype, int nchw,
                          cudaStream_t st) {
  return dispatch_dtype(dtype, [&](auto t) {
    using T = decltype(t);
    launch_k(unpack_output_k<T>, grid_for((int64_t)B * C * H * W), kThreads, 0, st, (const T*)in, out, B, C, H, W, Cp, nchw);
    return note_launch(), cudaGetLastError();
  });
}

}  // namespace dsp
