// Implicit-GEMM convolution / dense layer on 5th-gen tensor cores (tcgen05, sm_100a).
//
// One kernel family covers the three GEMMs of a conv (or dense) layer:
//
//   FPROP  D[M=n*P*Q][N=Cout]       = sum_k X_im2col[m][k=(r,s,ci)] * W[co][k]
//   DGRAD  D[M=n*H*W][N=Cin]        = sum_k dY_gather[m][k=(r,s,co)] * W[co][r][s][ci]
//   WGRAD  D[M=(r,s,ci)][N=Cout]    = sum_k X_im2col[k=pixel][m] * dY[k][co]   (split-K)
//
// These replace the reference's dense `matmul` calls inside block_forward /
// block_backward (/root/reference/pkg/src/stalepipe/blocks.py:105-116,
// 147-151; tensor.py:40-56) generalised from dense to conv layers (a dense
// layer is the 1x1 conv on a 1x1 image).
//
// Structure (per CTA, 128 threads, one 128 x BN output tile):
//   * all 4 warps gather the A/B operand tiles with 16-byte cp.async (zero-fill
//     implements padding, ragged edges and stride-2 dgrad holes) straight into
//     the UMMA canonical SWIZZLE_NONE layout, STAGES-deep ring;
//   * one thread issues tcgen05.mma (kind::f16 for bf16 / kind::tf32 for fp32)
//     with the accumulator in TMEM, and tcgen05.commit releases each ring slot;
//   * the epilogue reads TMEM with tcgen05.ld (32 lanes per warp) and fuses
//     bias / residual add / dtype conversion / BatchNorm partial statistics
//     (FPROP, DGRAD) or writes split-K fp32 partials (WGRAD).
//
// Shared-memory operand layout (both K-major and MN-major, 16-byte "chunks"):
//   core matrix = 128 contiguous bytes (8 rows x 16 B), core (mn_grp, k_grp)
//   at k_grp * LBO + mn_grp * 128, LBO = E * 16 (E = rows of the tile).
//   K-major:  row = M/N index, 16 B = EPC consecutive K elements.
//   MN-major: row = K index,   16 B = EPC consecutive M/N elements.
#include "common.cuh"
#include "kernels.cuh"
#include "../../include/dsp_b200.h"

#include <stdio.h>

namespace dsp {

constexpr int IG_BM = 128;
constexpr int IG_STAGES = 4;
constexpr int IG_THREADS = 128;

template <typename T>
struct MmaTraits;
template <>
struct MmaTraits<bf16> {
  static constexpr int MMA_K = 16;
  static constexpr uint32_t FMT = 1;
  __device__ static void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t i, uint32_t acc) { umma_bf16(d, a, b, i, acc); }
};
template <>
struct MmaTraits<float> {
  static constexpr int MMA_K = 8;
  static constexpr uint32_t FMT = 2;
  __device__ static void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t i, uint32_t acc) { umma_tf32(d, a, b, i, acc); }
};

template <typename T, int MODE, int BN>
__global__ void __launch_bounds__(IG_THREADS) igemm_kernel(const dsp_igemm_args_t a) {
  constexpr int EPC = 16 / (int)sizeof(T);   // elements per 16-byte chunk
  constexpr int KS = 8 * EPC;                // K extent of one ring stage (128 B per row)
  constexpr int A_BYTES = IG_BM * 128;
  constexpr int B_BYTES = BN * 128;
  constexpr int TMEM_COLS = BN < 32 ? 32 : BN;
  constexpr bool A_MN = (MODE == DSP_IGEMM_WGRAD);
  constexpr bool B_MN = (MODE != DSP_IGEMM_FPROP);

  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t mma_bar[IG_STAGES];
  __shared__ uint32_t tmem_base_s;
  __shared__ float red[4][BN][2];

  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const int lane = tid & 31;
  const dsp_conv_geom_t g = a.geom;
  const int M = a.M, N = a.N, Kd = a.Kd;
  const int m0 = blockIdx.x * IG_BM;
  const int n0 = blockIdx.y * BN;

  const T* __restrict__ Asrc = reinterpret_cast<const T*>(a.A);
  const T* __restrict__ Bsrc = reinterpret_cast<const T*>(a.B);

  const int nkb_total = (Kd + KS - 1) / KS;
  int kb_begin = 0, kb_end = nkb_total;
  if (MODE == DSP_IGEMM_WGRAD) {
    kb_begin = blockIdx.z * a.kb_per_split;
    kb_end = min(nkb_total, kb_begin + a.kb_per_split);
  }
  const int nk = kb_end - kb_begin;

  if (tid == 0) {
    for (int s = 0; s < IG_STAGES; ++s) mbar_init(&mma_bar[s], 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc(&tmem_base_s, TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_d = tmem_base_s;

  const uint32_t sA0 = smem_u32(smem);
  const uint32_t sB0 = sA0 + IG_STAGES * A_BYTES;

  // ---------------- per-tile precompute for the A gather ----------------
  // K-major A (FPROP / DGRAD): thread owns chunk column j and rows (tid>>3)+16*i.
  const int aj = tid & 7;
  int a_h[8], a_w[8];
  long long a_img[8];
  // MN-major A (WGRAD): thread owns MN group ag and k-rows.
  constexpr int AG = IG_BM / EPC;  // MN groups in the A tile
  const int ag = tid % AG;
  int wg_r = 0, wg_s = 0, wg_c = 0;
  bool wg_ok = false;
  if (MODE == DSP_IGEMM_FPROP || MODE == DSP_IGEMM_DGRAD) {
    const int PQ = (MODE == DSP_IGEMM_FPROP) ? g.P * g.Q : g.H * g.W;
    const int QQ = (MODE == DSP_IGEMM_FPROP) ? g.Q : g.W;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int m = m0 + (tid >> 3) + 16 * i;
      if (m < M) {
        const int img = m / PQ;
        const int rem = m - img * PQ;
        const int y = rem / QQ;
        const int x = rem - y * QQ;
        if (MODE == DSP_IGEMM_FPROP) {
          a_h[i] = y * g.stride - g.pad;
          a_w[i] = x * g.stride - g.pad;
          a_img[i] = (long long)img * g.H * g.W * g.C;
        } else {
          a_h[i] = y + g.pad;
          a_w[i] = x + g.pad;
          a_img[i] = (long long)img * g.P * g.Q * g.K;
        }
      } else {
        a_h[i] = -(1 << 28);  // forces the bounds check to fail
        a_w[i] = -(1 << 28);
        a_img[i] = 0;
      }
    }
  } else {
    const int m = m0 + ag * EPC;
    if (m < M) {
      const int tap = m / g.C;
      wg_c = m - tap * g.C;
      wg_r = tap / g.S;
      wg_s = tap - wg_r * g.S;
      wg_ok = true;
    }
  }

  auto load_stage = [&](int kb, uint32_t sA, uint32_t sB) {
    // ---------------- A operand ----------------
    if (MODE == DSP_IGEMM_FPROP || MODE == DSP_IGEMM_DGRAD) {
      const int k0 = kb * KS + aj * EPC;
      const bool kok = k0 < Kd;
      const int cdim = (MODE == DSP_IGEMM_FPROP) ? g.C : g.K;
      const int tap = kok ? k0 / cdim : 0;
      const int c0 = k0 - tap * cdim;
      const int r = tap / g.S;
      const int s = tap - r * g.S;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int row = (tid >> 3) + 16 * i;
        const T* src = Asrc;
        bool ok = kok;
        if (MODE == DSP_IGEMM_FPROP) {
          const int ih = a_h[i] + r, iw = a_w[i] + s;
          ok = ok && (unsigned)ih < (unsigned)g.H && (unsigned)iw < (unsigned)g.W;
          if (ok) src = Asrc + a_img[i] + ((long long)ih * g.W + iw) * g.C + c0;
        } else {
          int hh = a_h[i] - r, ww = a_w[i] - s;
          if (g.stride != 1) {
            ok = ok && hh >= 0 && ww >= 0 && (hh % g.stride) == 0 && (ww % g.stride) == 0;
            hh /= g.stride;
            ww /= g.stride;
          }
          ok = ok && (unsigned)hh < (unsigned)g.P && (unsigned)ww < (unsigned)g.Q;
          if (ok) src = Asrc + a_img[i] + ((long long)hh * g.Q + ww) * g.K + c0;
        }
        cp_async_16(sA + aj * (IG_BM * 16) + row * 16, src, ok ? 16u : 0u);
      }
    } else {
      // WGRAD: A[m=(r,s,ci)][k=pixel] from X, MN-major
      const int PQ = g.P * g.Q;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int kr = tid / AG + (IG_THREADS / AG) * i;
        const int p = kb * KS + kr;
        const T* src = Asrc;
        bool ok = wg_ok && p < Kd;
        if (ok) {
          const int img = p / PQ;
          const int rem = p - img * PQ;
          const int oh = rem / g.Q;
          const int ow = rem - oh * g.Q;
          const int ih = oh * g.stride - g.pad + wg_r;
          const int iw = ow * g.stride - g.pad + wg_s;
          ok = (unsigned)ih < (unsigned)g.H && (unsigned)iw < (unsigned)g.W;
          if (ok) src = Asrc + (((long long)img * g.H + ih) * g.W + iw) * g.C + wg_c;
        }
        cp_async_16(sA + (kr >> 3) * (AG * 128) + ag * 128 + (kr & 7) * 16, src, ok ? 16u : 0u);
      }
    }
    // ---------------- B operand ----------------
    constexpr int BCH = 8 * BN;  // chunks per stage
    if (MODE == DSP_IGEMM_FPROP) {
      // K-major weights Wb[n][Kd]
#pragma unroll
      for (int c = tid; c < BCH; c += IG_THREADS) {
        const int n = c >> 3, j = c & 7;
        const int k0 = kb * KS + j * EPC;
        const bool ok = (n0 + n) < N && k0 < Kd;
        const T* src = ok ? Bsrc + (long long)(n0 + n) * Kd + k0 : Bsrc;
        cp_async_16(sB + j * (BN * 16) + n * 16, src, ok ? 16u : 0u);
      }
    } else {
      constexpr int BG = BN / EPC;  // MN groups in the B tile
#pragma unroll
      for (int c = tid; c < BCH; c += IG_THREADS) {
        const int gg = c % BG, kr = c / BG;
        const int k = kb * KS + kr;
        const int n = n0 + gg * EPC;
        bool ok = n < N && k < Kd;
        const T* src = Bsrc;
        if (ok) {
          if (MODE == DSP_IGEMM_DGRAD) {
            // B[n=ci][k=(r,s,co)] = Wb[co][r][s][ci]
            const int tap = k / g.K;
            const int co = k - tap * g.K;
            src = Bsrc + ((long long)co * g.R * g.S + tap) * g.C + n;
          } else {
            // WGRAD: B[n=co][k=pixel] = dY[pixel][co]
            src = Bsrc + (long long)k * g.K + n;
          }
        }
        cp_async_16(sB + (kr >> 3) * (BG * 128) + gg * 128 + (kr & 7) * 16, src, ok ? 16u : 0u);
      }
    }
  };

  const uint32_t idesc = umma_idesc(MmaTraits<T>::FMT, A_MN ? 1u : 0u, B_MN ? 1u : 0u, IG_BM, BN);

  // ---------------- main pipelined K loop ----------------
  for (int it = 0; it < nk + IG_STAGES - 1; ++it) {
    if (it < nk) {
      const int s = it % IG_STAGES;
      if (it >= IG_STAGES) mbar_wait(&mma_bar[s], ((it / IG_STAGES) - 1) & 1);
      load_stage(kb_begin + it, sA0 + s * A_BYTES, sB0 + s * B_BYTES);
    }
    cp_async_commit();
    const int kc = it - (IG_STAGES - 1);
    if (kc >= 0) {
      cp_async_wait<IG_STAGES - 1>();
      fence_proxy_async_smem();
      __syncthreads();
      if (tid == 0) {
        tc_fence_after();
        const int s = kc % IG_STAGES;
        const uint32_t sa = sA0 + s * A_BYTES;
        const uint32_t sb = sB0 + s * B_BYTES;
#pragma unroll
        for (int kk = 0; kk < KS / MmaTraits<T>::MMA_K; ++kk) {
          const uint64_t ad = umma_sdesc(sa + kk * 32 * IG_BM, A_MN ? (IG_BM / EPC) * 128 : IG_BM * 16, 128);
          const uint64_t bd = umma_sdesc(sb + kk * 32 * BN, B_MN ? (BN / EPC) * 128 : BN * 16, 128);
          MmaTraits<T>::mma(tmem_d, ad, bd, idesc, (kc > 0 || kk > 0) ? 1u : 0u);
        }
        umma_commit(&mma_bar[s]);
      }
    }
  }
  if (nk > 0) {
    const int last = nk - 1;
    mbar_wait(&mma_bar[last % IG_STAGES], (last / IG_STAGES) & 1);
  }
  tc_fence_after();

  // ---------------- epilogue ----------------
  const int row = warp * 32 + lane;
  const int m = m0 + row;
  const bool mok = m < M;
  const uint32_t tl = tmem_d + ((uint32_t)(warp * 32) << 16);
  const bool want_stats = (MODE != DSP_IGEMM_WGRAD) && a.stats != nullptr;

#pragma unroll 1
  for (int cc = 0; cc < BN / 16; ++cc) {
    float v[16];
    if (nk > 0) {
      tmem_ld16(tl + cc * 16, v);
    } else {
#pragma unroll
      for (int i = 0; i < 16; ++i) v[i] = 0.f;
    }
    const int nb = n0 + cc * 16;
    if (MODE == DSP_IGEMM_WGRAD) {
      float* out = reinterpret_cast<float*>(a.D) + (size_t)blockIdx.z * M * N + (size_t)m * N;
      if (mok) {
        if (nb + 16 <= N && (N & 3) == 0) {
#pragma unroll
          for (int q = 0; q < 4; ++q)
            *reinterpret_cast<float4*>(out + nb + 4 * q) = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
        } else {
#pragma unroll
          for (int i = 0; i < 16; ++i)
            if (nb + i < N) out[nb + i] = v[i];
        }
      }
    } else {
      const int nvalid = a.n_valid > 0 ? a.n_valid : N;
      if (a.bias != nullptr) {
#pragma unroll
        for (int i = 0; i < 16; ++i)
          if (nb + i < nvalid) v[i] += a.bias[nb + i];
      }
      if (a.residual != nullptr && mok) {
        const T* res = reinterpret_cast<const T*>(a.residual) + (size_t)m * a.ldd;
#pragma unroll
        for (int i = 0; i < 16; ++i)
          if (nb + i < N) v[i] += to_f<T>(res[nb + i]);
      }
#pragma unroll
      for (int i = 0; i < 16; ++i)
        if (nb + i >= nvalid) v[i] = 0.f;
      if (a.out_f32) {
        float* out = reinterpret_cast<float*>(a.D) + (size_t)m * a.ldd;
        if (mok) {
#pragma unroll
          for (int i = 0; i < 16; ++i)
            if (nb + i < N) out[nb + i] = v[i];
        }
      } else {
        T* out = reinterpret_cast<T*>(a.D) + (size_t)m * a.ldd;
        // round to the storage type first so BN statistics describe the stored tensor
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = to_f<T>(from_f<T>(v[i]));
        if (mok) {
          if (nb + 16 <= N && (a.ldd % EPC) == 0) {
#pragma unroll
            for (int q = 0; q < 16 / EPC; ++q) {
              T tmp[EPC];
#pragma unroll
              for (int e = 0; e < EPC; ++e) tmp[e] = from_f<T>(v[q * EPC + e]);
              *reinterpret_cast<uint4*>(out + nb + q * EPC) = *reinterpret_cast<uint4*>(tmp);
            }
          } else {
#pragma unroll
            for (int i = 0; i < 16; ++i)
              if (nb + i < N) out[nb + i] = from_f<T>(v[i]);
          }
        }
      }
      if (want_stats) {
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const float x = mok ? v[i] : 0.f;
          const float s1 = warp_sum(x);
          const float s2 = warp_sum(x * x);
          if (lane == 0) {
            red[warp][cc * 16 + i][0] = s1;
            red[warp][cc * 16 + i][1] = s2;
          }
        }
      }
    }
  }
  if (want_stats) {
    __syncthreads();
    for (int c = tid; c < BN; c += IG_THREADS) {
      const int n = n0 + c;
      if (n < N) {
        const float s1 = (red[0][c][0] + red[1][c][0]) + (red[2][c][0] + red[3][c][0]);
        const float s2 = (red[0][c][1] + red[1][c][1]) + (red[2][c][1] + red[3][c][1]);
        a.stats[((size_t)blockIdx.x * 2 + 0) * N + n] = s1;
        a.stats[((size_t)blockIdx.x * 2 + 1) * N + n] = s2;
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem_d, TMEM_COLS);
  }
}

template <typename T, int MODE, int BN>
static cudaError_t launch_bn(const dsp_igemm_args_t& a, int splits, cudaStream_t st) {
  const int smem = IG_STAGES * (IG_BM * 128 + BN * 128);
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(igemm_kernel<T, MODE, BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  dim3 grid((a.M + IG_BM - 1) / IG_BM, (a.N + BN - 1) / BN, MODE == DSP_IGEMM_WGRAD ? splits : 1);
  igemm_kernel<T, MODE, BN><<<grid, IG_THREADS, smem, st>>>(a);
  note_launch();
  return cudaGetLastError();
}

template <typename T, int MODE>
static cudaError_t launch_mode(const dsp_igemm_args_t& a, int splits, cudaStream_t st) {
  if (a.N <= 16) return launch_bn<T, MODE, 16>(a, splits, st);
  if (a.N <= 32) return launch_bn<T, MODE, 32>(a, splits, st);
  if (a.N <= 64) return launch_bn<T, MODE, 64>(a, splits, st);
  if (a.N <= 128) return launch_bn<T, MODE, 128>(a, splits, st);
  return launch_bn<T, MODE, 256>(a, splits, st);
}

cudaError_t igemm_launch(int mode, int dtype, const dsp_igemm_args_t& a, int splits, cudaStream_t st) {
  if (dtype == DSP_DTYPE_BF16) {
    if (mode == DSP_IGEMM_FPROP) return launch_mode<bf16, DSP_IGEMM_FPROP>(a, splits, st);
    if (mode == DSP_IGEMM_DGRAD) return launch_mode<bf16, DSP_IGEMM_DGRAD>(a, splits, st);
    if (mode == DSP_IGEMM_WGRAD) return launch_mode<bf16, DSP_IGEMM_WGRAD>(a, splits, st);
  } else if (dtype == DSP_DTYPE_F32) {
    if (mode == DSP_IGEMM_FPROP) return launch_mode<float, DSP_IGEMM_FPROP>(a, splits, st);
    if (mode == DSP_IGEMM_DGRAD) return launch_mode<float, DSP_IGEMM_DGRAD>(a, splits, st);
    if (mode == DSP_IGEMM_WGRAD) return launch_mode<float, DSP_IGEMM_WGRAD>(a, splits, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace dsp
