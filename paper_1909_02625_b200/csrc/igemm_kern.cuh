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
// Persistent, warp-specialised CTA (288 threads), one or two CTAs per SM:
//   warps 0-3  producers: gather A/B operand tiles with 16-byte cp.async
//              (zero-fill = conv padding, ragged edges, stride-2 dgrad holes)
//              straight into the UMMA canonical SWIZZLE_NONE layout, through a
//              STAGES-deep smem ring that runs continuously across output tiles;
//   warp 4     allocates TMEM; lane 0 issues tcgen05.mma (kind::f16 / kind::tf32)
//              into a double-buffered TMEM accumulator and tcgen05.commit's the
//              ring slots / accumulators back;
//   warps 5-8  epilogue: tcgen05.ld 32 lanes each, fuse bias / residual add /
//              dtype conversion / BatchNorm statistics (FPROP, with the per-channel
//              finalize done by the last CTA to finish) or write split-K fp32
//              partials (WGRAD), while the MMA works on the next tile.
//
// Shared-memory operand layout (both K-major and MN-major, 16-byte "chunks"):
//   core matrix = 128 contiguous bytes (8 rows x 16 B), core (mn_grp, k_grp)
//   at k_grp * LBO + mn_grp * 128.
//   K-major:  row = M/N index, 16 B = EPC consecutive K elements.
//   MN-major: row = K index,   16 B = EPC consecutive M/N elements.
#pragma once
#include "common.cuh"
#include "kernels.cuh"
#include "../../include/dsp_b200.h"

#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <type_traits>
#include <cstdlib>
#include <cstring>

namespace dsp {

constexpr int IG_BM = 128;

// Stride-2 DGRAD, output parity ph: the taps r of an R-tap (pad (R-1)/2) kernel that reach
// output rows 2i+ph, i.e. (ph + pad - r) even; they read dY row i + (ph + pad - r) / 2.
__device__ __forceinline__ int s2_taps(int R, int pad, int ph, int (&list)[2]) {
  int n = 0;
  for (int r = 0; r < R && n < 2; ++r)
    if (((ph + pad - r) & 1) == 0) list[n++] = r;
  return n;
}

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

#ifndef IG_STAGES_SMALL
#define IG_STAGES_SMALL 3
#endif
#ifndef IG_DEEP64_STAGES  // im2col kernels with 64-wide tiles (ResNet-50 stage 1)
#define IG_DEEP64_STAGES 3
#endif
#ifndef IG_STAGES_MID
#define IG_STAGES_MID 2
#endif
// WGRAD ring depth for 128 / 64-wide tiles (its grid is ~one CTA per SM, so a deeper ring only costs
// the SM's co-residency with the other block streams' kernels)
#ifndef IG_WG_STAGES_128
#define IG_WG_STAGES_128 3
#endif
#ifndef IG_WG_STAGES_64
#define IG_WG_STAGES_64 4
#endif
template <int MODE, int BN, int CFG_STAGES>
struct IgStages {
  static constexpr int value = MODE != DSP_IGEMM_WGRAD ? CFG_STAGES
                               : BN == 128           ? (IG_WG_STAGES_128 > CFG_STAGES ? IG_WG_STAGES_128 : CFG_STAGES)
                               : BN == 64            ? (IG_WG_STAGES_64 > CFG_STAGES ? IG_WG_STAGES_64 : CFG_STAGES)
                                                     : CFG_STAGES;
};
#ifndef IG_REG_BLOCKS  // register budget as if this many CTAs shared an SM (headroom for other streams)
#define IG_REG_BLOCKS 3
#endif
// rows in flight per thread in the fused finalize's partial-row load (trace experiments vary it)
#ifndef IG_FIN_DEPTH
#define IG_FIN_DEPTH 4
#endif
#ifndef IG_MAX_CTAS_PER_SM
#define IG_MAX_CTAS_PER_SM 2
#endif
// Instrumentation (clock64 pipeline stamps of CTA 0, per-CTA %globaltimer timeline into
// a.trace) is compiled in only with -DIG_TRACE_BUILD: it costs registers, and register
// headroom decides how many of the other blocks' CTAs fit beside a conv CTA.
#ifdef IG_TRACE_BUILD
constexpr bool kTrace = true;
#else
constexpr bool kTrace = false;
#endif

// DEEP: the im2col kernel variant (ImageNet-sized launches that own the GPU) keeps a 4-stage
// ring at every width <= 64; the CIFAR variants stay shallow so concurrent block streams fit
template <int BN, bool DEEP = false>
struct IgCfg {
  static constexpr int STAGES = (DEEP && BN <= 32) ? 4 : (DEEP && BN == 64) ? IG_DEEP64_STAGES
                                : BN <= 32 ? IG_STAGES_SMALL : (BN <= 128 ? IG_STAGES_MID : 4);
  static constexpr int RING = STAGES * (IG_BM * 128 + BN * 128);
#ifdef IG_TMA_STORE
  static constexpr int OUT_BYTES = IG_BM * BN * 2;  // bf16 output tile staged for the TMA store
#else
  static constexpr int OUT_BYTES = 0;
#endif
  // wide tiles: per-epilogue-warp double-buffered 32-row x 16-column bf16 staging slabs for
  // TMA stores (8 warps x 2 x 1 KB)
  static constexpr int DW_BYTES = (BN >= 128 || (DEEP && BN == 64)) ? 8 * 2 * 1024 : 0;
  static constexpr int SMEM = RING + OUT_BYTES + DW_BYTES;
  // TMEM accumulators (MMA runs NACC-1 tiles ahead); BN=128 keeps two so two CTAs share an SM
  static constexpr int NACC = BN < 128 ? 4 : 2;
  static constexpr int TMEM_COLS = NACC * BN < 32 ? 32 : NACC * BN;
  static constexpr int BY_SMEM = SMEM <= 70 * 1024 ? 3 : SMEM <= 100 * 1024 ? 2 : 1;
  static constexpr int BY_TMEM = 512 / TMEM_COLS;
  static constexpr int CTAS_PER_SM = IG_MAX_CTAS_PER_SM < BY_SMEM ? (IG_MAX_CTAS_PER_SM < BY_TMEM ? IG_MAX_CTAS_PER_SM : BY_TMEM)
                                                                  : (BY_SMEM < BY_TMEM ? BY_SMEM : BY_TMEM);
};

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
template <int NT>
__device__ __forceinline__ void epi_barrier() { asm volatile("bar.sync 1, %0;" ::"n"(NT) : "memory"); }

// bf16 pair (one 32-bit word: element 2j in the low half) -> float2, for the packed FP32x2
// (FFMA2 / FADD2) statistics arithmetic of the fast epilogues
__device__ __forceinline__ float2 bf2f2(uint32_t w) {
  return make_float2(__uint_as_float(w << 16), __uint_as_float(w & 0xffff0000u));
}

// Reduce-scatter over the 8 lanes sharing lane % 4 (lane bits 4, 3, 2; fixed tree) of two 8-column
// partial-sum vectors a, b: each step keeps the half of the columns selected by the lane bit and
// adds the partner's copy, so lane (k4, cg = lane >> 2) ends with column cg's totals in ra / rb --
// 14 shuffles instead of a 48-shuffle butterfly. with_a = false skips a (rb only, 7 shuffles).
__device__ __forceinline__ void rs8_pair(const float (&a)[8], const float (&b)[8], int lane, bool with_a, float& ra,
                                         float& rb) {
  const int cg = lane >> 2;
  float v[8];
  {
    const bool hb = (cg >> 2) & 1;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float k1 = hb ? a[4 + i] : a[i], o1 = hb ? a[i] : a[4 + i];
      const float k2 = hb ? b[4 + i] : b[i], o2 = hb ? b[i] : b[4 + i];
      v[2 * i] = k1 + (with_a ? __shfl_xor_sync(0xffffffffu, o1, 16) : 0.f);
      v[2 * i + 1] = k2 + __shfl_xor_sync(0xffffffffu, o2, 16);
    }
  }
  {
    const bool hb = (cg >> 1) & 1;
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const float k1 = hb ? v[2 * (2 + i)] : v[2 * i], o1 = hb ? v[2 * i] : v[2 * (2 + i)];
      const float k2 = hb ? v[2 * (2 + i) + 1] : v[2 * i + 1], o2 = hb ? v[2 * i + 1] : v[2 * (2 + i) + 1];
      v[2 * i] = k1 + (with_a ? __shfl_xor_sync(0xffffffffu, o1, 8) : 0.f);
      v[2 * i + 1] = k2 + __shfl_xor_sync(0xffffffffu, o2, 8);
    }
  }
  const bool hb = cg & 1;
  const float k1 = hb ? v[2] : v[0], o1 = hb ? v[0] : v[2];
  const float k2 = hb ? v[3] : v[1], o2 = hb ? v[1] : v[3];
  ra = k1 + (with_a ? __shfl_xor_sync(0xffffffffu, o1, 4) : 0.f);
  rb = k2 + __shfl_xor_sync(0xffffffffu, o2, 4);
}

// Column sums of a 32-row x 16-column register tile (one row per lane) with 16
// shuffles: halve the column set at each butterfly step. Lane l ends holding the
// full sum of column (l >> 1) & 15.
__device__ __forceinline__ float colsum16(const float (&v)[16], int lane) {
  float w8[8], w4[4], w2[2];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const bool up = lane & 16;
    const float send = up ? v[i] : v[i + 8];
    const float keep = up ? v[i + 8] : v[i];
    w8[i] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const bool up = lane & 8;
    const float send = up ? w8[i] : w8[i + 4];
    const float keep = up ? w8[i + 4] : w8[i];
    w4[i] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
  }
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const bool up = lane & 4;
    const float send = up ? w4[i] : w4[i + 2];
    const float keep = up ? w4[i + 2] : w4[i];
    w2[i] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
  }
  const bool up = lane & 2;
  float w1 = (up ? w2[1] : w2[0]) + __shfl_xor_sync(0xffffffffu, up ? w2[0] : w2[1], 2);
  w1 += __shfl_xor_sync(0xffffffffu, w1, 1);
  return w1;
}

// tf32 operands stored MN-major (WGRAD A and B, DGRAD B in fp32 storage). kind::tf32 reads an
// MN-major operand only in the SWIZZLE_128B_BASE32B layout (measured with
// tools/gpu/umma_layout_probe.cu: SWIZZLE_NONE / 32B / 64B / 128B MN-major tf32 operands read as
// zeros): atoms of 4 K rows x 32 MN elements (128-byte rows), the 16-byte chunk c of row r stored
// at chunk c ^ 2r (bits [7,9) of the byte offset XORed into bits [5,7)). Here the K atoms of one
// 32-element MN slice lie 512 B apart (descriptor SBO) and the MN slices 32 K rows = 4 KB apart
// (LBO), so a 32-row ring stage holds 8 K atoms per MN slice.
constexpr uint32_t TF32_MN_LBO = 4096, TF32_MN_SBO = 512;

// 3xTF32 operand split of one 16-byte smem chunk: hi = x rounded to tf32 (exact in the MMA),
// lo = x - hi (exact in fp32; the MMA keeps its top 11 bits)
__device__ __forceinline__ void tf32_split16(uint32_t src_hi, uint32_t dst_lo) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(src_hi));
  uint32_t h[4];
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(h[0]) : "f"(v.x));
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(h[1]) : "f"(v.y));
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(h[2]) : "f"(v.z));
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(h[3]) : "f"(v.w));
  const float l0 = v.x - __uint_as_float(h[0]), l1 = v.y - __uint_as_float(h[1]), l2 = v.z - __uint_as_float(h[2]),
              l3 = v.w - __uint_as_float(h[3]);
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(src_hi), "r"(h[0]), "r"(h[1]), "r"(h[2]), "r"(h[3])
               : "memory");
  asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(dst_lo), "f"(l0), "f"(l1), "f"(l2), "f"(l3)
               : "memory");
}
__device__ __forceinline__ uint32_t tf32_mn_off(int mnchunk, int krow) {
  const int r = krow & 3;
  return (uint32_t)((mnchunk >> 3) * (int)TF32_MN_LBO + (krow >> 2) * (int)TF32_MN_SBO + r * 128 +
                    (((mnchunk & 7) ^ (r << 1)) << 4));
}

// 16 consecutive columns [nb, nb + 16) of row m of a [M][ld] storage-dtype tensor as
// floats (zeros for rows the tile does not own and columns >= N).
template <typename T>
__device__ __forceinline__ void ld_row16(const void* base, bool mok, int m, int ld, int nb, int N, float (&out)[16]) {
  constexpr int EPC = 16 / (int)sizeof(T);
  const T* p = reinterpret_cast<const T*>(base) + (size_t)m * ld + nb;
  if (mok && nb + 16 <= N && (ld % EPC) == 0) {
#pragma unroll
    for (int qq = 0; qq < 16 / EPC; ++qq) {
      const uint4 raw = *reinterpret_cast<const uint4*>(p + qq * EPC);
      const T* e8 = reinterpret_cast<const T*>(&raw);
#pragma unroll
      for (int e = 0; e < EPC; ++e) out[qq * EPC + e] = to_f<T>(e8[e]);
    }
  } else {
#pragma unroll
    for (int e = 0; e < 16; ++e) out[e] = (mok && nb + e < N) ? to_f<T>(p[e]) : 0.f;
  }
}

// TMA configuration of one launch (host-decided, see tma_plan()).
//   A (FPROP / stride-1 DGRAD): per k-block, 64/cbox boxes, one per (tap, channel
//   chunk), each a 128-pixel im2col tile of cbox channels at tap-shifted
//   coordinates; out-of-image taps are zero-filled by the TMA unit.
//   B (FPROP weights [Cout][Kd]): one 64 x BN box per k-block, SWIZZLE_128B.
struct IgTma {
  int on_a, on_b;
  int cbox;       // channels per A box (8, 16, 32, 64)
  int hb, nb;     // A box extent in output rows / images (box = OW x hb x nb pixels)
  int box_a;      // bytes per A box = 128 rows x cbox x 2
  int swz_a;      // UMMA layout type of A (0 none, 6 SW32, 4 SW64, 2 SW128)
  int box_b;      // bytes per B box (FPROP: BN rows x 128; WGRAD: 64 pixels x cbox_b x 2)
  // WGRAD (both operands MN-major, k = 64 output pixels per stage):
  int cbox_b;     // channels per B (dY) box
  int swz_b;      // UMMA layout type of B
  int kb_rows, kb_imgs;  // a 64-pixel k-block = Q x kb_rows x kb_imgs output pixels
  // D (bf16 FPROP / DGRAD output): epilogue stages the 128 x BN tile in smem, one TMA
  // store per box of d_cols columns (rows of d_cols*2 bytes, swizzle mask d_swz)
  int on_d, d_cols, d_swz;
  // FPROP halo tiles (stride-1 RxS convs, C <= 64, one image per tile): one stage per tile =
  // S boxes of (hb + R - 1) input rows x W x C (one per horizontal tap offset, OOB = padding);
  // tap (r, s) is the box-s view shifted down r rows. Weights stay resident in smem.
  int halo;
  int h_box;    // bytes of one A box
  int h_nst;    // ring depth (stages = tiles in flight)
  int h_nwb;    // resident weight boxes of 64 K x BN (SWIZZLE_128B)
  int h_rowb;   // bytes per A row (C * 2)
  int h_swz;    // UMMA layout type of A
  // im2col-mode A (any output width; FPROP stride 1/2, stride-1 DGRAD on dY with the per-tap
  // transposed weights B_t, WGRAD): one box of 128 (WGRAD: 64) consecutive output pixels x 64
  // channels per (tap, channel chunk); the tap is the instruction's im2col offset
  int i2c;
  int s2;       // stride-2 DGRAD split by output parity (ph, pw) into stride-1 sub-convolutions of dY
  int a2d;      // im2col plan of a 1x1 stride-1 conv: A is a plain [pixels][C] matrix (2-D tiled boxes)
  int d_warp;   // wide-tile epilogue: per-warp 32-row x 64-byte slabs staged in smem
  int d_tma;    // ... and stored by TMA from the slab (tmD: box {32 columns, 32 rows}, SWIZZLE_64B)
  int i2c_pad;  // start coordinate of output pixel (p, q) = (p * st - i2c_pad, q * st - i2c_pad)
  // FastDiv multipliers computed on the host (64-bit divisions are slow on device):
  // [0] output pixels / image, [1] output row width, [2] gathered channels, [3] S, [4] K
  uint32_t fd_d[5], fd_mul[5], fd_shr[5];
  int fin1;     // 1: single-level BN finalize (DSP_B200_FIN_1LEVEL A/B switch)
};

static void fastdiv_host(uint32_t d, uint32_t& mul, uint32_t& shr) {
  if (d <= 1) {
    mul = 0;
    shr = 0;
    return;
  }
  uint32_t l = 0;
  while ((1u << l) < d) ++l;
  mul = (uint32_t)((((uint64_t)1 << (31 + l)) + d - 1) / d);
  shr = 31 + l - 32;
}

// Warp roles for NPW producer warps: 4 when operands are gathered with cp.async (128
// threads), 1 when every operand comes through TMA (one lane issues the boxes).
// Registers are budgeted as if REG_BLOCKS CTAs shared an SM, leaving room for the other
// block streams' kernels beside a conv CTA (<= 75 regs at 288 threads, <= 68 at 192).
template <int NPW, int BN, bool I2C = false>
struct IgWarps {
  static constexpr bool WIDE = BN >= 128 || (I2C && BN == 64);
  // 8 epilogue warps (two per TMEM lane quadrant, each half the columns) for the wide tiles of
  // the tensor-bound shapes, whose epilogue would otherwise bound small-Kd (1x1) convs
  static constexpr int NEPI = WIDE ? 8 : 4;
  static constexpr int THREADS = (NPW + 1 + NEPI) * 32;
  static constexpr int MMA_WARP = NPW;
  static constexpr int EPI_WARP0 = NPW + 1;
  static constexpr int REG_BLOCKS = WIDE ? 1 : (NPW == 4 ? IG_REG_BLOCKS : IG_REG_BLOCKS + 2);
};

// I2C: the im2col-operand variant (its producer branches are compiled only into it: extra
// never-taken producer code measurably slowed the halo / tiled kernels of the CIFAR step)
template <typename T, int MODE, int BN, int NPW, bool I2C = false>
__global__ void __launch_bounds__(IgWarps<NPW, BN, I2C>::THREADS, IgWarps<NPW, BN, I2C>::REG_BLOCKS > IgCfg<BN, I2C>::CTAS_PER_SM
                                                             ? IgWarps<NPW, BN, I2C>::REG_BLOCKS
                                                             : IgCfg<BN, I2C>::CTAS_PER_SM)
    igemm_kernel(const dsp_igemm_args_t a, const __grid_constant__ CUtensorMap tmA,
                 const __grid_constant__ CUtensorMap tmB, const __grid_constant__ CUtensorMap tmD,
                 const IgTma tm) {
  using Cfg = IgCfg<BN, I2C>;
  constexpr int IG_THREADS = IgWarps<NPW, BN, I2C>::THREADS;
  constexpr int IG_MMA_WARP = IgWarps<NPW, BN, I2C>::MMA_WARP;
  constexpr int IG_EPI_WARP0 = IgWarps<NPW, BN, I2C>::EPI_WARP0;
  constexpr int NEPI = IgWarps<NPW, BN, I2C>::NEPI;
  constexpr int EPI_T = NEPI * 32;
  // fp32 storage runs 3xTF32 (see F32_SPLIT below): hi and lo copies of every stage, 2 stages
  constexpr int STAGES = sizeof(T) == 4 ? 2 : IgStages<MODE, BN, Cfg::STAGES>::value;
  constexpr int NACC = Cfg::NACC;
  constexpr int EPC = 16 / (int)sizeof(T);  // elements per 16-byte chunk
  constexpr int KS = 8 * EPC;               // K extent of one ring stage (128 B per row)
  constexpr int A_BYTES = IG_BM * 128;
  constexpr bool A_MN = (MODE == DSP_IGEMM_WGRAD);
  constexpr bool B_MN = (MODE != DSP_IGEMM_FPROP);
  constexpr bool TF_MN = sizeof(T) == 4;  // MN-major operands in the tf32 swizzled layout (tf32_mn_off)
  // a tf32 MN-major stage spans whole 32-element MN slices (4 KB each)
  constexpr int B_BYTES = (TF_MN && B_MN && BN < 32) ? 32 * 128 : BN * 128;
  // fp32 storage: fp32-faithful 3xTF32. The producers split every landed stage in place into
  // hi = tf32_rna(x) and lo = x - hi (lo copy LO bytes further on), and the MMA issuer accumulates
  // lo*hi + hi*lo + hi*hi: kind::tf32 alone keeps ~11 mantissa bits (a ~1e-3 step-1 loss error
  // that 24 DSP steps amplify ~100x, tests/test_configs_gpu.py); the split keeps ~21.
  constexpr bool F32_SPLIT = sizeof(T) == 4;
  constexpr uint32_t LO = (uint32_t)STAGES * (A_BYTES + B_BYTES);
  constexpr int AG = IG_BM / EPC;  // MN groups in the A tile (MN-major)
  constexpr int BG = BN / EPC;     // MN groups in the B tile (MN-major)

  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t full_bar[STAGES], empty_bar[STAGES], tfull_bar[NACC], tempty_bar[NACC], wbar;
  __shared__ uint32_t tmem_base_s;
  __shared__ int last_cta_s;
  __shared__ float red[4][BN][3];
  __shared__ float bst[2][2][BN];  // DGRAD BN-backward targets: mean / invstd of this CTA's columns

  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const int lane = tid & 31;
  if (kTrace && a.trace != nullptr && tid == 0) a.trace[192 + 8 * blockIdx.x] = (int64_t)globaltimer_ns();
  const dsp_conv_geom_t g = a.geom;
  // s2: the launch covers 4 output parities of M/4 pixels each (a.M = all dX pixels)
  const bool s2 = I2C && MODE == DSP_IGEMM_DGRAD && tm.s2;
  const int M = s2 ? a.M / 4 : a.M, N = a.N, Kd = a.Kd;
  const T* __restrict__ Asrc = reinterpret_cast<const T*>(a.A);
  const T* __restrict__ Bsrc = reinterpret_cast<const T*>(a.B);

  const int nkb_total = (Kd + KS - 1) / KS;
  const int mt = (M + IG_BM - 1) / IG_BM;
  const int nt = (N + BN - 1) / BN;
  const int kbps = MODE == DSP_IGEMM_WGRAD ? a.kb_per_split : nkb_total;
  const int ns = MODE == DSP_IGEMM_WGRAD ? (nkb_total + kbps - 1) / kbps : 1;
  const int units = mt * nt * ns;
  // FPROP: BatchNorm forward statistics of the output (sum, sum of squares).
  // DGRAD: BatchNorm backward statistics of the layer below (sum g, sum g*xhat_t).
  const bool bnb = MODE == DSP_IGEMM_DGRAD && a.bnb_count > 0;
  const bool want_stats = a.stats != nullptr && (MODE == DSP_IGEMM_FPROP || bnb);
  const int NS = MODE == DSP_IGEMM_FPROP ? 2 : 1 + a.bnb_count;  // statistics per column

  // Work assignment. FPROP/DGRAD: CTA c owns n-tile c % nt (so per-column BN
  // statistics can accumulate in registers) and m-tiles c/nt, c/nt + G/nt, ...
  // (the launcher makes gridDim.x a multiple of nt). WGRAD: round-robin units.
  auto get_unit = [&](int j, int& m0, int& n0, int& z, int& kb0, int& kb1) -> bool {
    if (MODE == DSP_IGEMM_WGRAD) {
      const int u = blockIdx.x + j * gridDim.x;
      if (u >= units) return false;
      m0 = (u % mt) * IG_BM;
      n0 = ((u / mt) % nt) * BN;
      z = u / (mt * nt);
      kb0 = z * kbps;
      kb1 = min(nkb_total, kb0 + kbps);
      return true;
    }
    const int mtile = blockIdx.x / nt + j * (gridDim.x / nt);
    if (mtile >= (s2 ? 4 * mt : mt)) return false;
    n0 = (blockIdx.x % nt) * BN;
    kb0 = 0;
    if (s2) {  // z = output parity (ph, pw) = (z >> 1, z & 1); k-blocks = its taps x K/64
      z = mtile / mt;
      m0 = (mtile - z * mt) * IG_BM;
      int rl[2], sl[2];
      kb1 = s2_taps(g.R, g.pad, z >> 1, rl) * s2_taps(g.S, g.pad, z & 1, sl) * (g.K / KS);
      return true;
    }
    m0 = mtile * IG_BM;
    z = 0;
    kb1 = nkb_total;
    return true;
  };
  (void)units;

  // full[s] arrivals: the TMA thread's arrive.expect_tx (if A uses TMA) plus one
  // cp.async arrival per producer thread (if any operand is still gathered)
  const bool gather = !(tm.on_a && tm.on_b);
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_bar[s], (tm.on_a ? 1 : 0) + (gather ? 128 : 0));
      mbar_init(&empty_bar[s], 1);
    }
    for (int s = 0; s < NACC; ++s) {
      mbar_init(&tfull_bar[s], 1);
      mbar_init(&tempty_bar[s], EPI_T);
    }
    mbar_init(&wbar, 1);
    fence_barrier_init();
  }
  if (warp == IG_MMA_WARP) tmem_alloc(&tmem_base_s, Cfg::TMEM_COLS);
  // programmatic dependent launch: everything above overlapped the predecessor's tail; no
  // global memory is touched before it has completed
  pdl_wait();
  if (want_stats && warp >= IG_EPI_WARP0) {
    for (int c = lane; c < BN; c += 32) red[warp & 3][c][0] = red[warp & 3][c][1] = red[warp & 3][c][2] = 0.f;
    if (bnb && warp == IG_EPI_WARP0) {
      const int n0c = (blockIdx.x % nt) * BN;  // the n-tile this CTA owns
      for (int c = lane; c < BN; c += 32)
        for (int t = 0; t < 2; ++t) {
          const bool ok = t < a.bnb_count && n0c + c < N;
          bst[t][0][c] = ok ? a.bnb[t].stat[n0c + c] : 0.f;
          bst[t][1][c] = ok ? a.bnb[t].stat[N + n0c + c] : 0.f;
        }
      if (a.bnb_mask == nullptr && a.bnb_mask_bits == nullptr)  // one target, mask from y: its scale / shift
                                                                 // in the unused second slot
        for (int c = lane; c < BN; c += 32) {
          const bool ok = n0c + c < N;
          bst[1][0][c] = ok ? a.bnb[0].stat[2 * N + n0c + c] : 0.f;
          bst[1][1][c] = ok ? a.bnb[0].stat[3 * N + n0c + c] : 0.f;
        }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_d = tmem_base_s;
  int64_t* const trace = (kTrace && a.trace != nullptr && blockIdx.x == 0) ? a.trace : nullptr;
#define IG_TRACE(slot, cond)                                   \
  do {                                                          \
    if (trace != nullptr && (cond) && (slot) < 192) trace[(slot)] = clock64(); \
  } while (0)
  IG_TRACE(176, tid == 0);
  // per-CTA global timeline (ns) after CTA 0's detail slots: start, setup done, work done, end
  int64_t* const ctat = (kTrace && a.trace != nullptr) ? a.trace + 192 + 8 * blockIdx.x : nullptr;
  if (ctat != nullptr && tid == 0) ctat[1] = (int64_t)globaltimer_ns();
  const uint32_t sA0 = smem_u32(smem);
  const uint32_t sB0 = sA0 + STAGES * A_BYTES;

  // halo layout: [h_nst stages of S boxes][resident weights]
  const uint32_t h_stage = (uint32_t)(tm.h_box * g.S);
  const uint32_t sW = sA0 + (uint32_t)tm.h_nst * h_stage;
  if (warp < NPW && !I2C && tm.halo) {
    // ============================ halo producer ============================
    if (warp == 0 && lane == 0) {
      tma_prefetch_desc(&tmA);
      tma_prefetch_desc(&tmB);
      const int n0c = (blockIdx.x % nt) * BN;
      mbar_arrive_expect_tx(&wbar, (uint32_t)(tm.h_nwb * BN * 128));
      for (int j = 0; j < tm.h_nwb; ++j) tma_load_2d(sW + j * (BN * 128), &tmB, &wbar, j * KS, n0c);
      int m0, n0, z, kb0, kb1;
      for (int t = 0; get_unit(t, m0, n0, z, kb0, kb1); ++t) {
        const int st = t % tm.h_nst;
        IG_TRACE(2 * t, t < 32);
        if (t >= tm.h_nst) mbar_wait(&empty_bar[st], ((t / tm.h_nst) - 1) & 1);
        IG_TRACE(2 * t + 1, t < 32);
        const int oh = MODE == DSP_IGEMM_FPROP ? g.P : g.H, ow = MODE == DSP_IGEMM_FPROP ? g.Q : g.W;
        const int img = m0 / (oh * ow);
        const int h0 = (m0 - img * oh * ow) / ow;
        mbar_arrive_expect_tx(&full_bar[st], h_stage);
        for (int sx = 0; sx < g.S; ++sx)
          tma_load_4d(sA0 + st * h_stage + sx * tm.h_box, &tmA, &full_bar[st], 0, sx - g.pad, h0 - g.pad, img);
      }
    }
  } else if (warp < NPW) {
    // =============================== producers ===============================
    // (all-TMA launches: only thread 0 produces; the other producer threads go idle)
    if (gather || warp == 0) {
    const int aj = tid & 7;
    const int ag = tid % AG;
    // every runtime divisor of the gathers as a multiply-shift (FastDiv)
    FastDiv fd_pix{tm.fd_d[0], tm.fd_mul[0], tm.fd_shr[0]}, fd_row{tm.fd_d[1], tm.fd_mul[1], tm.fd_shr[1]},
        fd_ch{tm.fd_d[2], tm.fd_mul[2], tm.fd_shr[2]}, fd_s{tm.fd_d[3], tm.fd_mul[3], tm.fd_shr[3]},
        fd_k{tm.fd_d[4], tm.fd_mul[4], tm.fd_shr[4]};
    const int sh = g.stride == 2 ? 1 : 0;  // stride is 1 or 2
    const int img_stride = MODE == DSP_IGEMM_DGRAD ? g.P * g.Q * g.K : g.H * g.W * g.C;
    const int out_hw = (MODE == DSP_IGEMM_DGRAD && !s2) ? g.H * g.W : g.P * g.Q;
    const int out_w = (MODE == DSP_IGEMM_DGRAD && !s2) ? g.W : g.Q;
    if (tm.on_a && tid == 0) {
      tma_prefetch_desc(&tmA);
      if (tm.on_b) tma_prefetch_desc(&tmB);
    }
    int gcount = 0;
    int m0, n0, z, kb0, kb1;
    for (int j = 0; get_unit(j, m0, n0, z, kb0, kb1); ++j) {
      const int t_n0 = m0 / out_hw;              // TMA tile origin: image, output row, column
      const int t_h0 = (m0 - t_n0 * out_hw) / out_w;
      const int t_q0 = m0 - t_n0 * out_hw - t_h0 * out_w;
      // per-tile A-row precompute
      int a_h[8], a_w[8], a_img[8];
      int wg_r = 0, wg_s = 0, wg_c = 0;
      bool wg_ok = false;
      if (tm.on_a) {
        // TMA computes the im2col addresses: nothing to decode per row
      } else if (MODE != DSP_IGEMM_WGRAD) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int m = m0 + (tid >> 3) + 16 * i;
          if (m < M) {
            int rem, x;
            const int img = fd_pix.divmod(m, rem);
            const int y = fd_row.divmod(rem, x);
            if (MODE == DSP_IGEMM_FPROP) {
              a_h[i] = (y << sh) - g.pad;
              a_w[i] = (x << sh) - g.pad;
            } else {
              a_h[i] = y + g.pad;
              a_w[i] = x + g.pad;
            }
            a_img[i] = img * img_stride;
          } else {
            a_h[i] = -(1 << 28);
            a_w[i] = -(1 << 28);
            a_img[i] = 0;
          }
        }
      } else {
        const int m = m0 + ag * EPC;
        if (m < M) {
          int c, ss;
          const int tap = fd_ch.divmod(m, c);
          wg_c = c;
          wg_r = fd_s.divmod(tap, ss);
          wg_s = ss;
          wg_ok = true;
        }
      }
      for (int kb = kb0; kb < kb1; ++kb, ++gcount) {
        const int s = gcount % STAGES;
        IG_TRACE(2 * gcount, tid == 0 && gcount < 32);
        if (gcount >= STAGES) mbar_wait(&empty_bar[s], ((gcount / STAGES) - 1) & 1);
        const uint32_t sA = sA0 + s * A_BYTES;
        const uint32_t sB = sB0 + s * B_BYTES;
        if (kTrace && (a.out_f32 & 2)) {  // ablation (trace builds only): skip operand loads
          if (tm.on_a && tid == 0) mbar_arrive_expect_tx(&full_bar[s], 0);
          if (gather) cp_async_arrive_noinc(&full_bar[s]);
          continue;
        }
        // ---------------- A operand ----------------
        if (I2C && MODE == DSP_IGEMM_WGRAD) {
          // k-block = 64 output pixels from kb*KS on (crossing rows / images); A boxes = one per
          // 64-channel M group (tap, c0) as im2col offsets; B = dY [pixels][K] 2-D boxes
          const int nbox_a = IG_BM / tm.cbox, nbox_b = BN / tm.cbox_b;
          if (warp == 0) {
            if (lane == 0) mbar_arrive_expect_tx(&full_bar[s], (uint32_t)(nbox_a * tm.box_a + nbox_b * tm.box_b));
            __syncwarp();
            if (lane < nbox_a) {
              int rem, kq;
              const int kn = fd_pix.divmod(kb * KS, rem);
              const int kh = fd_row.divmod(rem, kq);
              const int mm = m0 + lane * tm.cbox;
              int c0 = 0, rr = 0, ss2 = 0;
              if (mm < M) {
                const int tap = fd_ch.divmod(mm, c0);
                rr = fd_s.divmod(tap, ss2);
              }
              // rows past R*S*C read channels >= C: zero filled (their D rows are never stored)
              if (tm.a2d)
                tma_load_2d(sA + lane * tm.box_a, &tmA, &full_bar[s], mm < M ? c0 : g.C, kb * KS);
              else
                tma_load_im2col_4d(sA + lane * tm.box_a, &tmA, &full_bar[s], mm < M ? c0 : g.C,
                                   kq * g.stride - tm.i2c_pad, kh * g.stride - tm.i2c_pad, kn, (uint16_t)ss2,
                                   (uint16_t)rr);
            } else if (lane >= 32 - nbox_b) {
              const int jb = lane - (32 - nbox_b);
              tma_load_2d(sB + jb * tm.box_b, &tmB, &full_bar[s], n0 + jb * tm.cbox_b, kb * KS);
            }
          }
        } else if (I2C) {
          // one im2col box per (tap, cbox-channel chunk) of the stage (128 output pixels each),
          // one lane per box, plus the weight box; K beyond Kd reads channel cdim (zero fill)
          // (64-channel boxes: one box per stage, issued by lane 0 alone with no warp handshake --
          // the warp-parallel form measured 30% slower on the ResNet-50 stage-3 3x3)
          // (wide tiles compile only the 64-channel form: the extra producer code measured
          // 20% slower on the ResNet-50 stage-3 3x3 even when never executed)
          const int nbox = BN >= 128 ? 1 : KS / tm.cbox;
          if (s2) {
            if (warp == 0 && lane == 0) {
              // tap t of parity z: dY rows/cols i + dr, j + ds against weight tap (r, s)
              mbar_arrive_expect_tx(&full_bar[s], (uint32_t)(tm.box_a + tm.box_b));
              const int kpb = g.K / KS;
              const int tsub = kb / kpb, kc = (kb - tsub * kpb) * KS;
              int rl[2], sl[2];
              s2_taps(g.R, g.pad, z >> 1, rl);
              const int ns = s2_taps(g.S, g.pad, z & 1, sl);
              const int r = rl[tsub / ns], sx = sl[tsub % ns];
              const int dr = ((z >> 1) + g.pad - r) >> 1, ds = ((z & 1) + g.pad - sx) >> 1;
              tma_load_im2col_4d(sA, &tmA, &full_bar[s], kc, t_q0, t_h0, t_n0, (uint16_t)ds, (uint16_t)dr);
              tma_load_2d(sB, &tmB, &full_bar[s], (r * g.S + sx) * g.K + kc, n0);
            }
          } else if (nbox == 1) {
            if (warp == 0 && lane == 0) {
              mbar_arrive_expect_tx(&full_bar[s], (uint32_t)(tm.box_a + tm.box_b));
              const int k0 = kb * KS;
              int c0, ss2;
              const int tap = fd_ch.divmod(k0, c0);
              const int rr = fd_s.divmod(tap, ss2);
              const int st2 = MODE == DSP_IGEMM_FPROP ? g.stride : 1;
              const int ow = MODE == DSP_IGEMM_FPROP ? ss2 : g.S - 1 - ss2;
              const int oh = MODE == DSP_IGEMM_FPROP ? rr : g.R - 1 - rr;
              if (tm.a2d)
                tma_load_2d(sA, &tmA, &full_bar[s], c0, m0);
              else
                tma_load_im2col_4d(sA, &tmA, &full_bar[s], c0, t_q0 * st2 - tm.i2c_pad, t_h0 * st2 - tm.i2c_pad,
                                   t_n0, (uint16_t)ow, (uint16_t)oh);
              tma_load_2d(sB, &tmB, &full_bar[s], k0, n0);
            }
          } else if (warp == 0) {
            if (lane == 0) mbar_arrive_expect_tx(&full_bar[s], (uint32_t)(nbox * tm.box_a + tm.box_b));
            __syncwarp();
            if (lane < nbox) {
              const int k0 = kb * KS + lane * tm.cbox;
              const int cdim = MODE == DSP_IGEMM_FPROP ? g.C : g.K;
              int c0 = cdim, ss2 = 0, rr = 0;
              if (k0 < Kd) {
                const int tap = fd_ch.divmod(k0, c0);
                rr = fd_s.divmod(tap, ss2);
              }
              const int st2 = MODE == DSP_IGEMM_FPROP ? g.stride : 1;
              // DGRAD = conv of dY with the flipped kernel: weight tap (r, s) meets offset (R-1-r, S-1-s)
              const int ow = MODE == DSP_IGEMM_FPROP ? ss2 : g.S - 1 - ss2;
              const int oh = MODE == DSP_IGEMM_FPROP ? rr : g.R - 1 - rr;
              if (tm.a2d)
                tma_load_2d(sA + lane * tm.box_a, &tmA, &full_bar[s], c0, m0);
              else
                tma_load_im2col_4d(sA + lane * tm.box_a, &tmA, &full_bar[s], c0, t_q0 * st2 - tm.i2c_pad,
                                   t_h0 * st2 - tm.i2c_pad, t_n0, (uint16_t)ow, (uint16_t)oh);
            }
            if (lane == 31) tma_load_2d(sB, &tmB, &full_bar[s], kb * KS, n0);
          }
        } else if (!I2C && tm.on_a && MODE == DSP_IGEMM_WGRAD) {
          // WGRAD: k-block = 64 output pixels; A box j = tap-shifted X pixels x cbox
          // channels of MN range [m0 + j*cbox, +cbox); B box j = dY pixels x cbox_b
          const int nbox_a = IG_BM / tm.cbox, nbox_b = BN / tm.cbox_b;
          if (warp == 0) {
            if (lane == 0) mbar_arrive_expect_tx(&full_bar[s], (uint32_t)(nbox_a * tm.box_a + nbox_b * tm.box_b));
            __syncwarp();
            int rem;
            const int kn = fd_pix.divmod(kb * KS, rem);  // k-block origin: image, output row
            const int kh = fd_row.div(rem);
            if (lane < nbox_a) {
              const int mm = m0 + lane * tm.cbox;
              int c0 = 0, rr = 0, ss2 = 0;
              const bool ok = mm < M;
              if (ok) {
                const int tap = fd_ch.divmod(mm, c0);
                rr = fd_s.divmod(tap, ss2);
              }
              const int cw = ok ? ss2 - g.pad : -(1 << 20);  // rows past R*S*C: zero box
              tma_load_4d(sA + lane * tm.box_a, &tmA, &full_bar[s], c0, cw, kh * g.stride + rr - g.pad, kn);
            } else if (lane >= 32 - nbox_b) {
              const int jb = lane - (32 - nbox_b);
              tma_load_4d(sB + jb * tm.box_b, &tmB, &full_bar[s], n0 + jb * tm.cbox_b, 0, kh, kn);
            }
          }
        } else if (!I2C && tm.on_a) {
          // warp 0 issues the stage's TMA boxes in parallel, one per lane
          const int nbox = KS / tm.cbox;
          if (warp == 0) {
            if (lane == 0)
              mbar_arrive_expect_tx(&full_bar[s], (uint32_t)(nbox * tm.box_a + (tm.on_b ? tm.box_b : 0)));
            __syncwarp();
            if (lane < nbox) {
              const int jb = lane;
              const int k0 = kb * KS + jb * tm.cbox;
              int c0 = 0, rr = 0, ss2 = 0;
              if (k0 < Kd) {
                const int tap = fd_ch.divmod(k0, c0);
                rr = fd_s.divmod(tap, ss2);
              }
              int cw, ch;
              if (MODE == DSP_IGEMM_FPROP) {
                cw = ss2 - g.pad;
                ch = t_h0 * g.stride + rr - g.pad;
              } else {
                cw = g.pad - ss2;
                ch = t_h0 + g.pad - rr;
              }
              if (k0 >= Kd) cw = -(1 << 20);  // no such tap: a fully out-of-bounds (zero) box
              tma_load_4d(sA + jb * tm.box_a, &tmA, &full_bar[s], c0, cw, ch, t_n0);
            }
            if (tm.on_b && lane == 31) tma_load_2d(sB, &tmB, &full_bar[s], kb * KS, n0);
          }
        } else if (!I2C && MODE != DSP_IGEMM_WGRAD) {
          const int k0 = kb * KS + aj * EPC;
          const bool kok = k0 < Kd;
          int c0 = 0, s2 = 0, r = 0;
          if (kok) {
            const int tap = fd_ch.divmod(k0, c0);
            r = fd_s.divmod(tap, s2);
          }
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int row = (tid >> 3) + 16 * i;
            int off = 0;
            bool ok = kok;
            if (MODE == DSP_IGEMM_FPROP) {
              const int ih = a_h[i] + r, iw = a_w[i] + s2;
              ok = ok && (unsigned)ih < (unsigned)g.H && (unsigned)iw < (unsigned)g.W;
              off = a_img[i] + (ih * g.W + iw) * g.C + c0;
            } else {
              int hh = a_h[i] - r, ww = a_w[i] - s2;
              if (sh) {
                ok = ok && hh >= 0 && ww >= 0 && ((hh | ww) & 1) == 0;
                hh >>= 1;
                ww >>= 1;
              }
              ok = ok && (unsigned)hh < (unsigned)g.P && (unsigned)ww < (unsigned)g.Q;
              off = a_img[i] + (hh * g.Q + ww) * g.K + c0;
            }
            cp_async_16(sA + aj * (IG_BM * 16) + row * 16, ok ? Asrc + off : Asrc, ok ? 16u : 0u);
          }
        } else if (!I2C) {
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int kr = tid / AG + (128 / AG) * i;
            const int p = kb * KS + kr;
            int off = 0;
            bool ok = wg_ok && p < Kd;
            if (ok) {
              int rem, ow;
              const int img = fd_pix.divmod(p, rem);
              const int oh = fd_row.divmod(rem, ow);
              const int ih = (oh << sh) - g.pad + wg_r;
              const int iw = (ow << sh) - g.pad + wg_s;
              ok = (unsigned)ih < (unsigned)g.H && (unsigned)iw < (unsigned)g.W;
              off = ((img * g.H + ih) * g.W + iw) * g.C + wg_c;
            }
            const uint32_t soff = TF_MN ? tf32_mn_off(ag, kr) : (uint32_t)((kr >> 3) * (AG * 128) + ag * 128 + (kr & 7) * 16);
            cp_async_16(sA + soff, ok ? Asrc + off : Asrc, ok ? 16u : 0u);
          }
        }
        // ---------------- B operand ----------------
        constexpr int BCH = 8 * BN;
        if (I2C || tm.on_b) {
          // loaded by the TMA thread above
        } else if (MODE == DSP_IGEMM_FPROP) {
#pragma unroll
          for (int c = tid; c < BCH; c += 128) {
            const int n = c >> 3, jj = c & 7;
            const int k0 = kb * KS + jj * EPC;
            const bool ok = (n0 + n) < N && k0 < Kd;
            cp_async_16(sB + jj * (BN * 16) + n * 16, ok ? Bsrc + (n0 + n) * Kd + k0 : Bsrc, ok ? 16u : 0u);
          }
        } else {
#pragma unroll
          for (int c = tid; c < BCH; c += 128) {
            const int gg = c % BG, kr = c / BG;
            const int k = kb * KS + kr;
            const int n = n0 + gg * EPC;
            const bool ok = n < N && k < Kd;
            int off = 0;
            if (MODE == DSP_IGEMM_DGRAD) {
              int co;
              const int tap = fd_k.divmod(k, co);
              off = (co * g.R * g.S + tap) * g.C + n;
            } else {
              off = k * g.K + n;
            }
            const uint32_t soff = TF_MN ? tf32_mn_off(gg, kr) : (uint32_t)((kr >> 3) * (BG * 128) + gg * 128 + (kr & 7) * 16);
            cp_async_16(sB + soff, ok ? Bsrc + off : Bsrc, ok ? 16u : 0u);
          }
        }
        if constexpr (F32_SPLIT) {
          // every producer's copies of this stage have landed -> split the stage into hi / lo
          cp_async_commit();
          cp_async_wait<0>();
          asm volatile("bar.sync 2, 128;" ::: "memory");
          for (uint32_t o = tid * 16; o < (uint32_t)A_BYTES; o += 128 * 16) tf32_split16(sA + o, sA + LO + o);
          for (uint32_t o = tid * 16; o < (uint32_t)B_BYTES; o += 128 * 16) tf32_split16(sB + o, sB + LO + o);
          fence_proxy_async_smem();
          mbar_arrive(&full_bar[s]);
        } else if (gather) {
          // arrive on full[s] when this thread's copies land; never block the producer
          cp_async_arrive_noinc(&full_bar[s]);
        }
        IG_TRACE(2 * gcount + 1, tid == 0 && gcount < 32);
      }
    }
    cp_async_wait<0>();
    }
  } else if (warp == IG_MMA_WARP && !I2C && tm.halo) {
    // ============================ halo MMA issuer ============================
    if (lane == 0) {
      const uint32_t idesc = umma_idesc(MmaTraits<T>::FMT, 0u, 0u, IG_BM, BN);
      const uint64_t a_tpl = umma_sdesc(0, 16, 8 * tm.h_rowb, tm.h_swz);
      const uint64_t b_tpl = umma_sdesc(0, 16, 1024, 2);  // [BN][128 B] SWIZZLE_128B boxes
      // FPROP: tap (r, s) = box s shifted down r rows; DGRAD (flipped taps): box S-1-s, R-1-r
      const int C = MODE == DSP_IGEMM_FPROP ? g.C : g.K;  // channels of the A rows
      const int ow = MODE == DSP_IGEMM_FPROP ? g.Q : g.W;
      const uint32_t row_step = (uint32_t)(ow * tm.h_rowb);
      const bool unrolled = g.R == 3 && g.S == 3;
      mbar_wait(&wbar, 0);
      int m0, n0, z, kb0, kb1;
      for (int i = 0; get_unit(i, m0, n0, z, kb0, kb1); ++i) {
        const int acc = i % NACC;
        if (i >= NACC) mbar_wait(&tempty_bar[acc], ((i / NACC) - 1) & 1);
        const int st = i % tm.h_nst;
        IG_TRACE(128 + i, i < 16);
        mbar_wait(&full_bar[st], (i / tm.h_nst) & 1);
        IG_TRACE(64 + 2 * i, i < 32);
        tc_fence_after();
        const uint32_t td = tmem_d + acc * BN;
        const uint32_t base = sA0 + st * h_stage;
        // per-tile MMA sequence: 3x3 taps fully unrolled per channel count (compile-time tap and
        // K offsets; only the stage base and two runtime strides remain), generic loop otherwise
        auto issue = [&](auto cch) {
          constexpr int CC = decltype(cch)::value;
#pragma unroll
          for (int t = 0; t < 9; ++t) {
            const int r = t / 3, sx = t % 3;
            const int ro = MODE == DSP_IGEMM_FPROP ? r : 2 - r;
            const int bx = MODE == DSP_IGEMM_FPROP ? sx : 2 - sx;
            const uint32_t arow = base + bx * tm.h_box + ro * row_step;
#pragma unroll
            for (int kc = 0; kc < CC; kc += MmaTraits<T>::MMA_K) {
              const int k = t * CC + kc;
              const uint32_t aa = arow + kc * 2;
              const uint32_t ba = sW + (k / KS) * (BN * 128) + (k % KS) * 2;
              MmaTraits<T>::mma(td, a_tpl | (uint64_t)((aa >> 4) & 0x3FFF), b_tpl | (uint64_t)((ba >> 4) & 0x3FFF),
                                idesc, k > 0 ? 1u : 0u);
            }
          }
        };
        if (unrolled && C == 16) {
          issue(std::integral_constant<int, 16>{});
        } else if (unrolled && C == 32) {
          issue(std::integral_constant<int, 32>{});
        } else if (unrolled && C == 64) {
          issue(std::integral_constant<int, 64>{});
        } else {
          uint32_t k = 0;
          for (int r = 0; r < g.R; ++r) {
            const int ro = MODE == DSP_IGEMM_FPROP ? r : g.R - 1 - r;
            for (int sx = 0; sx < g.S; ++sx) {
              const int bx = MODE == DSP_IGEMM_FPROP ? sx : g.S - 1 - sx;
              const uint32_t arow = base + bx * tm.h_box + ro * row_step;
              for (int kc = 0; kc < C; kc += MmaTraits<T>::MMA_K, k += MmaTraits<T>::MMA_K) {
                const uint32_t aa = arow + kc * 2;
                const uint32_t ba = sW + (k / KS) * (BN * 128) + (k % KS) * 2;
                MmaTraits<T>::mma(td, a_tpl | (uint64_t)((aa >> 4) & 0x3FFF),
                                  b_tpl | (uint64_t)((ba >> 4) & 0x3FFF), idesc, k > 0 ? 1u : 0u);
              }
            }
          }
        }
        umma_commit(&empty_bar[st]);
        umma_commit(&tfull_bar[acc]);
        IG_TRACE(65 + 2 * i, i < 32);
      }
    }
    __syncwarp();
  } else if (warp == IG_MMA_WARP) {
    // =============================== MMA issuer ===============================
    if (lane == 0) {
      // im2col DGRAD reads the transposed weights B_t [C][R][S][K]: K-major like FPROP
      const bool b_mn = B_MN && !(I2C && MODE == DSP_IGEMM_DGRAD);
      const uint32_t idesc = umma_idesc(MmaTraits<T>::FMT, A_MN ? 1u : 0u, b_mn ? 1u : 0u, IG_BM, BN);
      constexpr int NKK = KS / MmaTraits<T>::MMA_K;
      // descriptor templates (start address 0) and per-MMA byte offsets, hoisted
      // out of the loop: the issuing thread only adds the stage base.
      uint64_t a_tpl, b_tpl;
      uint32_t a_off[NKK], b_off[NKK];
      // MN-major TMA tiles (WGRAD): rows = 64 pixels of rowbytes = cbox*2; an MMA
      // reads 16 pixel rows; MN groups (boxes) are box bytes apart.
      auto mn_tpl = [](int cbox, int box, int swz) -> uint64_t {
        return swz == 0 ? umma_sdesc(0, 128, box, 0)                 // NONE: LBO = K-group, SBO = MN-group
                        : umma_sdesc(0, box, 8 * cbox * 2, swz);     // swizzled: LBO = MN-group, SBO = 8 rows
      };
      if (tm.on_a && MODE == DSP_IGEMM_WGRAD) {
        a_tpl = mn_tpl(tm.cbox, tm.box_a, tm.swz_a);
        b_tpl = mn_tpl(tm.cbox_b, tm.box_b, tm.swz_b);
#pragma unroll
        for (int kk = 0; kk < NKK; ++kk) {
          a_off[kk] = kk * 16 * tm.cbox * 2;
          b_off[kk] = kk * 16 * tm.cbox_b * 2;
        }
      } else if (tm.on_a) {
        if (tm.cbox == 8) {  // two 16-byte-row boxes per MMA, SWIZZLE_NONE
          a_tpl = umma_sdesc(0, tm.box_a, 128, 0);
        } else {
          a_tpl = umma_sdesc(0, 16, 8 * tm.cbox * 2, tm.swz_a);
        }
#pragma unroll
        for (int kk = 0; kk < NKK; ++kk) {
          const int e = kk * MmaTraits<T>::MMA_K;  // MMA kk reads K elements [e, e+16) of the stage
          a_off[kk] = tm.cbox == 8 ? (e / 8) * tm.box_a : (e / tm.cbox) * tm.box_a + (e % tm.cbox) * 2;
        }
      } else if (TF_MN && A_MN) {
        a_tpl = umma_sdesc(0, TF32_MN_LBO, TF32_MN_SBO, 1);  // SWIZZLE_128B_BASE32B
#pragma unroll
        for (int kk = 0; kk < NKK; ++kk) a_off[kk] = kk * 2 * TF32_MN_SBO;  // 8 K rows = 2 atoms per MMA
      } else {
        a_tpl = umma_sdesc(0, A_MN ? (IG_BM / EPC) * 128 : IG_BM * 16, 128);
#pragma unroll
        for (int kk = 0; kk < NKK; ++kk) a_off[kk] = kk * 32 * IG_BM;
      }
      if (MODE == DSP_IGEMM_WGRAD && tm.on_a) {
        // set above
      } else if (tm.on_b) {
        b_tpl = umma_sdesc(0, 16, 1024, 2);  // [BN][128 B] SWIZZLE_128B
#pragma unroll
        for (int kk = 0; kk < NKK; ++kk) b_off[kk] = kk * 32;
      } else if (TF_MN && B_MN) {
        b_tpl = umma_sdesc(0, TF32_MN_LBO, TF32_MN_SBO, 1);
#pragma unroll
        for (int kk = 0; kk < NKK; ++kk) b_off[kk] = kk * 2 * TF32_MN_SBO;
      } else {
        b_tpl = umma_sdesc(0, B_MN ? (BN / EPC) * 128 : BN * 16, 128);
#pragma unroll
        for (int kk = 0; kk < NKK; ++kk) b_off[kk] = kk * 32 * BN;
      }
      const bool skip_mma = kTrace && (a.out_f32 & 4) != 0;  // ablation (trace builds only)
      int gcount = 0, i = 0;
      int m0, n0, z, kb0, kb1;
      for (; get_unit(i, m0, n0, z, kb0, kb1); ++i) {
        const int acc = i % NACC;
        if (i >= NACC) mbar_wait(&tempty_bar[acc], ((i / NACC) - 1) & 1);
        IG_TRACE(128 + i, i < 16);
        tc_fence_after();
        const uint32_t td = tmem_d + acc * BN;
        for (int kb = kb0; kb < kb1; ++kb, ++gcount) {
          const int s = gcount % STAGES;
          mbar_wait(&full_bar[s], (gcount / STAGES) & 1);
          IG_TRACE(64 + 2 * gcount, gcount < 32);
          tc_fence_after();
          const uint32_t sa = sA0 + s * A_BYTES;
          const uint32_t sb = sB0 + s * B_BYTES;
          if (!skip_mma) {
#pragma unroll
            for (int kk = 0; kk < NKK; ++kk) {
              const uint64_t ad = a_tpl | (uint64_t)(((sa + a_off[kk]) >> 4) & 0x3FFF);
              const uint64_t bd = b_tpl | (uint64_t)(((sb + b_off[kk]) >> 4) & 0x3FFF);
              if constexpr (F32_SPLIT) {
                const uint64_t adl = a_tpl | (uint64_t)(((sa + LO + a_off[kk]) >> 4) & 0x3FFF);
                const uint64_t bdl = b_tpl | (uint64_t)(((sb + LO + b_off[kk]) >> 4) & 0x3FFF);
                MmaTraits<T>::mma(td, adl, bd, idesc, (kb > kb0 || kk > 0) ? 1u : 0u);
                MmaTraits<T>::mma(td, ad, bdl, idesc, 1u);
                MmaTraits<T>::mma(td, ad, bd, idesc, 1u);
              } else {
                MmaTraits<T>::mma(td, ad, bd, idesc, (kb > kb0 || kk > 0) ? 1u : 0u);
              }
            }
          }
          umma_commit(&empty_bar[s]);
          IG_TRACE(65 + 2 * gcount, gcount < 32);
        }
        umma_commit(&tfull_bar[acc]);
      }
    }
    __syncwarp();
  } else {
    // =============================== epilogue ===============================
    const int q = warp & 3;  // TMEM lane quadrant this warp may access
    const int row = q * 32 + lane;
    const int et = tid - IG_EPI_WARP0 * 32;  // 0..EPI_T-1
    const int half = (warp - IG_EPI_WARP0) >> 2;  // column half (8 epilogue warps)
    const bool tma_out = Cfg::OUT_BYTES > 0 && MODE != DSP_IGEMM_WGRAD && sizeof(T) == 2 && tm.on_d;
    const uint32_t sOut = sA0 + Cfg::RING;  // 1024-aligned staging tile, boxes of 128 x d_cols
    // per-warp slab staging (wide tiles): slab = 32 rows x 32 B, two per warp
    const bool dw = Cfg::DW_BYTES > 0 && NEPI == 8 && MODE != DSP_IGEMM_WGRAD && sizeof(T) == 2 && tm.d_warp &&
                    !(a.out_f32 & 1);
    const uint32_t sDW = sA0 + Cfg::RING + Cfg::OUT_BYTES + (uint32_t)(warp - IG_EPI_WARP0) * 2048;
    int dwc = 0;  // slabs this warp has staged
    // FPROP fast path with <= 2 column chunks per warp: each lane's BN partial sums (8 columns x
    // its rows) stay in registers across all of the CTA's tiles (the CTA owns one n-tile, so a
    // lane's columns never change) and are reduced across lanes once, after the last tile
    constexpr int FCH = (MODE == DSP_IGEMM_FPROP && sizeof(T) == 2) ? BN / 16 / (NEPI / 4) / 2 : 0;
    constexpr bool FACC = FCH >= 1 && FCH <= 2;
    float fa1[FACC ? FCH : 1][8], fa2[FACC ? FCH : 1][8];
#pragma unroll
    for (int c = 0; c < (FACC ? FCH : 1); ++c)
#pragma unroll
      for (int j = 0; j < 8; ++j) fa1[c][j] = fa2[c][j] = 0.f;
    int i = 0;
    int m0, n0, z, kb0, kb1;
    for (; get_unit(i, m0, n0, z, kb0, kb1); ++i) {
      const int acc = i % NACC;
      mbar_wait(&tfull_bar[acc], (i / NACC) & 1);
      IG_TRACE(144 + 2 * i, et == 0 && i < 16);
      tc_fence_after();
      if (tma_out && i > 0) {  // the previous tile's store must have read the staging tile
        if (et == 0) bulk_wait_read0();
        epi_barrier<EPI_T>();
      }
      const int m = m0 + row;
      const bool mok = m < M;
      // dX row of tile row mm (s2: parity z's pixel (n, i, j) -> (n, 2i + ph, 2j + pw))
      auto rowmap = [&](int mm) -> int {
        if (!s2) return mm;
        const int PQ = g.P * g.Q;
        const int n = mm / PQ, rem = mm - n * PQ, ii = rem / g.Q, jj = rem - ii * g.Q;
        return (n * g.H + 2 * ii + (z >> 1)) * g.W + 2 * jj + (z & 1);
      };
      const int mr = rowmap(m);
      const bool zacc = s2 && kb1 == 0;  // a parity no tap reaches (1x1 stride 2): D = residual
      const uint32_t tl = tmem_d + acc * BN + ((uint32_t)(q * 32) << 16);
      // each warp: CPW 16-column chunks of its half; wide tiles load 32 TMEM columns per wait
      constexpr int CPW = BN / 16 / (NEPI / 4);
      constexpr int LDW = (BN >= 128 && CPW % 2 == 0) ? 2 : 1;
      // Fast path: a full bf16 FPROP tile of the wide (slab) epilogue without bias / residual (the
      // ResNet-50 convs): each 32-column chunk is packed with cvt.rn.bf16x2, staged as one 32-row x
      // 64-byte slab per warp (16-byte chunks XOR-swizzled by row pair: conflict-free), stored four
      // lanes per row, and its BN statistics come from the staged bf16 pairs -- ~150 instead of ~565
      // warp instructions per 32 x 32 chunk (ncu source counters, profiles/r02_epilogue.md).
      bool fast = false, fastd = false;
      if constexpr (MODE == DSP_IGEMM_FPROP && CPW % 2 == 0 && sizeof(T) == 2) {
        fast = dw && !s2 && a.bias == nullptr && a.residual == nullptr && m0 + IG_BM <= M &&
               n0 + BN <= (a.n_valid > 0 ? a.n_valid : N);
      }
      if constexpr (MODE == DSP_IGEMM_DGRAD && CPW % 2 == 0 && sizeof(T) == 2) {
        fastd = dw && !s2 && !zacc && a.bias == nullptr && m0 + IG_BM <= M && n0 + BN <= (a.n_valid > 0 ? a.n_valid : N) &&
                !(want_stats && a.bnb_mask != nullptr && a.bnb_mask_bits == nullptr);
      }
      if (fastd) {
        // DGRAD fast path (same slab scheme): optional residual add (lane = row, its four 16-byte
        // loads issued before the accumulator wait) and the fused BatchNorm-backward statistics
        // of the BN(s) below, g = stored dX * (mask > 0): lane = (column pair, row parity) reads
        // dX from the slab and mask / y straight from global -- two rows of 64 contiguous bytes per
        // warp load -- with all 16 rows' loads in flight before they are used.
        const int rbase = m0 + q * 32;
        const int nbt = a.bnb_count;
#pragma unroll 1
        for (int c2 = 0; c2 < CPW; c2 += 2) {
          const int col0 = (half * CPW + c2) * 16;
          // residual: copied coalesced (cp.async, no registers) as (row lane / 4 + 8 it, 16-byte chunk
          // lane % 4) -- 8 rows of 64 contiguous bytes per warp request -- into the slab, then read
          // back as lane = row (a lane-per-row global load touched 32 lines per instruction: the L1
          // was the bottleneck, 87% busy, and register-held prefetches spilled;
          // profiles/r02_dgrad_epilogue.md)
          // the accumulator chunk's TMEM load is issued first and waited for after the residual /
          // mask requests are out, so its latency overlaps theirs (16% of this epilogue's stall
          // samples waited on tcgen05.wait::ld right behind the load)
          uint32_t tr[32];
          tmem_ld32_issue(tl + col0, tr);
          if (tm.d_tma) {  // the previous chunk's TMA store has read the slab
            if (lane == 0) bulk_wait_read0();
            __syncwarp();
          }
          if (a.residual != nullptr) {
#pragma unroll
            for (int it = 0; it < 4; ++it) {
              const int r = (lane >> 2) + 8 * it, k = lane & 3;
              cp_async_16_cg(sDW + r * 64 + ((k ^ ((r >> 1) & 3)) << 4),
                             reinterpret_cast<const T*>(a.residual) + (size_t)(rbase + r) * a.ldd + n0 + col0 + k * 8);
            }
            cp_async_commit();
          }
          // mask bits with 32-aligned rows: lane l loads the chunk's 32-bit mask word of row l (one
          // coalesced load, issued here so it lands under the TMEM load / staging) and each row's
          // word is shuffled to the lanes that need it -- instead of 16 one-byte loads per lane (30%
          // of this epilogue's stall samples, profiles/r02_dgrad_epilogue.md)
          const bool mword = want_stats && a.bnb_mask_bits != nullptr && (a.ldd & 31) == 0;
          const uint32_t mw = mword ? __ldg(reinterpret_cast<const uint32_t*>(a.bnb_mask_bits) +
                                            (((size_t)(rbase + lane) * a.ldd + n0 + col0) >> 5))
                                    : 0u;
          // y (and mask-byte) row chunks of the statistics, requested before the accumulator wait too
          const int k4 = lane & 3;
          const bool mbits = a.bnb_mask_bits != nullptr;  // else the mask is recomputed from y (fastd)
          uint4 yr[4];
          uint32_t mb8[4];
          auto load_y = [&](const void* y) {
#pragma unroll
            for (int it = 0; it < 4; ++it) {
              const size_t o = (size_t)(rbase + (lane >> 2) + 8 * it) * a.ldd + n0 + col0 + k4 * 8;
              yr[it] = __ldg(reinterpret_cast<const uint4*>(reinterpret_cast<const T*>(y) + o));
            }
          };
          if (want_stats) {
            load_y(a.bnb[0].y);
            if (mbits && !mword) {
#pragma unroll
              for (int it = 0; it < 4; ++it)
                mb8[it] = __ldg(a.bnb_mask_bits +
                                (((size_t)(rbase + (lane >> 2) + 8 * it) * a.ldd + n0 + col0 + k4 * 8) >> 3));
            }
          }
          tmem_ld_wait(tr);
          float vb[32];
#pragma unroll
          for (int e = 0; e < 32; ++e) vb[e] = __uint_as_float(tr[e]);
          if (a.residual != nullptr) {
            cp_async_wait<0>();
            __syncwarp();
          }
          if (a.residual != nullptr) {  // row `lane` of the staged residual, one 16-byte chunk at a time
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              uint4 rk;
              asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                           : "=r"(rk.x), "=r"(rk.y), "=r"(rk.z), "=r"(rk.w)
                           : "r"(sDW + lane * 64 + ((k ^ ((lane >> 1) & 3)) << 4))
                           : "memory");
              const uint32_t w4[4] = {rk.x, rk.y, rk.z, rk.w};
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                vb[8 * k + 2 * j] += __uint_as_float(w4[j] << 16);
                vb[8 * k + 2 * j + 1] += __uint_as_float(w4[j] & 0xffff0000u);
              }
            }
            __syncwarp();  // every lane has its residual row before the slab takes the output
          }
          uint32_t pk[16];
#pragma unroll
          for (int j = 0; j < 16; ++j)
            asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(pk[j]) : "f"(vb[2 * j + 1]), "f"(vb[2 * j]));
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const uint32_t ad = sDW + lane * 64 + ((k ^ ((lane >> 1) & 3)) << 4);
            asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(ad), "r"(pk[4 * k]), "r"(pk[4 * k + 1]),
                         "r"(pk[4 * k + 2]), "r"(pk[4 * k + 3])
                         : "memory");
          }
          if (tm.d_tma) fence_proxy_async_smem();
          __syncwarp();
          if (tm.d_tma && lane == 0) {
            tma_store_2d(&tmD, sDW, n0 + col0, rbase);
            bulk_commit();
          }
          // lane = (row r = lane / 4 + 8 it, 16-byte chunk k4): the slab read that feeds the store
          // also feeds the statistics, with y (and mask) read as the same 16-byte row chunks --
          // coalesced 64-byte row segments, 4 (8 for two targets) loads per lane per chunk, all in
          // flight before the slab reads -- and the 8 lanes of a chunk reduced by shuffles in fixed
          // order (the 2-column-per-lane form issued 4-byte loads in two latency-bound batches)
          // this lane's slab chunk of row r (the stored dX; re-read for the statistics rather than
          // held in registers across the y loads' latency)
          auto slab = [&](int it) {
            const int r = (lane >> 2) + 8 * it;
            uint4 v;
            asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                         : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                         : "r"(sDW + r * 64 + ((k4 ^ ((r >> 1) & 3)) << 4)));
            return v;
          };
          if (!tm.d_tma) {
#pragma unroll
            for (int it = 0; it < 4; ++it) {
              const int r = (lane >> 2) + 8 * it;
              *reinterpret_cast<uint4*>(reinterpret_cast<T*>(a.D) + (size_t)(rbase + r) * a.ldd + n0 + col0 + k4 * 8) =
                  slab(it);
            }
          }
          if (want_stats) {
            const int cl = col0 + k4 * 8;  // tile columns cl .. cl + 7
            if (mword) {
#pragma unroll
              for (int it = 0; it < 4; ++it) mb8[it] = __shfl_sync(0xffffffffu, mw, (lane >> 2) + 8 * it) >> (8 * k4);
            }
            auto bf = [](uint32_t w, int j) { return __uint_as_float((j & 1) ? (w & 0xffff0000u) : (w << 16)); };
            // g = dX where the mask is on: the unit output's bits, or relu(y*scale + shift) > 0 (y of
            // target 0, whose scale / shift sit in bst[1] then); gate bits per (row, column)
            uint32_t on[4];
#pragma unroll
            for (int it = 0; it < 4; ++it) {
              if (mbits) {
                on[it] = mb8[it] & 0xffu;
              } else {
                const uint32_t yw[4] = {yr[it].x, yr[it].y, yr[it].z, yr[it].w};
                uint32_t b8 = 0u;
#pragma unroll
                for (int jp = 0; jp < 4; ++jp) {
                  const float2 z = __ffma2_rn(bf2f2(yw[jp]), make_float2(bst[1][0][cl + 2 * jp], bst[1][0][cl + 2 * jp + 1]),
                                              make_float2(bst[1][1][cl + 2 * jp], bst[1][1][cl + 2 * jp + 1]));
                  b8 |= ((z.x > 0.f ? 1u : 0u) | (z.y > 0.f ? 2u : 0u)) << (2 * jp);
                }
                on[it] = b8;
              }
            }
            // target t: per column, sum g and sum g * xhat_t over this lane's 4 rows, then over the 8
            // lanes of the chunk (fixed shuffle order); target 1's y row replaces target 0's in the
            // same registers as soon as that row is summed
            for (int t = 0; t < nbt; ++t) {
              float s1[8], s2[8];
#pragma unroll
              for (int j = 0; j < 8; ++j) s1[j] = s2[j] = 0.f;
#pragma unroll
              for (int it = 0; it < 4; ++it) {
                const uint4 gv = slab(it);
                const uint32_t gw[4] = {gv.x, gv.y, gv.z, gv.w};
                const uint32_t yw[4] = {yr[it].x, yr[it].y, yr[it].z, yr[it].w};
#pragma unroll
                for (int jp = 0; jp < 4; ++jp) {  // packed FP32x2: columns 2jp, 2jp + 1
                  const float2 gv2 = bf2f2(gw[jp]);
                  const float2 g = make_float2(((on[it] >> (2 * jp)) & 1u) ? gv2.x : 0.f,
                                               ((on[it] >> (2 * jp + 1)) & 1u) ? gv2.y : 0.f);
                  const float2 xh = __fmul2_rn(
                      __fadd2_rn(bf2f2(yw[jp]), make_float2(-bst[t][0][cl + 2 * jp], -bst[t][0][cl + 2 * jp + 1])),
                      make_float2(bst[t][1][cl + 2 * jp], bst[t][1][cl + 2 * jp + 1]));
                  const float2 a1 = __fadd2_rn(make_float2(s1[2 * jp], s1[2 * jp + 1]), g);
                  const float2 a2 = __ffma2_rn(g, xh, make_float2(s2[2 * jp], s2[2 * jp + 1]));
                  s1[2 * jp] = a1.x;
                  s1[2 * jp + 1] = a1.y;
                  s2[2 * jp] = a2.x;
                  s2[2 * jp + 1] = a2.y;
                }
                if (t + 1 < nbt) {
                  const size_t o = (size_t)(rbase + (lane >> 2) + 8 * it) * a.ldd + n0 + col0 + k4 * 8;
                  yr[it] = __ldg(reinterpret_cast<const uint4*>(reinterpret_cast<const T*>(a.bnb[1].y) + o));
                }
              }
              // 8-lane reduce-scatter: lane (k4, cg) ends with column cl + cg's sums; every lane
              // updates the CTA partials at once
              const int cg = lane >> 2;
              float v[2];
              rs8_pair(s1, s2, lane, t == 0, v[0], v[1]);
              if (t == 0) red[q][cl + cg][0] += v[0];
              red[q][cl + cg][1 + t] += v[1];
            }
          }
          __syncwarp();
        }
      } else if (fast) {
        const int rbase = m0 + q * 32;
#pragma unroll
        for (int c2 = 0; c2 < CPW; c2 += 2) {
          const int col0 = (half * CPW + c2) * 16;  // this chunk: tile columns [col0, col0 + 32)
          float vb[32];
          tmem_ld32(tl + col0, vb);
          uint32_t pk[16];
#pragma unroll
          for (int j = 0; j < 16; ++j)
            asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(pk[j]) : "f"(vb[2 * j + 1]), "f"(vb[2 * j]));
          // row `lane`: 4 x 16-byte chunks, chunk k at position k ^ ((lane >> 1) & 3) (= the TMA
          // SWIZZLE_64B layout of a 32-row x 64-byte box)
          if (tm.d_tma) {  // the previous chunk's TMA store has read the slab
            if (lane == 0) bulk_wait_read0();
            __syncwarp();
          }
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const uint32_t ad = sDW + lane * 64 + ((k ^ ((lane >> 1) & 3)) << 4);
            asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(ad), "r"(pk[4 * k]), "r"(pk[4 * k + 1]),
                         "r"(pk[4 * k + 2]), "r"(pk[4 * k + 3])
                         : "memory");
          }
          if (tm.d_tma) fence_proxy_async_smem();
          __syncwarp();
          if (tm.d_tma && lane == 0) {
            tma_store_2d(&tmD, sDW, n0 + col0, rbase);
            bulk_commit();
          }
          // lane = (row r = lane / 4 + 8 it, 16-byte chunk k4): each slab read feeds both the store
          // (8 rows of 64 contiguous bytes per warp store) and the BN statistics of its 8 columns,
          // reduced over the chunk's 8 lanes by reduce-scatter (the column-pair form re-read the slab
          // with 16 4-byte loads per lane: L1 84% busy, profiles/r02_fprop_epilogue.md)
          const int k4 = lane & 3;
          float s1[8], s2[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            s1[j] = FACC ? fa1[FACC ? c2 / 2 : 0][j] : 0.f;
            s2[j] = FACC ? fa2[FACC ? c2 / 2 : 0][j] : 0.f;
          }
#pragma unroll
          for (int it = 0; it < 4; ++it) {
            const int r = (lane >> 2) + 8 * it;
            uint4 raw;
            asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                         : "=r"(raw.x), "=r"(raw.y), "=r"(raw.z), "=r"(raw.w)
                         : "r"(sDW + r * 64 + ((k4 ^ ((r >> 1) & 3)) << 4)));
            if (!tm.d_tma)
              *reinterpret_cast<uint4*>(reinterpret_cast<T*>(a.D) + (size_t)(rbase + r) * a.ldd + n0 + col0 + k4 * 8) = raw;
            if (want_stats) {  // packed FP32x2: columns 2jp, 2jp + 1 per instruction
              const uint32_t w4[4] = {raw.x, raw.y, raw.z, raw.w};
#pragma unroll
              for (int jp = 0; jp < 4; ++jp) {
                const float2 y = bf2f2(w4[jp]);
                const float2 a1 = __fadd2_rn(make_float2(s1[2 * jp], s1[2 * jp + 1]), y);
                const float2 a2 = __ffma2_rn(y, y, make_float2(s2[2 * jp], s2[2 * jp + 1]));
                s1[2 * jp] = a1.x;
                s1[2 * jp + 1] = a1.y;
                s2[2 * jp] = a2.x;
                s2[2 * jp + 1] = a2.y;
              }
            }
          }
          if (want_stats) {
            if constexpr (FACC) {
#pragma unroll
              for (int j = 0; j < 8; ++j) {
                fa1[c2 / 2][j] = s1[j];
                fa2[c2 / 2][j] = s2[j];
              }
            } else {
              float v0, v1;
              rs8_pair(s1, s2, lane, true, v0, v1);
              const int c = col0 + k4 * 8 + (lane >> 2);
              red[q][c][0] += v0;
              red[q][c][1] += v1;
            }
          }
          __syncwarp();  // the slab is rewritten by the next chunk
        }
      } else
#pragma unroll 1
      for (int c2 = 0; c2 < CPW; c2 += LDW) {
        float vb[16 * LDW];
        if (zacc) {
#pragma unroll
          for (int e = 0; e < 16 * LDW; ++e) vb[e] = 0.f;
        } else if constexpr (LDW == 2) {
          tmem_ld32(tl + (half * CPW + c2) * 16, vb);
        } else {
          tmem_ld16(tl + (half * CPW + c2) * 16, vb);
        }
#pragma unroll
        for (int h = 0; h < LDW; ++h) {
        const int cc = half * CPW + c2 + h;
        float v[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) v[e] = vb[h * 16 + e];
        const int nb = n0 + cc * 16;
        if (MODE == DSP_IGEMM_WGRAD) {
          float* out = reinterpret_cast<float*>(a.D) + (size_t)z * M * N + (size_t)m * N;
          if (mok) {
            if (nb + 16 <= N && (N & 3) == 0) {
#pragma unroll
              for (int qq = 0; qq < 4; ++qq)
                *reinterpret_cast<float4*>(out + nb + 4 * qq) =
                    make_float4(v[4 * qq], v[4 * qq + 1], v[4 * qq + 2], v[4 * qq + 3]);
            } else {
#pragma unroll
              for (int e = 0; e < 16; ++e)
                if (nb + e < N) out[nb + e] = v[e];
            }
          }
        } else {
          const int nvalid = a.n_valid > 0 ? a.n_valid : N;
          if (a.bias != nullptr) {
#pragma unroll
            for (int e = 0; e < 16; ++e)
              if (nb + e < nvalid) v[e] += a.bias[nb + e];
          }
          if (a.residual != nullptr && mok) {
            const T* res = reinterpret_cast<const T*>(a.residual) + (size_t)mr * a.ldd;
            if (nb + 16 <= N && (a.ldd % EPC) == 0) {
#pragma unroll
              for (int qq = 0; qq < 16 / EPC; ++qq) {
                uint4 raw = *reinterpret_cast<const uint4*>(res + nb + qq * EPC);
                const T* e8 = reinterpret_cast<const T*>(&raw);
#pragma unroll
                for (int e = 0; e < EPC; ++e) v[qq * EPC + e] += to_f<T>(e8[e]);
              }
            } else {
#pragma unroll
              for (int e = 0; e < 16; ++e)
                if (nb + e < N) v[e] += to_f<T>(res[nb + e]);
            }
          }
#pragma unroll
          for (int e = 0; e < 16; ++e)
            if (nb + e >= nvalid) v[e] = 0.f;
          if (a.out_f32 & 1) {
            float* out = reinterpret_cast<float*>(a.D) + (size_t)mr * a.ldd;
            if (mok) {
#pragma unroll
              for (int e = 0; e < 16; ++e)
                if (nb + e < N) out[nb + e] = v[e];
            }
          } else if (dw) {
            // stage this warp's 32 x 16 slab (row = lane) in smem, then store it row-contiguously:
            // lane = (row l >> 1 (+16), 16-byte half l & 1), so each warp store writes 16 whole
            // 32-byte sectors instead of 32 half sectors in 32 rows
            const uint32_t buf = sDW + (uint32_t)(dwc & 1) * 1024;
#pragma unroll
            for (int e = 0; e < 16; ++e) v[e] = to_f<T>(from_f<T>(v[e]));
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
              uint4 raw;
              T* e8 = reinterpret_cast<T*>(&raw);
#pragma unroll
              for (int e = 0; e < 8; ++e) e8[e] = from_f<T>(v[hh * 8 + e]);
              asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(buf + lane * 32 + hh * 16), "r"(raw.x),
                           "r"(raw.y), "r"(raw.z), "r"(raw.w)
                           : "memory");
            }
            __syncwarp();
            {
              const int rvalid = M - (m0 + q * 32);
#pragma unroll
              for (int k2 = 0; k2 < 2; ++k2) {
                const int r = (lane >> 1) + 16 * k2;
                uint4 raw;
                asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                             : "=r"(raw.x), "=r"(raw.y), "=r"(raw.z), "=r"(raw.w)
                             : "r"(buf + r * 32 + (lane & 1) * 16));
                if (r < rvalid && nb < N)  // N % 16 == 0: a slab is wholly inside or outside
                  *reinterpret_cast<uint4*>(reinterpret_cast<T*>(a.D) + (size_t)rowmap(m0 + q * 32 + r) * a.ldd + nb +
                                            (lane & 1) * 8) = raw;
              }
            }
            if (want_stats && MODE == DSP_IGEMM_FPROP) {
              // column sums from the staged slab: lane = (column l & 15, row parity l >> 4)
              const int col = lane & 15;
              float s1 = 0.f, s2 = 0.f;
              const int rvalid = M - (m0 + q * 32);  // rows of this slab inside M
#pragma unroll
              for (int r2 = 0; r2 < 16; ++r2) {
                const int r = (lane >> 4) + 2 * r2;
                uint16_t raw16;
                asm volatile("ld.shared.u16 %0, [%1];" : "=h"(raw16) : "r"(buf + r * 32 + col * 2));
                const float y = r < rvalid ? __bfloat162float(__ushort_as_bfloat16(raw16)) : 0.f;
                s1 += y;
                s2 = fmaf(y, y, s2);
              }
              s1 += __shfl_xor_sync(0xffffffffu, s1, 16);
              s2 += __shfl_xor_sync(0xffffffffu, s2, 16);
              if (lane < 16) {
                red[q][cc * 16 + col][0] += s1;
                red[q][cc * 16 + col][1] += s2;
              }
            }
            ++dwc;
          } else if (tma_out) {
            // round to bf16 (BN statistics describe the stored tensor) and stage two 16-byte
            // chunks of this row in the TMA swizzle pattern (conflict-free across lanes)
#pragma unroll
            for (int e = 0; e < 16; ++e) v[e] = to_f<T>(from_f<T>(v[e]));
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int col = cc * 16 + h * 8;
              const uint32_t off = (uint32_t)((col / tm.d_cols) * (IG_BM * tm.d_cols * 2) + row * tm.d_cols * 2 +
                                              (col % tm.d_cols) * 2);
              const uint32_t sw = off ^ (((off >> 7) & (uint32_t)tm.d_swz) << 4);
              uint4 raw;
              T* e8 = reinterpret_cast<T*>(&raw);
#pragma unroll
              for (int e = 0; e < 8; ++e) e8[e] = from_f<T>(v[h * 8 + e]);
              asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(sOut + sw), "r"(raw.x), "r"(raw.y),
                           "r"(raw.z), "r"(raw.w)
                           : "memory");
            }
          } else {
            T* out = reinterpret_cast<T*>(a.D) + (size_t)mr * a.ldd;
            // round to the storage type first so BN statistics describe the stored tensor
#pragma unroll
            for (int e = 0; e < 16; ++e) v[e] = to_f<T>(from_f<T>(v[e]));
            if (mok) {
              if (nb + 16 <= N && (a.ldd % EPC) == 0) {
#pragma unroll
                for (int qq = 0; qq < 16 / EPC; ++qq) {
                  uint4 raw;
                  T* e8 = reinterpret_cast<T*>(&raw);
#pragma unroll
                  for (int e = 0; e < EPC; ++e) e8[e] = from_f<T>(v[qq * EPC + e]);
                  *reinterpret_cast<uint4*>(out + nb + qq * EPC) = raw;
                }
              } else {
#pragma unroll
                for (int e = 0; e < 16; ++e)
                  if (nb + e < N) out[nb + e] = from_f<T>(v[e]);
              }
            }
          }
          if (want_stats && MODE == DSP_IGEMM_FPROP && dw) {
            // accumulated from the staged slab above
          } else if (want_stats && MODE == DSP_IGEMM_FPROP) {
            float sq[16];
#pragma unroll
            for (int e = 0; e < 16; ++e) {
              v[e] = mok ? v[e] : 0.f;
              sq[e] = v[e] * v[e];
            }
            const float s1 = colsum16(v, lane);
            const float s2 = colsum16(sq, lane);
            if ((lane & 1) == 0) {  // this warp's private running sums (same n-tile every tile)
              red[q][cc * 16 + (lane >> 1)][0] += s1;
              red[q][cc * 16 + (lane >> 1)][1] += s2;
            }
          } else if (want_stats) {
            // g = stored dX * (mask > 0); xhat_t = (y_t - mean_t) * invstd_t of the BN below
            const int cl = cc * 16;  // column within the CTA's n-tile
            float g[16], pr[16];
            float yv[16];
            ld_row16<T>(a.bnb[0].y, mok, mr, a.ldd, nb, N, yv);
            if (a.bnb_mask_bits != nullptr) {  // two mask bytes: columns nb .. nb + 15 of row mr
              const uint32_t b16 = mok ? (uint32_t)a.bnb_mask_bits[((size_t)mr * a.ldd + nb) >> 3] |
                                             ((uint32_t)a.bnb_mask_bits[(((size_t)mr * a.ldd + nb) >> 3) + 1] << 8)
                                       : 0u;
#pragma unroll
              for (int e = 0; e < 16; ++e) g[e] = (b16 >> e) & 1u ? v[e] : 0.f;
            } else if (a.bnb_mask != nullptr) {
              float mk[16];
              ld_row16<T>(a.bnb_mask, mok, mr, a.ldd, nb, N, mk);
#pragma unroll
              for (int e = 0; e < 16; ++e) g[e] = mk[e] > 0.f ? v[e] : 0.f;
            } else {  // mask from y (one target): relu(y*scale + shift) > 0
#pragma unroll
              for (int e = 0; e < 16; ++e) g[e] = fmaf(yv[e], bst[1][0][cl + e], bst[1][1][cl + e]) > 0.f ? v[e] : 0.f;
            }
            const float s1 = colsum16(g, lane);
#pragma unroll
            for (int e = 0; e < 16; ++e) pr[e] = g[e] * ((yv[e] - bst[0][0][cl + e]) * bst[0][1][cl + e]);
            const float s2 = colsum16(pr, lane);
            float s3 = 0.f;
            if (a.bnb_count > 1) {
              ld_row16<T>(a.bnb[1].y, mok, mr, a.ldd, nb, N, yv);
#pragma unroll
              for (int e = 0; e < 16; ++e) pr[e] = g[e] * ((yv[e] - bst[1][0][cl + e]) * bst[1][1][cl + e]);
              s3 = colsum16(pr, lane);
            }
            if ((lane & 1) == 0) {
              red[q][cl + (lane >> 1)][0] += s1;
              red[q][cl + (lane >> 1)][1] += s2;
              red[q][cl + (lane >> 1)][2] += s3;
            }
          }
        }
        }
      }
      tc_fence_before();
      mbar_arrive(&tempty_bar[acc]);
      if (tma_out) {  // whole tile staged: one thread stores it (rows >= M / cols >= N are clipped)
        fence_proxy_async_smem();
        epi_barrier<EPI_T>();
        if (et == 0) {
          for (int b = 0; b * tm.d_cols < BN; ++b)
            tma_store_2d(&tmD, sOut + b * (IG_BM * tm.d_cols * 2), n0 + b * tm.d_cols, m0);
          bulk_commit();
        }
      }
      IG_TRACE(145 + 2 * i, et == 0 && i < 16);
    }
    if (tma_out && et == 0) bulk_wait0();
    if (tm.d_tma && lane == 0) bulk_wait_read0();  // slab reads only: the stores complete after the ticket
    if constexpr (FACC) {
      if (want_stats && dw) {  // the register-held fast-path partials (zeros if no tile took it)
#pragma unroll
        for (int c = 0; c < FCH; ++c) {
          float v0, v1;
          rs8_pair(fa1[c], fa2[c], lane, true, v0, v1);
          const int col = (half * (BN / 16 / (NEPI / 4)) + 2 * c) * 16 + (lane & 3) * 8 + (lane >> 2);
          red[q][col][0] += v0;
          red[q][col][1] += v1;
        }
      }
    }
    if (want_stats) {
      epi_barrier<EPI_T>();
      const int n0c = (blockIdx.x % nt) * BN;
      for (int c = et; c < BN; c += EPI_T) {
        const int n = n0c + c;
        if (n < N) {
          for (int k = 0; k < NS; ++k)
            a.stats[((size_t)blockIdx.x * NS + k) * N + n] = (red[0][c][k] + red[1][c][k]) + (red[2][c][k] + red[3][c][k]);
        }
      }
    }
  }

  // No early trigger by default: successors launch as our CTAs exit (programmatic launch still
  // overlaps their launch + prologue with our teardown). Triggering here, before the BN-finalize
  // tail, measured 10% slower in the concurrent step: waiting successor CTAs hold SM slots the
  // other block streams need (73.1k vs 63.5k samples/s; no PDL at all: 70.5k).
#ifdef IG_PDL_TRIGGER
  pdl_trigger();
#endif

  // ---------------- fused BatchNorm finalize by the last CTA ----------------
  if (ctat != nullptr) {
    __syncthreads();
    if (tid == 0) ctat[2] = (int64_t)globaltimer_ns();
  }
  const bool fuse_fin = want_stats && a.sem != nullptr && (bnb || a.stat_out != nullptr);
  // Two-level finalize: the G/nt CTAs owning an n-tile form groups of FIN_GS; the last CTA of a
  // group sums its group's partial rows (fixed order, double) into the group leader's row, and the
  // last group to finish reduces the ngr leader rows and finalizes. The single-CTA form loaded all
  // G/nt rows at one SM's bandwidth: 6-12 us of every ResNet-50 FPROP (--fprop-stats finalize vs
  // partials, tools/conv_tc.py). Level-1 tickets live at sem[64 + 32 t + g].
  constexpr int FIN_GS = 16;
  const int per_tile = (int)gridDim.x / nt;
  const int ngr = (per_tile + FIN_GS - 1) / FIN_GS;
  // Same-box A/B (tools/gpu/ab_fin_conv.sh): pays off for >= 64 partial rows of >= 128 columns
  // (2-4 us off ResNet-50's s2-s4 3x3 / reduce convs); the extra ticket costs more than it saves
  // on short rows (CIFAR widths) or few rows (wide 1x1 expansions).
  const bool two_level = fuse_fin && (N & 3) == 0 && per_tile >= 64 && min(BN, N) >= 128 && ngr <= 32 &&
                         nt <= 30 && !tm.fin1 && !kTrace;
  if (two_level) {
    const int t_own = (int)(blockIdx.x % nt);
    const int j = (int)(blockIdx.x / nt), gi = j / FIN_GS;
    const int gsize = min(FIN_GS, per_tile - gi * FIN_GS);
    const int cbeg = t_own * BN, cend = min(N, cbeg + BN), cols = cend - cbeg;
    if (last_cta_ticket(a.sem + 64 + 32 * t_own + gi, gsize, &last_cta_s)) {
      // level 1: rows of CTAs t_own + (gi*FIN_GS + r)*nt, r < gsize -> the leader's row (r = 0)
      const size_t lead = (size_t)t_own + (size_t)gi * FIN_GS * nt;
      for (int it = tid; it < NS * cols; it += IG_THREADS) {
        const int st = it / cols, c = cbeg + it % cols;
        float v[FIN_GS];
#pragma unroll
        for (int r = 0; r < FIN_GS; ++r)
          v[r] = r < gsize ? __ldcg(&a.stats[((lead + (size_t)r * nt) * NS + st) * N + c]) : 0.f;
        double acc = 0.0;
#pragma unroll
        for (int r = 0; r < FIN_GS; ++r) acc += (double)v[r];
        a.stats[(lead * NS + st) * N + c] = (float)acc;
      }
      if (tid == 0) a.sem[64 + 32 * t_own + gi] = 0;
      if (last_cta_ticket(a.sem + t_own, ngr, &last_cta_s)) {
        // level 2: the ngr leader rows, in group order
        const int nvalid = a.n_valid > 0 ? a.n_valid : N;
        const double count = (double)a.M;
        for (int cc = tid; cc < cols; cc += IG_THREADS) {
          const int c = cbeg + cc;
          double sv[3] = {0.0, 0.0, 0.0};
          for (int g2 = 0; g2 < ngr; ++g2) {
            const size_t row = (size_t)t_own + (size_t)g2 * FIN_GS * nt;
            for (int st = 0; st < NS; ++st) sv[st] += (double)__ldcg(&a.stats[(row * NS + st) * N + c]);
          }
          if (MODE == DSP_IGEMM_FPROP) {
            float mean = 0.f, inv = 0.f, scale = 0.f, shift = 0.f;
            if (c < nvalid) {
              const double mu = sv[0] / count;
              double var = sv[1] / count - mu * mu;
              if (var < 0.0) var = 0.0;
              const double iv = 1.0 / sqrt(var + 1e-5);
              mean = (float)mu;
              inv = (float)iv;
              scale = (float)((double)a.gamma[c] * iv);
              shift = (float)((double)a.beta[c] - mu * (double)a.gamma[c] * iv);
            }
            a.stat_out[c] = mean;
            a.stat_out[N + c] = inv;
            a.stat_out[2 * N + c] = scale;
            a.stat_out[3 * N + c] = shift;
          } else {
            for (int t = 0; t + 1 < NS; ++t) {  // DGRAD: target t's sum g * xhat_t is statistic t + 1
              const dsp_bnb_target_t& tg = a.bnb[t];
              const bool real = c < a.bnb_c_real;
              if (real) {
                tg.dbeta[c] = (float)sv[0];
                tg.dgamma[c] = (float)sv[t + 1];
              }
              tg.coef[c] = real ? tg.gamma[c] * __ldcg(&tg.stat[N + c]) : 0.f;
              tg.coef[N + c] = real ? (float)(sv[0] / count) : 0.f;
              tg.coef[2 * N + c] = real ? (float)(sv[t + 1] / count) : 0.f;
            }
          }
        }
        if (tid == 0) a.sem[t_own] = 0;
      }
    }
  } else if (fuse_fin) {
    // one ticket per n-tile (sem[t], t = blockIdx.x % nt): the last of the G/nt CTAs owning
    // n-tile t finalizes its BN columns, so wide outputs finalize on nt CTAs in parallel
    const int t_own = (int)(blockIdx.x % nt);
    int* const sem_t = a.sem + t_own;
    if (last_cta_ticket(sem_t, (int)gridDim.x / nt, &last_cta_s, kTrace ? (a.out_f32 >> 8) & 7 : 0,
                        ctat != nullptr ? a.trace + 192 + 8 * 1024 + 4 * blockIdx.x : nullptr)) {
      const int cbeg = t_own * BN, cend = min(N, cbeg + BN);
      if (kTrace && a.trace != nullptr && tid == 0) a.trace[186] = (int64_t)globaltimer_ns();
      const int nvalid = a.n_valid > 0 ? a.n_valid : N;
      const double count = (double)a.M;
      const int G = (int)gridDim.x;
      auto finish = [&](int c, double s1, double s2) {
        float mean = 0.f, inv = 0.f, scale = 0.f, shift = 0.f;
        if (c < nvalid) {
          const double mu = s1 / count;
          double var = s2 / count - mu * mu;
          if (var < 0.0) var = 0.0;
          const double iv = 1.0 / sqrt(var + 1e-5);
          mean = (float)mu;
          inv = (float)iv;
          scale = (float)((double)a.gamma[c] * iv);
          shift = (float)((double)a.beta[c] - mu * (double)a.gamma[c] * iv);
        }
        a.stat_out[c] = mean;
        a.stat_out[N + c] = inv;
        a.stat_out[2 * N + c] = scale;
        a.stat_out[3 * N + c] = shift;
      };
      // DGRAD: what bn_bwd_stats' finalize writes, per target t (g shared)
      auto finish_bnb = [&](int c, double sg, double sgx, int t) {
        const dsp_bnb_target_t& tg = a.bnb[t];
        const bool real = c < a.bnb_c_real;
        if (real) {
          tg.dbeta[c] = (float)sg;
          tg.dgamma[c] = (float)sgx;
        }
        tg.coef[c] = real ? tg.gamma[c] * __ldcg(&tg.stat[N + c]) : 0.f;
        tg.coef[N + c] = real ? (float)(sg / count) : 0.f;
        tg.coef[2 * N + c] = real ? (float)(sgx / count) : 0.f;
      };
      if ((N & 3) == 0) {
        // One L2 round trip per 4 rows: NTH threads = (part, lane), lane = (statistic,
        // 4-column group) reading float4s of every owning CTA's partial row; then a
        // fixed-order sum over parts (deterministic).
        double* fin4 = reinterpret_cast<double*>(smem);  // operand ring is idle by now
        constexpr int NTH = IG_THREADS >= 256 ? 256 : 128;  // threads of the load phase
        const int win = part_sums_window(NTH, NS);
        for (int w0 = cbeg; w0 < cend; w0 += win) {
          const int cols = min(win, cend - w0);
          part_sums_load<IG_FIN_DEPTH, NTH>(a.stats, G, N, NS, w0, cols, BN, nt, fin4);
          __syncthreads();
          if (kTrace && a.trace != nullptr && tid == 0 && w0 == cbeg) a.trace[187] = (int64_t)globaltimer_ns();
          for (int cc = tid; cc < cols; cc += IG_THREADS) {
            const double s1 = part_sums_get<NTH>(fin4, NS, cols, cc, 0);
            const double s2 = part_sums_get<NTH>(fin4, NS, cols, cc, 1);
            if (MODE == DSP_IGEMM_FPROP) {
              finish(w0 + cc, s1, s2);
            } else {
              finish_bnb(w0 + cc, s1, s2, 0);
              if (NS > 2) finish_bnb(w0 + cc, s1, part_sums_get<NTH>(fin4, NS, cols, cc, 2), 1);
            }
          }
          __syncthreads();
        }
      } else if (MODE == DSP_IGEMM_FPROP) {
        double(*fin)[2] = reinterpret_cast<double(*)[2]>(smem);
        constexpr int NTH = IG_THREADS >= 256 ? 256 : 128;
        for (int cb = cbeg; cb < cend; cb += NTH) {
          const int cols = min(NTH, cend - cb);
          const int parts = NTH / cols;
          if (tid < parts * cols) {
            const int c = cb + tid % cols, p = tid / cols;
            const int step = parts * nt;
            double s1 = 0.0, s2 = 0.0;
            for (int b = c / BN + p * nt; b < G; b += step) {
              s1 += (double)__ldcg(&a.stats[((size_t)b * 2 + 0) * N + c]);
              s2 += (double)__ldcg(&a.stats[((size_t)b * 2 + 1) * N + c]);
            }
            fin[tid][0] = s1;
            fin[tid][1] = s2;
          }
          __syncthreads();
          if (tid < cols) {
            double s1 = 0.0, s2 = 0.0;
            for (int p = 0; p < parts; ++p) {
              s1 += fin[p * cols + tid][0];
              s2 += fin[p * cols + tid][1];
            }
            finish(cb + tid, s1, s2);
          }
          __syncthreads();
        }
      }
      if (tid == 0) *sem_t = 0;
      if (kTrace && a.trace != nullptr && tid == 0) a.trace[188] = (int64_t)globaltimer_ns();
    }
  }

  if (ctat != nullptr && tid == 0) ctat[4] = (int64_t)globaltimer_ns();
  tc_fence_before();
  __syncthreads();
  if (ctat != nullptr && tid == 0) ctat[5] = (int64_t)globaltimer_ns();
  if (warp == IG_MMA_WARP) {
    if (ctat != nullptr && lane == 0) ctat[6] = (int64_t)globaltimer_ns();
    tc_fence_after();
    tmem_dealloc(tmem_d, Cfg::TMEM_COLS);
    IG_TRACE(177, lane == 0);
    if (ctat != nullptr && lane == 0) ctat[3] = (int64_t)globaltimer_ns();
  }
}

static PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

static PFN_cuTensorMapEncodeIm2col_v12000 im2col_encoder() {
  static PFN_cuTensorMapEncodeIm2col_v12000 fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeIm2col_v12000>(p);
  }
  return fn;
}

constexpr int IG_HALO_SMEM_MAX = 100 * 1024;  // keeps two conv CTAs per SM

// im2col-mode A operand (any output width, 64-channel multiples): FPROP (stride 1/2) on X,
// stride-1 DGRAD on dY with the transposed weights B_t (flipped-kernel conv, padding R-1-pad),
// WGRAD on X (64-pixel k-blocks) with dY as a plain [pixels][K] matrix. The tensor map's
// bounding box per image is [-pad, dim + pad - (R-1)) in W and H, walked with the conv stride,
// so the n-th pixel of a box is output pixel m0 + n whatever the rows / images it crosses.
template <int MODE, int BN>
static bool i2c_plan(const dsp_igemm_args_t& a, IgTma& tm, CUtensorMap& tmA, CUtensorMap& tmB,
                     PFN_cuTensorMapEncodeTiled_v12000 enc) {
  static const bool disabled = getenv("DSP_B200_NO_IM2COL") != nullptr;
  PFN_cuTensorMapEncodeIm2col_v12000 enc2 = im2col_encoder();
  const dsp_conv_geom_t& g = a.geom;
  if (disabled || enc2 == nullptr || g.R != g.S) return false;
  const int st = MODE == DSP_IGEMM_DGRAD ? 1 : g.stride;
  if (MODE == DSP_IGEMM_DGRAD && g.stride == 2) {
    // parity split: 4 stride-1 sub-convolutions of dY (dr, ds in {0, 1}) against the taps of
    // B_t that reach each output parity; one launch, units = 4 parities x m-tiles
    static const bool no_s2 = getenv("DSP_B200_NO_S2DGRAD") != nullptr;
    if (no_s2 || a.B_t == nullptr || g.R != g.S || (g.R != 1 && g.R != 3) || g.pad != (g.R - 1) / 2 ||
        g.H != 2 * g.P || g.W != 2 * g.Q || g.K % 64 || a.Kd % 64 || a.M % 4)
      return false;
    if ((reinterpret_cast<uintptr_t>(a.A) & 15) || (reinterpret_cast<uintptr_t>(a.B_t) & 15)) return false;
    cuuint64_t dims[4] = {(cuuint64_t)g.K, (cuuint64_t)g.Q, (cuuint64_t)g.P, (cuuint64_t)g.nimg};
    cuuint64_t strides[3] = {(cuuint64_t)g.K * 2, (cuuint64_t)g.Q * g.K * 2, (cuuint64_t)g.P * g.Q * g.K * 2};
    int lower[2] = {0, 0}, upper[2] = {0, 0};
    cuuint32_t es[4] = {1, 1, 1, 1};
    if (enc2(&tmA, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(a.A), dims, strides, lower, upper, 64,
             (cuuint32_t)IG_BM, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return false;
    cuuint64_t bd[2] = {(cuuint64_t)a.Kd, (cuuint64_t)a.N};
    cuuint64_t bs[1] = {(cuuint64_t)a.Kd * 2};
    cuuint32_t bb[2] = {64, (cuuint32_t)BN};
    cuuint32_t be[2] = {1, 1};
    if (enc(&tmB, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(a.B_t), bd, bs, bb, be,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return false;
    tm.on_a = tm.on_b = 1;
    tm.i2c = 1;
    tm.s2 = 1;
    tm.i2c_pad = 0;
    tm.cbox = 64;
    tm.box_a = IG_BM * 128;
    tm.swz_a = 2;
    tm.box_b = BN * 128;
    return true;
  }
  if (MODE == DSP_IGEMM_DGRAD && (g.stride != 1 || a.B_t == nullptr)) return false;
  if (st != 1 && st != 2) return false;
  const int cdim = MODE == DSP_IGEMM_DGRAD ? g.K : g.C;  // channels of the im2col'd tensor
  const int cbox = std::min(cdim, 64);  // channels per A box (one tap each)
  if ((cbox != 8 && cbox != 16 && cbox != 32 && cbox != 64) || cdim % cbox) return false;
  if (MODE != DSP_IGEMM_WGRAD && BN >= 128 && cbox != 64) return false;  // wide tiles: 64-channel boxes only
  const CUtensorMapSwizzle swz = cbox == 8 ? CU_TENSOR_MAP_SWIZZLE_NONE
                                 : cbox == 16 ? CU_TENSOR_MAP_SWIZZLE_32B
                                 : cbox == 32 ? CU_TENSOR_MAP_SWIZZLE_64B
                                              : CU_TENSOR_MAP_SWIZZLE_128B;
  const int uswz = cbox == 8 ? 0 : cbox == 16 ? 6 : cbox == 32 ? 4 : 2;
  const int pad = MODE == DSP_IGEMM_DGRAD ? g.R - 1 - g.pad : g.pad;
  if (pad < 0 || pad > 64 || g.R > 64) return false;
  const int ih = MODE == DSP_IGEMM_DGRAD ? g.P : g.H, iw = MODE == DSP_IGEMM_DGRAD ? g.Q : g.W;
  const int oh = MODE == DSP_IGEMM_DGRAD ? g.H : g.P, ow = MODE == DSP_IGEMM_DGRAD ? g.W : g.Q;
  const int lo = -pad, hi = pad - (g.R - 1);
  // positions walked per row / column must be exactly the output extent
  if ((iw + hi - lo + st - 1) / st != ow || (ih + hi - lo + st - 1) / st != oh) return false;
  const void* asrc = a.A;
  const void* bsrc = MODE == DSP_IGEMM_DGRAD ? a.B_t : a.B;
  if ((reinterpret_cast<uintptr_t>(asrc) & 15) || (reinterpret_cast<uintptr_t>(bsrc) & 15)) return false;
  const int ppc = MODE == DSP_IGEMM_WGRAD ? 64 : IG_BM;
  // 1x1 stride-1: output pixel m reads input pixel m, so A is a plain [pixels][channels] matrix
  static const bool no_a2d = getenv("DSP_B200_NO_A2D") != nullptr;
  const bool a2d = !no_a2d && g.R == 1 && st == 1 && pad == 0;
  if (a2d) {
    cuuint64_t dims[2] = {(cuuint64_t)cdim, (cuuint64_t)g.nimg * ih * iw};
    cuuint64_t strides[1] = {(cuuint64_t)cdim * 2};
    cuuint32_t box[2] = {(cuuint32_t)cbox, (cuuint32_t)ppc};
    cuuint32_t es[2] = {1, 1};
    if (enc(&tmA, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(asrc), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return false;
  } else {
    cuuint64_t dims[4] = {(cuuint64_t)cdim, (cuuint64_t)iw, (cuuint64_t)ih, (cuuint64_t)g.nimg};
    cuuint64_t strides[3] = {(cuuint64_t)cdim * 2, (cuuint64_t)iw * cdim * 2, (cuuint64_t)ih * iw * cdim * 2};
    int lower[2] = {lo, lo}, upper[2] = {hi, hi};
    cuuint32_t es[4] = {1, (cuuint32_t)st, (cuuint32_t)st, 1};
    if (enc2(&tmA, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(asrc), dims, strides, lower, upper, cbox,
             (cuuint32_t)ppc, es, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return false;
  }
  tm.a2d = a2d ? 1 : 0;
  if (MODE == DSP_IGEMM_WGRAD) {
    const int cb = std::min(std::min(g.K, 64), BN);
    if ((cb != 16 && cb != 32 && cb != 64) || g.K % cb || BN % cb) return false;
    const int64_t npix = (int64_t)g.nimg * g.P * g.Q;
    cuuint64_t bd[2] = {(cuuint64_t)g.K, (cuuint64_t)npix};  // dY [pixels][K]
    cuuint64_t bs[1] = {(cuuint64_t)g.K * 2};
    cuuint32_t bb[2] = {(cuuint32_t)cb, 64};
    cuuint32_t be[2] = {1, 1};
    const CUtensorMapSwizzle swz = cb == 16 ? CU_TENSOR_MAP_SWIZZLE_32B
                                   : cb == 32 ? CU_TENSOR_MAP_SWIZZLE_64B
                                              : CU_TENSOR_MAP_SWIZZLE_128B;
    if (enc(&tmB, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(a.B), bd, bs, bb, be,
            CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return false;
    tm.on_a = tm.on_b = 1;
    tm.i2c = 1;
    tm.i2c_pad = pad;
    tm.cbox = cbox;
    tm.box_a = 64 * cbox * 2;
    tm.swz_a = uswz;
    tm.cbox_b = cb;
    tm.box_b = 64 * cb * 2;
    tm.swz_b = cb == 16 ? 6 : cb == 32 ? 4 : 2;
    return true;
  }
  if (a.Kd % 8) return false;
  cuuint64_t bd[2] = {(cuuint64_t)a.Kd, (cuuint64_t)a.N};  // FPROP W [Cout][Kd]; DGRAD B_t [C][Kd]
  cuuint64_t bs[1] = {(cuuint64_t)a.Kd * 2};
  cuuint32_t bb[2] = {64, (cuuint32_t)BN};
  cuuint32_t be[2] = {1, 1};
  if (enc(&tmB, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(bsrc), bd, bs, bb, be,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return false;
  tm.on_a = tm.on_b = 1;
  tm.i2c = 1;
  tm.i2c_pad = pad;
  tm.cbox = cbox;
  tm.box_a = IG_BM * cbox * 2;
  tm.swz_a = uswz;
  tm.box_b = BN * 128;
  return true;
}

// FPROP halo tiles: stride-1 'same' RxS conv, C in {16, 32, 64} (one A box covers all
// channels), output rows of 8k pixels with a 128-pixel tile = hb whole rows of one image.
template <int MODE, int BN>
static bool halo_plan(const dsp_igemm_args_t& a, IgTma& tm, CUtensorMap& tmA, CUtensorMap& tmB,
                      PFN_cuTensorMapEncodeTiled_v12000 enc) {
  static const bool disabled = getenv("DSP_B200_NO_HALO") != nullptr;
  const dsp_conv_geom_t& g = a.geom;
  if (disabled || g.stride != 1 || g.R != g.S || g.pad != (g.R - 1) / 2 || g.R % 2 == 0) return false;
  static const int max_c = getenv("DSP_B200_HALO_MAXC") ? atoi(getenv("DSP_B200_HALO_MAXC")) : 64;
  // a 2-deep ring (stage 1: 42 KB) measured best in the concurrent step: 3 stages were
  // faster alone but left less smem for the other blocks' kernels
  static const int max_nst = getenv("DSP_B200_HALO_NST") ? atoi(getenv("DSP_B200_HALO_NST")) : 2;
  // A rows: FPROP = X pixels with C channels; DGRAD = dY pixels with K channels (weights B_t)
  const int cch = MODE == DSP_IGEMM_FPROP ? g.C : g.K;
  const void* bsrc = MODE == DSP_IGEMM_FPROP ? a.B : a.B_t;
  if ((cch != 16 && cch != 32 && cch != 64) || cch > max_c || bsrc == nullptr) return false;
  if (g.P != g.H || g.Q != g.W || g.Q % 8 || IG_BM % g.Q) return false;
  const int hb = IG_BM / g.Q;
  if (hb > g.P || g.P % hb) return false;
  if ((a.Kd % 8) || (reinterpret_cast<uintptr_t>(a.A) & 15) || (reinterpret_cast<uintptr_t>(bsrc) & 15)) return false;
  const int rows = hb + g.R - 1;
  if (rows > 256 || g.W > 256) return false;
  const int rowb = cch * 2;
  const int box = rowb * g.W * rows;
  const int nwb = (a.Kd + 63) / 64;
  const int wbytes = nwb * BN * 128;
  const int nst = std::min(std::min(IgCfg<BN>::STAGES, max_nst), (IG_HALO_SMEM_MAX - wbytes) / (box * g.S));
  if (nst < 2) return false;
  const CUtensorMapSwizzle swz = cch == 16 ? CU_TENSOR_MAP_SWIZZLE_32B
                                 : cch == 32 ? CU_TENSOR_MAP_SWIZZLE_64B
                                             : CU_TENSOR_MAP_SWIZZLE_128B;
  cuuint64_t dims[4] = {(cuuint64_t)cch, (cuuint64_t)g.W, (cuuint64_t)g.H, (cuuint64_t)g.nimg};
  cuuint64_t strides[3] = {(cuuint64_t)rowb, (cuuint64_t)g.W * rowb, (cuuint64_t)g.H * g.W * rowb};
  cuuint32_t bx[4] = {(cuuint32_t)cch, (cuuint32_t)g.W, (cuuint32_t)rows, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  if (enc(&tmA, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(a.A), dims, strides, bx, es,
          CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return false;
  cuuint64_t bd[2] = {(cuuint64_t)a.Kd, (cuuint64_t)a.N};  // weights [N rows][Kd], K-major
  cuuint64_t bs[1] = {(cuuint64_t)a.Kd * 2};
  cuuint32_t bb[2] = {64, (cuuint32_t)BN};
  cuuint32_t be[2] = {1, 1};
  if (enc(&tmB, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(bsrc), bd, bs, bb, be,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return false;
  tm.on_a = tm.on_b = 1;
  tm.halo = 1;
  tm.h_box = box;
  tm.h_nst = nst;
  tm.h_nwb = nwb;
  tm.h_rowb = rowb;
  tm.h_swz = cch == 16 ? 6 : cch == 32 ? 4 : 2;
  return true;
}

template <int BN>
static void tma_plan_wgrad_tiled(const dsp_igemm_args_t& a, IgTma& tm, CUtensorMap& tmA, CUtensorMap& tmB,
                                 PFN_cuTensorMapEncodeTiled_v12000 enc) {
  const dsp_conv_geom_t& g = a.geom;
  auto swz_of = [](int cbox, int& umma) {
    umma = cbox == 8 ? 0 : cbox == 16 ? 6 : cbox == 32 ? 4 : 2;
    return cbox == 8 ? CU_TENSOR_MAP_SWIZZLE_NONE
           : cbox == 16 ? CU_TENSOR_MAP_SWIZZLE_32B
           : cbox == 32 ? CU_TENSOR_MAP_SWIZZLE_64B
                        : CU_TENSOR_MAP_SWIZZLE_128B;
  };
  {
    // k-block = 64 output pixels = Q x rows x imgs; A = X boxes per (tap, channel chunk), B = dY boxes
    if (g.stride != 1 && g.stride != 2) return;
    const int ca = std::min(g.C, 64), cb = std::min(std::min(g.K, 64), BN);
    auto okc = [](int c) { return c == 8 || c == 16 || c == 32 || c == 64; };
    if (!okc(ca) || !okc(cb) || g.C % ca || g.K % cb || BN % cb || IG_BM % ca) return;
    if (64 % g.Q) return;
    int rows = 64 / g.Q, imgs = 1;
    if (rows <= g.P) {
      if (g.P % rows) return;
    } else {
      if (64 % (g.P * g.Q) || g.nimg % (64 / (g.P * g.Q))) return;
      imgs = 64 / (g.P * g.Q);
      rows = g.P;
    }
    if (g.Q * g.stride > 256 || rows * g.stride > 256 || imgs > 256) return;
    if ((reinterpret_cast<uintptr_t>(a.A) & 15) || (reinterpret_cast<uintptr_t>(a.B) & 15)) return;
    int ua, ub;
    cuuint64_t xd[4] = {(cuuint64_t)g.C, (cuuint64_t)g.W, (cuuint64_t)g.H, (cuuint64_t)g.nimg};
    cuuint64_t xs[3] = {(cuuint64_t)g.C * 2, (cuuint64_t)g.W * g.C * 2, (cuuint64_t)g.H * g.W * g.C * 2};
    cuuint32_t xb[4] = {(cuuint32_t)ca, (cuuint32_t)(g.Q * g.stride), (cuuint32_t)(rows * g.stride), (cuuint32_t)imgs};
    cuuint32_t xe[4] = {1, (cuuint32_t)g.stride, (cuuint32_t)g.stride, 1};
    cuuint64_t yd[4] = {(cuuint64_t)g.K, (cuuint64_t)g.Q, (cuuint64_t)g.P, (cuuint64_t)g.nimg};
    cuuint64_t ys[3] = {(cuuint64_t)g.K * 2, (cuuint64_t)g.Q * g.K * 2, (cuuint64_t)g.P * g.Q * g.K * 2};
    cuuint32_t yb[4] = {(cuuint32_t)cb, (cuuint32_t)g.Q, (cuuint32_t)rows, (cuuint32_t)imgs};
    cuuint32_t ye[4] = {1, 1, 1, 1};
    if (enc(&tmA, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(a.A), xd, xs, xb, xe,
            CU_TENSOR_MAP_INTERLEAVE_NONE, swz_of(ca, ua), CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return;
    if (enc(&tmB, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(a.B), yd, ys, yb, ye,
            CU_TENSOR_MAP_INTERLEAVE_NONE, swz_of(cb, ub), CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return;
    tm.on_a = tm.on_b = 1;
    tm.cbox = ca;
    tm.box_a = 64 * ca * 2;
    tm.swz_a = ua;
    tm.cbox_b = cb;
    tm.box_b = 64 * cb * 2;
    tm.swz_b = ub;
    tm.kb_rows = rows;
    tm.kb_imgs = imgs;
    return;
  }
}

template <int MODE, int BN>
static void tma_plan_tiled(const dsp_igemm_args_t& a, IgTma& tm, CUtensorMap& tmA, CUtensorMap& tmB,
                           PFN_cuTensorMapEncodeTiled_v12000 enc) {
  const dsp_conv_geom_t& g = a.geom;
  if (MODE == DSP_IGEMM_DGRAD && g.stride != 1) return;
  if (g.stride != 1 && g.stride != 2) return;
  const int cdim = MODE == DSP_IGEMM_FPROP ? g.C : g.K;  // channels of the gathered tensor
  const int oh = MODE == DSP_IGEMM_FPROP ? g.P : g.H, ow = MODE == DSP_IGEMM_FPROP ? g.Q : g.W;
  const int ih = MODE == DSP_IGEMM_FPROP ? g.H : g.P, iw = MODE == DSP_IGEMM_FPROP ? g.W : g.Q;
  const int st = MODE == DSP_IGEMM_FPROP ? g.stride : 1;
  const int cbox = std::min(cdim, 64);
  if (cdim % cbox || (cbox != 8 && cbox != 16 && cbox != 32 && cbox != 64)) return;
  if (IG_BM % ow) return;
  int hb = IG_BM / ow, nb = 1;
  if (hb <= oh) {
    if (oh % hb) return;
  } else {
    if (IG_BM % (oh * ow) || g.nimg % (IG_BM / (oh * ow))) return;
    nb = IG_BM / (oh * ow);
    hb = oh;
  }
  if (ow * st > 256 || hb * st > 256 || (reinterpret_cast<uintptr_t>(a.A) & 15)) return;
  cuuint64_t dims[4] = {(cuuint64_t)cdim, (cuuint64_t)iw, (cuuint64_t)ih, (cuuint64_t)g.nimg};
  cuuint64_t strides[3] = {(cuuint64_t)cdim * 2, (cuuint64_t)iw * cdim * 2, (cuuint64_t)ih * iw * cdim * 2};
  cuuint32_t box[4] = {(cuuint32_t)cbox, (cuuint32_t)(ow * st), (cuuint32_t)(hb * st), (cuuint32_t)nb};
  cuuint32_t estr[4] = {1, (cuuint32_t)st, (cuuint32_t)st, 1};
  const CUtensorMapSwizzle swz = cbox == 8 ? CU_TENSOR_MAP_SWIZZLE_NONE
                                 : cbox == 16 ? CU_TENSOR_MAP_SWIZZLE_32B
                                 : cbox == 32 ? CU_TENSOR_MAP_SWIZZLE_64B
                                              : CU_TENSOR_MAP_SWIZZLE_128B;
  if (enc(&tmA, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(a.A), dims, strides, box, estr,
          CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return;
  tm.on_a = 1;
  tm.cbox = cbox;
  tm.hb = hb;
  tm.nb = nb;
  tm.box_a = IG_BM * cbox * 2;
  tm.swz_a = cbox == 8 ? 0 : cbox == 16 ? 6 : cbox == 32 ? 4 : 2;
  if (MODE == DSP_IGEMM_FPROP && (a.Kd % 8) == 0 && (reinterpret_cast<uintptr_t>(a.B) & 15) == 0) {
    cuuint64_t bd[2] = {(cuuint64_t)a.Kd, (cuuint64_t)g.K};
    cuuint64_t bs[1] = {(cuuint64_t)a.Kd * 2};
    cuuint32_t bb[2] = {64, (cuuint32_t)BN};
    cuuint32_t be[2] = {1, 1};
    if (enc(&tmB, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(a.B), bd, bs, bb, be,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS) {
      tm.on_b = 1;
      tm.box_b = BN * 128;
    }
  }
}

// Decide whether this launch's A (and B) operands can be fetched with TMA and build the
// tensor maps: FPROP / DGRAD halo tiles, else tiled boxes when a 128-row M tile is whole output
// rows (OW | 128) or images, else im2col mode (64-channel multiples); WGRAD tiled, else im2col.
template <typename T, int MODE, int BN>
static void tma_plan(const dsp_igemm_args_t& a, IgTma& tm, CUtensorMap& tmA, CUtensorMap& tmB) {
  tm = IgTma{};
  memset(&tmA, 0, sizeof(tmA));
  memset(&tmB, 0, sizeof(tmB));
  static const bool disabled = getenv("DSP_B200_NO_TMA") != nullptr;
  if (disabled || sizeof(T) != 2) return;
  PFN_cuTensorMapEncodeTiled_v12000 enc = tensor_map_encoder();
  if (enc == nullptr) return;
  if (MODE == DSP_IGEMM_WGRAD) {
    tma_plan_wgrad_tiled<BN>(a, tm, tmA, tmB, enc);
  } else if (!halo_plan<MODE, BN>(a, tm, tmA, tmB, enc)) {
    tma_plan_tiled<MODE, BN>(a, tm, tmA, tmB, enc);
  }
  // im2col wherever an operand would otherwise be gathered
  if (!(tm.on_a && tm.on_b)) {
    IgTma t2{};
    CUtensorMap a2, b2;
    if (i2c_plan<MODE, BN>(a, t2, a2, b2, enc)) {
      tm = t2;
      tmA = a2;
      tmB = b2;
    }
  }
}

// D through TMA stores: bf16 FPROP / DGRAD outputs with 16-byte aligned rows.
template <typename T, int MODE, int BN>
static void tma_out_plan(const dsp_igemm_args_t& a, IgTma& tm, CUtensorMap& tmD) {
  memset(&tmD, 0, sizeof(tmD));
  tm.on_d = 0;
  // Measured on B200 (ResNet-56 shapes): no gain over per-row st.global.v4 once the
  // staging tile costs ring stages, so it is compiled in only with -DIG_TMA_STORE.
  if (IgCfg<BN>::OUT_BYTES == 0) return;
  if (MODE == DSP_IGEMM_WGRAD || sizeof(T) != 2 || (a.out_f32 & 1)) return;
  if ((reinterpret_cast<uintptr_t>(a.D) & 15) || (a.ldd % 8) || a.N % 8) return;
  PFN_cuTensorMapEncodeTiled_v12000 enc = tensor_map_encoder();
  if (enc == nullptr) return;
  const int cols = std::min(BN, 64);
  const CUtensorMapSwizzle swz = cols == 16 ? CU_TENSOR_MAP_SWIZZLE_32B
                                 : cols == 32 ? CU_TENSOR_MAP_SWIZZLE_64B
                                              : CU_TENSOR_MAP_SWIZZLE_128B;
  cuuint64_t dims[2] = {(cuuint64_t)a.N, (cuuint64_t)a.M};
  cuuint64_t strides[1] = {(cuuint64_t)a.ldd * 2};
  cuuint32_t box[2] = {(cuuint32_t)cols, (cuuint32_t)IG_BM};
  cuuint32_t estr[2] = {1, 1};
  if (enc(&tmD, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, a.D, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
          CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return;
  tm.on_d = 1;
  tm.d_cols = cols;
  tm.d_swz = cols == 16 ? 1 : cols == 32 ? 3 : 7;
}

// Wide-tile epilogue stores (BN >= 128, bf16 FPROP / DGRAD): each epilogue warp stages
// 32-row x 16-column slabs of the tile in smem and stores them row-contiguously (whole 32-byte
// sectors per lane pair instead of 32 row-strided 16-byte stores per warp instruction).
template <typename T, int MODE, int BN>
static void dwarp_plan(const dsp_igemm_args_t& a, IgTma& tm, CUtensorMap& tmD) {
  static const bool disabled = getenv("DSP_B200_NO_DWARP") != nullptr;
  if (disabled || tm.halo || (tm.i2c ? IgCfg<BN, true>::DW_BYTES : IgCfg<BN>::DW_BYTES) == 0 || MODE == DSP_IGEMM_WGRAD || sizeof(T) != 2 || (a.out_f32 & 1))
    return;
  if ((reinterpret_cast<uintptr_t>(a.D) & 15) || (a.ldd % 8) || a.N % 16 || a.ldd < a.N) return;
  tm.d_warp = 1;
  // FPROP / DGRAD slabs leave through TMA stores: the async-proxy stores are not drained by the release
  // fence of the BN-finalize ticket, so the finalize no longer waits behind the CTA's last output
  // stores (4-8.5 us per launch, profiles/r01_fin_trace.log)
  static const bool no_dtma = getenv("DSP_B200_NO_DTMA") != nullptr;
  static const int dtma_min_bn = getenv("DSP_B200_DTMA_MIN_BN") ? atoi(getenv("DSP_B200_DTMA_MIN_BN")) : 64;
  if (no_dtma || (a.ldd * 2) % 16 || BN < dtma_min_bn) return;
  {  // only into this device's memory (a multi-device engine's DGRAD may write a peer's ring slot)
    cudaPointerAttributes pa{};
    int dev = -1;
    if (cudaPointerGetAttributes(&pa, a.D) != cudaSuccess || cudaGetDevice(&dev) != cudaSuccess ||
        pa.type != cudaMemoryTypeDevice || pa.device != dev) {
      cudaGetLastError();
      return;
    }
  }
  PFN_cuTensorMapEncodeTiled_v12000 enc = tensor_map_encoder();
  if (enc == nullptr) return;
  cuuint64_t dims[2] = {(cuuint64_t)a.N, (cuuint64_t)a.M};
  cuuint64_t strides[1] = {(cuuint64_t)a.ldd * 2};
  cuuint32_t box[2] = {32, 32};
  cuuint32_t estr[2] = {1, 1};
  if (enc(&tmD, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, a.D, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return;
  tm.d_tma = 1;
}

// fp32 storage (3xTF32): 2 stages of hi + lo operand tiles (igemm_kernel F32_SPLIT)
template <typename T, int MODE, int BN>
constexpr int f32_smem() {
  return sizeof(T) != 4 ? 0 : 2 * 2 * (IG_BM * 128 + ((MODE != DSP_IGEMM_FPROP && BN < 32) ? 32 : BN) * 128);
}

template <typename T, int MODE, int BN>
cudaError_t launch_bn(const dsp_igemm_args_t& a, int splits, cudaStream_t st) {
  using Cfg = IgCfg<BN>;
  // the kernel attributes are per device: set them the first time each device launches
  constexpr int kMaxDev = 64;
  static int attr_state[kMaxDev] = {};
  static int num_sms_dev[kMaxDev] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDev) return cudaErrorInvalidDevice;
  if (!attr_state[dev]) {
    constexpr int wg_extra = (IgStages<MODE, BN, IgCfg<BN, true>::STAGES>::value - IgCfg<BN, true>::STAGES) *
                             (IG_BM * 128 + BN * 128);
    const int smax = std::max(std::max(std::max(Cfg::SMEM, IgCfg<BN, true>::SMEM + std::max(wg_extra, 0)),
                                       IG_HALO_SMEM_MAX),
                              f32_smem<T, MODE, BN>());
    cudaError_t e = cudaFuncSetAttribute(igemm_kernel<T, MODE, BN, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         smax);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(igemm_kernel<T, MODE, BN, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smax);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(igemm_kernel<T, MODE, BN, 1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smax);
    if (e != cudaSuccess) return e;
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    num_sms_dev[dev] = sms;
    attr_state[dev] = 1;
  }
  const int num_sms = num_sms_dev[dev];
  const int EPC = 16 / (int)sizeof(T);
  const int KS = 8 * EPC;
  const int nkb = (a.Kd + KS - 1) / KS;
  const int ns = MODE == DSP_IGEMM_WGRAD ? (nkb + a.kb_per_split - 1) / a.kb_per_split : 1;
  const int units = ((a.M + IG_BM - 1) / IG_BM) * ((a.N + BN - 1) / BN) * ns;
  static const int cap = getenv("DSP_B200_GRID_CAP") ? atoi(getenv("DSP_B200_GRID_CAP")) : DSP_IGEMM_MAX_CTAS;
  static_assert(IgCfg<BN, true>::CTAS_PER_SM == Cfg::CTAS_PER_SM, "grid sizing assumes equal residency");
  int grid = std::min(units, std::min(cap, num_sms * Cfg::CTAS_PER_SM));
  // CIFAR-sized FPROP / DGRAD (<= 64-wide tiles, M <= 256 K rows): one CTA per SM. Half the CTAs
  // each run twice the tiles, so the concurrent block streams' kernels co-reside with more of
  // them (ResNet-56 step +3.4 % same-box A/B; the per-kernel latency alone is unchanged, ResNet-50
  // is not affected). DSP_B200_SMALL_CAP=0 disables.
  static const int small_cap = getenv("DSP_B200_SMALL_CAP") ? atoi(getenv("DSP_B200_SMALL_CAP")) : 1;
  static const int small_m = getenv("DSP_B200_SMALL_M") ? atoi(getenv("DSP_B200_SMALL_M")) : 131072;
  if (small_cap && MODE != DSP_IGEMM_WGRAD && BN <= 64 && a.M <= small_m) grid = std::min(grid, num_sms);
  {  // per-mode caps (A/B knobs): DSP_B200_FPROP_CAP / DSP_B200_DGRAD_CAP
    static const int fcap = getenv("DSP_B200_FPROP_CAP") ? atoi(getenv("DSP_B200_FPROP_CAP")) : 0;
    static const int dcap = getenv("DSP_B200_DGRAD_CAP") ? atoi(getenv("DSP_B200_DGRAD_CAP")) : 0;
    const int mc = MODE == DSP_IGEMM_FPROP ? fcap : MODE == DSP_IGEMM_DGRAD ? dcap : 0;
    if (mc > 0) grid = std::min(grid, mc);
  }
  if (MODE != DSP_IGEMM_WGRAD) {  // each CTA owns one n-tile: grid must be a multiple of nt
    const int nt = (a.N + BN - 1) / BN;
    grid = std::max(nt, grid / nt * nt);
  }
  IgTma tm;
  CUtensorMap tmA, tmB, tmD;
  tma_plan<T, MODE, BN>(a, tm, tmA, tmB);
  tma_out_plan<T, MODE, BN>(a, tm, tmD);
  if (!tm.on_d) dwarp_plan<T, MODE, BN>(a, tm, tmD);
  {
    const dsp_conv_geom_t& g = a.geom;
    const uint32_t divs[5] = {(uint32_t)(MODE == DSP_IGEMM_DGRAD ? g.H * g.W : g.P * g.Q),
                              (uint32_t)(MODE == DSP_IGEMM_DGRAD ? g.W : g.Q),
                              (uint32_t)(MODE == DSP_IGEMM_DGRAD ? g.K : g.C), (uint32_t)g.S, (uint32_t)g.K};
    for (int i = 0; i < 5; ++i) {
      tm.fd_d[i] = divs[i];
      fastdiv_host(divs[i], tm.fd_mul[i], tm.fd_shr[i]);
    }
  }
  static const bool fin1 = getenv("DSP_B200_FIN_1LEVEL") != nullptr;
  tm.fin1 = fin1 ? 1 : 0;
  static const bool force4 = getenv("DSP_B200_NPW4") != nullptr;
  int smem = tm.halo ? tm.h_nst * tm.h_box * a.geom.S + tm.h_nwb * BN * 128
                     : (tm.i2c ? IgCfg<BN, true>::SMEM + (IgStages<MODE, BN, IgCfg<BN, true>::STAGES>::value -
                                                            IgCfg<BN, true>::STAGES) * (IG_BM * 128 + BN * 128)
                               : Cfg::SMEM + (IgStages<MODE, BN, Cfg::STAGES>::value - Cfg::STAGES) *
                                                 (IG_BM * 128 + BN * 128));
  if (sizeof(T) == 4) smem = f32_smem<T, MODE, BN>();
  if (tm.on_a && tm.on_b && (!force4 || tm.i2c))  // nothing to gather: one producer warp
  {
    if (tm.i2c)
      launch_k(igemm_kernel<T, MODE, BN, 1, true>, grid, IgWarps<1, BN, true>::THREADS, smem, st, a, tmA, tmB, tmD, tm);
    else
      launch_k(igemm_kernel<T, MODE, BN, 1>, grid, IgWarps<1, BN>::THREADS, smem, st, a, tmA, tmB, tmD, tm);
  }
  else
    launch_k(igemm_kernel<T, MODE, BN, 4>, grid, IgWarps<4, BN>::THREADS, smem, st, a, tmA, tmB, tmD, tm);
  (void)splits;
  note_launch();
  return cudaGetLastError();
}

}  // namespace dsp
