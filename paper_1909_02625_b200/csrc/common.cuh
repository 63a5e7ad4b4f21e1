// Shared device helpers for the DSP B200 kernels (sm_100a only).
//
// Inline-PTX wrappers for the Blackwell pieces the kernels use: mbarriers,
// cp.async with zero-fill (im2col gathers with padding), tcgen05 TMEM
// allocation / MMA / commit / load, and the UMMA shared-memory + instruction
// descriptors. Layout conventions are documented in DESIGN.md §3.
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <cstdlib>

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "paper_1909_02625_b200 kernels target sm_100a only"
#endif

namespace dsp {

typedef __nv_bfloat16 bf16;

__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// ---------------------------------------------------------------- mbarrier
// Last-CTA ticket for fused grid reductions. Every thread of the CTA calls it after
// writing its partials; returns true (CTA-uniformly) in the CTA that arrives last, with
// every other CTA's earlier global writes visible to all of its threads (read them with
// ld.global.cg). One thread fences at gpu scope (release before the ticket, acquire
// after it), the bar.syncs extend the ordering to the rest of the CTA; a per-thread
// __threadfence() (MEMBAR.SC.GPU in every warp) cost 5-7 us per launch here.
// Diagnostics only: dbg bits 1/2/4 skip the release fence / the atomic / the acquire fence
// (results invalid); ts (trace builds) receives globaltimer stamps [0] after the release
// fence, [1] after the atomic returned, [2] after the acquire fence (winner only).
__device__ __forceinline__ bool last_cta_ticket(int* sem, int total, int* flag_smem, int dbg = 0,
                                                int64_t* ts = nullptr) {
  __syncthreads();
  if (threadIdx.x == 0) {
    int old = 0;
    if (!(dbg & 1)) asm volatile("fence.acq_rel.gpu;" ::: "memory");
    if (ts != nullptr) ts[0] = (int64_t)globaltimer_ns();
    if (!(dbg & 2)) asm volatile("atom.relaxed.gpu.global.add.s32 %0, [%1], 1;" : "=r"(old) : "l"(sem) : "memory");
    if (ts != nullptr) ts[1] = (int64_t)globaltimer_ns();
    const int last = old == total - 1;
    if (last && !(dbg & 4)) asm volatile("fence.acq_rel.gpu;" ::: "memory");
    if (ts != nullptr && last) ts[2] = (int64_t)globaltimer_ns();
    *flag_smem = last;
  }
  __syncthreads();
  return *flag_smem != 0;
}

// Fixed-order reduction of per-CTA partial rows part[b][NS][N] (NS statistics per column)
// over columns [w0, w0 + cols), cols % 4 == 0, NS * cols / 4 <= NTH, by the first NTH
// threads: thread = (part p, lane = (statistic, 4-column group)); a lane reads its float4
// of rows b = tile + (p + k * np) * nt (tile = column / BN: only those CTAs own the
// columns), DEPTH rows in flight per batch, into fin4[NTH][4] (smem). part_sums_get()
// then adds the np parts of one column in order. Deterministic: the assignment never
// depends on timing.
template <int DEPTH = 8, int NTH = 256>
__device__ __forceinline__ void part_sums_load(const float* part, int G, int N, int NS, int w0, int cols, int BN,
                                               int nt, double* fin4) {
  const int tid = threadIdx.x;
  const int g4 = cols / 4, lanes = NS * g4, np = NTH / lanes;
  if (tid >= np * lanes) return;
  const int ln = tid % lanes, p0 = tid / lanes;
  const int stat = ln / g4, c = w0 + (ln % g4) * 4;
  const int tile = c / BN;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  for (int b0 = tile + p0 * nt; b0 < G; b0 += DEPTH * np * nt) {
    float4 v[DEPTH];
#pragma unroll
    for (int e = 0; e < DEPTH; ++e) {
      const int b = b0 + e * np * nt;
      v[e] = b < G ? __ldcg(reinterpret_cast<const float4*>(&part[((size_t)b * NS + stat) * N + c]))
                   : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int e = 0; e < DEPTH; ++e) {
      acc[0] += (double)v[e].x;
      acc[1] += (double)v[e].y;
      acc[2] += (double)v[e].z;
      acc[3] += (double)v[e].w;
    }
  }
#pragma unroll
  for (int e = 0; e < 4; ++e) fin4[tid * 4 + e] = acc[e];
}
template <int NTH = 256>
__device__ __forceinline__ double part_sums_get(const double* fin4, int NS, int cols, int cc, int stat) {
  const int g4 = cols / 4, lanes = NS * g4, np = NTH / lanes;
  double s = 0.0;
  for (int p = 0; p < np; ++p) s += fin4[(p * lanes + stat * g4 + cc / 4) * 4 + (cc & 3)];
  return s;
}
// widest column window part_sums_load can cover with NTH threads
__host__ __device__ constexpr int part_sums_window(int NTH, int NS) { return NS <= 2 ? 2 * NTH : NTH; }

// Programmatic dependent launch. Kernels are launched with programmatic stream serialization
// (launch_k below) so a kernel's launch and prologue overlap its predecessor's teardown; every
// kernel calls pdl_wait() before its first global-memory access (reads and writes: the
// predecessor may still be reading). No kernel triggers early (pdl_trigger): successors are
// released as the predecessor's CTAs exit -- early triggers let waiting CTAs occupy SM slots
// the concurrent block streams need (measured, igemm.cu).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }


__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

// Blocking phase wait. The suspend-time hint lets the hardware park the warp
// until the phase flips instead of re-issuing try_wait, which would otherwise
// compete with the producers' cp.async for the MIO pipe.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t"
      ".reg .pred P1;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
      "@P1 bra DONE_%=;\n\t"
      "bra WAIT_%=;\n\t"
      "DONE_%=:\n\t"
      "}" ::"r"(smem_u32(bar)),
      "r"(parity), "r"(0x989680u)
      : "memory");
}

// ---------------------------------------------------------------- cp.async
// 16-byte global->shared copy; src_bytes == 0 zero-fills the destination
// (used for conv padding, ragged tiles and stride-2 dgrad holes).
// .ca: allocate in L1, so the k*k taps of an implicit-GEMM gather re-hit L1.
__device__ __forceinline__ void cp_async_16(uint32_t dst, const void* src, uint32_t src_bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(src_bytes)
               : "memory");
}
// .cg: L2 only (streamed once, e.g. an epilogue's residual rows)
__device__ __forceinline__ void cp_async_16_cg(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
// Arrive (count 1, no pending-count increment) on an mbarrier once every cp.async
// previously issued by this thread has landed in shared memory.
__device__ __forceinline__ void cp_async_arrive_noinc(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// generic-proxy smem writes -> visible to the async proxy (tcgen05.mma operand reads)
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// ---------------------------------------------------------------- tcgen05
__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// D[tmem] (+)= A[smem] * B[smem]^T, kind::f16 (bf16 inputs, fp32 accumulate)
__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n\t"
      ".reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t"
      "}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// D[tmem] (+)= A * B^T, kind::tf32 (fp32 storage, tf32 multiply, fp32 accumulate)
__device__ __forceinline__ void umma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n\t"
      ".reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t"
      "}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// Arrive on an mbarrier once every tcgen05 op previously issued by this thread completes.
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

// 32 TMEM lanes x 16 consecutive 32-bit columns -> 16 registers per thread.
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,"
      "%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// Split form of tmem_ld32: issue the TMEM load, do independent work, then wait. The wait takes the
// destination registers as read-write operands so no use can be scheduled above it.
__device__ __forceinline__ void tmem_ld32_issue(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,"
      "%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld_wait(uint32_t (&r)[32]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;"
               : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]),
                 "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]),
                 "+r"(r[15]), "+r"(r[16]), "+r"(r[17]), "+r"(r[18]), "+r"(r[19]), "+r"(r[20]), "+r"(r[21]),
                 "+r"(r[22]), "+r"(r[23]), "+r"(r[24]), "+r"(r[25]), "+r"(r[26]), "+r"(r[27]), "+r"(r[28]),
                 "+r"(r[29]), "+r"(r[30]), "+r"(r[31])
               :
               : "memory");
}

// UMMA shared-memory descriptor (sm_100 version=1).
//   lbo: byte stride between core matrices along K (SWIZZLE_NONE; 16 for swizzled K-major)
//   sbo: byte stride between 8-row core-matrix groups along M/N
//   layout: 0 SWIZZLE_NONE, 6 SWIZZLE_32B, 4 SWIZZLE_64B, 2 SWIZZLE_128B
__device__ __forceinline__ uint64_t umma_sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout = 0) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version 1 (Blackwell)
  d |= (uint64_t)(layout & 7) << 61;
  return d;
}

// ---------------------------------------------------------------- TMA
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void tma_load_4d(uint32_t dst, const void* tmap, uint64_t* bar, int c0, int c1, int c2,
                                            int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], "
      "[%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}
// im2col-mode 4-D load (NHWC): pixelsPerColumn output pixels starting at input position
// (w, h, n) (the traversal walks W, then H, then N inside the tensor map's bounding box),
// each pixel's channels [c, c + channelsPerPixel) read at (h + oh, w + ow); OOB reads are 0.
__device__ __forceinline__ void tma_load_im2col_4d(uint32_t dst, const void* tmap, uint64_t* bar, int c, int w, int h,
                                                   int n, uint16_t ow, uint16_t oh) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.im2col.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, "
      "%6}], [%2], {%7, %8};" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(smem_u32(bar)), "r"(c), "r"(w), "r"(h), "r"(n), "h"(ow), "h"(oh)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const void* tmap, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          dst),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
// TMA tensor store smem -> global (bulk-group completion), and its waits.
__device__ __forceinline__ void tma_store_2d(const void* tmap, uint32_t src, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(tmap), "r"(src),
               "r"(c0), "r"(c1)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read1() { asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

__device__ __forceinline__ void tma_prefetch_desc(const void* tmap) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(tmap)) : "memory");
}

// Instruction descriptor: fp32 accumulate, A/B format fmt (1 = bf16, 2 = tf32),
// a_mn / b_mn = operand is MN-major in smem, M x N tile.
__host__ __device__ __forceinline__ uint32_t umma_idesc(uint32_t fmt, uint32_t a_mn, uint32_t b_mn, uint32_t M,
                                                        uint32_t N) {
  uint32_t d = 0;
  d |= 1u << 4;             // c_format = F32
  d |= (fmt & 7u) << 7;     // a_format
  d |= (fmt & 7u) << 10;    // b_format
  d |= (a_mn & 1u) << 15;   // a_major
  d |= (b_mn & 1u) << 16;   // b_major
  d |= ((N >> 3) & 63u) << 17;
  d |= ((M >> 4) & 31u) << 24;
  return d;
}

// ---------------------------------------------------------------- fast division
// n / d for 0 <= n < 2^31 as umulhi(n, mul) >> shr (Granlund-Montgomery, as
// CUTLASS FastDivmod): the implicit-GEMM gathers decode pixel / tap indices per
// 16-byte chunk, and runtime 32-bit division would dominate the producer warps.
struct FastDiv {
  uint32_t d, mul, shr;
  __device__ __forceinline__ void init(uint32_t div) {
    d = div;
    if (div <= 1) {
      mul = 0;
      shr = 0;
    } else {
      uint32_t l = 0;  // ceil(log2(div))
      while ((1u << l) < div) ++l;
      const uint32_t p = 31 + l;  // 2^p / div < 2^32 since div > 2^(l-1)
      mul = (uint32_t)((((uint64_t)1 << p) + div - 1) / div);
      shr = p - 32;
    }
  }
  __device__ __forceinline__ int div(int n) const {
    return d <= 1 ? n : (int)(__umulhi((uint32_t)n, mul) >> shr);
  }
  __device__ __forceinline__ int divmod(int n, int& rem) const {
    const int q = div(n);
    rem = n - q * (int)d;
    return q;
  }
};

// ---------------------------------------------------------------- misc
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <typename T>
__device__ __forceinline__ float to_f(T v);
template <>
__device__ __forceinline__ float to_f<float>(float v) { return v; }
template <>
__device__ __forceinline__ float to_f<bf16>(bf16 v) { return __bfloat162float(v); }

template <typename T>
__device__ __forceinline__ T from_f(float v);
template <>
__device__ __forceinline__ float from_f<float>(float v) { return v; }
template <>
__device__ __forceinline__ bf16 from_f<bf16>(float v) { return __float2bfloat16_rn(v); }

// Kernel launch with programmatic stream serialization (see pdl_wait); DSP_B200_PDL=0 turns it
// off (plain stream order). Captured into CUDA graphs as programmatic edges.
inline bool pdl_enabled() {
  static const int on = [] {
    const char* e = getenv("DSP_B200_PDL");
    return (e == nullptr || e[0] != '0') ? 1 : 0;
  }();
  return on != 0;
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                            Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

}  // namespace dsp
