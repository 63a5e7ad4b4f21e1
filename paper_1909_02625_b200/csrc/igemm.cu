// Implicit-GEMM launch dispatch (the kernels live in igemm_kern.cuh; their launchers are
// instantiated one (MODE, BN) per translation unit by _build.py so the library compiles in
// parallel).
#include "common.cuh"
#include "kernels.cuh"
#include "../../include/dsp_b200.h"

#include <cstdlib>

namespace dsp {

template <typename T, int MODE, int BN>
cudaError_t launch_bn(const dsp_igemm_args_t& a, int splits, cudaStream_t st);
template <typename T, int MODE>
static cudaError_t launch_mode(const dsp_igemm_args_t& a, int splits, cudaStream_t st) {
  if (a.N <= 16) return launch_bn<T, MODE, 16>(a, splits, st);
  if (a.N <= 32) return launch_bn<T, MODE, 32>(a, splits, st);
  if (a.N <= 64) return launch_bn<T, MODE, 64>(a, splits, st);
  if (a.N <= 128) return launch_bn<T, MODE, 128>(a, splits, st);
  // short-K FPROP / DGRAD (1x1 convs over <= 128 channels) are epilogue-bound: 128-wide tiles at
  // two CTAs per SM give each SM twice the epilogue warps of one 256-wide CTA
  static const bool wide = getenv("DSP_B200_SHORTK_WIDE") != nullptr;
  if (!wide && MODE != DSP_IGEMM_WGRAD && a.Kd <= 128) return launch_bn<T, MODE, 128>(a, splits, st);
  // DGRADs with a residual or fused BN-backward statistics are epilogue-bound up to Kd = 512: 128-wide
  // tiles at two CTAs per SM (ResNet-50 unit-input DGRADs: stage 3 116 -> 105 us, stage 4 75 -> 67 us;
  // the Kd = 1024 reduce-conv DGRAD gets slower, 58 -> 64 us). DSP_B200_DGRAD_BN128_KD overrides.
  static const int dg_kd = getenv("DSP_B200_DGRAD_BN128_KD") ? atoi(getenv("DSP_B200_DGRAD_BN128_KD")) : 512;
  if (MODE == DSP_IGEMM_DGRAD && a.Kd <= dg_kd && (a.residual != nullptr || a.bnb_count > 0))
    return launch_bn<T, MODE, 128>(a, splits, st);
  return launch_bn<T, MODE, 256>(a, splits, st);
}

// Live-duration probe (bench.py roofline): CUDA event pairs around the launches of one shape.
struct Probe {
  int mode = -1, n = 0;
  int64_t m = 0;
  cudaEvent_t* ev = nullptr;
  int npairs = 0, next = 0;
};
static Probe g_probe;

static cudaError_t igemm_dispatch(int mode, int dtype, const dsp_igemm_args_t& a, int splits, cudaStream_t st);

cudaError_t igemm_launch(int mode, int dtype, const dsp_igemm_args_t& a, int splits, cudaStream_t st) {
  Probe& p = g_probe;
  // probe key: mode (low 8 bits of p.mode), N, M and, when bits 8+ are set, Kd
  if (p.ev == nullptr || mode != (p.mode & 0xff) || a.N != p.n || a.M != p.m || p.next >= p.npairs ||
      ((p.mode >> 8) != 0 && a.Kd != (p.mode >> 8)))
    return igemm_dispatch(mode, dtype, a, splits, st);
  const int i = p.next++;
  // while capturing, External makes an event-record node that fires on every replay (a plain
  // record would only be a capture-internal dependency); the flag is illegal outside capture
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaError_t e = cudaStreamIsCapturing(st, &cs);
  if (e != cudaSuccess) return e;
  const unsigned flags = cs == cudaStreamCaptureStatusActive ? cudaEventRecordExternal : cudaEventRecordDefault;
  e = cudaEventRecordWithFlags(p.ev[2 * i], st, flags);
  if (e != cudaSuccess) return e;
  e = igemm_dispatch(mode, dtype, a, splits, st);
  if (e != cudaSuccess) return e;
  return cudaEventRecordWithFlags(p.ev[2 * i + 1], st, flags);
}

int probe_arm(int mode, int n, int64_t m, void* const* events, int n_pairs) {
  g_probe = Probe{};
  if (events == nullptr || n_pairs <= 0) return 0;
  g_probe.mode = mode;
  g_probe.n = n;
  g_probe.m = m;
  g_probe.ev = reinterpret_cast<cudaEvent_t*>(const_cast<void**>(events));
  g_probe.npairs = n_pairs;
  return 0;
}
int probe_reset() {
  const int k = g_probe.next;
  g_probe.next = 0;
  return k;
}

static cudaError_t igemm_dispatch(int mode, int dtype, const dsp_igemm_args_t& a, int splits, cudaStream_t st) {
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
