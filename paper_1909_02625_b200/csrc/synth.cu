// On-device synthetic data supply.
//
// The reference's counter-based splitmix64 stream (/root/reference/pkg/src/stalepipe/rng.py:
// 47-88) is trivially parallel: draw t of a stream is a pure function of (seed, t). So batch i
// of the benchmark pool synthetic_batches(n, B, shape, C, seed) (SURVEY.md §8d:
// x ~ SeededRng(seed).normal, labels = floor(SeededRng(derive_seed(seed, 1)).uniform * C))
// is generated straight into its packed bf16 NHWC device slot -- no host generation, no H2D.
//   x stream: batch i starts at raw draw i * 2*ceil(B*D/2) (normal() consumes whole pairs);
//   element j (NCHW flat within the batch) is Box-Muller pair j/2, cos for even j, sin for odd.
//   labels:   batch i starts at raw draw i * B of the derived stream.
// Integer work is bit-exact; the Box-Muller transcendental math runs in fp64 like numpy and is
// then rounded fp64 -> fp32 -> bf16 exactly as the host path (np.float32 + pack) does, so the
// stored inputs equal the host pipeline's (tests/test_synth_gpu.py).
#include "abi_internal.h"
#include "common.cuh"
#include "kernels.cuh"

#include <cuda_runtime.h>

#include <algorithm>

namespace dsp {
namespace {

constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ull;

__device__ __forceinline__ uint64_t splitmix(uint64_t seed, uint64_t t) {  // draw t (0-based)
  uint64_t z = seed + (t + 1) * kGolden;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__device__ __forceinline__ double u53(uint64_t z) { return (double)(z >> 11) * 0x1.0p-53; }

template <typename T>
__global__ void synth_x_k(uint64_t seed, uint64_t base, int B, int C, int H, int W, int Cp, T* __restrict__ out) {
  pdl_wait();  // predecessor complete before any global access (successors launch at exit)
  const int64_t n = (int64_t)B * H * W * Cp;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(i % Cp);
    int64_t t = i / Cp;
    const int w = (int)(t % W);
    t /= W;
    const int h = (int)(t % H);
    const int b = (int)(t / H);
    float v = 0.f;
    if (c < C) {
      const int64_t j = (((int64_t)b * C + c) * H + h) * W + w;  // NCHW index within the batch
      const uint64_t p = (uint64_t)(j >> 1);
      double u1 = u53(splitmix(seed, base + 2 * p));
      const double u2 = u53(splitmix(seed, base + 2 * p + 1));
      if (u1 == 0.0) u1 = 0x1.0p-53;  // log(0) guard (rng.py:80)
      const double r = sqrt(-2.0 * log(u1));
      const double theta = 2.0 * 3.141592653589793 * u2;
      v = (float)(r * ((j & 1) ? sin(theta) : cos(theta)));
    }
    out[i] = from_f<T>(v);
  }
}

__global__ void synth_labels_k(uint64_t seed, uint64_t base, int B, int C, int64_t* __restrict__ out) {
  pdl_wait();  // predecessor complete before any global access (successors launch at exit)
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  const double u = u53(splitmix(seed, base + (uint64_t)b));
  int64_t l = (int64_t)(u * (double)C);
  out[b] = l < C - 1 ? l : C - 1;
}

// Straggler injection: one thread spins on %globaltimer for ns nanoseconds on the stream.
__global__ void device_sleep_k(int64_t ns) {
  pdl_wait();
  const uint64_t t0 = globaltimer_ns();
  while ((int64_t)(globaltimer_ns() - t0) < ns) __nanosleep(256);
}

uint64_t mix64_host(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

}  // namespace
}  // namespace dsp

using namespace dsp;

extern "C" int dsp_synth_batch(uint64_t seed, int64_t batch_no, int batch, int c, int h, int w, int c_pad,
                               int num_classes, int dtype, void* act_out, int64_t* labels_out, void* stream) {
  if (batch <= 0 || c <= 0 || h <= 0 || w <= 0 || c_pad < c || c_pad % 8 || num_classes <= 0 || batch_no < 0 ||
      (!act_out && !labels_out))
    return set_error(DSP_E_INVALID, "dsp_synth_batch: bad arguments");
  if (dtype != DSP_DTYPE_BF16 && dtype != DSP_DTYPE_F32) return set_error(DSP_E_INVALID, "dsp_synth_batch: bad dtype");
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t width = (int64_t)c * h * w;
  const uint64_t draws_per_batch = 2ull * (uint64_t)((batch * width + 1) / 2);
  if (act_out) {
    const int64_t n = (int64_t)batch * h * w * c_pad;
    const int grid = (int)std::min<int64_t>((n + 255) / 256, 148 * 16);
    if (dtype == DSP_DTYPE_BF16)
      launch_k(synth_x_k<bf16>, grid, 256, 0, st, seed, (uint64_t)batch_no * draws_per_batch, batch, c, h, w, c_pad,
                                           (bf16*)act_out);
    else
      launch_k(synth_x_k<float>, grid, 256, 0, st, seed, (uint64_t)batch_no * draws_per_batch, batch, c, h, w, c_pad,
                                            (float*)act_out);
    note_launch();
    DSP_CUDA(cudaGetLastError());
  }
  if (labels_out) {
    const uint64_t lseed = mix64_host(seed + kGolden * 2ull);  // derive_seed(seed, 1) (rng.py:38-44)
    launch_k(synth_labels_k, (batch + 255) / 256, 256, 0, st, lseed, (uint64_t)batch_no * batch, batch, num_classes,
                                                        labels_out);
    note_launch();
    DSP_CUDA(cudaGetLastError());
  }
  return DSP_OK;
}

extern "C" int dsp_device_sleep(int64_t ns, void* stream) {
  if (ns < 0) return set_error(DSP_E_INVALID, "dsp_device_sleep: negative duration");
  if (ns == 0) return DSP_OK;
  DSP_CUDA(launch_k(device_sleep_k, 1, 1, 0, (cudaStream_t)stream, ns));
  note_launch();
  return DSP_OK;
}
