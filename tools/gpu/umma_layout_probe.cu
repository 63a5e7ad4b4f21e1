// Probe how tcgen05.mma kind::tf32 reads an MN-major (transposed) shared-memory operand.
//
// A (128 x 8, tf32) is filled with its own word indices (A_smem[w] = w, exact in tf32 for w < 2048)
// and read through a descriptor with the given layout / LBO / SBO; B (N x 8) is K-major with
// B[n][k] = (k == n) for n < 8 (the known-good layout of the FPROP path), so D[m][n] = the smem
// word the tensor core took as A[m][k = n].  The B probe swaps the roles.
//   nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -I../../paper_1909_02625_b200/csrc \
//        umma_layout_probe.cu -o umma_probe && ./umma_probe
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "common.cuh"

using namespace dsp;

// which: 0 = probe A (A MN-major, B K-major one-hot), 1 = probe B (A K-major one-hot, B MN-major)
__global__ void probe(float* out, int which, uint32_t lbo, uint32_t sbo, uint32_t layout, int N) {
  __shared__ __align__(1024) float sA[128 * 8 * 4];  // 16 KB: words past the 4 KB tile read as -1
  __shared__ __align__(1024) float sB[256 * 8 * 2];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5;
  // known-good K-major SWIZZLE_NONE: row r, chunk j (4 K elements) at j * (rows * 16) + r * 16
  for (int i = tid; i < 128 * 8 * 4; i += blockDim.x) sA[i] = -1.f;
  for (int i = tid; i < 256 * 8 * 2; i += blockDim.x) sB[i] = -1.f;
  __syncthreads();
  if (which == 0 || which == 2) {
    for (int i = tid; i < 128 * 8; i += blockDim.x) sA[i] = (float)i;
    for (int i = tid; i < N * 8; i += blockDim.x) {
      const int j = i / (N * 4), rem = i % (N * 4), r = rem / 4, e = rem % 4;  // word -> (chunk, row, elem)
      const int k = j * 4 + e;
      sB[i] = (k == r) ? 1.f : 0.f;
    }
  } else {
    for (int i = tid; i < N * 8; i += blockDim.x) sB[i] = (float)i;  // N x 8 = 128 words
    for (int i = tid; i < 128 * 8; i += blockDim.x) {
      const int j = i / (128 * 4), rem = i % (128 * 4), r = rem / 4, e = rem % 4;
      const int k = j * 4 + e;
      sA[i] = (k == (r & 7)) ? 1.f : 0.f;  // D[m][n] = B[n][m & 7]
    }
  }
  fence_proxy_async_smem();
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc(&tbase, 256);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (tid == 0) {
    const uint32_t a = smem_u32(sA), b = smem_u32(sB);
    uint64_t ad, bd;
    uint32_t idesc;
    if (which == 2) {  // control: both K-major (the FPROP layout)
      ad = umma_sdesc(a, 128 * 16, 128, 0);
      bd = umma_sdesc(b, N * 16, 128, 0);
      idesc = umma_idesc(2, 0, 0, 128, N);
    } else if (which == 0) {
      ad = umma_sdesc(a, lbo, sbo, layout);
      bd = umma_sdesc(b, N * 16, 128, 0);
      idesc = umma_idesc(2, 1, 0, 128, N);
    } else {
      ad = umma_sdesc(a, 128 * 16, 128, 0);
      bd = umma_sdesc(b, lbo, sbo, layout);
      idesc = umma_idesc(2, 0, 1, 128, N);
    }
    umma_tf32(tbase, ad, bd, idesc, 0u);
    umma_commit(&bar);
  }
  __syncwarp();
  mbar_wait(&bar, 0);
  tc_fence_after();
  if (warp < 4) {
    for (int c = 0; c < N; c += 16) {
      float v[16];
      tmem_ld16(tbase + ((uint32_t)(warp * 32) << 16) + c, v);
      for (int e = 0; e < 16; ++e) out[(warp * 32 + (tid & 31)) * N + c + e] = v[e];
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tbase, 256);
  }
}

int main(int argc, char** argv) {
  const int N = 16;
  float* d;
  cudaMalloc(&d, 128 * N * sizeof(float));
  std::vector<float> h(128 * N);
  struct V { const char* name; uint32_t lbo, sbo, layout; };
  // A MN-major 128 x 8: our layout has MN groups (4 elems, 16 B) at +128 B, K groups (8 rows) at +4096
  V va[] = {{"SW128_BASE32B lbo=512 sbo=2048", 512, 2048, 1}, {"SW128_BASE32B lbo=2048 sbo=512", 2048, 512, 1},
            {"SW128 lbo=1024 sbo=4096", 1024, 4096, 2}, {"SW128 lbo=4096 sbo=1024", 4096, 1024, 2},
            {"SW64 lbo=512 sbo=4096", 512, 4096, 4}, {"SW32 lbo=256 sbo=4096", 256, 4096, 6}};
  for (int which : {0, 1}) {
    printf("==== probe %s\n", which == 2 ? "control (K-major A words)" : which == 0 ? "A MN-major" : "B MN-major");
    for (auto& v : va) {
      cudaMemset(d, 0, 128 * N * sizeof(float));
      probe<<<1, 128>>>(d, which, v.lbo, v.sbo, v.layout, N);
      cudaError_t e = cudaDeviceSynchronize();
      cudaMemcpy(h.data(), d, h.size() * 4, cudaMemcpyDeviceToHost);
      printf("%s: %s\n", v.name, cudaGetErrorString(e));
      if (e != cudaSuccess) return 1;
      // A probe: row m, col n<8 = word read for A[m][k=n]; B probe: row m<8: D[m][n] = word read for B[n][k=m]
      if (which != 1) {
        for (int m : {0, 1, 2, 3, 4, 5, 31, 32, 127}) {
          printf("  A[%3d][k=0..7] <- words", m);
          for (int k = 0; k < 8; ++k) printf(" %5.0f", h[m * N + k]);
          printf("\n");
        }
      } else {
        for (int n : {0, 1, 2, 3, 4, 5, 15}) {
          printf("  B[%3d][k=0..7] <- words", n);
          for (int k = 0; k < 8; ++k) printf(" %5.0f", h[k * N + n]);
          printf("\n");
        }
      }
    }
  }
  return 0;
}
