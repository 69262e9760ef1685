// NVLink ceiling of the exchange's SM-driven peer stores (profiles/README.md): GPU 0 pushes N bytes
// into GPU 1's memory with the push kernel's copy loop (16-B vectors, 8 loads in flight per thread,
// 1184 blocks of 256 threads, plain stores to the peer through UVA), one direction and both at once;
// the copy engines (cudaMemcpyPeerAsync) beside it.  Sizes span the C3 exchange slice (~29 MB per
// rank per VDI at N = 2) to 1 GiB.  Needs two GPUs with peer access.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o nvlink_probe profiles/nvlink_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(256, 4) push(const uint4* __restrict__ s, uint4* __restrict__ d, size_t n) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 7 * stride < n; i += 8 * stride) {
    uint4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = __ldg(s + i + u * stride);
#pragma unroll
    for (int u = 0; u < 8; ++u) d[i + u * stride] = v[u];
  }
  for (; i < n; i += stride) d[i] = __ldg(s + i);
}

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e_)); return 1; } } while (0)

int main() {
  setvbuf(stdout, nullptr, _IONBF, 0);
  int ng = 0;
  CK(cudaGetDeviceCount(&ng));
  if (ng < 2) { printf("needs 2 GPUs\n"); return 1; }
  const size_t maxb = 1ull << 30;
  char *src[2], *dst[2];
  cudaStream_t st[2];
  cudaEvent_t e0[2], e1[2];
  for (int g = 0; g < 2; ++g) {
    CK(cudaSetDevice(g));
    CK(cudaDeviceEnablePeerAccess(1 - g, 0));
    CK(cudaMalloc(&src[g], maxb));
    CK(cudaMalloc(&dst[g], maxb));
    CK(cudaMemset(src[g], 1, maxb));
    CK(cudaStreamCreateWithFlags(&st[g], cudaStreamNonBlocking));
    CK(cudaEventCreate(&e0[g]));
    CK(cudaEventCreate(&e1[g]));
  }
  const size_t sizes[] = {8ull << 20, 32ull << 20, 128ull << 20, 512ull << 20, 1ull << 30};
  for (int mode = 0; mode < 4; ++mode) {  // 0: SM push 0->1; 1: SM push both ways; 2: CE 0->1; 3: CE both ways
    const char* names[] = {"SM push, one direction", "SM push, both directions", "copy engine, one direction",
                           "copy engine, both directions"};
    for (size_t b : sizes) {
      float best = 1e30f;
      for (int rep = 0; rep < 6; ++rep) {
        const int ndir = (mode == 1 || mode == 3) ? 2 : 1;
        for (int g = 0; g < ndir; ++g) { CK(cudaSetDevice(g)); CK(cudaDeviceSynchronize()); }
        for (int g = 0; g < ndir; ++g) {
          CK(cudaSetDevice(g));
          CK(cudaEventRecord(e0[g], st[g]));
          if (mode < 2) push<<<148 * 8, 256, 0, st[g]>>>((const uint4*)src[g], (uint4*)dst[1 - g], b / 16);
          else CK(cudaMemcpyPeerAsync(dst[1 - g], 1 - g, src[g], g, b, st[g]));
          CK(cudaEventRecord(e1[g], st[g]));
        }
        float ms = 0.f;
        for (int g = 0; g < ndir; ++g) {
          CK(cudaSetDevice(g));
          CK(cudaEventSynchronize(e1[g]));
          float t;
          CK(cudaEventElapsedTime(&t, e0[g], e1[g]));
          if (t > ms) ms = t;
        }
        if (rep && ms < best) best = ms;
      }
      printf("%-30s %5zu MiB  %.4f ms  %.1f GB/s per direction\n", names[mode], b >> 20, best, b / best / 1e6);
    }
  }
  printf("status ok\n");
  return 0;
}
