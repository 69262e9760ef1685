// Write-bandwidth ceilings on B200 for the pass-through's output pattern (profiles/README.md):
// the full representation is ~0.91 of the pass-through's bytes and is almost all written, so
// copy bandwidth (read+write) is not the only meaningful ceiling. Measures, over 1 GiB:
//   memset    cudaMemsetAsync
//   st.v4     plain 16-B vector stores, grid-stride, 148 x 8 blocks of 256 threads
//   bulk      one warp per block, each warp TMA-bulk-stores 15 KB chunks (the pass-through's
//             group image at k = 20) from shared memory, 13 blocks per SM, wait_group.read
//             between chunks (as merge_fast does before re-zeroing its image)
//   copy      cudaMemcpyAsync D2D of 1 GiB (read + write bytes), the MEASURED_PEAKS recipe
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o write_probe profiles/write_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void st_v4(float4* p, size_t n) {
  const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) p[i] = z;
}

template <int CH>
__global__ void __launch_bounds__(32) bulk(char* p, size_t nchunks) {
  extern __shared__ __align__(128) char sm[];
  for (int i = threadIdx.x; i < CH / 16; i += 32) reinterpret_cast<float4*>(sm)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  __syncwarp();
  for (size_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
    if (threadIdx.x == 0) {
      asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(p + c * CH),
                   "r"((uint32_t)__cvta_generic_to_shared(sm)), "r"(CH)
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
    }
    __syncwarp();
  }
  if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
}

// the same 15 KB chunks written by the warp itself: ld.shared.v4 + st.global.v4 (512 B per warp store)
template <int CH>
__global__ void __launch_bounds__(32) lsu(char* p, size_t nchunks) {
  extern __shared__ __align__(128) char sm[];
  float4* s4 = reinterpret_cast<float4*>(sm);
  for (int i = threadIdx.x; i < CH / 16; i += 32) s4[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  __syncwarp();
  for (size_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
    float4* d = reinterpret_cast<float4*>(p + c * CH);
#pragma unroll 8
    for (int i = threadIdx.x; i < CH / 16; i += 32) d[i] = s4[i];
  }
}

// the pass-through's mix: per 15 KB chunk, first 1776 B of records (74 records x 24 B) are read into
// shared memory with cp.async (LDGSTS) and waited for, then the chunk is bulk-stored (reads ~11.6 %
// of the bytes, as merge_fast's 92 MB per 941 MB written)
template <int CH, int RB>
__global__ void __launch_bounds__(32) bulk_ld(char* p, const char* q, size_t nchunks) {
  extern __shared__ __align__(128) char sm[];
  for (int i = threadIdx.x; i < (CH + RB) / 16; i += 32) reinterpret_cast<float4*>(sm)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  __syncwarp();
  const uint32_t st = (uint32_t)__cvta_generic_to_shared(sm + CH);
  for (size_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
    for (int i = threadIdx.x; i < RB / 16; i += 32)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(st + i * 16), "l"(q + c * RB + i * 16) : "memory");
    asm volatile("cp.async.wait_all;\n" ::: "memory");
    __syncwarp();
    if (threadIdx.x == 0) {
      asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(p + c * CH),
                   "r"((uint32_t)__cvta_generic_to_shared(sm)), "r"(CH)
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
    }
    __syncwarp();
  }
  if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
}

static float time_it(void (*f)(void*), void* a, cudaStream_t s, int reps) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    cudaEventRecord(e0, s);
    f(a);
    cudaEventRecord(e1, s);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (r && ms < best) best = ms;  // first rep is warm-up
  }
  return best;
}

struct Args { char* p; char* q; size_t bytes; cudaStream_t s; };

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e_)); return 1; } } while (0)
int main() {
  setvbuf(stdout, nullptr, _IONBF, 0);
  const size_t bytes = 1ull << 30;
  Args a;
  a.bytes = bytes;
  CK(cudaMalloc(&a.p, bytes));
  CK(cudaMalloc(&a.q, bytes));
  CK(cudaStreamCreate(&a.s));
  const int reps = 11;
  float t;
  t = time_it([](void* v) { Args* a = (Args*)v; cudaMemsetAsync(a->p, 0, a->bytes, a->s); }, &a, a.s, reps);
  printf("memset   %.4f ms  %.1f GB/s (write)\n", t, bytes / t / 1e6);
  t = time_it([](void* v) { Args* a = (Args*)v; st_v4<<<148 * 8, 256, 0, a->s>>>((float4*)a->p, a->bytes / 16); }, &a, a.s, reps);
  printf("st.v4    %.4f ms  %.1f GB/s (write)\n", t, bytes / t / 1e6);
  cudaFuncSetAttribute(bulk<15360>, cudaFuncAttributeMaxDynamicSharedMemorySize, 15360);
  t = time_it([](void* v) { Args* a = (Args*)v; bulk<15360><<<148 * 13, 32, 15360, a->s>>>(a->p, a->bytes / 15360); }, &a, a.s, reps);
  printf("bulk15K  %.4f ms  %.1f GB/s (write, 13 warps/SM, wait.read per chunk)\n", t, (a.bytes / 15360) * 15360.0 / t / 1e6);
  for (int wps : {4, 8, 13}) {
    static int W;
    W = wps;
    t = time_it([](void* v) { Args* a = (Args*)v; bulk<15360><<<148 * W, 32, 15360, a->s>>>(a->p, a->bytes / 15360); }, &a, a.s, reps);
    printf("bulk15K  %.4f ms  %.1f GB/s (write, %d warps/SM)\n", t, (a.bytes / 15360) * 15360.0 / t / 1e6, wps);
  }
  cudaFuncSetAttribute(lsu<15360>, cudaFuncAttributeMaxDynamicSharedMemorySize, 15360);
  for (int wps : {4, 8, 13}) {
    static int W;
    W = wps;
    t = time_it([](void* v) { Args* a = (Args*)v; lsu<15360><<<148 * W, 32, 15360, a->s>>>(a->p, a->bytes / 15360); }, &a, a.s, reps);
    printf("lsu15K   %.4f ms  %.1f GB/s (write, ld.shared + st.global.v4, %d warps/SM)\n", t, (a.bytes / 15360) * 15360.0 / t / 1e6, wps);
  }
  cudaFuncSetAttribute(bulk_ld<15360, 1776>, cudaFuncAttributeMaxDynamicSharedMemorySize, 15360 + 1776);
  for (int wps : {4, 8, 13}) {
    static int W;
    W = wps;
    t = time_it([](void* v) { Args* a = (Args*)v; bulk_ld<15360, 1776><<<148 * W, 32, 15360 + 1776, a->s>>>(a->p, a->q, a->bytes / 15360); }, &a, a.s, reps);
    const double nch = (double)(a.bytes / 15360);
    printf("bulk+ld  %.4f ms  %.1f GB/s (write %.1f + read %.1f, %d warps/SM)\n", t, nch * (15360.0 + 1776.0) / t / 1e6,
           nch * 15360.0 / t / 1e6, nch * 1776.0 / t / 1e6, wps);
  }
  t = time_it([](void* v) { Args* a = (Args*)v; cudaMemcpyAsync(a->q, a->p, a->bytes, cudaMemcpyDeviceToDevice, a->s); }, &a, a.s, reps);
  printf("copy     %.4f ms  %.1f GB/s (read+write)\n", t, 2.0 * bytes / t / 1e6);
  cudaError_t e = cudaDeviceSynchronize();
  printf("status %s\n", cudaGetErrorString(e));
  return e != cudaSuccess;
}
