// render.cu — the limit case of the compositing and the VDI renderers
// (sm_100a, fp32, -fmad=false, explicit fmaf).
//
//   image_kernel      : the non-convex plain-image limit case:
//                       with one S~ per sub-domain intersection, the
//                       compositing places a list's S~ in depth order
//                        and over-composites along the list;
//   gen_view_kernel   : a full-representation VDI rendered from its
//                       generation viewpoint -- over of each list's
//                       supersegments, exact by associativity;
//   novel_view_kernel : a VDI rendered from another viewpoint (PAPER.md:213,
//                       :364): rays of the new camera are marched through the
//                       volume's box one voxel per step; each sample is
//                       projected into the generation camera, the
//                       supersegment of the nearest list that contains its
//                       depth is looked up, and contributes its opacity
//                       adjusted to the step length, 1 - (1 - a)^(dt / L)
//                       with L the supersegment's length (Eq. 2),
//                       and its colour scaled alike.
#include <cuda_runtime.h>
#include <math_constants.h>

#include "internal.h"
#include "render.h"

namespace vdi {

__device__ __forceinline__ void over_acc(float4& acc, float r, float g, float b, float a) {
  const float tr = 1.0f - acc.w;
  acc.x = fmaf(tr, r, acc.x);
  acc.y = fmaf(tr, g, acc.y);
  acc.z = fmaf(tr, b, acc.z);
  acc.w = fmaf(tr, a, acc.w);
}

// Limit case: a warp per 32 consecutive lists, lane = list.  Each source's
// first record of the lane's list comes from its group base (offset array,
// pushed group bases, or the receive-side scan -- as in merge_fast) plus a
// warp scan of the counts; the n sources' runs are merged by their head
// t_front (ties: lower PE id, Q11) and over-composited in that order.
__device__ __forceinline__ uint32_t warp_excl(uint32_t v, int lane) {
  uint32_t x = v;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t t = __shfl_up_sync(0xffffffffu, x, d);
    if (lane >= d) x += t;
  }
  return x - v;
}

__global__ void __launch_bounds__(128) image_kernel(MergeParams mp, float4* __restrict__ out) {
  const int n = mp.n_src, lane = threadIdx.x & 31;
  const uint32_t nw = gridDim.x * (blockDim.x >> 5);
  for (uint32_t g = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); g < mp.n_groups; g += nw) {
    const uint32_t p = g * 32 + lane;
    uint32_t pos[VDI_MAX_SRC], end[VDI_MAX_SRC];
    for (int s = 0; s < n; ++s) {
      const SrcDesc& sd = mp.src[s];
      const uint32_t c = p < mp.P ? __ldg(sd.count + p) : 0u;
      const uint32_t base = sd.offset ? __ldg(sd.offset + (size_t)g * 32)
                                      : sd.gbase ? __ldg(sd.gbase + g) : __ldg(mp.group_base + (size_t)s * mp.n_groups + g);
      pos[s] = base + warp_excl(c, lane);
      end[s] = pos[s] + c;
    }
    if (p >= mp.P) continue;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (;;) {
      int best = -1;
      float bt = 0.f;
      for (int s = 0; s < n; ++s)
        if (pos[s] < end[s]) {
          const float t = __ldg(&mp.src[s].depth[pos[s]].x);
          if (best < 0 || t < bt) {
            best = s;
            bt = t;
          }
        }
      if (best < 0) break;
      const float4 c = __ldg(mp.src[best].rgba + pos[best]);
      ++pos[best];
      over_acc(acc, c.x, c.y, c.z, c.w);
    }
    out[p] = acc;
  }
}

// Generation-view render of a full-representation VDI: over of each list
__global__ void __launch_bounds__(128) gen_view_kernel(const uint8_t* __restrict__ count,
                                                       const float4* __restrict__ rgba, uint32_t P, int k,
                                                       float4* __restrict__ out) {
  for (uint32_t p = blockIdx.x * blockDim.x + threadIdx.x; p < P; p += gridDim.x * blockDim.x) {
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    const uint32_t c = count[p];
    for (uint32_t j = 0; j < c; ++j) {
      const float4 s = __ldg(rgba + (size_t)p * k + j);
      over_acc(acc, s.x, s.y, s.z, s.w);
    }
    out[p] = acc;
  }
}

__device__ __forceinline__ float dot3(const float* a, const float* b) { return fmaf(a[2], b[2], fmaf(a[1], b[1], a[0] * b[0])); }

__global__ void __launch_bounds__(128) novel_view_kernel(NovelParams np) {
  const uint32_t P = np.W_out * np.H_out;
  for (uint32_t p = blockIdx.x * blockDim.x + threadIdx.x; p < P; p += gridDim.x * blockDim.x) {
    const int x = (int)(p % np.W_out), y = (int)(p / np.W_out);
    // ray of the new camera through the pixel centre (DESIGN.md §4 camera)
    const float sx = ((2.0f * ((float)x + 0.5f)) / (float)np.W_out - 1.0f) * np.view.tan_x;
    const float sy = (1.0f - (2.0f * ((float)y + 0.5f)) / (float)np.H_out) * np.view.tan_y;
    float d[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) d[c] = (np.view.fwd[c] + sx * np.view.right[c]) + sy * np.view.up[c];
    const float len = sqrtf((d[0] * d[0] + d[1] * d[1]) + d[2] * d[2]);
#pragma unroll
    for (int c = 0; c < 3; ++c) d[c] /= len;
    float tmin = 0.0f, tmax = CUDART_INF_F;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const float t0 = (-np.half[c] - np.view.eye[c]) / d[c];
      const float t1 = (np.half[c] - np.view.eye[c]) / d[c];
      tmin = fmaxf(tmin, fminf(t0, t1));
      tmax = fminf(tmax, fmaxf(t0, t1));
    }
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    if (tmax > tmin) {
      for (int i = 0;; ++i) {
        const float t = tmin + ((float)i + 0.5f) * np.dt;
        if (!(t < tmax)) break;
        float v[3];
#pragma unroll
        for (int c = 0; c < 3; ++c) v[c] = (np.view.eye[c] + t * d[c]) - np.gen.eye[c];
        const float a = dot3(v, np.gen.fwd);
        if (!(a > 0.0f)) continue;
        const float gx = dot3(v, np.gen.right) / a, gy = dot3(v, np.gen.up) / a;
        const float fx = (gx / np.gen.tan_x + 1.0f) * 0.5f * (float)np.W - 0.5f;
        const float fy = (1.0f - gy / np.gen.tan_y) * 0.5f * (float)np.H - 0.5f;
        const int lx = (int)rintf(fx), ly = (int)rintf(fy);
        if (lx < 0 || ly < 0 || lx >= (int)np.W || ly >= (int)np.H) continue;
        const float tg = sqrtf((v[0] * v[0] + v[1] * v[1]) + v[2] * v[2]);  // depth along the generation ray
        const size_t l = (size_t)ly * np.W + lx;
        const uint32_t c = np.count[l];
        for (uint32_t j = 0; j < c; ++j) {
          const float2 dp = __ldg(np.depth + l * np.k + j);
          if (tg < dp.x) break;
          if (tg < dp.y) {
            const float4 s = __ldg(np.rgba + l * np.k + j);
            const float as = 1.0f - powf(1.0f - s.w, np.dt / (dp.y - dp.x));
            const float sc = as / s.w;
            over_acc(acc, s.x * sc, s.y * sc, s.z * sc, as);
            break;
          }
        }
      }
    }
    np.out[p] = acc;
  }
}

// rows of an RGBA strip into the root's window (the image gather), one
// counter bump per block at the root
__global__ void __launch_bounds__(256) rows_push_kernel(const float4* __restrict__ src, float4* __restrict__ dst,
                                                        uint32_t n, uint32_t* flag) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) dst[i] = __ldg(src + i);
  __syncthreads();
  if (threadIdx.x == 0 && flag) {
    __threadfence_system();
    atomicAdd_system(flag, 1u);
  }
}

static unsigned grid_for(size_t n) {
  const size_t b = (n + 127) / 128;
  return (unsigned)(b < 1 ? 1 : (b > 148 * 32 ? 148 * 32 : b));
}

cudaError_t launch_image(const MergeParams& mp, float4* out, cudaStream_t st) {
  if (!mp.P) return cudaSuccess;
  image_kernel<<<grid_for((size_t)mp.n_groups * 32 / 4 + 1), 128, 0, st>>>(mp, out);
  return cudaGetLastError();
}

cudaError_t launch_gen_view(const uint8_t* count, const float4* rgba, uint32_t P, int k, float4* out, cudaStream_t st) {
  if (!P) return cudaSuccess;
  gen_view_kernel<<<grid_for(P), 128, 0, st>>>(count, rgba, P, k, out);
  return cudaGetLastError();
}

cudaError_t launch_novel_view(const NovelParams& np, cudaStream_t st) {
  novel_view_kernel<<<grid_for((size_t)np.W_out * np.H_out), 128, 0, st>>>(np);
  return cudaGetLastError();
}

cudaError_t launch_rows_push(const float4* src, float4* dst, uint32_t n, uint32_t blocks, uint32_t* flag,
                             cudaStream_t st) {
  rows_push_kernel<<<blocks, 256, 0, st>>>(src, dst, n, flag);
  return cudaGetLastError();
}

cudaError_t preload_render() {
  cudaFuncAttributes fa;
  cudaFuncGetAttributes(&fa, image_kernel);
  cudaFuncGetAttributes(&fa, gen_view_kernel);
  cudaFuncGetAttributes(&fa, novel_view_kernel);
  cudaFuncGetAttributes(&fa, rows_push_kernel);
  return cudaGetLastError();
}

}  // namespace vdi
