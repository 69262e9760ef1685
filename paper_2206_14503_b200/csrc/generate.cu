// generate.cu — Phase-1 reference raycaster producing dense sub-VDIs
// (SUPPORT, untimed).
//
// One thread per ray.  Pass 1 finds the per-ray gamma and the supersegment
// count it generates (gamma = 0 if count(0) <= k, else the bisection of
// PAPER.md:100-101; reading G1), an exclusive scan (CUB) turns the counts into
// offsets (PAPER.md:115 does it on the CPU), pass 2 re-runs the sweep at the
// stored gamma and writes the supersegments at their offsets.
// Samples lie on the global grid t_i = t_in + (i + 1/2) dt (dt = one voxel,
// Q18), so every PE sees the same samples; a sample owned by another PE (or
// outside the volume) forces the open supersegment to close.
// The loop is clipped to the PE's bounding box (samples outside it are not
// owned, so skipping them changes nothing).  fp32, -fmad=false, explicit fmaf.
#include <cub/device/device_scan.cuh>
#include <cuda_runtime.h>
#include <math_constants.h>

#include "internal.h"

namespace vdi {

struct RayG {
  float o[3], d[3], bmin[3], scale, t_in, t_out, dt;
};

__device__ __forceinline__ RayG make_ray(const GenParams& gp, int x, int y) {
  RayG r;
  const float sx = ((2.0f * ((float)x + 0.5f)) / (float)gp.W - 1.0f) * gp.tan_x;
  const float sy = (1.0f - (2.0f * ((float)y + 0.5f)) / (float)gp.H) * gp.tan_y;
  float v[3];
#pragma unroll
  for (int c = 0; c < 3; ++c) v[c] = (gp.fwd[c] + sx * gp.right[c]) + sy * gp.up[c];
  const float len = sqrtf((v[0] * v[0] + v[1] * v[1]) + v[2] * v[2]);
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    r.o[c] = gp.eye[c];
    r.d[c] = v[c] / len;
  }
  const int md = max(gp.dims[0], max(gp.dims[1], gp.dims[2]));
  r.scale = (float)md;
  float tmin = 0.0f, tmax = CUDART_INF_F;
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    const float half = (float)gp.dims[c] / (2.0f * (float)md);
    r.bmin[c] = -half;
    const float t0 = (-half - r.o[c]) / r.d[c];
    const float t1 = (half - r.o[c]) / r.d[c];
    tmin = fmaxf(tmin, fminf(t0, t1));
    tmax = fminf(tmax, fmaxf(t0, t1));
  }
  r.t_in = tmin;
  r.t_out = tmax;
  r.dt = 1.0f / (float)md;
  return r;
}

__device__ __forceinline__ float voxel(const GenParams& gp, int x, int y, int z) {
  if (x < 0 || y < 0 || z < 0 || x >= gp.dims[0] || y >= gp.dims[1] || z >= gp.dims[2]) return 0.0f;
  const int64_t i = ((int64_t)z * gp.dims[1] + y) * gp.dims[0] + x;
  if (gp.bytes == 1) return (float)__ldg(static_cast<const uint8_t*>(gp.vox) + i) / 255.0f;
  return (float)__ldg(static_cast<const uint16_t*>(gp.vox) + i) / 65535.0f;
}

__device__ __forceinline__ float lerpf(float a, float b, float t) { return fmaf(t, b - a, a); }

// trilinear on the global volume, voxel i centred at i + 0.5 (Q19)
__device__ float sample_trilinear(const GenParams& gp, const float c[3]) {
  float f[3];
  int i[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const float u = c[k] - 0.5f;
    const float fl = floorf(u);
    i[k] = (int)fl;
    f[k] = u - fl;
  }
  const float c00 = lerpf(voxel(gp, i[0], i[1], i[2]), voxel(gp, i[0] + 1, i[1], i[2]), f[0]);
  const float c10 = lerpf(voxel(gp, i[0], i[1] + 1, i[2]), voxel(gp, i[0] + 1, i[1] + 1, i[2]), f[0]);
  const float c01 = lerpf(voxel(gp, i[0], i[1], i[2] + 1), voxel(gp, i[0] + 1, i[1], i[2] + 1), f[0]);
  const float c11 = lerpf(voxel(gp, i[0], i[1] + 1, i[2] + 1), voxel(gp, i[0] + 1, i[1] + 1, i[2] + 1), f[0]);
  const float c0 = lerpf(c00, c10, f[1]);
  const float c1 = lerpf(c01, c11, f[1]);
  return lerpf(c0, c1, f[2]);
}

// 256-entry TF with linear interpolation, premultiplied (alpha' = alpha_TF, Q18)
__device__ __forceinline__ float4 classify(const GenParams& gp, float v) {
  const float x = v * 255.0f;
  int i = (int)floorf(x);
  i = min(max(i, 0), 254);
  const float f = x - (float)i;
  const float4 a = __ldg(gp.tf + i), b = __ldg(gp.tf + i + 1);
  const float r = lerpf(a.x, b.x, f), g = lerpf(a.y, b.y, f), bl = lerpf(a.z, b.z, f), al = lerpf(a.w, b.w, f);
  return make_float4(r * al, g * al, bl * al, al);
}

__device__ __forceinline__ int owner_of(const GenParams& gp, const float c[3]) {
  int iv[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const float fl = floorf(c[k]);
    if (!(fl >= 0.0f) || fl >= (float)gp.dims[k]) return -1;
    iv[k] = (int)fl;
  }
  int bx = 0, by = 0, bz = 0;
  while (bx + 1 < gp.grid[0] && iv[0] >= gp.xb[bx + 1]) ++bx;
  while (by + 1 < gp.grid[1] && iv[1] >= gp.yb[by + 1]) ++by;
  while (bz + 1 < gp.grid[2] && iv[2] >= gp.zb[bz + 1]) ++bz;
  return (int)__ldg(gp.owner + (bz * gp.grid[1] + by) * gp.grid[0] + bx);
}

// index range [i0, i1) of grid samples that can be owned by this PE
__device__ void clip_range(const GenParams& gp, const RayG& r, int64_t* i0, int64_t* i1) {
  *i0 = 0;
  *i1 = 0;
  if (!(r.t_out > r.t_in)) return;
  float te = r.t_in, tx = r.t_out;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const float c0 = (r.o[k] - r.bmin[k]) * r.scale;
    const float dc = r.d[k] * r.scale;
    const float lo = gp.lo[k] - 1.0f, hi = gp.hi[k] + 1.0f;
    if (dc == 0.0f) {
      if (c0 < lo || c0 > hi) return;
      continue;
    }
    const float ta = (lo - c0) / dc, tb = (hi - c0) / dc;
    te = fmaxf(te, fminf(ta, tb));
    tx = fminf(tx, fmaxf(ta, tb));
  }
  if (!(tx >= te)) return;
  const float a = floorf((te - r.t_in) / r.dt) - 2.0f;
  const float b = ceilf((tx - r.t_in) / r.dt) + 2.0f;
  *i0 = a > 0.0f ? (int64_t)a : 0;
  *i1 = (int64_t)b;
}

__device__ __forceinline__ float dist2g(const float4& a, const float4& s) {
  const float dr = a.x - s.x, dg = a.y - s.y, db = a.z - s.z, da = a.w - s.w;
  return fmaf(da, da, fmaf(db, db, fmaf(dg, dg, dr * dr)));
}

// Generator sweep for PE gp.pe (Q8 transparent samples).
// Count mode (od == nullptr) returns once cnt > k.  Write mode writes <= k.
__device__ int gen_sweep(const GenParams& gp, const RayG& r, int64_t i0, int64_t i1, float gamma, int k,
                         float2* od, float4* oc) {
  const float g2 = gamma * gamma;
  int cnt = 0;
  bool open = false;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  float tf = 0.f, tb = 0.f;
  for (int64_t i = i0; i < i1; ++i) {
    const float t = r.t_in + ((float)i + 0.5f) * r.dt;
    if (!(t < r.t_out)) break;
    float c[3];
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      const float p = r.o[q] + t * r.d[q];
      c[q] = (p - r.bmin[q]) * r.scale;
    }
    if (owner_of(gp, c) != gp.pe) {
      if (open) {
        if (od && cnt <= k) {
          od[cnt - 1] = make_float2(tf, tb);
          oc[cnt - 1] = acc;
        }
        open = false;
      }
      continue;
    }
    const float4 s = classify(gp, sample_trilinear(gp, c));
    const float t_hi = r.t_in + (float)(i + 1) * r.dt;
    if (s.w == 0.0f) {
      if (open && dist2g(acc, make_float4(0.f, 0.f, 0.f, 0.f)) > g2) {
        if (od && cnt <= k) {
          od[cnt - 1] = make_float2(tf, tb);
          oc[cnt - 1] = acc;
        }
        open = false;
      }
      continue;
    }
    if (open) {
      if (dist2g(acc, s) > g2) {
        if (od && cnt <= k) {
          od[cnt - 1] = make_float2(tf, tb);
          oc[cnt - 1] = acc;
        }
      } else {
        const float tr = 1.0f - acc.w;
        acc.x = fmaf(tr, s.x, acc.x);
        acc.y = fmaf(tr, s.y, acc.y);
        acc.z = fmaf(tr, s.z, acc.z);
        acc.w = fmaf(tr, s.w, acc.w);
        tb = t_hi;
        continue;
      }
    }
    ++cnt;
    if (!od && cnt > k) return cnt;
    open = true;
    acc = s;
    tf = r.t_in + (float)i * r.dt;
    tb = t_hi;
  }
  if (open && od && cnt <= k) {
    od[cnt - 1] = make_float2(tf, tb);
    oc[cnt - 1] = acc;
  }
  return cnt;
}

__global__ void gen_pass1_kernel(GenParams gp, uint32_t* __restrict__ count32, float* __restrict__ gamma_out,
                                 int* __restrict__ err) {
  const int64_t P = (int64_t)gp.W * gp.H;
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < P; p += (int64_t)gridDim.x * blockDim.x) {
    const RayG r = make_ray(gp, (int)(p % gp.W), (int)(p / gp.W));
    int64_t i0, i1;
    clip_range(gp, r, &i0, &i1);
    if (gp.limit) {  // one S~ per sub-domain intersection: gamma = inf, only domain exits split
      const int c = gen_sweep(gp, r, i0, i1, CUDART_INF_F, gp.k, nullptr, nullptr);
      if (c > gp.k) atomicOr(err, 2);  // capacity (Q20)
      count32[p] = (uint32_t)min(c, gp.k);
      gamma_out[p] = CUDART_INF_F;
      continue;
    }
    int c = gen_sweep(gp, r, i0, i1, 0.0f, gp.k, nullptr, nullptr);
    float g = 0.0f;
    if (c > gp.k) {
      float lo = 0.0f, hi = gp.gamma_max, best = gp.gamma_max;
      int cb = -1;
      for (int it = 0; it < gp.max_iters; ++it) {
        const float mid = 0.5f * (lo + hi);
        const int cc = gen_sweep(gp, r, i0, i1, mid, gp.k, nullptr, nullptr);
        if (cc <= gp.k) {
          best = hi = mid;
          cb = cc;
          if (cc == gp.k) break;
        } else {
          lo = mid;
        }
      }
      g = best;
      c = cb >= 0 ? cb : gen_sweep(gp, r, i0, i1, best, 1 << 30, nullptr, nullptr);
      if (c > gp.k) atomicOr(err, 2);  // capacity (Q20)
    }
    count32[p] = (uint32_t)min(c, gp.k);
    gamma_out[p] = g;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) count32[P] = 0;  // so the scan's last entry is the total
}

__global__ void gen_pass2_kernel(GenParams gp, const uint32_t* __restrict__ offset,
                                 const float* __restrict__ gamma, const uint32_t* __restrict__ count32,
                                 float2* __restrict__ depth, float4* __restrict__ rgba) {
  const int64_t P = (int64_t)gp.W * gp.H;
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < P; p += (int64_t)gridDim.x * blockDim.x) {
    if (count32[p] == 0) continue;
    const RayG r = make_ray(gp, (int)(p % gp.W), (int)(p / gp.W));
    int64_t i0, i1;
    clip_range(gp, r, &i0, &i1);
    const uint32_t o = offset[p];
    gen_sweep(gp, r, i0, i1, gamma[p], gp.k, depth + o, rgba + o);
  }
}

// Ground-truth direct volume rendering (A19): over of ALL
// samples of the global grid front to back, fp32, no early termination
// (Q21) -- the generator's sampling without segmentation.  One thread per ray.
__global__ void dvr_kernel(GenParams gp, float4* __restrict__ out) {
  const int64_t P = (int64_t)gp.W * gp.H;
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < P; p += (int64_t)gridDim.x * blockDim.x) {
    const RayG r = make_ray(gp, (int)(p % gp.W), (int)(p / gp.W));
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    if (r.t_out > r.t_in) {
      for (int64_t i = 0;; ++i) {
        const float t = r.t_in + ((float)i + 0.5f) * r.dt;
        if (!(t < r.t_out)) break;
        float c[3];
#pragma unroll
        for (int q = 0; q < 3; ++q) {
          const float pp = r.o[q] + t * r.d[q];
          c[q] = (pp - r.bmin[q]) * r.scale;
        }
        bool inside = true;
#pragma unroll
        for (int q = 0; q < 3; ++q) {
          const float fl = floorf(c[q]);
          inside &= fl >= 0.0f && fl < (float)gp.dims[q];
        }
        if (!inside) continue;
        const float4 s = classify(gp, sample_trilinear(gp, c));
        const float tr = 1.0f - acc.w;
        acc.x = fmaf(tr, s.x, acc.x);
        acc.y = fmaf(tr, s.y, acc.y);
        acc.z = fmaf(tr, s.z, acc.z);
        acc.w = fmaf(tr, s.w, acc.w);
      }
    }
    out[p] = acc;
  }
}

cudaError_t launch_dvr(const GenParams& gp, float4* out, cudaStream_t st) {
  const int64_t P = (int64_t)gp.W * gp.H;
  const unsigned blocks = (unsigned)((P + 127) / 128);
  dvr_kernel<<<blocks ? blocks : 1, 128, 0, st>>>(gp, out);
  return cudaGetLastError();
}

__global__ void u32_to_u8_kernel(const uint32_t* __restrict__ in, uint8_t* __restrict__ out, size_t n) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    out[i] = (uint8_t)in[i];
}

cudaError_t launch_gen_pass1(const GenParams& gp, uint32_t* count32, float* gamma, int* err, cudaStream_t st) {
  const int64_t P = (int64_t)gp.W * gp.H;
  const int threads = 128;
  const unsigned blocks = (unsigned)((P + threads - 1) / threads);
  gen_pass1_kernel<<<blocks ? blocks : 1, threads, 0, st>>>(gp, count32, gamma, err);
  return cudaGetLastError();
}

cudaError_t launch_gen_pass2(const GenParams& gp, const uint32_t* offset, const float* gamma,
                             const uint32_t* count32, float2* depth, float4* rgba, cudaStream_t st) {
  const int64_t P = (int64_t)gp.W * gp.H;
  const int threads = 128;
  const unsigned blocks = (unsigned)((P + threads - 1) / threads);
  gen_pass2_kernel<<<blocks ? blocks : 1, threads, 0, st>>>(gp, offset, gamma, count32, depth, rgba);
  return cudaGetLastError();
}

cudaError_t gen_scan(const uint32_t* count32, uint32_t* offset, size_t n, void** tmp, size_t* tmp_bytes,
                     cudaStream_t st) {
  size_t need = 0;
  cudaError_t e = cub::DeviceScan::ExclusiveSum(nullptr, need, count32, offset, (int)n, st);
  if (e != cudaSuccess) return e;
  if (need > *tmp_bytes) {
    if (*tmp) cudaFree(*tmp);
    *tmp = nullptr;
    e = cudaMalloc(tmp, need);
    if (e != cudaSuccess) {
      *tmp_bytes = 0;
      return e;
    }
    *tmp_bytes = need;
  }
  return cub::DeviceScan::ExclusiveSum(*tmp, *tmp_bytes, count32, offset, (int)n, st);
}

cudaError_t launch_u32_to_u8(const uint32_t* in, uint8_t* out, size_t n, cudaStream_t st) {
  u32_to_u8_kernel<<<(unsigned)std::min<size_t>((n + 255) / 256, 148 * 16), 256, 0, st>>>(in, out, n);
  return cudaGetLastError();
}

}  // namespace vdi
