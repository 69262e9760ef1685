// merge.cu — Phase-2 compositing kernels for sm_100a.
//
// Per strip of P lists and n sources (PEs):
//   group_sums / group_scan : receive-side exclusive scan of each source's
//                             count slice at 32-list granularity (PAPER.md:166
//                             ships prefix chunks; we re-derive them, Q17);
//   merge_fast              : one warp per 32 consecutive lists, lane = list.
//                             Lists with m <= k_out and no overlap / no
//                             transparent record are depth-ordered by a k-way
//                             merge of the per-PE sorted runs
//                             and written verbatim (Q9); every list of the
//                             group is staged in shared memory in the
//                             full-representation layout (zeros in unused
//                             slots) and streamed to HBM with
//                             coalesced 16-B stores.  Other lists are pushed
//                             to a work list;
//   merge_slow              : one thread per work-list entry: k-way merge,
//                             overlap subdivision (Eq. 2 generalised, Q12),
//                             gamma bisection and
//                             final sweep (Q1, Q2, Q8), written in place.
// The decision arithmetic (tau, the blend) is fp32 with explicit fmaf in the
// order DESIGN.md §2 fixes; the TU is compiled with -fmad=false so no other
// contraction happens.
#include <cuda_runtime.h>
#include <math_constants.h>

#include "internal.h"

namespace vdi {

static constexpr int kFastThreads = 128;  // 4 warps
static constexpr int kSlowThreads = 128;
static constexpr unsigned kFull = 0xffffffffu;

// ---------------------------------------------------------------------------
// Receive-side scan, stage 1: sum of each 32-list group of each source.
// ---------------------------------------------------------------------------
__global__ void group_sums_kernel(MergeParams mp, uint32_t* __restrict__ group_sum) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t gw = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const uint64_t n_work = (uint64_t)mp.n_groups * mp.n_src;
  if (gw >= n_work) return;
  const uint32_t s = (uint32_t)(gw / mp.n_groups);
  const uint32_t g = (uint32_t)(gw % mp.n_groups);
  const uint32_t p = g * 32 + lane;
  uint32_t c = 0;
  if (p < mp.P) c = __ldg(mp.src[s].count + p);
  c = __reduce_add_sync(kFull, c);
  if (lane == 0) group_sum[gw] = c;
}

// Stage 2: exclusive scan over the groups of one source (one block per source).
__global__ void group_scan_kernel(uint32_t n_groups, const uint32_t* __restrict__ group_sum,
                                  uint32_t* __restrict__ group_base, unsigned long long* __restrict__ totals) {
  __shared__ uint32_t warp_tot[32];
  __shared__ unsigned long long carry_s;
  const uint32_t s = blockIdx.x;
  const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const uint32_t* in = group_sum + (size_t)s * n_groups;
  uint32_t* out = group_base + (size_t)s * n_groups;
  if (threadIdx.x == 0) carry_s = 0;
  __syncthreads();
  for (uint32_t base = 0; base < n_groups; base += blockDim.x) {
    uint32_t i = base + threadIdx.x;
    uint32_t v = i < n_groups ? in[i] : 0;
    uint32_t incl = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      uint32_t t = __shfl_up_sync(kFull, incl, d);
      if (lane >= (uint32_t)d) incl += t;
    }
    if (lane == 31) warp_tot[w] = incl;
    __syncthreads();
    if (w == 0) {
      uint32_t t = lane < nw ? warp_tot[lane] : 0;
      uint32_t ti = t;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        uint32_t u = __shfl_up_sync(kFull, ti, d);
        if (lane >= (uint32_t)d) ti += u;
      }
      if (lane < nw) warp_tot[lane] = ti - t;  // exclusive warp offsets
    }
    __syncthreads();
    unsigned long long carry = carry_s;
    if (i < n_groups) out[i] = (uint32_t)(carry + warp_tot[w] + incl - v);
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry_s = carry + warp_tot[w] + incl;
    __syncthreads();
  }
  if (threadIdx.x == 0) totals[s] = carry_s;
}

// ---------------------------------------------------------------------------
// Eq. 1 distance, fixed order (Q2): D^2 = fma(da,da, fma(db,db, fma(dg,dg, dr*dr)))
// ---------------------------------------------------------------------------
__device__ __forceinline__ float dist2(float ar, float ag, float ab, float aa, float sr, float sg, float sb,
                                       float sa) {
  float dr = ar - sr, dg = ag - sg, db = ab - sb, da = aa - sa;
  return fmaf(da, da, fmaf(db, db, fmaf(dg, dg, dr * dr)));
}

// One greedy sweep over depth-ordered samples (
// Q1, Q2, Q8).  Count mode (od == nullptr) returns early once cnt > k.
// Write mode writes the closed segments to od/oc[0..cnt).
__device__ int sweep(const Rec* __restrict__ S, int m, float gamma, int k, float2* od, float4* oc) {
  const float g2 = gamma * gamma;
  int cnt = 0;
  bool open = false;
  float ar = 0.f, ag = 0.f, ab = 0.f, aa = 0.f, tf = 0.f, tb = 0.f, prev_tb = 0.f;
  for (int i = 0; i < m; ++i) {
    const Rec s = S[i];
    if (open && s.tf > prev_tb) {
      if (dist2(ar, ag, ab, aa, 0.f, 0.f, 0.f, 0.f) > g2) {
        if (od && cnt <= k) {
          od[cnt - 1] = make_float2(tf, tb);
          oc[cnt - 1] = make_float4(ar, ag, ab, aa);
        }
        open = false;
      }
    }
    bool start = !open;
    if (open) {
      if (dist2(ar, ag, ab, aa, s.r, s.g, s.b, s.a) > g2) {
        if (od && cnt <= k) {
          od[cnt - 1] = make_float2(tf, tb);
          oc[cnt - 1] = make_float4(ar, ag, ab, aa);
        }
        start = true;
      } else {
        const float tr = 1.0f - aa;
        ar = fmaf(tr, s.r, ar);
        ag = fmaf(tr, s.g, ag);
        ab = fmaf(tr, s.b, ab);
        aa = fmaf(tr, s.a, aa);
        tb = s.tb;
      }
    }
    if (start) {
      ++cnt;
      if (!od && cnt > k) return cnt;
      open = true;
      ar = s.r;
      ag = s.g;
      ab = s.b;
      aa = s.a;
      tf = s.tf;
      tb = s.tb;
    }
    prev_tb = s.tb;
  }
  if (open && od && cnt <= k) {
    od[cnt - 1] = make_float2(tf, tb);
    oc[cnt - 1] = make_float4(ar, ag, ab, aa);
  }
  return cnt;
}

// ---------------------------------------------------------------------------
// Fast path: warp per 32 lists, lane = list.
// ---------------------------------------------------------------------------
template <int NS>
__global__ void __launch_bounds__(kFastThreads) merge_fast_kernel(MergeParams mp) {
  extern __shared__ float4 smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const int k = mp.k_out;
  const int n = mp.n_src;
  float4* st_rgba = smem + (size_t)warp * (32 * k * 3 / 2);
  float2* st_depth = reinterpret_cast<float2*>(st_rgba + 32 * k);
  const unsigned lt_mask = (1u << lane) - 1u;
  unsigned long long rec_acc = 0;

  for (uint32_t g = blockIdx.x * nwarps + warp; g < mp.n_groups; g += gridDim.x * nwarps) {
    const uint32_t p0 = g * 32, p = p0 + lane;
    const bool valid = p < mp.P;
    uint32_t off[NS], cnt[NS];
    uint32_t m = 0;
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      off[s] = 0;
      cnt[s] = 0;
      if (s < n) {
        uint32_t c = valid ? (uint32_t)__ldg(mp.src[s].count + p) : 0u;
        uint32_t incl = c;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
          uint32_t t = __shfl_up_sync(kFull, incl, d);
          if (lane >= d) incl += t;
        }
        off[s] = __ldg(mp.group_base + (size_t)s * mp.n_groups + g) + incl - c;
        cnt[s] = c;
        m += c;
      }
    }
    rec_acc += m;

    // zero the staging area of the 32 lists (full representation zeros)
    const int stage_f4 = 32 * k * 3 / 2;
    for (int i = lane; i < stage_f4; i += 32) st_rgba[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    __syncwarp();

    bool slow = valid && (int)m > k;
    if (valid && m > 0 && !slow) {
      float htf[NS];
      uint32_t hp[NS];
#pragma unroll
      for (int s = 0; s < NS; ++s) {
        hp[s] = 0;
        htf[s] = (cnt[s] > 0) ? __ldg(&mp.src[s].depth[off[s]].x) : CUDART_INF_F;
      }
      float prev_tb = -CUDART_INF_F;
      uint32_t r = 0;
      for (; r < m; ++r) {
        int best = 0;
        float bt = htf[0];
#pragma unroll
        for (int s = 1; s < NS; ++s)
          if (htf[s] < bt) {  // strict: ties keep the lower PE id (Q11)
            bt = htf[s];
            best = s;
          }
        uint32_t q = 0;
#pragma unroll
        for (int s = 0; s < NS; ++s)
          if (s == best) q = off[s] + hp[s];
        const float2* dp = mp.src[best].depth;
        const float4* cp = mp.src[best].rgba;
        const float2 d = __ldg(dp + q);
        const float4 c = __ldg(cp + q);
        if (c.w == 0.f || d.x < prev_tb) {  // transparent record (Q23) or overlap (Q12): slow path
          slow = true;
          break;
        }
        prev_tb = d.y;
        st_depth[lane * k + r] = d;
        st_rgba[lane * k + r] = c;
#pragma unroll
        for (int s = 0; s < NS; ++s)
          if (s == best) {
            hp[s] += 1;
            htf[s] = (hp[s] < cnt[s]) ? __ldg(&dp[q + 1].x) : CUDART_INF_F;
          }
      }
      if (slow)
        for (uint32_t j = 0; j < r; ++j) {
          st_depth[lane * k + j] = make_float2(0.f, 0.f);
          st_rgba[lane * k + j] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
    }

    // slow lists -> work list (one atomic pair per warp)
    const unsigned slow_mask = __ballot_sync(kFull, slow);
    if (slow_mask) {
      uint32_t need = slow ? 4u * m : 0u;
      uint32_t incl = need;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        uint32_t t = __shfl_up_sync(kFull, incl, d);
        if (lane >= d) incl += t;
      }
      const uint32_t tot = __shfl_sync(kFull, incl, 31);
      uint32_t wl0 = 0;
      unsigned long long sc0 = 0;
      if (lane == 0) {
        wl0 = atomicAdd(mp.wl_count, (uint32_t)__popc(slow_mask));
        sc0 = atomicAdd(mp.scratch_used, (unsigned long long)tot);
      }
      wl0 = __shfl_sync(kFull, wl0, 0);
      sc0 = __shfl_sync(kFull, sc0, 0);
      if (slow) {
        const uint32_t idx = wl0 + __popc(slow_mask & lt_mask);
        const unsigned long long sb = sc0 + incl - need;
        if (idx < mp.wl_cap && sb + need <= mp.scratch_cap) {
          uint32_t* e = mp.wl + (size_t)idx * (3 + n);
          e[0] = p;
          e[1] = (uint32_t)sb;
          e[2] = m;
#pragma unroll
          for (int s = 0; s < NS; ++s)
            if (s < n) e[3 + s] = off[s];
        } else {
          atomicOr(mp.err, 1);
        }
      }
    }
    if (valid) {
      mp.out_count[p] = slow ? 0 : (uint8_t)m;
      if (mp.stat_m) mp.stat_m[p] = (uint16_t)m;
      if (mp.stat_gamma) mp.stat_gamma[p] = 0.f;
    }
    __syncwarp();

    // stream the staged lists to HBM (contiguous: lists p0.. p0+npix-1)
    const uint32_t npix = min(32u, mp.P - p0);
    float2* gd = mp.out_depth + (size_t)p0 * k;
    const uint32_t nd = npix * k;
    if ((reinterpret_cast<uintptr_t>(gd) & 15u) == 0 && (nd & 1u) == 0) {
      float4* gd4 = reinterpret_cast<float4*>(gd);
      const float4* sd4 = reinterpret_cast<const float4*>(st_depth);
      for (uint32_t i = lane; i < nd / 2; i += 32) gd4[i] = sd4[i];
    } else {
      for (uint32_t i = lane; i < nd; i += 32) gd[i] = st_depth[i];
    }
    float4* gc = mp.out_rgba + (size_t)p0 * k;
    for (uint32_t i = lane; i < nd; i += 32) gc[i] = st_rgba[i];
    __syncwarp();
  }

  // one atomic per warp for the "supersegments merged" counter
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) rec_acc += __shfl_down_sync(kFull, rec_acc, d);
  if (lane == 0 && rec_acc) atomicAdd(mp.records_in, rec_acc);
}

// ---------------------------------------------------------------------------
// Slow path: thread per work-list entry (general algorithm, steps 1-6).
// ---------------------------------------------------------------------------
__device__ void over_into(float* acc, const float* b) {
  const float tr = 1.0f - acc[3];
  for (int c = 0; c < 4; ++c) acc[c] = fmaf(tr, b[c], acc[c]);
}

__global__ void __launch_bounds__(kSlowThreads) merge_slow_kernel(MergeParams mp) {
  const int n = mp.n_src, k = mp.k_out;
  uint32_t total = *mp.wl_count;
  if (total > mp.wl_cap) total = mp.wl_cap;
  for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += gridDim.x * blockDim.x) {
    const uint32_t* ent = mp.wl + (size_t)e * (3 + n);
    const uint32_t p = ent[0];
    const uint32_t m0 = ent[2];
    Rec* A = mp.scratch + ent[1];
    Rec* B = A + m0;
    float* E = reinterpret_cast<float*>(B + 2 * m0);
    // step 1: k-way merge of the per-PE sorted runs, dropping alpha == 0
    uint32_t pos[VDI_MAX_SRC], end[VDI_MAX_SRC];
    for (int s = 0; s < n; ++s) {
      pos[s] = ent[3 + s];
      end[s] = pos[s] + __ldg(mp.src[s].count + p);
    }
    int m = 0;
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
      const float2 d = __ldg(mp.src[best].depth + pos[best]);
      const float4 c = __ldg(mp.src[best].rgba + pos[best]);
      pos[best]++;
      if (c.w != 0.f) A[m++] = Rec{d.x, d.y, c.x, c.y, c.z, c.w};
    }
    // step 2: subdivide overlapping clusters
    const Rec* S = A;
    int mm = 0;
    bool changed = false;
    for (int i = 1; i < m; ++i)
      if (A[i].tf < A[i - 1].tb) changed = true;
    if (changed) {
      int i = 0;
      while (i < m) {
        int j = i;
        float maxtb = A[i].tb;
        while (j + 1 < m && A[j + 1].tf < maxtb) {
          ++j;
          maxtb = fmaxf(maxtb, A[j].tb);
        }
        if (j == i) {
          B[mm++] = A[i];
          ++i;
          continue;
        }
        int ne = 0;
        for (int q = i; q <= j; ++q) {
          E[ne++] = A[q].tf;
          E[ne++] = A[q].tb;
        }
        for (int a = 1; a < ne; ++a) {  // insertion sort
          float v = E[a];
          int b = a - 1;
          while (b >= 0 && E[b] > v) {
            E[b + 1] = E[b];
            --b;
          }
          E[b + 1] = v;
        }
        int nu = 0;
        for (int a = 0; a < ne; ++a)
          if (nu == 0 || E[a] != E[nu - 1]) E[nu++] = E[a];
        for (int a = 0; a + 1 < nu; ++a) {
          const float e0 = E[a], e1 = E[a + 1];
          bool have = false;
          float acc[4] = {0.f, 0.f, 0.f, 0.f};
          for (int q = i; q <= j; ++q) {
            const Rec& r = A[q];
            if (!(r.tf <= e0 && r.tb >= e1)) continue;
            const float frac = (e1 - e0) / (r.tb - r.tf);
            const float ap = 1.0f - powf(1.0f - r.a, frac);
            const float scale = ap / r.a;
            float piece[4] = {r.r * scale, r.g * scale, r.b * scale, ap};
            if (!have) {
              for (int c = 0; c < 4; ++c) acc[c] = piece[c];
              have = true;
            } else {
              over_into(acc, piece);
            }
          }
          if (have) B[mm++] = Rec{e0, e1, acc[0], acc[1], acc[2], acc[3]};
        }
        i = j + 1;
      }
      S = B;
      m = mm;
    }
    // steps 3-6
    float2* od = mp.out_depth + (size_t)p * k;
    float4* oc = mp.out_rgba + (size_t)p * k;
    float gamma = 0.f;
    int cnt;
    if (m <= k) {
      for (int j = 0; j < m; ++j) {
        od[j] = make_float2(S[j].tf, S[j].tb);
        oc[j] = make_float4(S[j].r, S[j].g, S[j].b, S[j].a);
      }
      cnt = m;
    } else {
      float lo = 0.f, hi = mp.gamma_max, best = mp.gamma_max;
      for (int it = 0; it < mp.max_iters; ++it) {
        const float mid = 0.5f * (lo + hi);
        const int c = sweep(S, m, mid, k, nullptr, nullptr);
        if (c <= k) {
          best = hi = mid;
          if (c == k) break;
        } else {
          lo = mid;
        }
      }
      gamma = best;
      cnt = sweep(S, m, best, k, od, oc);
    }
    mp.out_count[p] = (uint8_t)cnt;
    if (mp.stat_m) mp.stat_m[p] = (uint16_t)m;
    if (mp.stat_gamma) mp.stat_gamma[p] = gamma;
  }
}

// ---------------------------------------------------------------------------
// Launchers
// ---------------------------------------------------------------------------
static int sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

cudaError_t launch_group_sums(const MergeParams& mp, uint32_t* group_sum, cudaStream_t st, int* launches) {
  const uint64_t warps = (uint64_t)mp.n_groups * mp.n_src;
  if (!warps) return cudaSuccess;
  const int wpb = 8;
  group_sums_kernel<<<(unsigned)((warps + wpb - 1) / wpb), wpb * 32, 0, st>>>(mp, group_sum);
  ++*launches;
  return cudaGetLastError();
}

cudaError_t launch_group_scan(const MergeParams& mp, const uint32_t* group_sum, uint32_t* group_base,
                              uint64_t* totals, cudaStream_t st, int* launches) {
  if (!mp.n_src) return cudaSuccess;
  group_scan_kernel<<<mp.n_src, 1024, 0, st>>>(mp.n_groups, group_sum, group_base,
                                                reinterpret_cast<unsigned long long*>(totals));
  ++*launches;
  return cudaGetLastError();
}

template <int NS>
static cudaError_t launch_fast_ns(const MergeParams& mp, cudaStream_t st) {
  const size_t smem = (size_t)(kFastThreads / 32) * 32 * mp.k_out * 24;
  static size_t configured = 0;
  if (smem > configured) {
    cudaError_t e = cudaFuncSetAttribute(merge_fast_kernel<NS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    configured = smem;
  }
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, merge_fast_kernel<NS>, kFastThreads, smem);
  if (per_sm < 1) per_sm = 1;
  const uint32_t want = (mp.n_groups + (kFastThreads / 32) - 1) / (kFastThreads / 32);
  uint32_t grid = (uint32_t)sm_count() * per_sm;
  if (grid > want) grid = want ? want : 1;
  merge_fast_kernel<NS><<<grid, kFastThreads, smem, st>>>(mp);
  return cudaGetLastError();
}

cudaError_t launch_merge(const MergeParams& mp, cudaStream_t st, int* launches) {
  cudaError_t e;
  if (mp.n_src <= 1) e = launch_fast_ns<1>(mp, st);
  else if (mp.n_src <= 2) e = launch_fast_ns<2>(mp, st);
  else if (mp.n_src <= 4) e = launch_fast_ns<4>(mp, st);
  else if (mp.n_src <= 8) e = launch_fast_ns<8>(mp, st);
  else if (mp.n_src <= 16) e = launch_fast_ns<16>(mp, st);
  else e = launch_fast_ns<VDI_MAX_SRC>(mp, st);
  if (e != cudaSuccess) return e;
  ++*launches;
  merge_slow_kernel<<<sm_count() * 4, kSlowThreads, 0, st>>>(mp);
  ++*launches;
  return cudaGetLastError();
}

}  // namespace vdi
