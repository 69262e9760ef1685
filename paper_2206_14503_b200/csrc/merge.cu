// merge.cu — Phase-2 compositing kernels for sm_100a.
//
// Per strip of P lists and n sources (PEs):
//   chunk_sums / group_base : receive-side exclusive scan of each source's
//                             count slice at 32-list granularity (PAPER.md:166
//                             ships prefix chunks; we re-derive them, Q17);
//   merge_fast              : one warp per 32 consecutive lists, lane = list.
//                             Lists with m <= k_out are copied (LDGSTS) into
//                             their slots of a shared-memory image of the
//                             output, depth-ordered there by a run-based k-way
//                             merge of the per-PE sorted runs
//                             and written verbatim (Q9); the 32 lists' full
//                             representation (zeros in unused
//                             slots) leaves with two TMA bulk stores.  Lists
//                             with m > k_out go to a search work list,
//                             bucketed by m;
//   search_gather           : lists with k_out < m <= 40, thread per list: the
//                             run-based merge with the run heads in registers,
//                             samples in depth order to a pool slot
//                             ([sample][lane], gap flag in the sign of alpha);
//   search_sweep            : warp per 32 of them: samples 0..15 in registers,
//                             16..39 in shared rows; memoised gamma bisection
//                              with count sweeps that
//                             stop once the answer is decided; final sweep;
//   long_search             : m > 40: gather + bisection + final sweep in one
//                             kernel from warp-private L2-resident slots (lane
//                             per list), or warp per list with five bisection
//                             levels per sweep when there are few long lists;
//   merge_general           : thread per list for overlapping records
//                             (subdivision, Eq. 2 generalised, Q12), alpha==0
//                             records (Q23) and lists whose pool slot could not
//                             be allocated.
// The decision arithmetic (tau, the blend) is fp32 with explicit fmaf in the
// order DESIGN.md §2 fixes; the TU is compiled with -fmad=false so no other
// contraction happens.
#include <algorithm>
#include <cuda_runtime.h>
#include <math_constants.h>

#include "internal.h"

namespace vdi {

static constexpr int kFastThreads = 32;  // 1 warp per block: 13 resident per SM at k = 20 (smem-bound)
static constexpr int kSlowThreads = 128;
static constexpr unsigned kFull = 0xffffffffu;
static constexpr int kChunk = 4096;       // lists per scan chunk (128 groups of 32)

__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t v, int lane) {
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t t = __shfl_up_sync(kFull, v, d);
    if (lane >= d) v += t;
  }
  return v;
}

// ---------------------------------------------------------------------------
// Receive-side scan.  Stage 1: sum of each 4096-list chunk of each source.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) chunk_sums_kernel(MergeParams mp, uint32_t* __restrict__ chunk_sum,
                                                         uint32_t n_chunks) {
  __shared__ uint32_t red[8];
  const uint32_t c = blockIdx.x, s = blockIdx.y;
  const uint8_t* cnt = mp.src[s].count;
  const uint32_t b0 = c * kChunk, b1 = min(b0 + kChunk, mp.P);
  const bool al = (reinterpret_cast<uintptr_t>(cnt) & 3u) == 0;
  uint32_t acc = 0;
  for (uint32_t i = b0 + threadIdx.x * 4; i < b1; i += blockDim.x * 4) {
    if (al && i + 4 <= b1) {
      acc = __dp4a(__ldg(reinterpret_cast<const unsigned int*>(cnt + i)), 0x01010101u, acc);
    } else {
      for (uint32_t j = i; j < min(i + 4, b1); ++j) acc += __ldg(cnt + j);
    }
  }
  acc = __reduce_add_sync(kFull, acc);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    uint32_t v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0u;
    v = __reduce_add_sync(kFull, v);
    if (threadIdx.x == 0) chunk_sum[(size_t)s * n_chunks + c] = v;
  }
}

// Stage 2: one block (128 threads = 128 groups) per chunk and source: chunk
// prefix + block scan of the 32-list group sums -> group_base[s][g].
__global__ void __launch_bounds__(128) group_base_kernel(MergeParams mp, const uint32_t* __restrict__ chunk_sum,
                                                         uint32_t n_chunks, uint32_t* __restrict__ group_base) {
  __shared__ uint32_t red[4];
  __shared__ uint32_t wtot[4];
  const uint32_t c = blockIdx.x, s = blockIdx.y;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t pre = 0;
  for (uint32_t i = threadIdx.x; i < c; i += blockDim.x) pre += __ldg(chunk_sum + (size_t)s * n_chunks + i);
  pre = __reduce_add_sync(kFull, pre);
  if (lane == 0) red[w] = pre;
  const uint32_t g = c * 128 + threadIdx.x;
  const uint8_t* cnt = mp.src[s].count;
  const uint32_t p0 = g * 32, p1 = min(p0 + 32, mp.P);
  uint32_t gs = 0;
  if (p0 < mp.P) {
    if ((reinterpret_cast<uintptr_t>(cnt) & 15u) == 0 && p1 == p0 + 32) {
      const uint4 a = __ldg(reinterpret_cast<const uint4*>(cnt + p0));
      const uint4 b = __ldg(reinterpret_cast<const uint4*>(cnt + p0 + 16));
      gs = __dp4a(a.x, 0x01010101u, gs);
      gs = __dp4a(a.y, 0x01010101u, gs);
      gs = __dp4a(a.z, 0x01010101u, gs);
      gs = __dp4a(a.w, 0x01010101u, gs);
      gs = __dp4a(b.x, 0x01010101u, gs);
      gs = __dp4a(b.y, 0x01010101u, gs);
      gs = __dp4a(b.z, 0x01010101u, gs);
      gs = __dp4a(b.w, 0x01010101u, gs);
    } else {
      for (uint32_t q = p0; q < p1; ++q) gs += __ldg(cnt + q);
    }
  }
  const uint32_t incl = warp_incl_scan(gs, lane);
  if (lane == 31) wtot[w] = incl;
  __syncthreads();
  const uint32_t base = red[0] + red[1] + red[2] + red[3];
  uint32_t woff = 0;
  for (int q = 0; q < w; ++q) woff += wtot[q];
  const uint32_t sb = mp.src_base ? __ldg(mp.src_base + s) : 0u;  // index of the strip's first record
  if (g < mp.n_groups) group_base[(size_t)s * mp.n_groups + g] = sb + base + woff + incl - gs;
}

// ---------------------------------------------------------------------------
// Eq. 1 distance, fixed order (Q2): D^2 = fma(da,da, fma(db,db, fma(dg,dg, dr*dr)))
// ---------------------------------------------------------------------------
__device__ __forceinline__ float dist2(float ar, float ag, float ab, float aa, float sr, float sg, float sb,
                                       float sa) {
  float dr = ar - sr, dg = ag - sg, db = ab - sb, da = aa - sa;
  return fmaf(da, da, fmaf(db, db, fmaf(dg, dg, dr * dr)));
}

// (|acc|^2, |acc - s|^2) as one packed f32x2 chain: the same four rounded
// steps as dist2 on each half (FMUL2 + 3 FFMA2 instead of 8 scalar ops).
__device__ __forceinline__ void n2d2_packed(float ar, float ag, float ab, float aa, float sr, float sg, float sb,
                                            float sa, float& n2, float& d2) {
  unsigned long long pr, pg, pb, pa, t;
  asm("mov.b64 %0, {%1, %2};" : "=l"(pr) : "f"(ar), "f"(ar - sr));
  asm("mov.b64 %0, {%1, %2};" : "=l"(pg) : "f"(ag), "f"(ag - sg));
  asm("mov.b64 %0, {%1, %2};" : "=l"(pb) : "f"(ab), "f"(ab - sb));
  asm("mov.b64 %0, {%1, %2};" : "=l"(pa) : "f"(aa), "f"(aa - sa));
  asm("mul.rn.f32x2 %0, %1, %1;" : "=l"(t) : "l"(pr));
  asm("fma.rn.f32x2 %0, %1, %1, %2;" : "=l"(t) : "l"(pg), "l"(t));
  asm("fma.rn.f32x2 %0, %1, %1, %2;" : "=l"(t) : "l"(pb), "l"(t));
  asm("fma.rn.f32x2 %0, %1, %1, %2;" : "=l"(t) : "l"(pa), "l"(t));
  asm("mov.b64 {%0, %1}, %2;" : "=f"(n2), "=f"(d2) : "l"(t));
}

// |sqrt(D^2) - gamma| in double (the tie margin of one executed comparison;
// VDI_FLAG_PIXEL_STATS only)
__device__ __forceinline__ void note_margin(double* mg, float d2, float gamma) {
  if (mg) *mg = fmin(*mg, fabs(sqrt((double)d2) - (double)gamma));
}

// One greedy sweep over depth-ordered samples (
// Q1, Q2, Q8).  get(i) returns sample i.  Count mode (od == nullptr) returns
// early once cnt > k.  Write mode writes the closed segments to od/oc[0..cnt).
// mg (optional) tracks the tie margin of the executed comparisons.
template <class Get>
__device__ __forceinline__ int sweep(Get get, int m, float gamma, int k, float2* od, float4* oc,
                                     double* mg = nullptr, unsigned long long* steps = nullptr) {
  const float g2 = gamma * gamma;
  int cnt = 0;
  bool open = false;
  float ar = 0.f, ag = 0.f, ab = 0.f, aa = 0.f, tf = 0.f, tb = 0.f, prev_tb = 0.f;
  for (int i = 0; i < m; ++i) {
    if (steps) ++*steps;
    const Rec s = get(i);
    if (open && s.tf > prev_tb) {
      const float n2 = dist2(ar, ag, ab, aa, 0.f, 0.f, 0.f, 0.f);
      note_margin(mg, n2, gamma);
      if (n2 > g2) {
        if (od && cnt <= k) {
          od[cnt - 1] = make_float2(tf, tb);
          oc[cnt - 1] = make_float4(ar, ag, ab, aa);
        }
        open = false;
      }
    }
    bool start = !open;
    if (open) {
      const float d2 = dist2(ar, ag, ab, aa, s.r, s.g, s.b, s.a);
      note_margin(mg, d2, gamma);
      if (d2 > g2) {
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

// Per-list gamma bisection (PAPER.md:100-101 re-used at :176; Q3-Q6):
// midpoints 0.5*(lo+hi) of [0, gamma_max], I iterations, stop at count == k.
template <class Get>
__device__ __forceinline__ float bisect(Get get, int m, int k, int iters, float gmax, double* mg = nullptr,
                                        unsigned long long* steps = nullptr) {
  float lo = 0.f, hi = gmax, best = gmax;
  for (int it = 0; it < iters; ++it) {
    const float mid = 0.5f * (lo + hi);
    const int c = sweep(get, m, mid, k, nullptr, nullptr, mg, steps);
    if (c <= k) {
      best = hi = mid;
      if (c == k) break;
    } else {
      lo = mid;
    }
  }
  return best;
}

// Per-list gamma bisection state (Q3-Q6) with
// memoised sweep paths.  A count sweep at g2 = fl(mid * mid) takes the same
// split/merge decisions -- hence returns the same count -- for every g2' with
// L <= g2' < U, where L is the largest D^2 it merged on (D^2 <= g2) and U the
// smallest D^2 it split on (D^2 > g2), both over the decisions it evaluated
// (a sweep that stopped early at count > k_out constrains only its prefix).
// A level whose midpoint falls inside the interval of the latest sweep on
// either side of the bracket is resolved without sweeping; the sequence of
// midpoints and counts is exactly the sequential procedure's.
struct Bisection {
  float lo, hi, best, mid, g2;
  float hL, hU, lL, lU;  // validity intervals (in g2) of the latest count <= k / count > k sweeps
  int hc, it;
  bool active;
  __device__ __forceinline__ void init(float gmax, bool act) {
    lo = 0.f;
    hi = best = gmax;
    hL = lL = 1.f;  // empty
    hU = lU = 0.f;
    hc = 0;
    it = 0;
    active = act;
    mid = g2 = 0.f;
  }
  __device__ __forceinline__ void step(int c, int k, int iters) {
    if (c <= k) {
      best = hi = mid;
      if (c == k) active = false;
    } else {
      lo = mid;
    }
    if (++it >= iters) active = false;
  }
  // resolve the levels whose count is known; leaves mid / g2 at the next level to sweep
  __device__ __forceinline__ void advance(int k, int iters) {
    while (active) {
      mid = 0.5f * (lo + hi);
      g2 = mid * mid;
      if (g2 >= hL && g2 < hU) step(hc, k, iters);
      else if (g2 >= lL && g2 < lU) step(k + 1, k, iters);
      else break;
    }
  }
  // record a sweep at g2 (count c, validity [L, U)) and take its level
  __device__ __forceinline__ void swept(int c, float L, float U, int k, int iters) {
    if (c <= k) {
      hL = L;
      hU = U;
      hc = c;
    } else {
      lL = L;
      lU = U;
    }
    step(c, k, iters);
  }
};

// One evaluated decision step of a count sweep: the interval bookkeeping of
// Bisection for the gap test (n2 vs g2, Q8) and the Eq. 1 test (d2 vs g2).
__device__ __forceinline__ void track(bool ev, bool gap, float n2, float d2, float g2, float& L, float& U) {
  const bool gcl = gap & (n2 > g2);  // the gap closed the segment: d2 not consulted
  const bool dsp = d2 > g2;
  const float up = gcl ? n2 : (dsp ? d2 : CUDART_INF_F);
  const float lw = fmaxf((gap & !gcl) ? n2 : -1.f, (!gcl & !dsp) ? d2 : -1.f);
  U = ev ? fminf(U, up) : U;
  L = ev ? fmaxf(L, lw) : L;
}

// Append the lanes with bk >= 0 to work-list bucket bk (one atomic per warp and
// bucket).  goff[s] = index of the list's first record in source s's payload.
template <int NS>
__device__ __forceinline__ void push_entries(const MergeParams& mp, int bk, uint32_t p, uint32_t m,
                                             const uint32_t (&goff)[NS], int lane) {
  const unsigned lt = (1u << lane) - 1u;
  {
    // lanes of the same bucket: one atomic per bucket present, by its lowest lane
    const unsigned mask = __match_any_sync(kFull, bk);
    const int leader = __ffs(mask) - 1;
    const int b = bk;
    uint32_t w0 = 0;
    if (b >= 0 && lane == leader) w0 = atomicAdd(mp.wl_count + b, (uint32_t)__popc(mask));
    w0 = __shfl_sync(kFull, w0, leader);
    if (b >= 0) {
      const uint32_t idx = w0 + __popc(mask & lt);
      if (idx < mp.wl_cap) {
        uint32_t* e = mp.wl[b] + (size_t)idx * (3 + mp.n_src);
        e[0] = p;
        e[1] = 0u;
        e[2] = m;
#pragma unroll
        for (int s = 0; s < NS; ++s)
          if (s < mp.n_src) e[3 + s] = goff[s];
      } else {
        atomicOr(mp.err, 1);
      }
    }
  }
}

__device__ __forceinline__ int bucket_of(uint32_t m) {
  return m <= 32 ? 0 : m <= 40 ? 1 : m <= 64 ? 2 : 3;
}

// Run-based k-way merge of NS sorted runs held in shared memory (PAPER.md:168:
// repeatedly take the run with the lowest starting depth; ties -> lower PE id,
// Q11).  Run s occupies depth[(start[s] + i) * stride] for i < cnt[s].  One
// selection per run of consecutive records from the same PE (disjoint domains
// give one run per PE).  Writes perm[r * pstride] = start index of the r-th
// record and returns false on a transparent record (alpha(idx) == 0, Q23) or
// an overlap (t_front < previous t_back, Q12).
template <int NS, class PermT, class Alpha>
__device__ __forceinline__ bool run_merge(const float2* __restrict__ depth, int stride, const uint32_t (&start)[NS],
                                          const uint32_t (&cnt)[NS], uint32_t m, PermT* perm, int pstride,
                                          Alpha alpha) {
  uint32_t hp[NS];
#pragma unroll
  for (int s = 0; s < NS; ++s) hp[s] = 0;
  float prev_tb = -CUDART_INF_F;
  uint32_t r = 0;
  while (r < m) {
    int b = -1, b2 = NS;
    float bt = CUDART_INF_F, b2t = CUDART_INF_F;
#pragma unroll
    for (int s = 0; s < NS; ++s)
      if (hp[s] < cnt[s]) {
        const float t = depth[(start[s] + hp[s]) * stride].x;
        if (b < 0 || t < bt) {
          if (b >= 0) {
            b2t = bt;
            b2 = b;
          }
          bt = t;
          b = s;
        } else if (t < b2t) {
          b2t = t;
          b2 = s;
        }
      }
    uint32_t i = 0, sb = 0, cb = 0;
#pragma unroll
    for (int s = 0; s < NS; ++s)
      if (s == b) {
        i = hp[s];
        sb = start[s];
        cb = cnt[s];
      }
    for (;;) {
      const float2 d = depth[(sb + i) * stride];
      if (!(alpha(sb + i) != 0.f) || d.x < prev_tb) return false;
      prev_tb = d.y;
      perm[r * pstride] = (PermT)(sb + i);
      ++r;
      ++i;
      if (i >= cb) break;
      const float tn = depth[(sb + i) * stride].x;
      if (!(tn < b2t || (tn == b2t && b < b2))) break;
    }
#pragma unroll
    for (int s = 0; s < NS; ++s)
      if (s == b) hp[s] = i;
  }
  return true;
}

// Direct (unstaged) pass-through of one list: k-way merge from global memory,
// records written to the list's first m slots.  Rare: only when the warp's
// staging buffer is full.  Source pointers are selected with compile-time
// indices so the kernel parameters stay in the constant bank.
template <int NS>
__device__ __forceinline__ bool direct_list(const MergeParams& mp, uint32_t p, const uint32_t (&gidx)[NS],
                                            const uint32_t (&cnt)[NS], uint32_t m) {
  const int k = mp.k_out;
  uint32_t hp[NS];
#pragma unroll
  for (int s = 0; s < NS; ++s) hp[s] = 0;
  float prev_tb = -CUDART_INF_F;
  for (uint32_t r = 0; r < m; ++r) {
    int b = -1;
    float bt = 0.f;
    const float2* dp = nullptr;
    const float4* cp = nullptr;
    uint32_t q = 0;
#pragma unroll
    for (int s = 0; s < NS; ++s)
      if (hp[s] < cnt[s]) {
        const float t = __ldg(&mp.src[s].depth[gidx[s] + hp[s]].x);
        if (b < 0 || t < bt) {
          b = s;
          bt = t;
          dp = mp.src[s].depth;
          cp = mp.src[s].rgba;
          q = gidx[s] + hp[s];
        }
      }
#pragma unroll
    for (int s = 0; s < NS; ++s)
      if (s == b) hp[s] += 1;
    const float2 d = __ldg(dp + q);
    const float4 c = __ldg(cp + q);
    if (c.w == 0.f || d.x < prev_tb) return false;
    prev_tb = d.y;
    mp.out_depth[(size_t)p * k + r] = d;
    mp.out_rgba[(size_t)p * k + r] = c;
  }
  return true;
}

// ---------------------------------------------------------------------------
// Fast path: warp per 32 consecutive lists, lane = list.
//   * counts of the n sources (coalesced bytes) + warp scans -> each list's
//     records inside the group's per-source payload ranges;
//   * the 32 lists' full representation is assembled in a
//     shared-memory image of the output that is all zeros except the slots
//     written; a list with 0 < m <= k_out loads its records (independent
//     loads, PE-concatenated order) straight into its own k_out slots and is
//     depth-ordered there in place (run-based k-way merge of the per-PE sorted
//     runs) -- verbatim pass-through, Q9;
//   * the image leaves with two TMA bulk stores (cp.async.bulk shared::cta ->
//     global) and the written slots are re-zeroed once the bulk engine has
//     read them (lazy zeroing: no per-slot store instructions);
//   * lists with m > k_out go to the search buckets, lists with transparent
//     or overlapping records to the general path (their slots go out as zeros
//     and are overwritten later).
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void bulk_store(void* gdst, const void* ssrc, uint32_t bytes) {
  unsigned long long pol;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(gdst),
               "r"(smem_u32(ssrc)), "r"(bytes), "l"(pol)
               : "memory");
}

// bytes of per-warp shared memory of the fast kernel for budget k
__host__ __device__ constexpr size_t fast_warp_bytes(int k) {
  return ((size_t)32 * k * 24         // output image: rgba [32k] float4 + depth [32k] float2
          + (size_t)32 * k * 2 + 15)  // permutation (u16 per slot)
         & ~(size_t)15;
}

#ifndef VDI_FAST_RUN
#define VDI_FAST_RUN 4
#endif
template <int NS>
__global__ void __launch_bounds__(kFastThreads) merge_fast_kernel(MergeParams mp) {
  extern __shared__ float4 smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const int k = mp.k_out;
  const int n = mp.n_src;
  float4* o_rgba = reinterpret_cast<float4*>(reinterpret_cast<char*>(smem) + (size_t)warp * fast_warp_bytes(k));
  float2* o_depth = reinterpret_cast<float2*>(o_rgba + 32 * k);
  uint16_t* perm = reinterpret_cast<uint16_t*>(o_depth + 32 * k);
  float4* my_rgba = o_rgba + lane * k;
  float2* my_depth = o_depth + lane * k;
  uint16_t* my_perm = perm + lane * k;
  const bool bulk_ok =
      ((reinterpret_cast<uintptr_t>(mp.out_depth) | reinterpret_cast<uintptr_t>(mp.out_rgba)) & 15u) == 0;
  unsigned long long rec_acc = 0, plain_acc = 0, srch_acc = 0;

  // the output image starts all-zero (full-representation zeros)
  for (int i = lane; i < 32 * k; i += 32) {
    o_rgba[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    o_depth[i] = make_float2(0.f, 0.f);
  }
  uint32_t written = 0;  // slots of this lane's list written into the image last time
  __syncwarp();

  // counts and group bases of the next group are loaded one iteration ahead
  // groups are taken in runs of kRun consecutive groups, the runs interleaved
  // over the warps (all warps write one window of the output at a time: DRAM
  // page locality); counts are loaded one group ahead.  Group bases: from
  // the receive-side scan, or -- when the sources carry their offset arrays --
  // read at the start of a run and carried along as base + the group's count
  // total (one offset sector per source and run instead of per group)
  constexpr uint32_t kRun = VDI_FAST_RUN;
  const uint32_t nw_all = gridDim.x * nwarps, w_id = blockIdx.x * nwarps + warp;
  // per source: offset array (bases read at run starts and carried), pushed
  // group bases (read per group), or the receive-side scan (mp.group_base)
  auto next_group = [&](uint32_t gg) -> uint32_t {  // the group after gg in this warp's sequence
    const uint32_t r = (gg - mp.g_begin) % kRun;
    return r + 1 < kRun ? gg + 1 : gg + 1 + (nw_all - 1) * kRun;
  };
  // nb: bases loaded by the prefetch (in flight until the next iteration);
  // nbc: bases carried along a run.  Separate registers, so that the carry
  // written during group g never waits on (or overwrites) a load in flight
  uint32_t nc[NS], nb[NS], nbc[NS];
#pragma unroll
  for (int s = 0; s < NS; ++s) nb[s] = nbc[s] = 0;
  auto prefetch = [&](uint32_t gg) {
    const uint32_t pp = gg * 32 + lane;
    const bool run_start = (gg - mp.g_begin) % kRun == 0;
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      nc[s] = 0;
      if (s < n && gg < mp.g_end) {
        if (pp < mp.P) nc[s] = __ldg(mp.src[s].count + pp);
        if (mp.src[s].offset) {
          if (run_start) nb[s] = __ldg(mp.src[s].offset + (size_t)gg * 32);
        } else if (mp.src[s].gbase) {
          nb[s] = __ldg(mp.src[s].gbase + gg);
        } else {
          nb[s] = __ldg(mp.group_base + (size_t)s * mp.n_groups + gg);
        }
      }
    }
  };
  const uint32_t g_first = mp.g_begin + w_id * kRun;
  prefetch(g_first);

  for (uint32_t g = g_first; g < mp.g_end; g = next_group(g)) {
    const uint32_t p0 = g * 32, p = p0 + lane;
    const bool valid = p < mp.P;
    uint32_t cnt[NS], gidx[NS];
    uint32_t m = 0;
    const bool mid_run = (g - mp.g_begin) % kRun != 0;
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      cnt[s] = nc[s];
      gidx[s] = (mp.src[s].offset && mid_run) ? nbc[s] : nb[s];
    }
    prefetch(next_group(g));
    // the warp scans of the sources' counts, two sources per scan: 16-bit
    // halves hold the running sums (<= 32 x 255 < 2^16); the (NS + 1) / 2
    // scans advance step by step together, so their shuffle latencies overlap
    const bool carry = (g - mp.g_begin) % kRun + 1 < kRun;
    constexpr int NP = (NS + 1) / 2;
    uint32_t pc[NP], incl[NP];
#pragma unroll
    for (int q = 0; q < NP; ++q) {
      const int s0 = 2 * q, s1 = 2 * q + 1 < NS ? 2 * q + 1 : 2 * q;
      const uint32_t c0 = s0 < n ? cnt[s0] : 0u, c1 = (2 * q + 1 < NS && s1 < n) ? cnt[s1] : 0u;
      pc[q] = c0 | (c1 << 16);
      incl[q] = pc[q];
    }
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      uint32_t t[NP];
#pragma unroll
      for (int q = 0; q < NP; ++q) t[q] = (2 * q < n) ? __shfl_up_sync(kFull, incl[q], d) : 0u;
#pragma unroll
      for (int q = 0; q < NP; ++q)
        if (lane >= d) incl[q] += t[q];
    }
    uint32_t tot[NP];  // the group's count totals (lane 31's inclusive sums), all shuffles issued together
#pragma unroll
    for (int q = 0; q < NP; ++q) tot[q] = (carry && 2 * q < n) ? __shfl_sync(kFull, incl[q], 31) : 0u;
#pragma unroll
    for (int q = 0; q < NP; ++q) {
      const int s0 = 2 * q, s1 = 2 * q + 1 < NS ? 2 * q + 1 : 2 * q;
      if (s0 < n) {
        const bool two = 2 * q + 1 < NS && s1 < n;
        const uint32_t c0 = pc[q] & 0xffffu, c1 = pc[q] >> 16;
        const uint32_t i0 = incl[q] & 0xffffu, i1 = incl[q] >> 16;
        if (carry) {
          if (mp.src[s0].offset) nbc[s0] = gidx[s0] + (tot[q] & 0xffffu);  // base of group g + 1 (same run)
          if (two && mp.src[s1].offset) nbc[s1] = gidx[s1] + (tot[q] >> 16);
        }
        gidx[s0] += i0 - c0;
        m += c0;
        if (two) {
          gidx[s1] += i1 - c1;
          m += c1;
        }
      }
    }
    rec_acc += m;
#pragma unroll
    for (int s = 0; s < NS; ++s)
      if (s < n) VDI_CHECK(!mp.src[s].nrec || gidx[s] + cnt[s] <= mp.src[s].nrec, "merge_fast: record index past the source");
    const bool cand = valid && m > 0 && (int)m <= k;
    int bk = (valid && (int)m > k) ? bucket_of(m) : -1;
    const bool bulk = bulk_ok && p0 + 32 <= mp.P;  // tail group / unaligned output: plain stores
    bool pass = cand;
    if (bulk) {
      // the bulk engine must have read the previous image before we touch it
      if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      __syncwarp();
      for (uint32_t j = 0; j < written; ++j) {  // lazy re-zero of last time's slots
        my_depth[j] = make_float2(0.f, 0.f);
        my_rgba[j] = make_float4(0.f, 0.f, 0.f, 0.f);
      }
      written = 0;
      if (cand) {
        uint32_t start[NS];
        uint32_t j = 0;
#pragma unroll
        for (int s = 0; s < NS; ++s) {
          start[s] = j;
          j += cnt[s];
        }
        // every record straight into its slot of the image with async copies
        // (LDGSTS): all of the list's loads in flight at once, no registers,
        // no per-record source selection
#pragma unroll
        for (int s = 0; s < NS; ++s) {
          if (s < n) {
            const float2* dp = mp.src[s].depth + gidx[s];
            const float4* cp = mp.src[s].rgba + gidx[s];
            const uint32_t sd0 = smem_u32(my_depth + start[s]), sc0 = smem_u32(my_rgba + start[s]);
            for (uint32_t jj = 0; jj < cnt[s]; ++jj) {
              asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sd0 + jj * 8), "l"(dp + jj) : "memory");
              asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sc0 + jj * 16), "l"(cp + jj) : "memory");
            }
          }
        }
        asm volatile("cp.async.wait_all;" ::: "memory");
        written = m;
        // already in depth order (e.g. a single PE's run)?  then only validate
        bool sorted = true;
        float prev_tb = -CUDART_INF_F;
        for (uint32_t i = 0; i < m; ++i) {
          const float2 d = my_depth[i];
          if (my_rgba[i].w == 0.f || d.x < prev_tb) sorted = false;
          prev_tb = d.y;
        }
        if (!sorted) {
          pass = run_merge<NS>(my_depth, 1, start, cnt, m, my_perm, 1, [&](uint32_t idx) { return my_rgba[idx].w; });
          if (pass) {  // apply the permutation in place (cycle following, bit 15 marks done)
            for (uint32_t r = 0; r < m; ++r) {
              if (my_perm[r] & 0x8000u) continue;
              const uint32_t r0 = r;
              const float2 td = my_depth[r0];
              const float4 tc = my_rgba[r0];
              uint32_t cur = r0;
              for (;;) {
                const uint32_t src = my_perm[cur] & 0x7fffu;
                my_perm[cur] = (uint16_t)(src | 0x8000u);
                if (src == r0) {
                  my_depth[cur] = td;
                  my_rgba[cur] = tc;
                  break;
                }
                my_depth[cur] = my_depth[src];
                my_rgba[cur] = my_rgba[src];
                cur = src;
              }
            }
          } else {  // transparent / overlapping records: zeros now, general path later
            for (uint32_t i = 0; i < m; ++i) {
              my_depth[i] = make_float2(0.f, 0.f);
              my_rgba[i] = make_float4(0.f, 0.f, 0.f, 0.f);
            }
          }
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) {
        bulk_store(mp.out_depth + (size_t)p0 * k, o_depth, 32u * k * 8u);
        bulk_store(mp.out_rgba + (size_t)p0 * k, o_rgba, 32u * k * 16u);
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
    } else {
      // plain-store path (tail group or unaligned output): per-list stores
      if (lane == 0) ++plain_acc;
      if (cand) pass = direct_list<NS>(mp, p, gidx, cnt, m);
      if (valid) {
        float2* od = mp.out_depth + (size_t)p * k;
        float4* oc = mp.out_rgba + (size_t)p * k;
        for (int jj = pass ? (int)m : 0; jj < k; ++jj) {
          od[jj] = make_float2(0.f, 0.f);
          oc[jj] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
      }
    }
    if (cand && !pass) bk = VDI_BUCKET_GENERAL;  // transparent or overlapping records
    if (__any_sync(kFull, bk >= 0)) push_entries<NS>(mp, bk, p, m, gidx, lane);
    if (bk >= 0) srch_acc += m;
    if (valid) {
      mp.out_count[p] = pass ? (uint8_t)m : (uint8_t)0;
      if (mp.stat_m) mp.stat_m[p] = (uint16_t)m;
      if (mp.stat_gamma) mp.stat_gamma[p] = 0.f;
      if (mp.stat_margin) mp.stat_margin[p] = CUDART_INF_F;  // no comparison executed (overwritten if searched)
    }
  }
  if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    rec_acc += __shfl_down_sync(kFull, rec_acc, d);
    plain_acc += __shfl_down_sync(kFull, plain_acc, d);
    srch_acc += __shfl_down_sync(kFull, srch_acc, d);
  }
  if (lane == 0) {
    if (rec_acc) atomicAdd(mp.records_in, rec_acc);
    if (plain_acc) atomicAdd(mp.fallback_groups, plain_acc);
    if (srch_acc && mp.records_search) atomicAdd(mp.records_search, srch_acc);
  }
}

// ---------------------------------------------------------------------------
// Search path for short lists (m <= 40), in two kernels:
//   search_gather : thread per list (16 warps per SM hide the latency): the
//                   run-based k-way merge over the per-PE runs,
//                   the samples written in depth order to a pool slot in
//                   [batch][sample][lane] layout, the gap flag in alpha's sign;
//                   transparent / overlapping records -> general path;
//   search_sweep  : warp per batch of 32 lists: each lane's first samples in a
//                   statically indexed register array, the rest in the warp's
//                   shared rows (cp.async); the bisection (PAPER.md:100-101,
//                   :176) as predicated lock-step sweeps, and the final write
//                   sweep.
// ---------------------------------------------------------------------------

// Gather of one batch of short search lists (k_out < m <= 40), thread per
// list: the run-based k-way merge over the per-PE runs, their
// heads in registers (long_gather_lane), writes the samples in depth order to
// the batch's pool slot in [sample][lane] layout with the gap flag in the sign
// of alpha; transparent / overlapping records -> general path.
template <int NS, int CH = 8, int RS = 0>
__device__ __forceinline__ bool long_gather_lane(const MergeParams& mp, uint32_t m, const uint32_t (&goff)[NS],
                                                 const uint32_t (&cnt)[NS], float4* orgba, float2* odep,
                                                 float4* srgba = nullptr);
#ifndef VDI_SGATHER_CH
#define VDI_SGATHER_CH 8  // records loaded per trip in the short gather
#endif
#ifndef VDI_SGATHER_MINB
#define VDI_SGATHER_MINB 1
#endif
template <int NS>
__device__ __forceinline__ void gather_short_batch(const MergeParams& mp, uint32_t b, uint32_t nb1, uint32_t c0,
                                                   uint32_t c1, uint32_t lane) {
  const int n = mp.n_src;
  const int bucket = b < nb1 ? 1 : 0;
  const uint32_t i = (bucket == 1 ? b : b - nb1) * 32 + lane;
  const bool valid = i < (bucket == 0 ? c0 : c1);
  const uint32_t* ent = mp.wl[bucket] + (size_t)(valid ? i : 0) * (3 + n);
  const uint32_t p = valid ? ent[0] : 0u, m = valid ? ent[2] : 0u;
  uint32_t goff[NS], cnt[NS];
#pragma unroll
  for (int s = 0; s < NS; ++s) {
    goff[s] = cnt[s] = 0;
    if (valid && s < n) {
      goff[s] = ent[3 + s];
      cnt[s] = __ldg(mp.src[s].count + p);
    }
  }
#pragma unroll
  for (int s = 0; s < NS; ++s)
    if (s < n) VDI_CHECK(!mp.src[s].nrec || goff[s] + cnt[s] <= mp.src[s].nrec, "short gather: record index past the source");
  VDI_CHECK(!valid || (m > (uint32_t)mp.k_out && m <= 40), "short gather: m outside (k_out, 40]");
  // one pool slot per batch of 32 entries (a warp here = one batch)
  uint32_t slot = 0;
  if (lane == 0) {
    slot = atomicAdd(mp.pool_next, 1u);
    mp.batch_slot[bucket][i >> 5] = slot;  // >= pool_cap: the sweep skips the batch
  }
  slot = __shfl_sync(kFull, slot, 0);
  if (slot >= mp.pool_cap) {  // pool exhausted: the batch's lists take the general path
    if (__any_sync(kFull, valid)) push_entries<NS>(mp, valid ? VDI_BUCKET_GENERAL : -1, p, m, goff, lane);
    return;
  }
  float4* orgba = mp.pool_rgba + (size_t)slot * 40 * 32 + lane;
  float2* odep = mp.pool_depth + (size_t)slot * 40 * 32 + lane;
  // run-based k-way merge with the run heads in registers, straight into the
  // slot columns (measured C3 search stage 0.152 -> 0.142 ms vs staging the
  // depths in shared memory and merging there)
  bool bad = false;
  if (valid) {
    bad = !long_gather_lane<NS, VDI_SGATHER_CH>(mp, m, goff, cnt, orgba, odep);
    uint32_t* og = mp.pool_gap + (size_t)slot * 64 + lane;
    og[0] = bad ? 0xffffffffu : 0u;  // skip marker
    og[32] = bad ? 0xffffffffu : 0u;
  }
  const int bk = (valid && bad) ? VDI_BUCKET_GENERAL : -1;
  if (__any_sync(kFull, bk >= 0)) push_entries<NS>(mp, bk, p, m, goff, lane);
}

// Short-list sweep of one batch (32 work-list entries, lane = list): the
// samples are loaded once -- the first R into a statically indexed register
// file, the rest (cp.async) into the warp's shared-memory rows [q - R][lane]
// -- then the memoised bisection (see Bisection) sweeps while any lane still
// needs a count; (|acc|^2, |acc - s|^2) are one packed f32x2 chain.  Keeping
// only R samples in registers raises the resident warps per SM (8 at 40
// register samples, 16 at 16); the shared rows are swept by a rolled loop of
// 8-step chunks, which keeps the kernel's code (and instruction-cache misses)
// small.
#ifndef VDI_UB_EXIT
#define VDI_UB_EXIT 1  // count sweeps also stop once the count can no longer reach k
#endif
#ifndef VDI_MEMO
#define VDI_MEMO 1  // 0: plain bisection in the short sweep (A/B of the memo's cost)
#endif
#ifndef VDI_SWEEP_R
// measured (C3 search stage; shared part rolled): R = 8 / 16 / 24 -> 0.146 / 0.138 / 0.143 ms
// (fully unrolled: R = 8 / 16 / 24 / 40 -> 0.160 / 0.161 / 0.153 / 0.160)
#define VDI_SWEEP_R 16
#endif
__device__ __forceinline__ void cp_async16(void* sdst, const void* gsrc) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(sdst)), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

// The sweeps of one batch whose samples are in place: rows 0..R-1 in the
// register array S, row q >= R at sm[(q - OFF) * 32 + lane] (NaN past m).
template <int MS, int R, int OFF>
__device__ __forceinline__ void sweep_rows(const MergeParams& mp, uint32_t p, int mi, bool valid, bool bad,
                                           const float4 (&S)[R], const float4* __restrict__ sm,
                                           const float2* __restrict__ dcol) {
  const int lane = threadIdx.x & 31;
  const int k = mp.k_out;
  const float qnan = __int_as_float(0x7fc00000);
  {
    // memoised bisection: a count sweep at g2 takes the same decisions for
    // every g2' in [L, U), so a later midpoint inside the interval of the
    // latest sweep on either side of the bracket reuses its count; each lane
    // resolves such levels on its own and the warp sweeps while any lane
    // still needs a sweep
    Bisection bs;
    bs.init(mp.gamma_max, valid && !bad && mp.max_iters > 0);
    for (;;) {
      bs.advance(k, mp.max_iters);
      if (!__any_sync(kFull, bs.active)) break;
      const float g2 = bs.g2;
      float ar = 0.f, ag = 0.f, ab = 0.f, aa = 0.f, L = -1.f, U = CUDART_INF_F;
      int sc = 0;
      auto cstep = [&](const float4 sv, bool first) {
        const bool gap = sv.w < 0.f;  // NaN padding: false
        const float sa = fabsf(sv.w);
        float n2, d2;
        n2d2_packed(ar, ag, ab, aa, sv.x, sv.y, sv.z, sa, n2, d2);
        // the comparisons of this step: v1 = |acc|^2 at a gap (Q8), v2 = D^2
        // unless the gap closed the segment; NaN = not made (ignored below)
        const float v1 = gap ? n2 : qnan;
        const bool gcl = v1 > g2;
        const float v2 = gcl ? qnan : d2;
        const bool dsp = v2 > g2;
        if (!first && VDI_MEMO) {  // a split tightens U, a merge raises L
          U = gcl ? fminf(U, v1) : U;
          L = gcl ? L : fmaxf(L, v1);
          U = dsp ? fminf(U, v2) : U;
          L = dsp ? L : fmaxf(L, v2);
        }
        const bool st = first | gcl | dsp;
        const float tr = 1.0f - aa;
        ar = st ? sv.x : fmaf(tr, sv.x, ar);
        ag = st ? sv.y : fmaf(tr, sv.y, ag);
        ab = st ? sv.z : fmaf(tr, sv.z, ab);
        aa = st ? sa : fmaf(tr, sa, aa);
        sc += st ? 1 : 0;
      };
      // a lane still needs samples while its count can still reach k: past
      // k the sweep's answer is "> k"; with sc + (samples left) < k it is
      // "< k" (each sample opens at most one segment) -- both decide the level
      auto needs = [&](int q) { return bs.active && q < mi && sc <= k && sc + (mi - q) >= k; };
      bool more = true;
      int qe = MS;  // samples swept
#pragma unroll
      for (int q = 0; q < R; ++q) {  // the register samples: static indices
        if ((q & 7) == 0 && q > 0 && !__any_sync(kFull, VDI_UB_EXIT ? needs(q) : (bs.active && q < mi && sc <= k))) {
          more = false;
          qe = q;
          break;
        }
        cstep(S[q], q == 0);
      }
      if (more) {
#pragma unroll 1
        for (int q0 = R; q0 < MS; q0 += 8) {  // the shared rows: a rolled loop of 8-step chunks (code size)
          if (!__any_sync(kFull, VDI_UB_EXIT ? needs(q0) : (bs.active && q0 < mi && sc <= k))) {
            qe = q0;
            break;
          }
#pragma unroll
          for (int u = 0; u < 8; ++u) cstep(sm[(q0 - OFF + u) * 32 + lane], false);
        }
      }
      // an unfinished sweep below k records its bound sc + (samples left) < k
      // (<= k and != k: the same decision as the exact count)
      const int cr = (qe < mi && sc <= k) ? sc + (mi - qe) : sc;
      if (bs.active) bs.swept(cr, VDI_MEMO ? L : 1.f, VDI_MEMO ? U : 0.f, k, mp.max_iters);
    }
    const float best = bs.best;
    if (valid && !bad) {  // final write sweep
      const float gg = best * best;
      float2* od = mp.out_depth + (size_t)p * k;
      float4* oc = mp.out_rgba + (size_t)p * k;
      float ar = 0.f, ag = 0.f, ab = 0.f, aa = 0.f, tf = 0.f, tb = 0.f;
      int c = 0;
      auto wstep = [&](const float4 sv, const float2 d, int q) {
        const bool gap = sv.w < 0.f;
        const float sa = fabsf(sv.w);
        const float n2 = fmaf(aa, aa, fmaf(ab, ab, fmaf(ag, ag, ar * ar)));
        const float d2 = dist2(ar, ag, ab, aa, sv.x, sv.y, sv.z, sa);
        const bool st = (q == 0) | (gap & (n2 > gg)) | (d2 > gg);
        if (st && q > 0 && c <= k) {  // close the open segment (ends at its last content sample)
          od[c - 1] = make_float2(tf, tb);
          oc[c - 1] = make_float4(ar, ag, ab, aa);
        }
        const float tr = 1.0f - aa;
        ar = st ? sv.x : fmaf(tr, sv.x, ar);
        ag = st ? sv.y : fmaf(tr, sv.y, ag);
        ab = st ? sv.z : fmaf(tr, sv.z, ab);
        aa = st ? sa : fmaf(tr, sa, aa);
        tf = st ? d.x : tf;
        tb = d.y;
        c += st ? 1 : 0;
      };
      float2 dq[8];
#pragma unroll
      for (int q = 0; q < R; ++q) {
        if ((q & 7) == 0) {  // depth of the next 8 samples: loads issued together, before the stores
#pragma unroll
          for (int u = 0; u < 8; ++u)
            if (q + u < mi) dq[u] = dcol[(q + u) * 32];
        }
        if (q < mi) wstep(S[q], dq[q & 7], q);
      }
#pragma unroll 1
      for (int q0 = R; q0 < mi; q0 += 8) {
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (q0 + u < mi) dq[u] = dcol[(q0 + u) * 32];
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (q0 + u < mi) wstep(sm[(q0 - OFF + u) * 32 + lane], dq[u], q0 + u);
      }
      if (mi > 0 && c <= k) {
        od[c - 1] = make_float2(tf, tb);
        oc[c - 1] = make_float4(ar, ag, ab, aa);
      }
      mp.out_count[p] = (uint8_t)c;
      if (mp.stat_gamma) mp.stat_gamma[p] = best;
    }
  }
}

// Short-list sweep of one batch of the pool (two-kernel path): samples
// 0..R-1 into registers, R..MS-1 into the warp's shared rows (cp.async).
template <int MS, int R>
__device__ __forceinline__ void sweep_batch(const MergeParams& mp, int bucket, uint32_t batch, float4* __restrict__ sm) {
  const int lane = threadIdx.x;
  const int n = mp.n_src;
  const uint32_t total = min(mp.wl_count[bucket], mp.wl_cap);
  const uint32_t* wl = mp.wl[bucket];
  const uint32_t e = batch * 32 + lane;
  const bool valid = e < total;
  const uint32_t* ent = wl + (size_t)(valid ? e : 0) * (3 + n);
  const uint32_t p = valid ? ent[0] : 0u;
  const int mi = valid ? (int)ent[2] : 0;
  const uint32_t slot = mp.batch_slot[bucket][batch];
  if (slot >= mp.pool_cap) return;
  const uint32_t* gp = mp.pool_gap + (size_t)slot * 64 + lane;
  const uint32_t gw0 = valid ? gp[0] : 0u, gw1 = valid ? gp[32] : 0u;
  const bool bad = valid && gw0 == 0xffffffffu && gw1 == 0xffffffffu;  // sent to the general path
  const float4* col = mp.pool_rgba + (size_t)slot * 40 * 32 + lane;
  const float2* dcol = mp.pool_depth + (size_t)slot * 40 * 32 + lane;
  // samples past m are NaN: D^2 = NaN never exceeds g^2 and their gap bits
  // are 0, so they never split and the count sweeps need no "q < m" test
  float4 S[R];
  const float qnan = __int_as_float(0x7fc00000);
  const float4 nan4 = make_float4(qnan, qnan, qnan, qnan);
  __syncwarp();  // the previous batch's reads of the shared rows are done
#pragma unroll
  for (int q = R; q < MS; ++q) {
    if (q < mi && !bad) cp_async16(sm + (q - R) * 32 + lane, col + q * 32);
    else sm[(q - R) * 32 + lane] = nan4;
  }
#pragma unroll
  for (int q = 0; q < R; ++q) S[q] = (q < mi && !bad) ? col[q * 32] : nan4;
  cp_async_wait_all();  // each lane reads only its own column: no warp barrier needed
  sweep_rows<MS, R, R>(mp, p, mi, valid, bad, S, sm, dcol);
}

#ifndef VDI_SWEEP_MINB
#define VDI_SWEEP_MINB 16  // 128 registers at R = 16: 16 warps per SM
#endif

// ---------------------------------------------------------------------------
// Search path for long lists (m > 40), one fused kernel: every warp owns a
// private slot of global memory ([sample][lane] layout: rgba with the gap flag
// in the sign of alpha, then depth) that it refills batch after batch, so the
// slots in flight stay resident in L2 while the bisection sweeps re-read them
// (PAPER.md:176's "multiple passes" do not become HBM passes); the lists'
// records are read from the sources once.
// ---------------------------------------------------------------------------
// L2 eviction priorities of the long search (VDI_LONG_POLICY): the slot rows
// re-read by every bisection sweep evict last, the streamed source records and
// output slots evict first.
#ifndef VDI_LONG_POLICY
#define VDI_LONG_POLICY 1  // measured C5 long search 16.03 -> 15.43 ms (2: slots only, 16.06), C2 neutral
#endif
__device__ __forceinline__ unsigned long long pol_last() {
  unsigned long long p;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ unsigned long long pol_first() {
  unsigned long long p;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ float4 slot_ld(const float4* a) {
#if VDI_LONG_POLICY
  float4 v;
  asm volatile("ld.global.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(a), "l"(pol_last()));
  return v;
#else
  return *a;
#endif
}
__device__ __forceinline__ void slot_st(float4* a, float4 v) {
#if VDI_LONG_POLICY
  asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1,%2,%3,%4}, %5;" ::"l"(a), "f"(v.x), "f"(v.y), "f"(v.z),
               "f"(v.w), "l"(pol_last())
               : "memory");
#else
  *a = v;
#endif
}
__device__ __forceinline__ float4 src_ld4(const float4* a) {
#if VDI_LONG_POLICY == 1
  float4 v;
  asm volatile("ld.global.nc.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(a), "l"(pol_first()));
  return v;
#else
  return __ldg(a);
#endif
}
// the slots' depth column: written by the gather, read once by the final
// write sweep -- evict first, so the rgba rows the sweeps re-read stay in L2
__device__ __forceinline__ void dep_st(float2* a, float2 v) {
#if VDI_LONG_POLICY == 1
  asm volatile("st.global.L2::cache_hint.v2.f32 [%0], {%1,%2}, %3;" ::"l"(a), "f"(v.x), "f"(v.y), "l"(pol_first())
               : "memory");
#else
  *a = v;
#endif
}
__device__ __forceinline__ float2 dep_ld(const float2* a) {
#if VDI_LONG_POLICY == 1
  float2 v;
  asm volatile("ld.global.L2::cache_hint.v2.f32 {%0,%1}, [%2], %3;" : "=f"(v.x), "=f"(v.y) : "l"(a), "l"(pol_first()));
  return v;
#else
  return *a;
#endif
}
__device__ __forceinline__ void out_st4(float4* a, float4 v) {
#if VDI_LONG_POLICY == 1
  asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1,%2,%3,%4}, %5;" ::"l"(a), "f"(v.x), "f"(v.y), "f"(v.z),
               "f"(v.w), "l"(pol_first())
               : "memory");
#else
  *a = v;
#endif
}

// Gather of the lanes' lists (valid lanes) into the slot columns orgba/odep
// (stride 32): run-based k-way merge over the runs' head
// t_front kept in registers, 8 records loaded per trip.  Returns false for a
// transparent or overlapping record (Q23, Q12: the general path).  RS > 0:
// rgba rows r < RS go to the shared-memory column srgba instead of orgba.
template <int NS, int CH, int RS>
__device__ __forceinline__ bool long_gather_lane(const MergeParams& mp, uint32_t m, const uint32_t (&goff)[NS],
                                                 const uint32_t (&cnt)[NS], float4* orgba, float2* odep,
                                                 float4* srgba) {
  bool bad = false;
  uint32_t hp[NS];
  float ht[NS];  // t_front of each run's head, kept in registers (one load per record)
#pragma unroll
  for (int s = 0; s < NS; ++s) {
    hp[s] = 0;
    ht[s] = cnt[s] ? __ldg(&mp.src[s].depth[goff[s]].x) : CUDART_INF_F;
  }
  float prev_tb = -CUDART_INF_F;
  uint32_t r = 0;
  while (r < m) {
    int b = -1, b2 = NS;
    float bt = CUDART_INF_F, b2t = CUDART_INF_F;
#pragma unroll
    for (int s = 0; s < NS; ++s)
      if (hp[s] < cnt[s]) {
        const float t = ht[s];
        if (b < 0 || t < bt) {
          if (b >= 0) {
            b2t = bt;
            b2 = b;
          }
          bt = t;
          b = s;
        } else if (t < b2t) {
          b2t = t;
          b2 = s;
        }
      }
    uint32_t ii = 0, cb = 0, gb = 0;
    const float2* dp = nullptr;
    const float4* cp = nullptr;
#pragma unroll
    for (int s = 0; s < NS; ++s)
      if (s == b) {
        ii = hp[s];
        cb = cnt[s];
        gb = goff[s];
        dp = mp.src[s].depth;
        cp = mp.src[s].rgba;
      }
    // take records of run b while they precede the next run's head (ties:
    // lower PE first, Q11), 8 loaded per trip (the ones past the cut are
    // reloaded, from L1/L2, when b is chosen again)
    float tn = CUDART_INF_F;
    // two chunks of CH/2 records: the next chunk of the run is loaded
    // (speculatively) before the current one is merged, so a run longer than
    // a chunk costs one round trip, not one per chunk
    constexpr int CQ = CH / 2;
    float2 dv[CQ], dn[CQ];
    float4 cv[CQ], cn[CQ];
    uint32_t nch = min((uint32_t)CQ, cb - ii);
#pragma unroll
    for (int u = 0; u < CQ; ++u)
      if ((uint32_t)u < nch) {
        dv[u] = __ldg(dp + gb + ii + u);
        cv[u] = src_ld4(cp + gb + ii + u);
      }
    for (bool first = true;;) {
      const uint32_t ii2 = ii + nch;
      const uint32_t nch2 = ii2 < cb ? min((uint32_t)CQ, cb - ii2) : 0u;
#pragma unroll
      for (int u = 0; u < CQ; ++u)
        if ((uint32_t)u < nch2) {
          dn[u] = __ldg(dp + gb + ii2 + u);
          cn[u] = src_ld4(cp + gb + ii2 + u);
        }
      uint32_t taken = 0;
      bool stop = false;
#pragma unroll
      for (int u = 0; u < CQ; ++u)
        if (!stop && (uint32_t)u < nch) {
          const float2 d = dv[u];
          if (!(first && u == 0) && !(d.x < b2t || (d.x == b2t && b < b2))) {
            stop = true;
            tn = d.x;
          } else {
            float4 c = cv[u];
            bad |= c.w == 0.f || d.x < prev_tb;  // Q23 / Q12
            if (r > 0 && d.x > prev_tb) c.w = -c.w;  // gap before this sample: sign of alpha
            prev_tb = d.y;
            if (RS > 0 && r < (uint32_t)RS) srgba[r * 32] = c;
            else slot_st(orgba + r * 32, c);
            dep_st(odep + r * 32, d);
            ++r;
            ++taken;
          }
        }
      ii += taken;
      first = false;
      if (stop) break;  // tn = head of run b
      if (ii >= cb) {
        tn = CUDART_INF_F;
        break;
      }
#pragma unroll
      for (int u = 0; u < CQ; ++u) {  // the whole chunk was taken: the next one is current
        dv[u] = dn[u];
        cv[u] = cn[u];
      }
      nch = nch2;
    }
#pragma unroll
    for (int s = 0; s < NS; ++s)
      if (s == b) {
        hp[s] = ii;
        ht[s] = tn;
      }
  }
  return !bad;
}

// Eight steps of a count-mode sweep over a pool column (same decisions as
// sweep()) with the validity-interval bookkeeping of Bisection: a comparison
// that split tightens U, one that merged raises L; comparisons that did not
// happen contribute NaN, which fminf / fmaxf ignore.  Samples past m (rows of
// longer lists of the batch, or the pool's slack) may be evaluated: their
// splits are not counted and their extra constraints only shrink [L, U),
// which keeps it valid.
__device__ __forceinline__ void long_step8(const float4 (&v)[8], int q0, int m, float g2, float& ar, float& ag,
                                           float& ab, float& aa, int& sc, float& L, float& U) {
  const float qn = __int_as_float(0x7fc00000);
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const float4 sv = v[u];
    const bool first = u == 0 && q0 == 0;  // the first sample opens without a comparison
    const bool gap = sv.w < 0.f;
    const float sa = fabsf(sv.w);
    const float n2 = fmaf(aa, aa, fmaf(ab, ab, fmaf(ag, ag, ar * ar)));
    const float d2 = dist2(ar, ag, ab, aa, sv.x, sv.y, sv.z, sa);
    const bool gcl = gap & (n2 > g2);  // the gap closed the segment: d2 not consulted (Q8)
    const bool dsp = d2 > g2;
    const bool dev = !gcl & !first;
    U = fminf(U, fminf(gcl ? n2 : qn, (dev & dsp) ? d2 : qn));
    L = fmaxf(L, fmaxf((gap & !gcl) ? n2 : qn, (dev & !dsp) ? d2 : qn));
    const bool st = first | gcl | dsp;
    const float tr = 1.0f - aa;
    ar = st ? sv.x : fmaf(tr, sv.x, ar);
    ag = st ? sv.y : fmaf(tr, sv.y, ag);
    ab = st ? sv.z : fmaf(tr, sv.z, ab);
    aa = st ? sa : fmaf(tr, sa, aa);
    sc += (st & (q0 + u < m)) ? 1 : 0;
  }
}

#ifndef VDI_LONG_SROWS
#define VDI_LONG_SROWS 32  // rgba rows of each long-search slot column kept in shared memory (multiple of 8)
#endif
// Rows q..q+7 of a slot column (q a multiple of 8, the same on every lane that
// shares the call): rows below RS from the warp's shared-memory column scol,
// the rest from the global slot column col.
template <int RS>
__device__ __forceinline__ void rows8(float4 (&X)[8], const float4* scol, const float4* __restrict__ col, int q) {
  if (RS > 0 && q < RS) {
#pragma unroll
    for (int u = 0; u < 8; ++u) X[u] = scol[(q + u) * 32];
  } else {
#pragma unroll
    for (int u = 0; u < 8; ++u) X[u] = slot_ld(col + (q + u) * 32);
  }
}

// One count-mode sweep over a pool column: chunks of 8 samples in two register
// buffers (the next chunk's loads are in flight while one is swept; ping-pong,
// no copies), leaving as soon as the count exceeds k.  Reads up to 24 rows past
// m (the pool has slack for that).
template <int RS>
__device__ __forceinline__ int long_count(const float4* scol, const float4* __restrict__ col, int m, float g2, int k,
                                          float& L, float& U) {
  float ar = 0.f, ag = 0.f, ab = 0.f, aa = 0.f;
  int sc = 0;
  L = -1.f;
  U = CUDART_INF_F;
  // three register chunks in rotation: the loads run two chunks (16 samples)
  // ahead of the sweep, which covers the L2 latency of the pool
  float4 A[8], B[8], C[8];
  rows8<RS>(A, scol, col, 0);
  rows8<RS>(B, scol, col, 8);
  int qn = 16;  // next row to load
  int q0 = 0;
  for (;;) {
    rows8<RS>(C, scol, col, qn);
    qn += 8;
    long_step8(A, q0, m, g2, ar, ag, ab, aa, sc, L, U);
    q0 += 8;
    if (q0 >= m || sc > k || (VDI_UB_EXIT && sc + (m - q0) < k)) break;
    rows8<RS>(A, scol, col, qn);
    qn += 8;
    long_step8(B, q0, m, g2, ar, ag, ab, aa, sc, L, U);
    q0 += 8;
    if (q0 >= m || sc > k || (VDI_UB_EXIT && sc + (m - q0) < k)) break;
    rows8<RS>(B, scol, col, qn);
    qn += 8;
    long_step8(C, q0, m, g2, ar, ag, ab, aa, sc, L, U);
    q0 += 8;
    if (q0 >= m || sc > k || (VDI_UB_EXIT && sc + (m - q0) < k)) break;
  }
  return (q0 < m && sc <= k) ? sc + (m - q0) : sc;  // unfinished below k: the bound (< k), see sweep_rows
}

// long_count with the warp in lock step: every lane sweeps the same rows at
// the same time (coalesced 512-B row loads of the slot), the loop ends when
// no lane still needs a sample (its bisection active, q < m, count <= k).
// Lanes that went past their end keep stepping harmlessly: samples past m are
// not counted, and extra constraints only shrink the memo interval.
template <int RS>
__device__ __forceinline__ int long_count_sync(const float4* scol, const float4* __restrict__ col, int m, float g2,
                                               int k, bool act, float& L, float& U) {
  float ar = 0.f, ag = 0.f, ab = 0.f, aa = 0.f;
  int sc = 0;
  L = -1.f;
  U = CUDART_INF_F;
  float4 A[8], B[8], C[8];
  rows8<RS>(A, scol, col, 0);
  rows8<RS>(B, scol, col, 8);
  int qn = 16;
  int q0 = 0;
  for (;;) {
    rows8<RS>(C, scol, col, qn);
    qn += 8;
    long_step8(A, q0, m, g2, ar, ag, ab, aa, sc, L, U);
    q0 += 8;
    if (!__any_sync(kFull, act && q0 < m && sc <= k && (!VDI_UB_EXIT || sc + (m - q0) >= k))) break;
    rows8<RS>(A, scol, col, qn);
    qn += 8;
    long_step8(B, q0, m, g2, ar, ag, ab, aa, sc, L, U);
    q0 += 8;
    if (!__any_sync(kFull, act && q0 < m && sc <= k && (!VDI_UB_EXIT || sc + (m - q0) >= k))) break;
    rows8<RS>(B, scol, col, qn);
    qn += 8;
    long_step8(C, q0, m, g2, ar, ag, ab, aa, sc, L, U);
    q0 += 8;
    if (!__any_sync(kFull, act && q0 < m && sc <= k && (!VDI_UB_EXIT || sc + (m - q0) >= k))) break;
  }
  return (q0 < m && sc <= k) ? sc + (m - q0) : sc;  // unfinished below k: the bound (< k), see sweep_rows
}

// The final write sweep over a pool column (same decisions and output as
// sweep(), the gap taken from the sign of alpha): rgba and depth in chunks of
// 8 with the next chunk's loads in flight, so the sweep does not wait on one
// L2 round trip per sample.
template <int RS>
__device__ __forceinline__ int long_write(const float4* scol, const float4* __restrict__ col,
                                          const float2* __restrict__ dcol, int m, float gamma, int k, float2* od,
                                          float4* oc) {
  const float gg = gamma * gamma;
  float ar = 0.f, ag = 0.f, ab = 0.f, aa = 0.f, tf = 0.f, tb = 0.f;
  int c = 0;
  float4 cv[8], cn[8];
  float2 dv[8], dn[8];
  rows8<RS>(cv, scol, col, 0);
#pragma unroll
  for (int u = 0; u < 8; ++u) dv[u] = dep_ld(dcol + u * 32);
  for (int q0 = 0; q0 < m; q0 += 8) {
    rows8<RS>(cn, scol, col, q0 + 8);
#pragma unroll
    for (int u = 0; u < 8; ++u) dn[u] = dep_ld(dcol + (q0 + 8 + u) * 32);
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int q = q0 + u;
      if (q < m) {
        const float4 sv = cv[u];
        const float2 d = dv[u];
        const bool gap = sv.w < 0.f;
        const float sa = fabsf(sv.w);
        const float n2 = fmaf(aa, aa, fmaf(ab, ab, fmaf(ag, ag, ar * ar)));
        const float d2 = dist2(ar, ag, ab, aa, sv.x, sv.y, sv.z, sa);
        const bool st = (q == 0) | (gap & (n2 > gg)) | (d2 > gg);
        if (st && q > 0 && c <= k) {  // close the open segment (ends at its last content sample)
          od[c - 1] = make_float2(tf, tb);
          out_st4(oc + (c - 1), make_float4(ar, ag, ab, aa));
        }
        const float tr = 1.0f - aa;
        ar = st ? sv.x : fmaf(tr, sv.x, ar);
        ag = st ? sv.y : fmaf(tr, sv.y, ag);
        ab = st ? sv.z : fmaf(tr, sv.z, ab);
        aa = st ? sa : fmaf(tr, sa, aa);
        tf = st ? d.x : tf;
        tb = d.y;
        c += st ? 1 : 0;
      }
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      cv[u] = cn[u];
      dv[u] = dn[u];
    }
  }
  if (m > 0 && c <= k) {
    od[c - 1] = make_float2(tf, tb);
    out_st4(oc + (c - 1), make_float4(ar, ag, ab, aa));
  }
  return c;
}

// Few long lists (C4: ~1000 at 1080p) would leave a lane-per-list sweep
// latency bound (~34 warps on the whole GPU, each lane running ~10 dependent
// sweeps).  Then every list gets a warp: lane j (heap node j + 1 of the next
// five bisection levels) evaluates the midpoint the sequential procedure would
// reach along that path (the same fp32 mid = 0.5 (lo + hi) recurrence), all
// lanes sweep the same samples (broadcast loads), and the warp walks the five
// levels with the counts, stopping where the procedure stops (count == k_out,
// or I iterations).  Same gamma*, same output.
#ifndef VDI_SPEC_MAX
#define VDI_SPEC_MAX 8192
#endif
template <int RS>
__device__ __forceinline__ float long_spec_bisect(const MergeParams& mp, const float4* scol, const float4* col, int m,
                                                  int lane) {
  const int k = mp.k_out;
  const uint32_t jn = lane < 31 ? (uint32_t)lane + 1 : 1u;  // heap node of this lane
  const int depth = 31 - __clz(jn);
  float lo = 0.f, hi = mp.gamma_max, best = mp.gamma_max;
  int it = 0;
  bool done = mp.max_iters <= 0;
  while (!done) {
    float lw = lo, hg = hi, md = 0.5f * (lw + hg);
    for (int b = depth - 1; b >= 0; --b) {  // bit 1: count > k (lo = mid), bit 0: count <= k (hi = mid)
      if ((jn >> b) & 1u) lw = md;
      else hg = md;
      md = 0.5f * (lw + hg);
    }
    float L, U;
    const int c = long_count<RS>(scol, col, m, md * md, k, L, U);
    uint32_t node = 1;
    for (int lev = 0; lev < 5 && !done; ++lev) {
      const int cn = __shfl_sync(kFull, c, (int)node - 1);
      const float mid = __shfl_sync(kFull, md, (int)node - 1);
      if (cn <= k) {
        best = hi = mid;
        if (cn == k) done = true;
        node = 2 * node;
      } else {
        lo = mid;
        node = 2 * node + 1;
      }
      if (++it >= mp.max_iters) done = true;
    }
  }
  return best;
}

#ifndef VDI_LONG_WPS
#define VDI_LONG_WPS 8  // resident long-search warps per SM (their slots in flight stay in L2)
#endif
template <int NS>
__global__ void __launch_bounds__(32) long_search_kernel(MergeParams mp) {
  const int lane = threadIdx.x;
  const int k = mp.k_out, n = mp.n_src;
  const uint32_t c2 = min(mp.wl_count[2], mp.wl_cap), c3 = min(mp.wl_count[3], mp.wl_cap);
  if (mp.long_hint && blockIdx.x == 0 && lane == 0) {  // zero-copy note for the host's frames schedule,
    const uint32_t h = c2 + c3 > kSerialLong ? 1u : 0u;  // written only when it changes
    if (*mp.long_hint_dev != h) {
      *mp.long_hint_dev = h;
      *(volatile uint32_t*)mp.long_hint = h;
    }
  }
  if (c2 + c3 == 0) return;  // no long lists: leave before the claim atomics
  const uint32_t cap = mp.long_maxm;  // rows of a slot
  char* slot = mp.long_pool + (size_t)blockIdx.x * mp.long_slot;
  float4* col0 = reinterpret_cast<float4*>(slot);
  float2* dcol0 = reinterpret_cast<float2*>(slot + (size_t)(cap + 32) * 32 * 16);
  constexpr int RS = VDI_LONG_SROWS;
  extern __shared__ float4 lsm[];  // rgba rows 0..RS-1 of the slot columns (RS x 32 float4)
  const bool spec = c2 + c3 <= VDI_SPEC_MAX;
  const uint32_t nb2 = (c2 + 31) / 32, nb3 = (c3 + 31) / 32;
  for (;;) {
    // claim: a batch of 32 lists (lane = list), or one list (spec: the warp)
    uint32_t t = 0;
    if (lane == 0) t = atomicAdd(&mp.search_ticket[spec ? 4 : 3], 1u);
    t = __shfl_sync(kFull, t, 0);
    if (t >= (spec ? c2 + c3 : nb2 + nb3)) break;
    uint32_t e;
    int bucket;
    bool valid;
    if (spec) {
      bucket = t < c3 ? 3 : 2;  // the longest bucket first
      e = t < c3 ? t : t - c3;
      valid = lane == 0;        // lane 0 gathers the list into column 0
    } else {
      bucket = t < nb3 ? 3 : 2;
      e = (t < nb3 ? t : t - nb3) * 32 + lane;
      valid = e < (bucket == 2 ? c2 : c3);
    }
    const uint32_t* ent = mp.wl[bucket] + (size_t)(valid ? e : (spec ? e : 0)) * (3 + n);
    const uint32_t p = (valid || spec) ? ent[0] : 0u, m = (valid || spec) ? ent[2] : 0u;
    uint32_t goff[NS], cnt[NS];
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      goff[s] = cnt[s] = 0;
      if (valid && s < n) {
        goff[s] = ent[3 + s];
        cnt[s] = __ldg(mp.src[s].count + p);
      }
    }
#pragma unroll
    for (int s = 0; s < NS; ++s)
      if (s < n) VDI_CHECK(!mp.src[s].nrec || goff[s] + cnt[s] <= mp.src[s].nrec, "long search: record index past the source");
    bool bad = valid && m > cap;  // cannot hold it: general path
    if (valid && !bad)
      bad = !long_gather_lane<NS, 8, RS>(mp, m, goff, cnt, col0 + (spec ? 0 : lane), dcol0 + (spec ? 0 : lane),
                                         lsm + (spec ? 0 : lane));
    __syncwarp();  // the slot columns are complete (and visible to the warp)
    if (__any_sync(kFull, bad)) push_entries<NS>(mp, bad ? VDI_BUCKET_GENERAL : -1, p, m, goff, lane);
    if (spec) {
      if (__shfl_sync(kFull, bad ? 1 : 0, 0)) continue;
      const float best = long_spec_bisect<RS>(mp, lsm, col0, (int)m, lane);
      if (lane == 0) {
        const int c = long_write<RS>(lsm, col0, dcol0, (int)m, best, k, mp.out_depth + (size_t)p * k,
                                     mp.out_rgba + (size_t)p * k);
        mp.out_count[p] = (uint8_t)c;
        if (mp.stat_gamma) mp.stat_gamma[p] = best;
      }
    } else {
      // bisection (Q3-Q6), memoised per lane, the
      // warp sweeping in lock step (coalesced slot rows)
      const bool ok = valid && !bad;
      const float4* col = col0 + lane;
      const float4* scol = lsm + lane;
      Bisection bs;
      bs.init(mp.gamma_max, ok && mp.max_iters > 0);
      for (;;) {
        bs.advance(k, mp.max_iters);
        if (!__any_sync(kFull, bs.active)) break;
        float L, U;
        const int c = long_count_sync<RS>(scol, col, ok ? (int)m : 0, bs.g2, k, bs.active, L, U);
        if (bs.active) bs.swept(c, L, U, k, mp.max_iters);
      }
      if (ok) {
        const int c = long_write<RS>(scol, col, dcol0 + lane, (int)m, bs.best, k, mp.out_depth + (size_t)p * k,
                                     mp.out_rgba + (size_t)p * k);
        mp.out_count[p] = (uint8_t)c;
        if (mp.stat_gamma) mp.stat_gamma[p] = bs.best;
      }
    }
    __syncwarp();  // every lane is done with the slot before the next batch overwrites it
  }
}

// ---------------------------------------------------------------------------
// General path: thread per work-list entry (steps 1-6 with subdivision),
// samples in global scratch.  Used for overlapping / transparent records, for
// lists longer than a long-search slot (m > 1024) and when a pool is full.
// ---------------------------------------------------------------------------
__device__ void over_into(float* acc, const float* b) {
  const float tr = 1.0f - acc[3];
  for (int c = 0; c < 4; ++c) acc[c] = fmaf(tr, b[c], acc[c]);
}

__device__ __forceinline__ void general_body(const MergeParams& mp, uint32_t tid, uint32_t nthreads) {
  const int n = mp.n_src, k = mp.k_out;
  const uint32_t total = min(mp.wl_count[VDI_BUCKET_GENERAL], mp.wl_cap);
  const uint32_t* wl = mp.wl[VDI_BUCKET_GENERAL];
  // this thread's scratch slice: A [m0] sorted records, B [2 m0] subdivided
  // samples, E [2 m0] endpoints (m0 <= n_src k_in, gen_stride = 4 n_src k_in)
  Rec* A = mp.scratch + (size_t)tid * mp.gen_stride;
  for (uint32_t e = tid; e < total; e += nthreads) {
    const uint32_t* ent = wl + (size_t)e * (3 + n);
    const uint32_t p = ent[0];
    const uint32_t m0 = ent[2];
    Rec* B = A + m0;
    float* E = reinterpret_cast<float*>(B + 2 * m0);
    // step 1: k-way merge of the per-PE sorted runs, dropping alpha == 0 (Q23)
    uint32_t pos[VDI_MAX_SRC], end[VDI_MAX_SRC];
    VDI_CHECK(4 * m0 <= mp.gen_stride, "general: list longer than its scratch slice");
    for (int s = 0; s < n; ++s) {
      pos[s] = ent[3 + s];
      end[s] = pos[s] + __ldg(mp.src[s].count + p);
      VDI_CHECK(!mp.src[s].nrec || end[s] <= mp.src[s].nrec, "general: record index past the source");
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
    // step 2: subdivide overlapping clusters (Eq. 2 generalised, Q12)
    const Rec* S = A;
    bool changed = false;
    for (int i = 1; i < m; ++i)
      if (A[i].tf < A[i - 1].tb) changed = true;
    if (changed) {
      int mm = 0, i = 0;
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
        for (int a = 1; a < ne; ++a) {  // insertion sort of the endpoints
          const float v = E[a];
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
    auto get = [&](int i) { return S[i]; };
    float gamma = 0.f;
    int cnt;
    double mgn = CUDART_INF;
    double* mg = mp.stat_margin ? &mgn : nullptr;
    if (m <= k) {
      for (int j = 0; j < m; ++j) {
        od[j] = make_float2(S[j].tf, S[j].tb);
        oc[j] = make_float4(S[j].r, S[j].g, S[j].b, S[j].a);
      }
      for (int j = m; j < k; ++j) {
        od[j] = make_float2(0.f, 0.f);
        oc[j] = make_float4(0.f, 0.f, 0.f, 0.f);
      }
      cnt = m;
    } else {
      unsigned long long st = 0;
      gamma = bisect(get, m, k, mp.max_iters, mp.gamma_max, mg, mp.sweep_steps ? &st : nullptr);
      cnt = sweep(get, m, gamma, k, od, oc, mg, mp.sweep_steps ? &st : nullptr);
      if (st) atomicAdd(mp.sweep_steps, st);
    }
    mp.out_count[p] = (uint8_t)cnt;
    if (mp.stat_m) mp.stat_m[p] = (uint16_t)m;
    if (mp.stat_gamma) mp.stat_gamma[p] = gamma;
    if (mp.stat_margin) mp.stat_margin[p] = (float)mgn;
  }
}

__global__ void __launch_bounds__(kSlowThreads) merge_general_kernel(MergeParams mp) {
  const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
  if (tid < mp.gen_threads) general_body(mp, tid, mp.gen_threads);
}

// Tie margins of the searched lists (VDI_FLAG_PIXEL_STATS, debug): thread per
// work-list entry of buckets 0-3 (scratch slice of the general path), the
// list gathered in depth order from its sources (step 1) and its bisection and
// final sweep replayed (the same procedure as the search kernels: same gamma*,
// same comparisons), with the margin min |sqrt(D^2) - gamma| of every
// executed comparison in double.  Lists with transparent or overlapping
// records are the general path's (it records their margins).
__global__ void __launch_bounds__(kSlowThreads) margins_kernel(MergeParams mp) {
  const uint32_t c[4] = {min(mp.wl_count[0], mp.wl_cap), min(mp.wl_count[1], mp.wl_cap),
                         min(mp.wl_count[2], mp.wl_cap), min(mp.wl_count[3], mp.wl_cap)};
  const uint32_t tot = c[0] + c[1] + c[2] + c[3];
  const int n = mp.n_src, k = mp.k_out;
  const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long steps = 0;
  Rec* A = mp.scratch + (size_t)tid * mp.gen_stride;
  const uint32_t t_end = (tot + 31) / 32 * 32;  // whole warps iterate (warp reduction below)
  for (uint32_t t = tid; t < t_end && tid < mp.gen_threads; t += mp.gen_threads) {
    if (t >= tot) continue;
    int b = 0;
    uint32_t e = t;
    while (e >= c[b]) e -= c[b++];
    const uint32_t* ent = mp.wl[b] + (size_t)e * (3 + n);
    const uint32_t p = ent[0];
    uint32_t pos[VDI_MAX_SRC], end[VDI_MAX_SRC];
    for (int s = 0; s < n; ++s) {
      pos[s] = ent[3 + s];
      end[s] = pos[s] + __ldg(mp.src[s].count + p);
    }
    int m = 0;
    bool bad = false;
    for (;;) {
      int best = -1;
      float bt = 0.f;
      for (int s = 0; s < n; ++s)
        if (pos[s] < end[s]) {
          const float tt = __ldg(&mp.src[s].depth[pos[s]].x);
          if (best < 0 || tt < bt) {
            best = s;
            bt = tt;
          }
        }
      if (best < 0) break;
      const float2 d = __ldg(mp.src[best].depth + pos[best]);
      const float4 cc = __ldg(mp.src[best].rgba + pos[best]);
      pos[best]++;
      bad |= cc.w == 0.f || (m > 0 && d.x < A[m - 1].tb);
      A[m++] = Rec{d.x, d.y, cc.x, cc.y, cc.z, cc.w};
    }
    if (bad) continue;
    auto get = [&](int i) { return A[i]; };
    double mgn = CUDART_INF;
    unsigned long long st = 0;
    const float g = bisect(get, m, k, mp.max_iters, mp.gamma_max, &mgn, &st);
    sweep(get, m, g, k, nullptr, nullptr, &mgn, &st);
    mp.stat_margin[p] = (float)mgn;
    steps += st;
  }
  // algorithmic sample-steps of the procedure (count sweeps to their early
  // exit + the final sweep), the unit of the search's ALU roofline
  for (int d = 16; d > 0; d >>= 1) steps += __shfl_down_sync(kFull, steps, d);
  if ((threadIdx.x & 31) == 0 && steps && mp.sweep_steps) atomicAdd(mp.sweep_steps, steps);
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

uint32_t scan_chunks(uint32_t P) { return (P + kChunk - 1) / kChunk; }

cudaError_t launch_scan(const MergeParams& mp, uint32_t* chunk_sum, uint32_t* group_base, cudaStream_t st,
                        int* launches) {
  if (!mp.n_src || !mp.P) return cudaSuccess;
  const uint32_t nc = scan_chunks(mp.P);
  chunk_sums_kernel<<<dim3(nc, mp.n_src), 256, 0, st>>>(mp, chunk_sum, nc);
  ++*launches;
  group_base_kernel<<<dim3(nc, mp.n_src), 128, 0, st>>>(mp, chunk_sum, nc, group_base);
  ++*launches;
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Dense gather support: compaction of a composited
// full-representation strip into the dense layout before
// it crosses NVLink; the root re-inflates with the pass-through kernel.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) sum_u32_kernel(const uint32_t* __restrict__ a, uint32_t n,
                                                      unsigned long long* __restrict__ out) {
  __shared__ unsigned long long red[8];
  unsigned long long acc = 0;
  for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) acc += a[i];
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) acc += __shfl_down_sync(kFull, acc, d);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long t = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    *out = t;
  }
}

// Compaction of one 32-list group (warp): the group's records are contiguous
// in the dense output, so record d of the group goes to od/oc[base + d] --
// consecutive lanes store consecutive records (coalesced, also across NVLink);
// the lane whose list holds record d is found by a 5-step search over the
// lists' exclusive prefix (warp shuffles).
__device__ __forceinline__ void compact_group(const uint8_t* __restrict__ count, const float2* __restrict__ depth,
                                              const float4* __restrict__ rgba, uint32_t P, int k, uint32_t g,
                                              size_t base, float2* __restrict__ od, float4* __restrict__ oc, int lane) {
  const uint32_t p = g * 32 + lane;
  const uint32_t c = p < P ? count[p] : 0u;
  const uint32_t incl = warp_incl_scan(c, lane), excl = incl - c;
  const uint32_t tot = __shfl_sync(kFull, incl, 31);
  for (uint32_t d0 = 0; d0 < tot; d0 += 32) {
    const uint32_t d = d0 + lane;
    uint32_t l = 0;
#pragma unroll
    for (int step = 16; step > 0; step >>= 1) {
      const uint32_t e = __shfl_sync(kFull, excl, (int)(l + step));
      if (e <= d) l += step;
    }
    // empty lists share their successor's prefix: l is the last list starting at or before d
    const uint32_t el = __shfl_sync(kFull, excl, (int)l);
    if (d < tot) {
      const size_t src = ((size_t)g * 32 + l) * k + (d - el);
      od[base + d] = __ldg(depth + src);
      oc[base + d] = __ldg(rgba + src);
    }
  }
}

__global__ void __launch_bounds__(128) compact_kernel(const uint8_t* __restrict__ count, const float2* __restrict__ depth,
                                                      const float4* __restrict__ rgba, uint32_t P, int k,
                                                      const uint32_t* __restrict__ group_base, float2* __restrict__ od,
                                                      float4* __restrict__ oc) {
  const int lane = threadIdx.x & 31;
  const uint32_t ng = (P + 31) / 32;
  for (uint32_t g = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); g < ng; g += gridDim.x * (blockDim.x >> 5))
    compact_group(count, depth, rgba, P, k, g, group_base[g], od, oc, lane);
}

cudaError_t launch_total(const MergeParams& mp, const uint32_t* chunk_sum, unsigned long long* out, cudaStream_t st,
                         int* launches) {
  sum_u32_kernel<<<1, 256, 0, st>>>(chunk_sum, scan_chunks(mp.P) * mp.n_src, out);
  ++*launches;
  return cudaGetLastError();
}

cudaError_t launch_compact(const uint8_t* count, const float2* depth, const float4* rgba, uint32_t P, int k,
                           const uint32_t* group_base, float2* od, float4* oc, cudaStream_t st, int* launches) {
  const uint32_t ng = (P + 31) / 32;
  if (!ng) return cudaSuccess;
  compact_kernel<<<std::min<uint32_t>((ng + 3) / 4, (uint32_t)sm_count() * 16), 128, 0, st>>>(count, depth, rgba, P, k,
                                                                                             group_base, od, oc);
  ++*launches;
  return cudaGetLastError();
}

template <class K>
static cudaError_t prep(K kernel, size_t smem, int threads, int* per_sm) {
  cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(per_sm, kernel, threads, smem);
  if (*per_sm < 1) *per_sm = 1;
  return e;
}

// Short search as two kernels: a gather kernel (thread per list, 16 warps per
// SM) followed by a sweep-only kernel (register-heavy, warp per batch).
template <int NS>
__global__ void __launch_bounds__(128, VDI_SGATHER_MINB) search_gather_kernel(MergeParams mp) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t c0 = min(mp.wl_count[0], mp.wl_cap), c1 = min(mp.wl_count[1], mp.wl_cap);
  const uint32_t nb0 = (c0 + 31) / 32, nb1 = (c1 + 31) / 32;
  for (;;) {
    uint32_t v = 0;
    if (lane == 0) v = atomicAdd(&mp.search_ticket[1], 1u);
    v = __shfl_sync(kFull, v, 0);
    if (v >= nb0 + nb1) break;
    gather_short_batch<NS>(mp, v, nb1, c0, c1, lane);
  }
}

// Short-list sweeps, warp per batch (dynamic claims, longest bucket first).
static constexpr int kSweepSmem = (40 - VDI_SWEEP_R) * 32 * 16;  // shared rows of the warp's samples
__global__ void __launch_bounds__(32, VDI_SWEEP_MINB) search_sweep_kernel(MergeParams mp) {
  extern __shared__ float4 sweep_rows[];
  const uint32_t c0 = min(mp.wl_count[0], mp.wl_cap), c1 = min(mp.wl_count[1], mp.wl_cap);
  const uint32_t nb0 = (c0 + 31) / 32, nb1 = (c1 + 31) / 32;
  for (;;) {
    uint32_t v = 0;
    if (threadIdx.x == 0) v = atomicAdd(&mp.search_ticket[0], 1u);
    v = __shfl_sync(kFull, v, 0);
    if (v >= nb0 + nb1) break;
    sweep_batch<40, VDI_SWEEP_R>(mp, v < nb1 ? 1 : 0, v < nb1 ? v : v - nb1, sweep_rows);
  }
}

template <int NS>
static cudaError_t launch_fast_ns(const MergeParams& mp, cudaStream_t st, int* launches) {
  const size_t smem = (size_t)(kFastThreads / 32) * fast_warp_bytes(mp.k_out);
  static int per_sm = 0;
  static size_t prepared = 0;
  if (smem != prepared) {
    cudaError_t e = prep(merge_fast_kernel<NS>, smem, kFastThreads, &per_sm);
    if (e != cudaSuccess) return e;
    prepared = smem;
  }
  const uint32_t groups = mp.g_end - mp.g_begin;
  if (!groups) return cudaSuccess;
  const uint32_t want = (groups + (kFastThreads / 32) - 1) / (kFastThreads / 32);
  uint32_t grid = (uint32_t)sm_count() * per_sm;
  if (grid > want) grid = want;
  merge_fast_kernel<NS><<<grid, kFastThreads, smem, st>>>(mp);
  ++*launches;
  return cudaGetLastError();
}

template <int NS>
static cudaError_t launch_search_ns(const MergeParams& mp, cudaStream_t st, int* launches) {
  cudaError_t e;
  // the search kernels fill the GPU (a share of it for the next VDI's
  // pass-through beside them was measured slower: profiles/README.md)
  auto part = [&](uint32_t full) { return std::max<uint32_t>(1, full); };
  static int g_per_sm = 0;  // one static per NS instantiation
  if (!g_per_sm) {
    if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&g_per_sm, search_gather_kernel<NS>, 128, 0)) != cudaSuccess)
      return e;
    if (g_per_sm < 1) g_per_sm = 1;
  }
  search_gather_kernel<NS><<<part(sm_count() * g_per_sm), 128, 0, st>>>(mp);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  ++*launches;
  {
    static int per_sm = 0;
    if (!per_sm) {
      if ((e = prep(search_sweep_kernel, kSweepSmem, 32, &per_sm)) != cudaSuccess) return e;
    }
    search_sweep_kernel<<<part(sm_count() * per_sm), 32, kSweepSmem, st>>>(mp);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    ++*launches;
  }
  long_search_kernel<NS><<<part(mp.long_warps), 32, (size_t)VDI_LONG_SROWS * 32 * 16, st>>>(mp);
  ++*launches;
  return cudaGetLastError();
}

uint32_t long_warps(uint32_t m_max, size_t* slot_bytes) {
  // warp-private slots of min(m_max, 1024) rows (+32 rows of read slack in
  // both columns: the count and write sweeps load up to 24 / 16 rows ahead);
  // at most VDI_LONG_WPS warps per SM and ~1 GB of slots
  const uint32_t rows = std::min<uint32_t>(std::max<uint32_t>(m_max, 41), 1024);
  *slot_bytes = ((size_t)(rows + 32) * 32 * 16 + (size_t)(rows + 32) * 32 * 8 + 255) & ~(size_t)255;
  const uint64_t fit = (1ull << 30) / *slot_bytes;
  return (uint32_t)std::max<uint64_t>(148, std::min<uint64_t>(fit, (uint64_t)sm_count() * VDI_LONG_WPS));
}

uint32_t general_threads(uint32_t m_max) {
  // one scratch slice of 4 m_max records per thread; at most ~512 MB of scratch
  const uint64_t per = 4ull * std::max<uint32_t>(m_max, 1) * sizeof(Rec);
  const uint64_t cap = (512ull << 20) / per;
  return (uint32_t)std::max<uint64_t>(128, std::min<uint64_t>(cap, (uint64_t)sm_count() * 4 * kSlowThreads));
}

cudaError_t launch_general(const MergeParams& mp, cudaStream_t st, int* launches) {
  merge_general_kernel<<<(mp.gen_threads + kSlowThreads - 1) / kSlowThreads, kSlowThreads, 0, st>>>(mp);
  ++*launches;
  return cudaGetLastError();
}

cudaError_t launch_margins(const MergeParams& mp, cudaStream_t st, int* launches) {
  margins_kernel<<<(mp.gen_threads + kSlowThreads - 1) / kSlowThreads, kSlowThreads, 0, st>>>(mp);
  ++*launches;
  return cudaGetLastError();
}

#define VDI_DISPATCH_NS(F, ...)                                  \
  if (mp.n_src <= 1) return F<1>(__VA_ARGS__);                   \
  if (mp.n_src <= 2) return F<2>(__VA_ARGS__);                   \
  if (mp.n_src <= 4) return F<4>(__VA_ARGS__);                   \
  if (mp.n_src <= 8) return F<8>(__VA_ARGS__);                   \
  if (mp.n_src <= 16) return F<16>(__VA_ARGS__);                 \
  return F<VDI_MAX_SRC>(__VA_ARGS__);

cudaError_t launch_fast(const MergeParams& mp, cudaStream_t st, int* launches) {
  VDI_DISPATCH_NS(launch_fast_ns, mp, st, launches)
}

cudaError_t launch_search(const MergeParams& mp, cudaStream_t st, int* launches) {
  VDI_DISPATCH_NS(launch_search_ns, mp, st, launches)
}

// VDI_FLAG_VALIDATE: input checks of one dense sub-VDI (thread per list):
// bit 0 count > k_in, bit 1 offset[p+1] - offset[p] != count[p] (or the last
// offset != total), bit 2 t_front >= t_back or NaN, bit 3 alpha outside
// [0, 1] or NaN, bit 4 a list's records not front-to-back and disjoint
// (t_front < previous t_back) -- the dense layout of PAPER.md:113-115 and
// the record invariants the merge relies on (Q7, Q23).
__global__ void __launch_bounds__(256) validate_kernel(const uint8_t* __restrict__ count,
                                                       const uint32_t* __restrict__ offset,
                                                       const float2* __restrict__ depth,
                                                       const float4* __restrict__ rgba, uint32_t P, int k,
                                                       unsigned long long total, int* err) {
  int e = 0;
  for (uint32_t p = blockIdx.x * blockDim.x + threadIdx.x; p < P; p += gridDim.x * blockDim.x) {
    const uint32_t c = count[p];
    if ((int)c > k) e |= 1;
    if (!offset) continue;
    const uint32_t o = offset[p];
    if (offset[p + 1] - o != c) e |= 2;
    if (p + 1 == P && offset[P] != total) e |= 2;
    if (o + c > total) {
      e |= 2;
      continue;
    }
    float prev_tb = -CUDART_INF_F;
    for (uint32_t j = 0; j < c; ++j) {
      const float2 d = depth[o + j];
      const float a = rgba[o + j].w;
      if (!(d.x < d.y)) e |= 4;
      if (!(a >= 0.f && a <= 1.f)) e |= 8;
      if (d.x < prev_tb) e |= 16;
      prev_tb = d.y;
    }
  }
  if (e) atomicOr(err, e);
}

cudaError_t launch_validate(const uint8_t* count, const uint32_t* offset, const float2* depth, const float4* rgba,
                            uint32_t P, int k, unsigned long long total, int* err, cudaStream_t st) {
  if (!P) return cudaSuccess;
  validate_kernel<<<std::min<uint32_t>((P + 255) / 256, (uint32_t)sm_count() * 8), 256, 0, st>>>(count, offset, depth,
                                                                                               rgba, P, k, total, err);
  return cudaGetLastError();
}

// Load every merge kernel now (lazy module loading could otherwise try to
// load a kernel while a spinning wait kernel of another loopback context
// occupies the device)
template <int NS>
static void preload_ns(cudaFuncAttributes* fa) {
  cudaFuncGetAttributes(fa, merge_fast_kernel<NS>);
  cudaFuncGetAttributes(fa, search_gather_kernel<NS>);
  cudaFuncGetAttributes(fa, long_search_kernel<NS>);
}

cudaError_t preload_merge() {
  cudaFuncAttributes fa;
  preload_ns<1>(&fa);
  preload_ns<2>(&fa);
  preload_ns<4>(&fa);
  preload_ns<8>(&fa);
  preload_ns<16>(&fa);
  preload_ns<VDI_MAX_SRC>(&fa);
  cudaFuncGetAttributes(&fa, chunk_sums_kernel);
  cudaFuncGetAttributes(&fa, group_base_kernel);
  cudaFuncGetAttributes(&fa, search_sweep_kernel);
  cudaFuncGetAttributes(&fa, merge_general_kernel);
  cudaFuncGetAttributes(&fa, margins_kernel);
  cudaFuncGetAttributes(&fa, sum_u32_kernel);
  cudaFuncGetAttributes(&fa, compact_kernel);
  return cudaGetLastError();
}

}  // namespace vdi
