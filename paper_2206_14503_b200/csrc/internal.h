// internal.h — libvdi internals shared by the .cu translation units.
// Product code (sm_100a).  Shares nothing with oracle/.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "vdi.h"

#define VDI_MAX_SRC 64        // sources (PEs) supported by one composite

// Debug build (make debug, -DVDI_CHECKS): device-side bounds checks of every
// index computed from the inputs; a failed check prints and traps.
#ifdef VDI_CHECKS
#include <cstdio>
#define VDI_CHECK(c, what)                                                          \
  do {                                                                              \
    if (!(c)) {                                                                     \
      printf("VDI_CHECK failed %s:%d: %s (block %d thread %d)\n", __FILE__, __LINE__, what, \
             (int)blockIdx.x, (int)threadIdx.x);                                    \
      __trap();                                                                     \
    }                                                                               \
  } while (0)
#else
#define VDI_CHECK(c, what) \
  do {                     \
  } while (0)
#endif
#define VDI_MAX_GRID_AXIS 16  // bricks per axis in a decomposition

namespace vdi {
// 24-byte record of the sub-supersegment scratch (AoS).
struct Rec {
  float tf, tb, r, g, b, a;
};

// One composite source (PE) as seen by the merge kernels: the strip's count
// slice and the source's payload array; record indices are absolute in the
// payload array (the receive-side scan adds MergeParams::src_base[s], the
// index of the strip's first record, which only the device knows).
struct SrcDesc {
  const uint8_t* count;
  const float2* depth;
  const float4* rgba;
  const uint32_t* offset;  // the source's exclusive scan of count (indexed by list), or null
  const uint32_t* gbase;   // or: the index of the first record of each 32-list group of the strip (pushed by
                           // the sender / from its scan); neither: the merge scans the counts itself
                           // (receive-side scan)
  unsigned long long nrec; // records addressable in depth/rgba (0: unknown; bounds of the VDI_CHECKS build)
};

// Work-list buckets of lists that need more than the pass-through:
// 0, 1 = gamma search with m <= 32 / 40 samples (samples in registers);
// 2, 3 = gamma search with 40 < m <= 64 / m > 64 samples (samples in a pool);
// 4 = general path (overlap subdivision, alpha==0 records, and lists whose
// search-pool slot could not be allocated; thread per list, per-thread scratch).
#define VDI_N_BUCKETS 5
// frames in flight: a VDI with more long lists than this (~16 waves of the long
// kernel: 148 SMs x 8 warps x 32 lists) runs its search without the next VDI's
// pass-through beside it (vdi_composite_frames; measured C5 +7.4 %)
static constexpr uint32_t kSerialLong = 600000;
#define VDI_BUCKET_GENERAL 4

struct MergeParams {
  SrcDesc src[VDI_MAX_SRC];
  int n_src;
  int k_out;
  int max_iters;
  float gamma_max;
  uint32_t P;          // lists in the strip
  uint32_t n_groups;   // ceil(P / 32)
  uint32_t g_begin, g_end;  // 32-list groups of this launch's chunk of the strip
  const uint32_t* group_base;  // [n_src][n_groups] exclusive scan of 32-list group sums
  const uint32_t* src_base;    // optional device [n_src]: added to the receive-side scan (strip start)
  uint8_t* out_count;          // [P]
  float2* out_depth;           // [P][k_out]
  float4* out_rgba;            // [P][k_out]
  // work lists: entry i of bucket b = wl[b][i*(3+n_src) ...] = {p, 0, m, off[0..n_src)}
  uint32_t* wl[VDI_N_BUCKETS];
  uint32_t* wl_count;          // [VDI_N_BUCKETS]
  uint32_t* long_hint;         // mapped host word or null: 1 when the long buckets hold > kSerialLong lists
  uint32_t* long_hint_dev;     // device mirror of the last value written to long_hint
  uint32_t wl_cap;             // entries per bucket
  Rec* scratch;            // general path: gen_threads slices of gen_stride records
  uint32_t gen_threads;    // threads of the general kernel (one scratch slice each)
  uint32_t gen_stride;     // records per slice: 4 * (n_src * k_in)
  float* stat_gamma;   // optional [P]
  uint16_t* stat_m;    // optional [P]
  float* stat_margin;  // optional [P]: min |sqrt(D^2) - gamma| over the executed comparisons
  unsigned long long* records_in;
  unsigned long long* records_search;   // records of lists sent to the search / general paths
  unsigned long long* sweep_steps;      // optional: sample-steps of the plain procedure (PIXEL_STATS replay)
  unsigned long long* fallback_groups;  // groups written with plain stores
  uint32_t* search_ticket;              // [VDI_N_BUCKETS] per-bucket claim tickets of the search kernels
  // short-list search scratch (buckets 0, 1), a pool of batch slots shared by
  // all chunks: slot = [40][32] rgba + [40][32] depth + [2][32] gap words;
  // batch_slot[b][i] = slot of batch i (32 entries) of bucket b of this chunk
  float4* pool_rgba;
  float2* pool_depth;
  uint32_t* pool_gap;
  uint32_t* pool_next;
  uint32_t pool_cap;
  uint32_t* batch_slot[2];
  // long-list search (buckets 2, 3): long_warps warp-private slots of long_slot
  // bytes, each [long_maxm + 32][32] rgba then [long_maxm + 32][32] depth (32 rows of read slack)
  char* long_pool;
  size_t long_slot;
  uint32_t long_maxm;
  uint32_t long_warps;
  int* err;            // bit 0: work-list overflow (cannot happen: capacity = lists)
  int validate;
};

// Launchers (merge.cu)
uint32_t scan_chunks(uint32_t P);  // chunks of the receive-side scan
cudaError_t launch_scan(const MergeParams& mp, uint32_t* chunk_sum, uint32_t* group_base, cudaStream_t st,
                        int* launches);
// pass-through kernel over groups [mp.g_begin, mp.g_end) (stream st)
cudaError_t launch_fast(const MergeParams& mp, cudaStream_t st, int* launches);
// dense gather: total of the scanned counts (chunk sums) and compaction of a full-representation strip
cudaError_t launch_total(const MergeParams& mp, const uint32_t* chunk_sum, unsigned long long* out, cudaStream_t st,
                         int* launches);
cudaError_t launch_compact(const uint8_t* count, const float2* depth, const float4* rgba, uint32_t P, int k,
                           const uint32_t* group_base, float2* od, float4* oc, cudaStream_t st, int* launches);
// search kernels (buckets 0-3); after launch_fast (it zeroes their lists' slots)
cudaError_t launch_search(const MergeParams& mp, cudaStream_t st, int* launches);
// general path (bucket 4); after launch_fast and launch_search
cudaError_t launch_general(const MergeParams& mp, cudaStream_t st, int* launches);
// VDI_FLAG_PIXEL_STATS: tie margins of the searched lists (replays their bisection from the pools)
cudaError_t launch_margins(const MergeParams& mp, cudaStream_t st, int* launches);
uint32_t general_threads(uint32_t m_max);
uint32_t long_warps(uint32_t m_max, size_t* slot_bytes);  // warps (and slot bytes) of the long-list search
cudaError_t preload_merge();
// VDI_FLAG_VALIDATE: input checks of one dense sub-VDI; error bits ORed into *err (merge.cu)
cudaError_t launch_validate(const uint8_t* count, const uint32_t* offset, const float2* depth, const float4* rgba,
                            uint32_t P, int k, unsigned long long total, int* err, cudaStream_t st);  // load every merge kernel now (loopback groups spin-wait across contexts)  // threads of the general kernel for lists of <= m_max records

// Generator (generate.cu)
struct GenParams {
  const void* vox;
  int bytes;
  int dims[3];
  const float4* tf;
  float eye[3], fwd[3], right[3], up[3];
  float tan_x, tan_y;
  int W, H;
  int grid[3];
  int xb[VDI_MAX_GRID_AXIS + 1], yb[VDI_MAX_GRID_AXIS + 1], zb[VDI_MAX_GRID_AXIS + 1];
  const int8_t* owner;  // device [gx*gy*gz]
  float lo[3], hi[3];   // PE bounding box in continuous voxel coordinates
  int pe;
  int k;
  int max_iters;
  float gamma_max;
  int limit;  // 1: one S~ per sub-domain intersection (gamma = inf)
};
cudaError_t launch_dvr(const GenParams& gp, float4* out, cudaStream_t st);  // ground-truth DVR image [H][W]
cudaError_t launch_gen_pass1(const GenParams& gp, uint32_t* count32, float* gamma, int* err,
                             cudaStream_t st);
cudaError_t launch_gen_pass2(const GenParams& gp, const uint32_t* offset, const float* gamma,
                             const uint32_t* count32, float2* depth, float4* rgba, cudaStream_t st);
cudaError_t gen_scan(const uint32_t* count32, uint32_t* offset, size_t n, void** tmp, size_t* tmp_bytes,
                     cudaStream_t st);
cudaError_t launch_u32_to_u8(const uint32_t* in, uint8_t* out, size_t n, cudaStream_t st);

}  // namespace vdi
