// comm.h — device-driven exchange / gather kernels of libvdi (comm.cu).
// Product code (sm_100a).  Shares nothing with oracle/.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#define VDI_MAX_RANKS 64

namespace vdi {

// strip bounds of the local PEs (a2)
struct BoundsArgs {
  const uint32_t* offset[64];   // per local PE, or null (then count + gbase are used)
  const uint8_t* count[64];
  const uint32_t* gbase;        // [n_local][n_groups] 32-list group bases of the counts (receive-side scan)
  uint64_t total[64];           // per local PE (host-known totals; used past the last group)
  uint32_t rows[VDI_MAX_RANKS + 1];
  uint32_t n_groups;
  uint32_t W;
  int n_local, G;
  unsigned long long* bnd;      // out [n_local][G + 1]
  uint32_t* srcbase;            // out [n_pes]: srcbase[pe[l]] = bnd[l][me] (the merge reads its strip in place)
  uint32_t pe[64];
  int me;
};

// one (local PE, destination) slice of the strip exchange (a4)
struct PushSeg {
  const uint8_t* src_count;     // the strip's count slice
  const float2* src_depth;      // the PE's whole payload arrays (absolute record indices)
  const float4* src_rgba;
  const unsigned long long* bnd;  // &bnd[l][g]: records [bnd[0], bnd[1]); null -> [rec0, rec0 + nrec)
  unsigned long long rec0, nrec;
  unsigned long long n_count;   // bytes of the count slice
  const uint32_t* src_offset;   // group bases of the slice from the PE's offsets (at the slice start), or
  const uint32_t* src_gb32;     // from its 32-list scan (at the slice's first group); neither: none pushed
  uint32_t n_groups;            // 32-list groups of the destination strip
  uint32_t* dst_gbase;          // [n_groups]: index of each group's first record in the slice
  uint8_t* dst_count;           // destination window slot (peer memory)
  float2* dst_depth;
  float4* dst_rgba;
  unsigned long long* dst_hdr;  // receives the record count of the slice
  unsigned long long* bytes;    // local counter of pushed bytes (or null)
  uint32_t* flag;               // the destination's counter word for this sender
  unsigned long long src_total; // records of the source PE (bounds of the VDI_CHECKS build)
  unsigned long long cap_rec;   // records the destination slot holds
};

// the gather's compaction into the root's window (a11)
struct CompactPushArgs {
  const uint8_t* count;         // composited strip (full representation)
  const float2* depth;
  const float4* rgba;
  uint32_t P;
  int k;
  const uint32_t* group_base;   // local exclusive scan of the strip's counts per 32-list group
  uint32_t region;              // first record of this rank's region in the root window
  uint8_t* dst_count;           // root window (peer memory)
  uint32_t* dst_gbase;
  float2* dst_depth;
  float4* dst_rgba;
  unsigned long long* total_out;  // root window header: records pushed
  unsigned long long* bytes;    // local counter of pushed bytes (or null)
  uint32_t* flag;
  unsigned long long region_cap;  // records the root's region for this rank holds
};

struct WaitArgs {
  const uint32_t* addr[VDI_MAX_RANKS];
  uint32_t target[VDI_MAX_RANKS];
  int n;
};

struct SignalArgs {
  uint32_t* addr[VDI_MAX_RANKS];
  uint32_t value[VDI_MAX_RANKS];
  int n;
};

cudaError_t launch_bounds(const BoundsArgs& a, cudaStream_t st);
cudaError_t launch_push(const PushSeg* dsegs, uint32_t n_segs, uint32_t blocks_per_seg, cudaStream_t st);
cudaError_t launch_compact_push(const CompactPushArgs& a, uint32_t blocks, cudaStream_t st);
cudaError_t launch_wait(const WaitArgs& a, cudaStream_t st);
cudaError_t launch_signal(const SignalArgs& a, cudaStream_t st);
cudaError_t launch_check(const WaitArgs& a, unsigned long long* fails, cudaStream_t st);
cudaError_t preload_comm();   // load the comm kernels now (see preload_merge)

// blocks (256 threads) of the gather compaction of a P-list strip (both ends
// derive it): up to 8 per SM (full occupancy: the copy is latency bound), each
// looping over its share of 32-list groups
inline uint32_t compact_push_blocks(uint32_t P) {
  const uint32_t ng = (P + 31) / 32;
  const uint32_t b = (ng + 7) / 8;
  return b < 1 ? 1 : (b > 148 * 8 ? 148 * 8 : b);
}
// blocks per (PE, destination) segment of the exchange push (both ends derive it)
inline uint32_t push_blocks(uint32_t n_local, uint32_t G) {
  const uint32_t segs = n_local * (G > 1 ? G - 1 : 1);
  const uint32_t b = segs ? (148u * 8u) / segs : 1u;
  return b < 1 ? 1 : (b > 1024 ? 1024 : b);
}

}  // namespace vdi
