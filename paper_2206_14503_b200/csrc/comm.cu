// comm.cu — device-driven exchange and gather of libvdi (sm_100a).
//
// Every byte of the strip exchange (MPI_AllToAllv in the paper)
// and of the gather to the root (MPI_Gather) is moved by these
// kernels with plain stores into the receiving GPU's memory over NVLink 5 /
// NVSwitch (CUDA IPC mappings of ctx-owned windows, opened once at init) --
// no host round trip, no size exchange on the host:
//   * a sender reads its strip bounds from its own offset arrays (or a scan
//     of its counts) on the device and pushes the count slice and the packed
//     payload slice of every (local PE, strip) pair into the owner's window;
//   * every block, after its stores, bumps a per-sender counter word in the
//     receiver's flag array (bar.sync + fence.sc.sys + atomic add at system
//     scope), so the receiver knows its data has landed once the counter
//     reaches (call index) x (blocks per call) -- both ends derive the block
//     count from the config;
//   * receivers wait with a one-CTA spin kernel (ld.acquire.sys) and release
//     the sender's window slot with a one-CTA signal kernel after their merge.
#include <cuda_runtime.h>

#include <cstdlib>

#include "comm.h"
#include "internal.h"

namespace vdi {

__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// all of this block's stores are performed (at system scope) before the
// counter increment becomes visible
__device__ __forceinline__ void block_arrive(uint32_t* flag) {
  __syncthreads();
  if (threadIdx.x == 0 && flag) {
    __threadfence_system();
    atomicAdd_system(flag, 1u);
  }
}

template <class V>
__device__ __forceinline__ void copy_span(const V* __restrict__ s, V* __restrict__ d, unsigned long long n,
                                          unsigned long long i0, unsigned long long stride) {
  unsigned long long i = i0;
  for (; i + 7 * stride < n; i += 8 * stride) {  // 8 loads in flight per thread
    V v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = __ldg(s + i + u * stride);
#pragma unroll
    for (int u = 0; u < 8; ++u) d[i + u * stride] = v[u];
  }
  for (; i < n; i += stride) d[i] = __ldg(s + i);
}

// bytes [0, n) from s to d; the widest vector both addresses allow
__device__ __forceinline__ void copy_bytes(const void* s, void* d, unsigned long long n, unsigned long long i0,
                                           unsigned long long stride) {
  const uintptr_t al = reinterpret_cast<uintptr_t>(s) | reinterpret_cast<uintptr_t>(d);
  if (!(al & 15)) {
    const unsigned long long n16 = n / 16;
    copy_span(static_cast<const uint4*>(s), static_cast<uint4*>(d), n16, i0, stride);
    for (unsigned long long i = n16 * 16 + i0; i < n; i += stride)
      static_cast<uint8_t*>(d)[i] = static_cast<const uint8_t*>(s)[i];
  } else if (!(al & 3)) {
    const unsigned long long n4 = n / 4;
    copy_span(static_cast<const uint32_t*>(s), static_cast<uint32_t*>(d), n4, i0, stride);
    for (unsigned long long i = n4 * 4 + i0; i < n; i += stride)
      static_cast<uint8_t*>(d)[i] = static_cast<const uint8_t*>(s)[i];
  } else {
    copy_span(static_cast<const uint8_t*>(s), static_cast<uint8_t*>(d), n, i0, stride);
  }
}

// ---------------------------------------------------------------------------
// Strip bounds of the local PEs (a2): bnd[l][g] = index of the first record of
// strip g in PE l's payload, g = 0..G (bnd[l][G] = the PE's total).  From the
// PE's offset array when given, else from the 32-list group
// bases of a scan of its counts plus the partial group.
// ---------------------------------------------------------------------------
__global__ void bounds_kernel(BoundsArgs a) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.n_local * (a.G + 1)) return;
  const int l = i / (a.G + 1), g = i % (a.G + 1);
  const uint64_t p = (uint64_t)a.rows[g] * a.W;
  uint64_t v;
  if (a.offset[l]) {
    v = a.offset[l][p];
  } else {
    const uint64_t g32 = p / 32;
    v = g32 < a.n_groups ? a.gbase[(size_t)l * a.n_groups + g32] : a.total[l];
    if (g32 < a.n_groups)
      for (uint64_t q = g32 * 32; q < p; ++q) v += a.count[l][q];
  }
  a.bnd[(size_t)l * (a.G + 1) + g] = v;
  if (g == a.me && a.srcbase) a.srcbase[a.pe[l]] = (uint32_t)v;
}

// ---------------------------------------------------------------------------
// Push of (local PE, destination strip) slices into the destination windows
// (a4): blockIdx.y = segment, blockIdx.x = share of it.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256, 4) push_kernel(const PushSeg* __restrict__ segs) {
  const PushSeg sg = segs[blockIdx.y];
  const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
  const unsigned long long i0 = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long r0, nrec;
  if (sg.bnd) {  // dense slice [bnd[0], bnd[1]) of the payload
    r0 = sg.bnd[0];
    nrec = sg.bnd[1] - r0;
  } else {       // fixed-size slice (full representation)
    r0 = sg.rec0;
    nrec = sg.nrec;
  }
  VDI_CHECK(nrec <= sg.cap_rec, "push: slice larger than the destination slot");
  VDI_CHECK(!sg.src_total || r0 + nrec <= sg.src_total, "push: slice past the source's records");
  copy_bytes(sg.src_count, sg.dst_count, sg.n_count, i0, stride);
  if (sg.dst_gbase) {  // group bases relative to the slice's first record: the receiver needs no scan
    if (sg.src_offset) {
      const uint32_t b0 = sg.src_offset[0];
      for (unsigned long long i = i0; i < sg.n_groups; i += stride) sg.dst_gbase[i] = sg.src_offset[i * 32] - b0;
    } else if (sg.src_gb32) {
      const uint32_t b0 = sg.src_gb32[0];
      for (unsigned long long i = i0; i < sg.n_groups; i += stride) sg.dst_gbase[i] = sg.src_gb32[i] - b0;
    }
  }
  if (nrec) {
    copy_bytes(sg.src_depth + r0, sg.dst_depth, nrec * 8, i0, stride);
    copy_bytes(sg.src_rgba + r0, sg.dst_rgba, nrec * 16, i0, stride);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    if (sg.dst_hdr) *sg.dst_hdr = nrec;
    if (sg.bytes) atomicAdd(sg.bytes, sg.n_count + 24ull * nrec);
  }
  block_arrive(sg.flag);
}

// ---------------------------------------------------------------------------
// Gather (a11): compaction of a composited strip (full representation,
// PAPER.md:185) into the root's window -- counts at their image rows, the
// 32-list group bases of the packed records (+ region offset), the records
// packed in list order -- then one counter bump per block at the root.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t warp_incl_scan_c(uint32_t v, int lane) {
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t t = __shfl_up_sync(0xffffffffu, v, d);
    if (lane >= d) v += t;
  }
  return v;
}

__global__ void __launch_bounds__(256) compact_push_kernel(CompactPushArgs a) {
  const int lane = threadIdx.x & 31;
  const uint32_t ng = (a.P + 31) / 32;
  const uint32_t gstep = gridDim.x * (blockDim.x >> 5);
  uint32_t g = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  // the next group's count and base are loaded while this one is copied
  uint32_t c_nx = 0, gb_nx = 0;
  if (g < ng) {
    c_nx = g * 32 + lane < a.P ? __ldg(a.count + g * 32 + lane) : 0u;
    gb_nx = __ldg(a.group_base + g);
  }
  for (; g < ng; g += gstep) {
    const uint32_t p = g * 32 + lane;
    const uint32_t c = c_nx, gb = gb_nx;
    const uint32_t gn = g + gstep;
    if (gn < ng) {
      c_nx = gn * 32 + lane < a.P ? __ldg(a.count + gn * 32 + lane) : 0u;
      gb_nx = __ldg(a.group_base + gn);
    }
    if (p < a.P) a.dst_count[p] = (uint8_t)c;
    if (lane == 0) a.dst_gbase[g] = a.region + gb;
    // the group's records are contiguous in the root window: record d goes to
    // base + d, consecutive lanes -> consecutive records (coalesced stores over
    // NVLink); the list holding record d: 5-step search over the lists' prefix
    const uint32_t incl = warp_incl_scan_c(c, lane), excl = incl - c;
    const uint32_t tot = __shfl_sync(0xffffffffu, incl, 31);
    const size_t base = (size_t)a.region + gb;
    VDI_CHECK(gb + tot <= a.region_cap, "compact_push: records past the rank's region");
    for (uint32_t d0 = 0; d0 < tot; d0 += 32) {
      const uint32_t d = d0 + lane;
      uint32_t l = 0;
#pragma unroll
      for (int step = 16; step > 0; step >>= 1) {
        const uint32_t e = __shfl_sync(0xffffffffu, excl, (int)(l + step));
        if (e <= d) l += step;
      }
      const uint32_t el = __shfl_sync(0xffffffffu, excl, (int)l);
      if (d < tot) {
        const size_t src = ((size_t)g * 32 + l) * a.k + (d - el);
        a.dst_depth[base + d] = __ldg(a.depth + src);
        a.dst_rgba[base + d] = __ldg(a.rgba + src);
      }
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0 && a.total_out) {
    // records of the strip = the base of the last group + its count sum
    const uint32_t lg = ng ? ng - 1 : 0;
    uint32_t t = ng ? a.group_base[lg] : 0u;
    for (uint32_t q = lg * 32; q < a.P; ++q) t += a.count[q];
    *a.total_out = t;
    if (a.bytes) atomicAdd(a.bytes, (unsigned long long)a.P + 4ull * ng + 24ull * t);
  }
  block_arrive(a.flag);
}

// ---------------------------------------------------------------------------
// Flags: one-CTA wait (thread t spins until flag t reaches its target, wrap-
// aware) and one-CTA signal (release store of a value into peer flag words).
// ---------------------------------------------------------------------------
__global__ void wait_kernel(WaitArgs a) {
  const int t = threadIdx.x;
  if (t < a.n) {
    while ((int32_t)(ld_acquire_sys(a.addr[t]) - a.target[t]) < 0) __nanosleep(64);
  }
  __syncthreads();
}

// loopback: the flags must already be at their targets (the stream waited on
// the producers' events); count the shortfalls
__global__ void check_kernel(WaitArgs a, unsigned long long* fails) {
  const int t = threadIdx.x;
  if (t < a.n && (int32_t)(ld_acquire_sys(a.addr[t]) - a.target[t]) < 0) atomicAdd(fails, 1ull);
}

__global__ void signal_kernel(SignalArgs a) {
  const int t = threadIdx.x;
  if (t < a.n) {
    __threadfence_system();
    st_release_sys(a.addr[t], a.value[t]);
  }
}

cudaError_t launch_bounds(const BoundsArgs& a, cudaStream_t st) {
  const int n = a.n_local * (a.G + 1);
  if (!n) return cudaSuccess;
  bounds_kernel<<<(n + 127) / 128, 128, 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_push(const PushSeg* dsegs, uint32_t n_segs, uint32_t blocks_per_seg, cudaStream_t st) {
  if (!n_segs) return cudaSuccess;
  push_kernel<<<dim3(blocks_per_seg, n_segs), 256, 0, st>>>(dsegs);
  return cudaGetLastError();
}

cudaError_t launch_compact_push(const CompactPushArgs& a, uint32_t blocks, cudaStream_t st) {
  compact_push_kernel<<<blocks, 256, 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_wait(const WaitArgs& a, cudaStream_t st) {
  if (!a.n) return cudaSuccess;
  wait_kernel<<<1, 64, 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_check(const WaitArgs& a, unsigned long long* fails, cudaStream_t st) {
  if (!a.n) return cudaSuccess;
  check_kernel<<<1, 64, 0, st>>>(a, fails);
  return cudaGetLastError();
}

cudaError_t launch_signal(const SignalArgs& a, cudaStream_t st) {
  if (!a.n) return cudaSuccess;
  signal_kernel<<<1, 64, 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t preload_comm() {
  cudaFuncAttributes fa;
  cudaFuncGetAttributes(&fa, bounds_kernel);
  cudaFuncGetAttributes(&fa, push_kernel);
  cudaFuncGetAttributes(&fa, compact_push_kernel);
  cudaFuncGetAttributes(&fa, wait_kernel);
  cudaFuncGetAttributes(&fa, signal_kernel);
  cudaFuncGetAttributes(&fa, check_kernel);
  return cudaGetLastError();
}

}  // namespace vdi
