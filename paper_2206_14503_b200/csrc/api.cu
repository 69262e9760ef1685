// api.cu — libvdi C ABI (include/vdi.h): context, validation, the Phase-2
// orchestration (strip partition, size exchange, all-to-allv over NCCL,
// receive-side scan, merge) and the gather to the root.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <nccl.h>

#include <map>
#include <memory>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "internal.h"

using namespace vdi;

namespace {

thread_local std::string g_err;

vdi_status fail(vdi_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return s;
}

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  ~DevBuf() {
    if (p) cudaFree(p);
  }
  cudaError_t grow(size_t need) {
    if (need <= bytes) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
    size_t want = std::max(need, (size_t)256);
    cudaError_t e = cudaMalloc(&p, want);
    if (e == cudaSuccess) bytes = want;
    return e;
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

struct GenOut {
  DevBuf count32, count8, offset, gamma, depth, rgba, owner;
  uint64_t total = 0;
};

// device-side counters of one composite
#define VDI_MAX_CHUNKS 8
struct DevCounters {
  uint32_t wl_count[VDI_MAX_CHUNKS][VDI_N_BUCKETS];
  uint32_t search_ticket[VDI_MAX_CHUNKS][VDI_N_BUCKETS];
  int err;
  uint32_t pool_next;
  unsigned long long scratch_used;
  unsigned long long records_in;
  unsigned long long fallback_groups;
  unsigned long long records_search;
  unsigned long long long_used;
};

}  // namespace

struct vdi_ctx {
  vdi_config cfg{};
  cudaStream_t stream = nullptr;
  int device = 0;
  ncclComm_t comm = nullptr;
  bool poisoned = false;
  uint32_t row0 = 0, row1 = 0;
  uint64_t P = 0;  // lists in this rank's strip
  uint64_t mP = 0;  // lists of the last merge (strip, or whole frame in vdi_composite_frames)
  // merge scratch
  DevBuf group_sum, group_base, wl, scratch, dcnt, stat_gamma, stat_m, bounds, srch, slots;
  DevBuf g_sum, g_base, g_tot, g_dense, g_rcount, g_rpay, g_misc;  // dense gather
  DevBuf lpool, lbatch;  // long-list search pool
  std::map<std::string, void*> ipc_cache;  // IPC handle bytes -> mapped base of a peer allocation
  static constexpr int kXStreams = 4;      // copy-engine streams of the peer exchange
  cudaStream_t xs[4] = {};
  cudaEvent_t evx[5] = {};
  bool peer_reads = false;
  int n_chunks = 1;
  // exchange receive buffers per source
  std::vector<DevBuf> rcount, rdepth, rrgba;
  // vdi_composite_frames: receive buffers per (owned frame, source), chunk events
  std::vector<std::unique_ptr<DevBuf>> fcount, fdepth, frgba;
  static constexpr int kMaxChunks = 8;
  cudaEvent_t evc[8][4] = {};
  DevBuf fblob;
  // vdi_composite_fullrep: per-source dense scratch of the compaction + its scan
  std::vector<std::unique_ptr<DevBuf>> xdense;
  DevBuf xsum, xbase, xtot;
  DevBuf segbuf;  // peer_copy_kernel segment tables (grow-only, stream-ordered)
  size_t seg_used = 0;
  // generator outputs per pe
  std::vector<GenOut> gen;
  DevBuf gen_tmp;
  void* cub_tmp = nullptr;
  size_t cub_tmp_bytes = 0;
  // host e2e staging
  std::vector<DevBuf> hcount, hoffset, hdepth, hrgba;
  DevBuf hstrip_count, hstrip_depth, hstrip_rgba;
  // vdi_composite_host_dense_frames: the second input slot, per-slot dense
  // outputs, the H2D / D2H streams and their slot events
  std::vector<DevBuf> hcount1, hoffset1, hdepth1, hrgba1;
  DevBuf harena[2];  // input slots when the host arrays are packed in one span
  DevBuf pcount[2], pdense[2];
  cudaStream_t pin_st = nullptr, pout_st = nullptr;
  cudaEvent_t pev_in[2] = {}, pev_used[2] = {}, pev_tot[2] = {}, pev_comp[2] = {}, pev_out[2] = {};
  unsigned long long* ptot = nullptr;      // pinned, mapped host [2]: frame totals written by the kernel
  unsigned long long* ptot_dev = nullptr;  // its device alias
  // counters
  vdi_counters last{};
  bool have_stats = false;
  cudaEvent_t ev[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
  bool timing_pending = false;
  bool gather_timing_pending = false;
  cudaEvent_t gev[2] = {nullptr, nullptr};
  cudaEvent_t fev[2] = {nullptr, nullptr};  // frames mode: pull start / end
  bool frames_timing_pending = false;
  ~vdi_ctx() {
    if (pin_st) cudaStreamSynchronize(pin_st);
    if (pout_st) cudaStreamSynchronize(pout_st);
    if (pin_st) cudaStreamDestroy(pin_st);
    if (pout_st) cudaStreamDestroy(pout_st);
    for (cudaEvent_t* a : {pev_in, pev_used, pev_tot, pev_comp, pev_out})
      for (int i = 0; i < 2; ++i)
        if (a[i]) cudaEventDestroy(a[i]);
    if (ptot) cudaFreeHost(ptot);
    if (cub_tmp) cudaFree(cub_tmp);
    for (auto& x : xs)
      if (x) cudaStreamDestroy(x);
    for (auto& e : evx)
      if (e) cudaEventDestroy(e);
    for (auto& e : ev)
      if (e) cudaEventDestroy(e);
    for (auto& e : gev)
      if (e) cudaEventDestroy(e);
    for (auto& e : fev)
      if (e) cudaEventDestroy(e);
    for (auto& r : evc)
      for (auto& e : r)
        if (e) cudaEventDestroy(e);
    // local teardown: drain our stream, then abort (not finalize) the
    // communicator so destroying contexts never waits on other ranks
    if (stream || comm) cudaStreamSynchronize(stream);
    for (auto& kv : ipc_cache) cudaIpcCloseMemHandle(kv.second);
    if (comm) ncclCommAbort(comm);
  }
};

#define CUDA_TRY(ctx, expr)                                                                  \
  do {                                                                                       \
    cudaError_t e_ = (expr);                                                                 \
    if (e_ != cudaSuccess) {                                                                 \
      (ctx)->poisoned = true;                                                                \
      return fail(e_ == cudaErrorMemoryAllocation ? VDI_ERR_OUT_OF_MEMORY : VDI_ERR_CUDA,   \
                  "%s:%d %s: %s", __FILE__, __LINE__, #expr, cudaGetErrorString(e_));       \
    }                                                                                        \
  } while (0)

#define NCCL_TRY(ctx, expr)                                                                         \
  do {                                                                                              \
    ncclResult_t r_ = (expr);                                                                       \
    if (r_ != ncclSuccess) {                                                                        \
      (ctx)->poisoned = true;                                                                       \
      return fail(VDI_ERR_NCCL, "%s:%d %s: %s", __FILE__, __LINE__, #expr, ncclGetErrorString(r_)); \
    }                                                                                               \
  } while (0)

namespace {

// SM-driven copy of many segments (peer slices over NVLink through CUDA IPC
// mappings into local receive buffers): blockIdx.y = segment, 16/8/4/1-byte
// vectors by the common alignment of the segment, 4 loads in flight per thread.
#ifndef VDI_COPY_BPS
#define VDI_COPY_BPS 4
#endif
struct CopySeg {
  const void* src;
  void* dst;
  unsigned long long bytes;
};

template <class V>
__device__ __forceinline__ void copy_vec(const V* __restrict__ s, V* __restrict__ d, unsigned long long n) {
  const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
  unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n; i += 4 * stride) {
    const V a = s[i], b = s[i + stride], c = s[i + 2 * stride], e = s[i + 3 * stride];
    d[i] = a;
    d[i + stride] = b;
    d[i + 2 * stride] = c;
    d[i + 3 * stride] = e;
  }
  for (; i < n; i += stride) d[i] = s[i];
}

__global__ void __launch_bounds__(256) peer_copy_kernel(const CopySeg* __restrict__ segs) {
  const CopySeg sg = segs[blockIdx.y];
  const uintptr_t al = reinterpret_cast<uintptr_t>(sg.src) | reinterpret_cast<uintptr_t>(sg.dst) | sg.bytes;
  if (!(al & 15)) copy_vec(static_cast<const uint4*>(sg.src), static_cast<uint4*>(sg.dst), sg.bytes / 16);
  else if (!(al & 7)) copy_vec(static_cast<const uint2*>(sg.src), static_cast<uint2*>(sg.dst), sg.bytes / 8);
  else if (!(al & 3)) copy_vec(static_cast<const uint32_t*>(sg.src), static_cast<uint32_t*>(sg.dst), sg.bytes / 4);
  else copy_vec(static_cast<const uint8_t*>(sg.src), static_cast<uint8_t*>(sg.dst), sg.bytes);
}

__global__ void gather_bounds_kernel(const uint32_t* const* offs, const uint32_t* pes, int n_local,
                                     const uint32_t* rows, int G, uint32_t W, int n_pes,
                                     unsigned long long* bnd, size_t hdr_stride = 0, size_t bnd_stride = 0) {
  // bnd[pe][g] = offset_pe[rows[g] * W]  (g = 0..G); block b handles frame b
  // (headers hdr_stride bytes apart, bnd blocks bnd_stride entries apart)
  offs = reinterpret_cast<const uint32_t* const*>(reinterpret_cast<const char*>(offs) + blockIdx.x * hdr_stride);
  pes = reinterpret_cast<const uint32_t*>(reinterpret_cast<const char*>(pes) + blockIdx.x * hdr_stride);
  rows = reinterpret_cast<const uint32_t*>(reinterpret_cast<const char*>(rows) + blockIdx.x * hdr_stride);
  bnd += blockIdx.x * bnd_stride;
  for (int i = threadIdx.x; i < n_local * (G + 1); i += blockDim.x) {
    const int l = i / (G + 1), g = i % (G + 1);
    bnd[(size_t)pes[l] * (G + 1) + g] = offs[l][(size_t)rows[g] * W];
  }
}

// ---- CUDA IPC references to (sub-ranges of) cudaMalloc allocations ---------
struct IpcRef {
  cudaIpcMemHandle_t h;  // handle of the allocation's base
  uint64_t off;          // byte offset of the pointer inside the allocation
};
static_assert(sizeof(IpcRef) == 72, "IpcRef layout");

PFN_cuMemGetAddressRange_v3020 get_range_fn() {
  static PFN_cuMemGetAddressRange_v3020 fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", reinterpret_cast<void**>(&fn), cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      fn = nullptr;
  }
  return fn;
}

bool ipc_export(const void* p, IpcRef* r) {
  PFN_cuMemGetAddressRange_v3020 fn = get_range_fn();
  if (!fn) return false;
  CUdeviceptr base = 0;
  size_t size = 0;
  if (fn(&base, &size, reinterpret_cast<CUdeviceptr>(p)) != CUDA_SUCCESS) return false;
  if (cudaIpcGetMemHandle(&r->h, reinterpret_cast<void*>(base)) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  r->off = reinterpret_cast<uint64_t>(p) - base;
  return true;
}

cudaError_t ipc_import(vdi_ctx* ctx, const IpcRef& r, void** out) {
  const std::string key(reinterpret_cast<const char*>(&r.h), sizeof r.h);
  auto it = ctx->ipc_cache.find(key);
  void* base = nullptr;
  if (it == ctx->ipc_cache.end()) {
    cudaError_t e = cudaIpcOpenMemHandle(&base, r.h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) return e;
    ctx->ipc_cache.emplace(key, base);
  } else {
    base = it->second;
  }
  *out = static_cast<char*>(base) + r.off;
  return cudaSuccess;
}

vdi_status check_ctx(vdi_ctx* ctx) {
  if (!ctx) return fail(VDI_ERR_INVALID_ARG, "ctx is NULL");
  if (ctx->poisoned) return fail(VDI_ERR_STATE, "context poisoned by an earlier CUDA/NCCL error");
  return VDI_OK;
}

uint32_t strip_row(uint32_t H, uint32_t G, uint32_t g) { return (uint32_t)((uint64_t)g * H / G); }

}  // namespace

// Enqueue one peer_copy_kernel over `segs` on st.  The segment table goes
// through a pinned-less H2D copy into a ctx-owned slice (stream-ordered).
static int api_sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n < 1) n = 1;
  }
  return n;
}

static cudaError_t sm_copy(vdi_ctx* ctx, const std::vector<CopySeg>& segs, cudaStream_t st, int& launches,
                           int bps = VDI_COPY_BPS) {
  if (segs.empty()) return cudaSuccess;
  const size_t bytes = segs.size() * sizeof(CopySeg);
  cudaError_t e = ctx->segbuf.grow(std::max<size_t>(bytes, 64 * sizeof(CopySeg)));
  if (e != cudaSuccess) return e;
  if ((e = cudaMemcpyAsync(ctx->segbuf.p, segs.data(), bytes, cudaMemcpyHostToDevice, st)) != cudaSuccess) return e;
  // bps blocks of 256 threads per SM over all segments
  const unsigned gx = std::max<unsigned>(1u, (unsigned)(api_sm_count() * bps / (int)segs.size()));
  peer_copy_kernel<<<dim3(gx, (unsigned)segs.size()), 256, 0, st>>>(ctx->segbuf.as<CopySeg>());
  ++launches;
  return cudaGetLastError();
}

// Merge of P lists whose sources are set in mp.src[0..n_pes) (receive-side
// scan, pass-through + classification, gamma search, general path;
// PAPER.md:166-185) into the full representation `so` (P lists).  Scratch is
// ctx-owned and stream-ordered, so consecutive merges on the ctx stream reuse it.
static vdi_status merge_lists(vdi_ctx* ctx, MergeParams& mp, uint64_t P, uint64_t S_here, vdi_full_view* so,
                              bool timing, int& launches_ref) {
  const vdi_config& cf = ctx->cfg;
  const uint32_t n = cf.n_pes, k = cf.k_out;
  cudaStream_t st = ctx->stream;
  int launches = 0;
  mp.P = (uint32_t)P;
  mp.n_groups = (uint32_t)((P + 31) / 32);
  ctx->mP = P;
  // buffers of the merge
  const size_t ng = mp.n_groups;
  CUDA_TRY(ctx, ctx->group_sum.grow((size_t)scan_chunks(mp.P) * n * 4));
  CUDA_TRY(ctx, ctx->group_base.grow(ng * n * 4));
  // One chunk of 32-list groups, search kernels after the pass-through on
  // the same stream.  Measured on C3 (profiles/README.md): overlapping them
  // is slower -- chunked overlap on a second stream (C = 2: 1495 VDIs/s,
  // C = 8: 973, vs 1976) and a classify kernel + search concurrent with the
  // whole pass-through (2069-2124 vs 2120): the latency-bound search kernels
  // run ~2x slower beside the HBM-bound pass-through.
  const uint32_t C = 1;
  ctx->n_chunks = (int)C;
  std::vector<uint32_t> gb(C + 1);
  for (uint32_t c = 0; c <= C; ++c) gb[c] = (uint32_t)((uint64_t)ng * c / C);
  const size_t wl_words = std::max<size_t>(P, 1) * (3 + n) * VDI_N_BUCKETS + 64;
  CUDA_TRY(ctx, ctx->wl.grow(wl_words * 4));
  CUDA_TRY(ctx, ctx->slots.grow((2 * ng + 2 * C + 64) * 4));
  CUDA_TRY(ctx, ctx->scratch.grow(std::max<uint64_t>(4 * S_here, 1) * sizeof(Rec)));
  CUDA_TRY(ctx, ctx->dcnt.grow(sizeof(DevCounters)));
  const bool stats = cf.flags & VDI_FLAG_PIXEL_STATS;
  if (stats) {
    CUDA_TRY(ctx, ctx->stat_gamma.grow(P * 4));
    CUDA_TRY(ctx, ctx->stat_m.grow(P * 2));
  }
  // short-list search pool: a list in bucket 0/1 has m > k_out samples, so at
  // most S_here / (k_out + 1) such lists exist; + one partial batch per chunk and bucket
  const uint64_t pool_cap = (S_here / (k + 1) + 31) / 32 + 2 * C + 2;
  const size_t slot_bytes = 40 * 32 * 16 + 40 * 32 * 8 + 64 * 4;
  CUDA_TRY(ctx, ctx->srch.grow(pool_cap * slot_bytes + 256));
  {
    char* q = ctx->srch.as<char>();
    mp.pool_rgba = reinterpret_cast<float4*>(q);
    q += pool_cap * 40 * 32 * 16;
    mp.pool_depth = reinterpret_cast<float2*>(q);
    q += pool_cap * 40 * 32 * 8;
    mp.pool_gap = reinterpret_cast<uint32_t*>(q);
    mp.pool_cap = (uint32_t)pool_cap;
  }
  // long-list pool: slots of stride maxm per 32-list batch; a list of bucket
  // 2/3 has m > 40, so the pool needs at most 24 B x (S_here + 32 x batches
  // of padding); batches <= S_here / 41 / 32 + 1 per bucket
  const uint64_t lb = S_here / 41 / 32 + 2;
  // + 32 rows x 32 lanes x 16 B of slack: the long sweeps read up to 24 rows past a list's end
  const unsigned long long lcap = 24ull * S_here * 2 + lb * 2 * (128 + 24 * 32) + 4096 + 32 * 32 * 16;
  CUDA_TRY(ctx, ctx->lpool.grow(lcap));
  CUDA_TRY(ctx, ctx->lbatch.grow((size_t)(P / 32 + 2) * 2 * 16));
  mp.long_pool = ctx->lpool.as<char>();
  mp.long_cap = lcap;
  mp.long_batch[0] = ctx->lbatch.as<PoolBatch>();
  mp.long_batch[1] = ctx->lbatch.as<PoolBatch>() + (P / 32 + 2);
  DevCounters* dc = ctx->dcnt.as<DevCounters>();
  CUDA_TRY(ctx, cudaMemsetAsync(dc, 0, sizeof(DevCounters), st));
  mp.long_used = &dc->long_used;
  mp.group_base = ctx->group_base.as<uint32_t>();
  mp.out_count = so->count;
  mp.out_depth = reinterpret_cast<float2*>(so->depth);
  mp.out_rgba = reinterpret_cast<float4*>(so->rgba);
  mp.fallback_groups = &dc->fallback_groups;
  mp.pool_next = &dc->pool_next;
  mp.scratch_used = &dc->scratch_used;
  mp.scratch_cap = 4 * S_here;
  mp.scratch = ctx->scratch.as<Rec>();
  mp.stat_gamma = stats ? ctx->stat_gamma.as<float>() : nullptr;
  mp.stat_m = stats ? ctx->stat_m.as<uint16_t>() : nullptr;
  mp.records_in = &dc->records_in;
  mp.records_search = &dc->records_search;
  mp.err = &dc->err;
  mp.validate = (cf.flags & VDI_FLAG_VALIDATE) ? 1 : 0;
  if (P) {
    if (!mp.src[0].offset)
      CUDA_TRY(ctx, launch_scan(mp, ctx->group_sum.as<uint32_t>(), ctx->group_base.as<uint32_t>(), st, &launches));
    if (timing) CUDA_TRY(ctx, cudaEventRecord(ctx->ev[3], st));
    uint32_t* wlp = ctx->wl.as<uint32_t>();
    uint32_t* slp = ctx->slots.as<uint32_t>();
    for (uint32_t c = 0; c < C; ++c) {
      MergeParams mc = mp;
      mc.g_begin = gb[c];
      mc.g_end = gb[c + 1];
      const uint64_t Pc = std::min<uint64_t>((uint64_t)gb[c + 1] * 32, P) - (uint64_t)gb[c] * 32;
      mc.wl_cap = (uint32_t)std::max<uint64_t>(Pc, 1);
      for (int b = 0; b < VDI_N_BUCKETS; ++b) {
        mc.wl[b] = wlp;
        wlp += (size_t)mc.wl_cap * (3 + n);
      }
      for (int b = 0; b < 2; ++b) {
        mc.batch_slot[b] = slp;
        slp += (mc.wl_cap + 31) / 32 + 1;
      }
      mc.wl_count = dc->wl_count[c];
      mc.search_ticket = dc->search_ticket[c];
      // pass-through (writes every slot of the strip) -> search kernels -> general path
      CUDA_TRY(ctx, launch_fast(mc, st, &launches));
      if (timing) CUDA_TRY(ctx, cudaEventRecord(ctx->ev[4], st));
      CUDA_TRY(ctx, launch_search(mc, st, &launches));
      if (timing) CUDA_TRY(ctx, cudaEventRecord(ctx->ev[5], st));
      CUDA_TRY(ctx, launch_general(mc, st, &launches));
    }
  }
  launches_ref += launches;
  return VDI_OK;
}

extern "C" {

const char* vdi_version(void) { return "libvdi 0.1 (sm_100a)"; }

const char* vdi_status_string(vdi_status s) {
  switch (s) {
    case VDI_OK: return "VDI_OK";
    case VDI_ERR_INVALID_ARG: return "VDI_ERR_INVALID_ARG";
    case VDI_ERR_OUT_OF_MEMORY: return "VDI_ERR_OUT_OF_MEMORY";
    case VDI_ERR_CUDA: return "VDI_ERR_CUDA";
    case VDI_ERR_NCCL: return "VDI_ERR_NCCL";
    case VDI_ERR_STATE: return "VDI_ERR_STATE";
    case VDI_ERR_CAPACITY: return "VDI_ERR_CAPACITY";
    case VDI_ERR_INTERNAL: return "VDI_ERR_INTERNAL";
  }
  return "VDI_ERR_UNKNOWN";
}

const char* vdi_last_error(const vdi_ctx*) { return g_err.c_str(); }

vdi_status vdi_strip_rows(uint32_t height, uint32_t n_ranks, uint32_t g, uint32_t* row_begin,
                          uint32_t* row_end) {
  if (!n_ranks || g >= n_ranks || !row_begin || !row_end) return fail(VDI_ERR_INVALID_ARG, "bad strip query");
  *row_begin = strip_row(height, n_ranks, g);
  *row_end = strip_row(height, n_ranks, g + 1);
  return VDI_OK;
}

uint32_t vdi_pe_home(uint32_t n_pes, uint32_t n_ranks, uint32_t pe) {
  if (!n_pes) return 0;
  return (uint32_t)((uint64_t)pe * n_ranks / n_pes);
}

uint64_t vdi_full_bytes(uint32_t width, uint32_t rows, uint32_t k) {
  return (uint64_t)width * rows * (1ull + 24ull * k);
}

vdi_status vdi_get_unique_id(uint8_t out[128]) {
  if (!out) return fail(VDI_ERR_INVALID_ARG, "out is NULL");
  ncclUniqueId id;
  ncclResult_t r = ncclGetUniqueId(&id);
  if (r != ncclSuccess) return fail(VDI_ERR_NCCL, "ncclGetUniqueId: %s", ncclGetErrorString(r));
  static_assert(sizeof(id) == 128, "ncclUniqueId size");
  memcpy(out, &id, 128);
  return VDI_OK;
}

vdi_status vdi_composite_init(const vdi_config* cfg, vdi_ctx** out) {
  if (!cfg || !out) return fail(VDI_ERR_INVALID_ARG, "cfg/out is NULL");
  *out = nullptr;
  if (!cfg->width || !cfg->height) return fail(VDI_ERR_INVALID_ARG, "empty image");
  if (cfg->k_in < 1 || cfg->k_in > 255 || cfg->k_out < 1 || cfg->k_out > 255)
    return fail(VDI_ERR_INVALID_ARG, "k_in/k_out must be in 1..255");
  if (cfg->n_pes < 1 || cfg->n_pes > VDI_MAX_SRC)
    return fail(VDI_ERR_INVALID_ARG, "n_pes must be in 1..%d", VDI_MAX_SRC);
  if (cfg->n_ranks < 1 || cfg->rank >= cfg->n_ranks) return fail(VDI_ERR_INVALID_ARG, "bad rank/n_ranks");
  if (cfg->root >= cfg->n_ranks) return fail(VDI_ERR_INVALID_ARG, "root %u >= n_ranks %u", cfg->root, cfg->n_ranks);
  if (cfg->n_ranks > cfg->height) return fail(VDI_ERR_INVALID_ARG, "more ranks than image rows");
  if (cfg->n_ranks > 1 && !cfg->nccl_unique_id) return fail(VDI_ERR_INVALID_ARG, "nccl_unique_id required");
  if ((uint64_t)cfg->width * cfg->height > (1ull << 31)) return fail(VDI_ERR_INVALID_ARG, "image too large");
  vdi_ctx* ctx = new vdi_ctx();
  ctx->cfg = *cfg;
  if (!ctx->cfg.max_iters) ctx->cfg.max_iters = 16;
  if (!(ctx->cfg.gamma_max > 0.0f)) ctx->cfg.gamma_max = 2.0f;
  ctx->cfg.nccl_unique_id = nullptr;
  ctx->stream = static_cast<cudaStream_t>(cfg->cuda_stream);
  cudaError_t e = cudaGetDevice(&ctx->device);
  if (e != cudaSuccess) {
    delete ctx;
    return fail(VDI_ERR_CUDA, "cudaGetDevice: %s", cudaGetErrorString(e));
  }
  ctx->row0 = strip_row(cfg->height, cfg->n_ranks, cfg->rank);
  ctx->row1 = strip_row(cfg->height, cfg->n_ranks, cfg->rank + 1);
  ctx->P = (uint64_t)(ctx->row1 - ctx->row0) * cfg->width;
  ctx->rcount.resize(cfg->n_pes);
  ctx->rdepth.resize(cfg->n_pes);
  ctx->rrgba.resize(cfg->n_pes);
  ctx->gen.resize(cfg->n_pes);
  ctx->hcount.resize(cfg->n_pes);
  ctx->hoffset.resize(cfg->n_pes);
  ctx->hdepth.resize(cfg->n_pes);
  ctx->hrgba.resize(cfg->n_pes);
  ctx->hcount1.resize(cfg->n_pes);
  ctx->hoffset1.resize(cfg->n_pes);
  ctx->hdepth1.resize(cfg->n_pes);
  ctx->hrgba1.resize(cfg->n_pes);
  for (auto& ev : ctx->ev) cudaEventCreate(&ev);
  for (auto& ev : ctx->gev) cudaEventCreate(&ev);
  for (auto& ev : ctx->fev) cudaEventCreate(&ev);
  for (auto& ev : ctx->evx) cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
  for (auto& r : ctx->evc)
    for (auto& ev : r) cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
  for (auto& x : ctx->xs) cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking);
  if (cfg->n_ranks > 1) {
    ncclUniqueId id;
    memcpy(&id, cfg->nccl_unique_id, sizeof id);
    ncclResult_t r = ncclCommInitRank(&ctx->comm, (int)cfg->n_ranks, id, (int)cfg->rank);
    if (r != ncclSuccess) {
      ctx->comm = nullptr;
      delete ctx;
      return fail(VDI_ERR_NCCL, "ncclCommInitRank: %s", ncclGetErrorString(r));
    }
  }
  *out = ctx;
  return VDI_OK;
}

void vdi_composite_destroy(vdi_ctx* ctx) { delete ctx; }

// ---------------------------------------------------------------------------
// Phase 1 (SUPPORT)
// ---------------------------------------------------------------------------
vdi_status vdi_generate_subvdi(vdi_ctx* ctx, const vdi_volume_desc* vol, const vdi_tf_desc* tf,
                               const vdi_camera* cam, const vdi_decomp_desc* dec, uint32_t pe_id,
                               vdi_dense_view* out) {
  if (vdi_status s = check_ctx(ctx)) return s;
  if (!vol || !tf || !cam || !dec || !out || !vol->voxels || !tf->table)
    return fail(VDI_ERR_INVALID_ARG, "NULL argument");
  if (pe_id >= ctx->cfg.n_pes) return fail(VDI_ERR_INVALID_ARG, "pe_id out of range");
  if (vol->bytes_per_voxel != 1 && vol->bytes_per_voxel != 2)
    return fail(VDI_ERR_INVALID_ARG, "bytes_per_voxel must be 1 or 2");
  for (int a = 0; a < 3; ++a) {
    if (!vol->dims[a]) return fail(VDI_ERR_INVALID_ARG, "empty volume");
    if (dec->grid[a] < 1 || dec->grid[a] > VDI_MAX_GRID_AXIS)
      return fail(VDI_ERR_INVALID_ARG, "decomposition grid must be 1..%d per axis", VDI_MAX_GRID_AXIS);
  }
  if (!dec->xb || !dec->yb || !dec->zb || !dec->owner) return fail(VDI_ERR_INVALID_ARG, "NULL decomposition");
  GenParams gp{};
  gp.vox = vol->voxels;
  gp.bytes = (int)vol->bytes_per_voxel;
  for (int a = 0; a < 3; ++a) {
    gp.dims[a] = (int)vol->dims[a];
    gp.grid[a] = (int)dec->grid[a];
    gp.eye[a] = cam->eye[a];
    gp.fwd[a] = cam->fwd[a];
    gp.right[a] = cam->right[a];
    gp.up[a] = cam->up[a];
  }
  gp.tf = reinterpret_cast<const float4*>(tf->table);
  gp.tan_x = cam->tan_x;
  gp.tan_y = cam->tan_y;
  gp.W = (int)ctx->cfg.width;
  gp.H = (int)ctx->cfg.height;
  for (uint32_t i = 0; i <= dec->grid[0]; ++i) gp.xb[i] = dec->xb[i];
  for (uint32_t i = 0; i <= dec->grid[1]; ++i) gp.yb[i] = dec->yb[i];
  for (uint32_t i = 0; i <= dec->grid[2]; ++i) gp.zb[i] = dec->zb[i];
  const size_t nb = (size_t)dec->grid[0] * dec->grid[1] * dec->grid[2];
  std::vector<int8_t> own(nb);
  float lo[3] = {1e30f, 1e30f, 1e30f}, hi[3] = {-1e30f, -1e30f, -1e30f};
  bool any = false;
  for (uint32_t bz = 0; bz < dec->grid[2]; ++bz)
    for (uint32_t by = 0; by < dec->grid[1]; ++by)
      for (uint32_t bx = 0; bx < dec->grid[0]; ++bx) {
        const size_t b = ((size_t)bz * dec->grid[1] + by) * dec->grid[0] + bx;
        const int o = dec->owner[b];
        if (o < -1 || o >= 127) return fail(VDI_ERR_INVALID_ARG, "owner id out of range");
        own[b] = (int8_t)o;
        if (o == (int)pe_id) {
          any = true;
          const int l[3] = {dec->xb[bx], dec->yb[by], dec->zb[bz]};
          const int h[3] = {dec->xb[bx + 1], dec->yb[by + 1], dec->zb[bz + 1]};
          for (int a = 0; a < 3; ++a) {
            lo[a] = std::min(lo[a], (float)l[a]);
            hi[a] = std::max(hi[a], (float)h[a]);
          }
        }
      }
  if (!any)
    for (int a = 0; a < 3; ++a) lo[a] = hi[a] = -1e6f;  // empty domain: no samples
  for (int a = 0; a < 3; ++a) {
    gp.lo[a] = lo[a];
    gp.hi[a] = hi[a];
  }
  gp.pe = (int)pe_id;
  gp.k = (int)ctx->cfg.k_in;
  gp.max_iters = (int)ctx->cfg.max_iters;
  gp.gamma_max = ctx->cfg.gamma_max;

  GenOut& g = ctx->gen[pe_id];
  const size_t P = (size_t)ctx->cfg.width * ctx->cfg.height;
  CUDA_TRY(ctx, g.owner.grow(nb));
  CUDA_TRY(ctx, cudaMemcpyAsync(g.owner.p, own.data(), nb, cudaMemcpyHostToDevice, ctx->stream));
  gp.owner = g.owner.as<int8_t>();
  CUDA_TRY(ctx, g.count32.grow((P + 1) * 4));
  CUDA_TRY(ctx, g.count8.grow(P));
  CUDA_TRY(ctx, g.offset.grow((P + 1) * 4));
  CUDA_TRY(ctx, g.gamma.grow(P * 4));
  CUDA_TRY(ctx, ctx->gen_tmp.grow(16));
  int* derr = ctx->gen_tmp.as<int>();
  CUDA_TRY(ctx, cudaMemsetAsync(derr, 0, 4, ctx->stream));
  CUDA_TRY(ctx, launch_gen_pass1(gp, g.count32.as<uint32_t>(), g.gamma.as<float>(), derr, ctx->stream));
  CUDA_TRY(ctx, gen_scan(g.count32.as<uint32_t>(), g.offset.as<uint32_t>(), P + 1, &ctx->cub_tmp,
                         &ctx->cub_tmp_bytes, ctx->stream));
  uint32_t total32 = 0;
  int herr = 0;
  CUDA_TRY(ctx, cudaMemcpyAsync(&total32, g.offset.as<uint32_t>() + P, 4, cudaMemcpyDeviceToHost, ctx->stream));
  CUDA_TRY(ctx, cudaMemcpyAsync(&herr, derr, 4, cudaMemcpyDeviceToHost, ctx->stream));
  CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  if (herr & 2) return fail(VDI_ERR_CAPACITY, "a ray of PE %u needs more than k_in supersegments (Q20)", pe_id);
  g.total = total32;
  CUDA_TRY(ctx, g.depth.grow(std::max<size_t>(g.total, 1) * 8));
  CUDA_TRY(ctx, g.rgba.grow(std::max<size_t>(g.total, 1) * 16));
  CUDA_TRY(ctx, launch_gen_pass2(gp, g.offset.as<uint32_t>(), g.gamma.as<float>(), g.count32.as<uint32_t>(),
                                 g.depth.as<float2>(), g.rgba.as<float4>(), ctx->stream));
  CUDA_TRY(ctx, launch_u32_to_u8(g.count32.as<uint32_t>(), g.count8.as<uint8_t>(), P, ctx->stream));
  out->pe_id = pe_id;
  out->total = g.total;
  out->count = g.count8.as<uint8_t>();
  out->offset = g.offset.as<uint32_t>();
  out->depth = g.depth.as<float>();
  out->rgba = g.rgba.as<float>();
  return VDI_OK;
}

// ---------------------------------------------------------------------------
// Phase 2: the hot path
// ---------------------------------------------------------------------------
vdi_status vdi_composite(vdi_ctx* ctx, const vdi_dense_view* local, uint32_t n_local, vdi_full_view* so) {
  if (vdi_status s = check_ctx(ctx)) return s;
  const vdi_config& cf = ctx->cfg;
  const uint32_t G = cf.n_ranks, me = cf.rank, n = cf.n_pes, W = cf.width, k = cf.k_out;
  if (!so || !so->count || !so->depth || !so->rgba) return fail(VDI_ERR_INVALID_ARG, "strip_out is NULL");
  if (so->row_begin != ctx->row0 || so->row_end != ctx->row1)
    return fail(VDI_ERR_CAPACITY, "strip_out rows [%u,%u) != this rank's strip [%u,%u)", so->row_begin,
                so->row_end, ctx->row0, ctx->row1);
  if ((reinterpret_cast<uintptr_t>(so->rgba) & 15) || (reinterpret_cast<uintptr_t>(so->depth) & 7))
    return fail(VDI_ERR_INVALID_ARG, "strip_out depth/rgba must be 8/16-byte aligned");
  // which PEs are homed here (PAPER.md:218 block placement)
  std::vector<int> slot(n, -1);
  uint32_t expect = 0;
  for (uint32_t s = 0; s < n; ++s)
    if (vdi_pe_home(n, G, s) == me) ++expect;
  if (n_local != expect) return fail(VDI_ERR_INVALID_ARG, "rank %u homes %u PEs, got %u", me, expect, n_local);
  if (n_local && !local) return fail(VDI_ERR_INVALID_ARG, "local_pes is NULL");
  for (uint32_t l = 0; l < n_local; ++l) {
    const vdi_dense_view& v = local[l];
    if (v.pe_id >= n || vdi_pe_home(n, G, v.pe_id) != me || slot[v.pe_id] >= 0)
      return fail(VDI_ERR_INVALID_ARG, "pe_id %u not homed on rank %u or duplicated", v.pe_id, me);
    if (!v.count || (v.total && (!v.depth || !v.rgba)) || (G > 1 && !v.offset))
      return fail(VDI_ERR_INVALID_ARG, "dense view of PE %u has NULL arrays", v.pe_id);
    if ((reinterpret_cast<uintptr_t>(v.rgba) & 15) || (reinterpret_cast<uintptr_t>(v.depth) & 7))
      return fail(VDI_ERR_INVALID_ARG, "dense view of PE %u: depth/rgba misaligned", v.pe_id);
    slot[v.pe_id] = (int)l;
  }
  cudaStream_t st = ctx->stream;
  const bool timing = cf.flags & VDI_FLAG_STAGE_TIMING;
  int launches = 0;
  if (timing) CUDA_TRY(ctx, cudaEventRecord(ctx->ev[0], st));

  MergeParams mp{};
  mp.n_src = (int)n;
  mp.k_out = (int)k;
  mp.max_iters = (int)cf.max_iters;
  mp.gamma_max = cf.gamma_max;
  mp.P = (uint32_t)ctx->P;
  mp.n_groups = (uint32_t)((ctx->P + 31) / 32);
  uint64_t S_here = 0, sent = 0, recvd = 0;

  if (G == 1) {
    // every source is whole and local: when all carry their offset arrays
    // (Fig. 2) the group bases are read from them and the
    // receive-side scan is skipped
    bool all_off = true;
    for (uint32_t s = 0; s < n; ++s) all_off &= local[slot[s]].offset != nullptr;
    for (uint32_t s = 0; s < n; ++s) {
      const vdi_dense_view& v = local[slot[s]];
      mp.src[s] = SrcDesc{v.count, reinterpret_cast<const float2*>(v.depth), reinterpret_cast<const float4*>(v.rgba),
                          all_off ? v.offset : nullptr};
      S_here += v.total;
    }
  } else {
    // strip boundaries of every PE's dense payload: bnd[s][g] = offset_s[row_g * W]
    std::vector<uint32_t> rows(G + 1);
    for (uint32_t g = 0; g <= G; ++g) rows[g] = strip_row(cf.height, G, g);
    const size_t nb = (size_t)n * (G + 1);
    const size_t hdr = 64 * 8 + 64 * 4 + 64 * 4;  // ptrs, pes, rows
    // exchange blob: bnd (u64) | IPC references of every PE's count/depth/rgba
    const bool peer = !(cf.flags & VDI_FLAG_NCCL_EXCHANGE);
    const size_t refs_bytes = peer ? (size_t)n * 3 * sizeof(IpcRef) : 0;
    const size_t blob = nb * 8 + refs_bytes;
    CUDA_TRY(ctx, ctx->bounds.grow(blob + hdr));
    std::vector<uint8_t> h(hdr, 0);
    const uint32_t** hp = reinterpret_cast<const uint32_t**>(h.data());
    uint32_t* hpes = reinterpret_cast<uint32_t*>(h.data() + 64 * 8);
    uint32_t* hrows = reinterpret_cast<uint32_t*>(h.data() + 64 * 8 + 64 * 4);
    for (uint32_t l = 0; l < n_local; ++l) {
      hp[l] = local[l].offset;
      hpes[l] = local[l].pe_id;
    }
    for (uint32_t g = 0; g <= G; ++g) hrows[g] = rows[g];
    uint8_t* dh = ctx->bounds.as<uint8_t>() + blob;
    unsigned long long* dbnd = ctx->bounds.as<unsigned long long>();
    std::vector<IpcRef> myrefs;
    if (peer) {  // this rank's PEs, exported for the peers (zeros elsewhere: the sum is a gather)
      myrefs.assign((size_t)n * 3, IpcRef{});
      for (uint32_t l = 0; l < n_local; ++l) {
        const vdi_dense_view& v = local[l];
        const void* ptrs[3] = {v.count, v.depth, v.rgba};
        for (int a2 = 0; a2 < 3; ++a2) {
          if (!ptrs[a2]) continue;
          if (!ipc_export(ptrs[a2], &myrefs[(size_t)v.pe_id * 3 + a2]))
            return fail(VDI_ERR_INVALID_ARG, "PE %u: buffer is not IPC-exportable device memory (use "
                        "VDI_FLAG_NCCL_EXCHANGE)", v.pe_id);
        }
      }
    }
    CUDA_TRY(ctx, cudaMemcpyAsync(dh, h.data(), hdr, cudaMemcpyHostToDevice, st));
    CUDA_TRY(ctx, cudaMemsetAsync(dbnd, 0, nb * 8, st));
    if (peer)
      CUDA_TRY(ctx, cudaMemcpyAsync(reinterpret_cast<uint8_t*>(dbnd) + nb * 8, myrefs.data(), refs_bytes,
                                    cudaMemcpyHostToDevice, st));
    gather_bounds_kernel<<<1, 256, 0, st>>>(reinterpret_cast<const uint32_t* const*>(dh),
                                            reinterpret_cast<const uint32_t*>(dh + 64 * 8), (int)n_local,
                                            reinterpret_cast<const uint32_t*>(dh + 64 * 8 + 64 * 4), (int)G, W,
                                            (int)n, dbnd);
    ++launches;
    CUDA_TRY(ctx, cudaGetLastError());
    // size (+ IPC reference) exchange: every rank contributes its PEs' rows and
    // zeros elsewhere, so a byte-wise sum is a gather.  It is also the start
    // barrier of the peer reads: every rank's inputs are complete in its
    // stream order before it joins.
    NCCL_TRY(ctx, ncclAllReduce(dbnd, dbnd, blob, ncclUint8, ncclSum, ctx->comm, st));
    std::vector<unsigned long long> bnd(nb);
    std::vector<IpcRef> refs(peer ? (size_t)n * 3 : 0);
    CUDA_TRY(ctx, cudaMemcpyAsync(bnd.data(), dbnd, nb * 8, cudaMemcpyDeviceToHost, st));
    if (peer)
      CUDA_TRY(ctx, cudaMemcpyAsync(refs.data(), reinterpret_cast<uint8_t*>(dbnd) + nb * 8, refs_bytes,
                                    cudaMemcpyDeviceToHost, st));
    CUDA_TRY(ctx, cudaStreamSynchronize(st));
    auto T = [&](uint32_t s, uint32_t g) { return bnd[(size_t)s * (G + 1) + g + 1] - bnd[(size_t)s * (G + 1) + g]; };
    if (peer) {
      // Exchange over NVLink through CUDA IPC mappings of the peers' sub-VDIs:
      // default, the strip slices are pulled by the copy engines (peer
      // cudaMemcpyAsync on side streams) into local buffers; with
      // VDI_FLAG_PEER_READS the merge kernels read peer memory directly.
      const bool zero_copy = cf.flags & VDI_FLAG_PEER_READS;
      const bool sm_copies = !(cf.flags & VDI_FLAG_CE_COPIES) && !zero_copy;
      std::vector<CopySeg> segs;
      int q = 0;
      if (!zero_copy) CUDA_TRY(ctx, cudaEventRecord(ctx->evx[0], st));
      for (uint32_t s = 0; s < n; ++s) {
        if (slot[s] >= 0) continue;
        void* pc = nullptr;
        void* pd = nullptr;
        void* pr = nullptr;
        CUDA_TRY(ctx, ipc_import(ctx, refs[(size_t)s * 3 + 0], &pc));
        CUDA_TRY(ctx, ipc_import(ctx, refs[(size_t)s * 3 + 1], &pd));
        CUDA_TRY(ctx, ipc_import(ctx, refs[(size_t)s * 3 + 2], &pr));
        const uint64_t b0 = bnd[(size_t)s * (G + 1) + me], t = T(s, me);
        const uint8_t* rc = static_cast<const uint8_t*>(pc) + (size_t)ctx->row0 * W;
        const float2* rd = static_cast<const float2*>(pd) + b0;
        const float4* rr = static_cast<const float4*>(pr) + b0;
        if (zero_copy) {
          mp.src[s] = SrcDesc{rc, rd, rr};
        } else {
          CUDA_TRY(ctx, ctx->rcount[s].grow(ctx->P));
          CUDA_TRY(ctx, ctx->rdepth[s].grow(std::max<uint64_t>(t, 1) * 8));
          CUDA_TRY(ctx, ctx->rrgba[s].grow(std::max<uint64_t>(t, 1) * 16));
          if (sm_copies) {
            segs.push_back(CopySeg{rc, ctx->rcount[s].p, ctx->P});
            if (t) {
              segs.push_back(CopySeg{rd, ctx->rdepth[s].p, t * 8});
              segs.push_back(CopySeg{rr, ctx->rrgba[s].p, t * 16});
            }
          } else {
            cudaStream_t cs = ctx->xs[q % vdi_ctx::kXStreams];
            if (q < vdi_ctx::kXStreams) CUDA_TRY(ctx, cudaStreamWaitEvent(cs, ctx->evx[0], 0));
            CUDA_TRY(ctx, cudaMemcpyAsync(ctx->rcount[s].p, rc, ctx->P, cudaMemcpyDeviceToDevice, cs));
            if (t) {
              CUDA_TRY(ctx, cudaMemcpyAsync(ctx->rdepth[s].p, rd, t * 8, cudaMemcpyDeviceToDevice, cs));
              CUDA_TRY(ctx, cudaMemcpyAsync(ctx->rrgba[s].p, rr, t * 16, cudaMemcpyDeviceToDevice, cs));
            }
          }
          mp.src[s] = SrcDesc{ctx->rcount[s].as<uint8_t>(), ctx->rdepth[s].as<float2>(), ctx->rrgba[s].as<float4>()};
          ++q;
        }
        recvd += ctx->P + 24 * t;
      }
      // nothing overlaps the strip exchange: the whole GPU pulls (16 blocks per SM)
      if (sm_copies) CUDA_TRY(ctx, sm_copy(ctx, segs, st, launches, 16));
      for (int i = 0; i < (sm_copies ? 0 : std::min<int>(q, vdi_ctx::kXStreams)); ++i) {  // join the copy streams
        CUDA_TRY(ctx, cudaEventRecord(ctx->evx[1 + i], ctx->xs[i]));
        CUDA_TRY(ctx, cudaStreamWaitEvent(st, ctx->evx[1 + i], 0));
      }
      for (uint32_t s = 0; s < n; ++s)
        if (slot[s] >= 0)
          for (uint32_t g = 0; g < G; ++g)
            if (g != me) sent += (uint64_t)(rows[g + 1] - rows[g]) * W + 24 * T(s, g);
      ctx->peer_reads = true;
    } else {
      for (uint32_t s = 0; s < n; ++s) {
        if (slot[s] >= 0) continue;
        CUDA_TRY(ctx, ctx->rcount[s].grow(ctx->P));
        CUDA_TRY(ctx, ctx->rdepth[s].grow(std::max<uint64_t>(T(s, me), 1) * 8));
        CUDA_TRY(ctx, ctx->rrgba[s].grow(std::max<uint64_t>(T(s, me), 1) * 16));
      }
      // all-to-allv of count slices and dense payload slices
      NCCL_TRY(ctx, ncclGroupStart());
      for (uint32_t g = 0; g < G; ++g) {
        if (g == me) continue;
        const uint64_t Pg = (uint64_t)(rows[g + 1] - rows[g]) * W;
        for (uint32_t s = 0; s < n; ++s) {  // our PEs -> g
          if (slot[s] < 0) continue;
          const vdi_dense_view& v = local[slot[s]];
          const uint64_t b = bnd[(size_t)s * (G + 1) + g], t = T(s, g);
          NCCL_TRY(ctx, ncclSend(v.count + (size_t)rows[g] * W, Pg, ncclUint8, (int)g, ctx->comm, st));
          if (t) {
            NCCL_TRY(ctx, ncclSend(v.depth + b * 2, t * 2, ncclFloat32, (int)g, ctx->comm, st));
            NCCL_TRY(ctx, ncclSend(v.rgba + b * 4, t * 4, ncclFloat32, (int)g, ctx->comm, st));
          }
          sent += Pg + 24 * t;
        }
        for (uint32_t s = 0; s < n; ++s) {  // g's PEs -> us
          if (vdi_pe_home(n, G, s) != g) continue;
          const uint64_t t = T(s, me);
          NCCL_TRY(ctx, ncclRecv(ctx->rcount[s].p, ctx->P, ncclUint8, (int)g, ctx->comm, st));
          if (t) {
            NCCL_TRY(ctx, ncclRecv(ctx->rdepth[s].p, t * 2, ncclFloat32, (int)g, ctx->comm, st));
            NCCL_TRY(ctx, ncclRecv(ctx->rrgba[s].p, t * 4, ncclFloat32, (int)g, ctx->comm, st));
          }
          recvd += ctx->P + 24 * t;
        }
      }
      NCCL_TRY(ctx, ncclGroupEnd());
    }
    for (uint32_t s = 0; s < n; ++s) {
      S_here += T(s, me);
      if (slot[s] >= 0) {
        const vdi_dense_view& v = local[slot[s]];
        const uint64_t b = bnd[(size_t)s * (G + 1) + me];
        mp.src[s] = SrcDesc{v.count + (size_t)ctx->row0 * W, reinterpret_cast<const float2*>(v.depth) + b,
                            reinterpret_cast<const float4*>(v.rgba) + b};
      } else if (!peer) {
        mp.src[s] = SrcDesc{ctx->rcount[s].as<uint8_t>(), ctx->rdepth[s].as<float2>(), ctx->rrgba[s].as<float4>()};
      }  // peer: set above
    }
  }
  if (timing) CUDA_TRY(ctx, cudaEventRecord(ctx->ev[1], st));

  if (vdi_status s = merge_lists(ctx, mp, ctx->P, S_here, so, timing, launches)) return s;
  if (ctx->peer_reads) {
    // end barrier: no rank reuses its inputs before every peer finished reading them
    CUDA_TRY(ctx, ctx->bounds.grow(16));
    NCCL_TRY(ctx, ncclAllReduce(ctx->bounds.p, ctx->bounds.p, 1, ncclUint8, ncclSum, ctx->comm, st));
    ctx->peer_reads = false;
  }
  if (timing) {
    CUDA_TRY(ctx, cudaEventRecord(ctx->ev[2], st));
    ctx->timing_pending = true;
  }
  ctx->have_stats = cf.flags & VDI_FLAG_PIXEL_STATS;
  ctx->last = vdi_counters{};
  ctx->last.bytes_sent = sent;
  ctx->last.bytes_received = recvd;
  ctx->last.kernel_launches = (uint32_t)launches;
  return VDI_OK;
}

vdi_status vdi_composite_frames(vdi_ctx* ctx, uint32_t F, const vdi_dense_view* local, uint32_t n_local,
                                vdi_full_view* images, uint32_t chunks) {
  if (vdi_status s = check_ctx(ctx)) return s;
  const vdi_config& cf = ctx->cfg;
  const uint32_t G = cf.n_ranks, me = cf.rank, n = cf.n_pes, W = cf.width, H = cf.height;
  const uint64_t P = (uint64_t)W * H;
  if (F < 1) return fail(VDI_ERR_INVALID_ARG, "n_frames must be >= 1");
  if (!images) return fail(VDI_ERR_INVALID_ARG, "images is NULL");
  const uint32_t C = std::max<uint32_t>(1, std::min<uint32_t>(chunks ? chunks : 2, std::min<uint32_t>(vdi_ctx::kMaxChunks, H)));
  uint32_t expect = 0;
  for (uint32_t s = 0; s < n; ++s)
    if (vdi_pe_home(n, G, s) == me) ++expect;
  if (n_local != expect) return fail(VDI_ERR_INVALID_ARG, "rank %u homes %u PEs, got %u", me, expect, n_local);
  if (n_local && !local) return fail(VDI_ERR_INVALID_ARG, "local_pes is NULL");
  // slot[f][s]: index of PE s of frame f in local[], -1 if remote
  std::vector<int> slot((size_t)F * n, -1);
  for (uint32_t f = 0; f < F; ++f)
    for (uint32_t l = 0; l < n_local; ++l) {
      const vdi_dense_view& v = local[(size_t)f * n_local + l];
      if (v.pe_id >= n || vdi_pe_home(n, G, v.pe_id) != me || slot[(size_t)f * n + v.pe_id] >= 0)
        return fail(VDI_ERR_INVALID_ARG, "frame %u: pe_id %u not homed on rank %u or duplicated", f, v.pe_id, me);
      if (!v.count || !v.offset || (v.total && (!v.depth || !v.rgba)))
        return fail(VDI_ERR_INVALID_ARG, "frame %u: dense view of PE %u has NULL arrays", f, v.pe_id);
      if ((reinterpret_cast<uintptr_t>(v.rgba) & 15) || (reinterpret_cast<uintptr_t>(v.depth) & 7))
        return fail(VDI_ERR_INVALID_ARG, "frame %u: dense view of PE %u misaligned", f, v.pe_id);
      slot[(size_t)f * n + v.pe_id] = (int)l;
    }
  for (uint32_t f = me; f < F; f += G) {
    const vdi_full_view& im = images[f];
    if (!im.count || !im.depth || !im.rgba || im.row_begin != 0 || im.row_end != H)
      return fail(VDI_ERR_INVALID_ARG, "images[%u] (owned by rank %u) must cover rows [0, H)", f, me);
    if ((reinterpret_cast<uintptr_t>(im.rgba) & 15) || (reinterpret_cast<uintptr_t>(im.depth) & 7))
      return fail(VDI_ERR_INVALID_ARG, "images[%u]: depth/rgba must be 8/16-byte aligned", f);
  }
  cudaStream_t st = ctx->stream;
  const bool timing = cf.flags & VDI_FLAG_STAGE_TIMING;
  int launches = 0;
  uint64_t sent = 0, recvd = 0;
  if (timing) CUDA_TRY(ctx, cudaEventRecord(ctx->ev[0], st));
  std::vector<uint32_t> rows(C + 1);
  for (uint32_t c = 0; c <= C; ++c) rows[c] = strip_row(H, C, c);
  const size_t nb = (size_t)n * (C + 1);  // bnd[s][c] = offset_s[rows[c] * W] of one frame
  // exchange blob: per frame bnd (u64) | per frame IPC references of every PE's count/depth/rgba
  const size_t refs_off = (size_t)F * nb * 8;
  const size_t blob = refs_off + (G > 1 ? (size_t)F * n * 3 * sizeof(IpcRef) : 0);
  const size_t hdr = 64 * 8 + 64 * 4 + 64 * 4;  // per frame: ptrs, pes, rows
  CUDA_TRY(ctx, ctx->fblob.grow(blob + (size_t)F * hdr));
  uint8_t* dblob = ctx->fblob.as<uint8_t>();
  std::vector<uint8_t> h((size_t)F * hdr, 0);
  std::vector<IpcRef> myrefs(G > 1 ? (size_t)F * n * 3 : 0, IpcRef{});
  for (uint32_t f = 0; f < F; ++f) {
    uint8_t* hf = h.data() + (size_t)f * hdr;
    const uint32_t** hp = reinterpret_cast<const uint32_t**>(hf);
    uint32_t* hpes = reinterpret_cast<uint32_t*>(hf + 64 * 8);
    uint32_t* hrows = reinterpret_cast<uint32_t*>(hf + 64 * 8 + 64 * 4);
    for (uint32_t l = 0; l < n_local; ++l) {
      const vdi_dense_view& v = local[(size_t)f * n_local + l];
      hp[l] = v.offset;
      hpes[l] = v.pe_id;
      if (G > 1) {
        const void* ptrs[3] = {v.count, v.depth, v.rgba};
        for (int a2 = 0; a2 < 3; ++a2)
          if (ptrs[a2] && !ipc_export(ptrs[a2], &myrefs[((size_t)f * n + v.pe_id) * 3 + a2]))
            return fail(VDI_ERR_INVALID_ARG, "frame %u PE %u: buffer is not IPC-exportable device memory", f,
                        v.pe_id);
      }
    }
    for (uint32_t c = 0; c <= C; ++c) hrows[c] = rows[c];
  }
  CUDA_TRY(ctx, cudaMemcpyAsync(dblob + blob, h.data(), h.size(), cudaMemcpyHostToDevice, st));
  CUDA_TRY(ctx, cudaMemsetAsync(dblob, 0, refs_off, st));
  if (G > 1)
    CUDA_TRY(ctx, cudaMemcpyAsync(dblob + refs_off, myrefs.data(), myrefs.size() * sizeof(IpcRef),
                                  cudaMemcpyHostToDevice, st));
  {  // one launch for every frame
    const uint8_t* dh = dblob + blob;
    gather_bounds_kernel<<<F, 256, 0, st>>>(reinterpret_cast<const uint32_t* const*>(dh),
                                            reinterpret_cast<const uint32_t*>(dh + 64 * 8), (int)n_local,
                                            reinterpret_cast<const uint32_t*>(dh + 64 * 8 + 64 * 4), (int)C, W,
                                            (int)n, reinterpret_cast<unsigned long long*>(dblob), hdr, nb);
    ++launches;
  }
  CUDA_TRY(ctx, cudaGetLastError());
  // one size + IPC-reference exchange for all frames (each rank contributes
  // its PEs' entries, zeros elsewhere: the byte-wise sum is a gather); also
  // the start barrier of the peer copies
  if (G > 1) NCCL_TRY(ctx, ncclAllReduce(dblob, dblob, blob, ncclUint8, ncclSum, ctx->comm, st));
  std::vector<unsigned long long> bnd((size_t)F * nb);
  std::vector<IpcRef> refs(myrefs.size());
  CUDA_TRY(ctx, cudaMemcpyAsync(bnd.data(), dblob, refs_off, cudaMemcpyDeviceToHost, st));
  if (G > 1)
    CUDA_TRY(ctx, cudaMemcpyAsync(refs.data(), dblob + refs_off, refs.size() * sizeof(IpcRef),
                                  cudaMemcpyDeviceToHost, st));
  CUDA_TRY(ctx, cudaStreamSynchronize(st));
  auto B = [&](uint32_t f, uint32_t s, uint32_t c) { return bnd[(size_t)f * nb + (size_t)s * (C + 1) + c]; };
  for (uint32_t f = 0; f < F; ++f)  // bytes this rank's PEs send to the frames' owners
    if (f % G != me)
      for (uint32_t s = 0; s < n; ++s)
        if (slot[(size_t)f * n + s] >= 0) sent += P + 24 * B(f, s, C);
  // frames owned here: the copy engines pull every remote PE's sub-VDI over
  // NVLink chunk by chunk (rows [rows[c], rows[c+1])) while the merge of the
  // previous chunk runs on the compositing stream
  uint32_t j = 0;
  bool first = true;
  if (G > 1) CUDA_TRY(ctx, cudaEventRecord(ctx->evx[0], st));  // the copies wait only for the size exchange
  for (uint32_t f = me; f < F; f += G, ++j) {
    if (ctx->fcount.size() < (size_t)(j + 1) * n) {
      while (ctx->fcount.size() < (size_t)(j + 1) * n) {
        ctx->fcount.emplace_back(new DevBuf());
        ctx->fdepth.emplace_back(new DevBuf());
        ctx->frgba.emplace_back(new DevBuf());
      }
    }
    struct Src {
      const uint8_t* c;
      const float2* d;
      const float4* r;
    };
    std::vector<Src> src(n), rp(n);
    std::vector<int> qs(n, -1);
    int q = 0;
    for (uint32_t s = 0; s < n; ++s) {
      const int l = slot[(size_t)f * n + s];
      if (l >= 0) {
        const vdi_dense_view& v = local[(size_t)f * n_local + l];
        src[s] = Src{v.count, reinterpret_cast<const float2*>(v.depth), reinterpret_cast<const float4*>(v.rgba)};
        continue;
      }
      void *pc = nullptr, *pd = nullptr, *pr = nullptr;
      CUDA_TRY(ctx, ipc_import(ctx, refs[((size_t)f * n + s) * 3 + 0], &pc));
      CUDA_TRY(ctx, ipc_import(ctx, refs[((size_t)f * n + s) * 3 + 1], &pd));
      CUDA_TRY(ctx, ipc_import(ctx, refs[((size_t)f * n + s) * 3 + 2], &pr));
      const uint64_t T = B(f, s, C);
      DevBuf& bc = *ctx->fcount[(size_t)j * n + s];
      DevBuf& bd = *ctx->fdepth[(size_t)j * n + s];
      DevBuf& br = *ctx->frgba[(size_t)j * n + s];
      recvd += P + 24 * T;
      if (cf.flags & VDI_FLAG_PEER_READS) {  // zero copy: the merge kernels load the peer's arrays over NVLink
        src[s] = Src{static_cast<const uint8_t*>(pc), static_cast<const float2*>(pd), static_cast<const float4*>(pr)};
        continue;
      }
      CUDA_TRY(ctx, bc.grow(P));
      CUDA_TRY(ctx, bd.grow(std::max<uint64_t>(T, 1) * 8));
      CUDA_TRY(ctx, br.grow(std::max<uint64_t>(T, 1) * 16));
      src[s] = Src{bc.as<uint8_t>(), bd.as<float2>(), br.as<float4>()};
      const int xi = q % vdi_ctx::kXStreams;
      qs[s] = xi;
      rp[s] = Src{static_cast<const uint8_t*>(pc), static_cast<const float2*>(pd), static_cast<const float4*>(pr)};
      ++q;
    }
    const int nq = std::min<int>(q, vdi_ctx::kXStreams);
    for (int xi = 0; xi < nq; ++xi) CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->xs[xi], ctx->evx[0], 0));
    const bool smc = !(cf.flags & VDI_FLAG_CE_COPIES) && j == 0 && q;
    if (smc) {
      // the first owned frame: nothing else runs yet, so the SMs pull its
      // remote sources (faster than the copy engines); later frames' copies
      // go to the copy engines after it, overlapping the merges
      std::vector<CopySeg> segs;
      for (uint32_t s = 0; s < n; ++s) {
        if (qs[s] < 0) continue;
        const uint64_t T = B(f, s, C);
        segs.push_back(CopySeg{rp[s].c, const_cast<uint8_t*>(src[s].c), P});
        if (T) {
          segs.push_back(CopySeg{rp[s].d, const_cast<float2*>(src[s].d), T * 8});
          segs.push_back(CopySeg{rp[s].r, const_cast<float4*>(src[s].r), T * 16});
        }
      }
      if (timing) CUDA_TRY(ctx, cudaEventRecord(ctx->fev[0], st));
      CUDA_TRY(ctx, sm_copy(ctx, segs, st, launches));
      if (timing) {
        CUDA_TRY(ctx, cudaEventRecord(ctx->fev[1], st));
        ctx->frames_timing_pending = true;
      }
      CUDA_TRY(ctx, cudaEventRecord(ctx->evx[0], st));  // later frames' copies start after it
    }
    // chunk-major issue: chunk c of every remote source, then one event per
    // copy stream, so the merge of chunk c waits only for chunk c's copies
    for (uint32_t c = 0; c < C && q && !smc; ++c) {
      const size_t r0 = (size_t)rows[c] * W, r1 = (size_t)rows[c + 1] * W;
      for (uint32_t s = 0; s < n; ++s) {
        if (qs[s] < 0) continue;
        cudaStream_t cs = ctx->xs[qs[s]];
        const uint64_t b0 = B(f, s, c), b1 = B(f, s, c + 1);
        CUDA_TRY(ctx, cudaMemcpyAsync(const_cast<uint8_t*>(src[s].c) + r0, rp[s].c + r0, r1 - r0,
                                      cudaMemcpyDeviceToDevice, cs));
        if (b1 > b0) {
          CUDA_TRY(ctx, cudaMemcpyAsync(const_cast<float2*>(src[s].d) + b0, rp[s].d + b0, (b1 - b0) * 8,
                                        cudaMemcpyDeviceToDevice, cs));
          CUDA_TRY(ctx, cudaMemcpyAsync(const_cast<float4*>(src[s].r) + b0, rp[s].r + b0, (b1 - b0) * 16,
                                        cudaMemcpyDeviceToDevice, cs));
        }
      }
      for (int xi = 0; xi < nq; ++xi) CUDA_TRY(ctx, cudaEventRecord(ctx->evc[c][xi], ctx->xs[xi]));
    }
    for (uint32_t c = 0; c < C; ++c) {
      MergeParams mp{};
      mp.n_src = (int)n;
      mp.k_out = (int)cf.k_out;
      mp.max_iters = (int)cf.max_iters;
      mp.gamma_max = cf.gamma_max;
      uint64_t S_c = 0;
      for (uint32_t s = 0; s < n; ++s) {
        const uint64_t b0 = B(f, s, c);
        mp.src[s] = SrcDesc{src[s].c + (size_t)rows[c] * W, src[s].d + b0, src[s].r + b0};
        S_c += B(f, s, c + 1) - b0;
      }
      vdi_full_view so{rows[c], rows[c + 1], images[f].count + (size_t)rows[c] * W,
                       images[f].depth + (size_t)rows[c] * W * cf.k_out * 2,
                       images[f].rgba + (size_t)rows[c] * W * cf.k_out * 4};
      if (!smc)
        for (int xi = 0; xi < nq; ++xi) CUDA_TRY(ctx, cudaStreamWaitEvent(st, ctx->evc[c][xi], 0));
      if (first && timing) CUDA_TRY(ctx, cudaEventRecord(ctx->ev[1], st));
      first = false;
      if (vdi_status e = merge_lists(ctx, mp, (uint64_t)(rows[c + 1] - rows[c]) * W, S_c, &so, timing, launches))
        return e;
    }
  }
  if (first && timing) CUDA_TRY(ctx, cudaEventRecord(ctx->ev[1], st));
  if (G > 1) {
    // end barrier: no rank reuses its inputs before every owner finished copying them
    for (int xi = 0; xi < vdi_ctx::kXStreams; ++xi) {
      CUDA_TRY(ctx, cudaEventRecord(ctx->evx[1 + xi], ctx->xs[xi]));
      CUDA_TRY(ctx, cudaStreamWaitEvent(st, ctx->evx[1 + xi], 0));
    }
    CUDA_TRY(ctx, ctx->bounds.grow(16));
    NCCL_TRY(ctx, ncclAllReduce(ctx->bounds.p, ctx->bounds.p, 1, ncclUint8, ncclSum, ctx->comm, st));
  }
  if (timing) {
    CUDA_TRY(ctx, cudaEventRecord(ctx->ev[2], st));
    ctx->timing_pending = true;
  }
  ctx->have_stats = cf.flags & VDI_FLAG_PIXEL_STATS;
  ctx->last = vdi_counters{};
  ctx->last.bytes_sent = sent;
  ctx->last.bytes_received = recvd;
  ctx->last.kernel_launches = (uint32_t)launches;
  return VDI_OK;
}

vdi_status vdi_dense_to_full(vdi_ctx* ctx, const vdi_dense_view* in, vdi_full_view* out) {
  if (vdi_status s = check_ctx(ctx)) return s;
  const vdi_config& cf = ctx->cfg;
  if (!in || !out || !in->count || (in->total && (!in->depth || !in->rgba)))
    return fail(VDI_ERR_INVALID_ARG, "in/out is NULL");
  if (!out->count || !out->depth || !out->rgba || out->row_begin != 0 || out->row_end != cf.height)
    return fail(VDI_ERR_INVALID_ARG, "out must cover rows [0, H)");
  if ((reinterpret_cast<uintptr_t>(out->rgba) & 15) || (reinterpret_cast<uintptr_t>(out->depth) & 7) ||
      (reinterpret_cast<uintptr_t>(in->rgba) & 15) || (reinterpret_cast<uintptr_t>(in->depth) & 7))
    return fail(VDI_ERR_INVALID_ARG, "depth/rgba misaligned");
  cudaStream_t st = ctx->stream;
  const size_t P = (size_t)cf.width * cf.height;
  int launches = 0;
  CUDA_TRY(ctx, ctx->g_sum.grow(((size_t)scan_chunks((uint32_t)P) + 8) * 4));
  CUDA_TRY(ctx, ctx->g_base.grow((P / 32 + 8) * 4));
  CUDA_TRY(ctx, ctx->g_misc.grow(sizeof(DevCounters) + 256));
  DevCounters* gc = ctx->g_misc.as<DevCounters>();
  CUDA_TRY(ctx, cudaMemsetAsync(gc, 0, sizeof(DevCounters), st));
  MergeParams mi{};
  mi.n_src = 1;
  mi.k_out = (int)cf.k_in;  // k_in slots per list: every list passes through verbatim (m <= k_in)
  mi.max_iters = (int)cf.max_iters;
  mi.gamma_max = cf.gamma_max;
  mi.P = (uint32_t)P;
  mi.n_groups = (uint32_t)((P + 31) / 32);
  mi.g_begin = 0;
  mi.g_end = mi.n_groups;
  mi.src[0] = SrcDesc{in->count, reinterpret_cast<const float2*>(in->depth), reinterpret_cast<const float4*>(in->rgba)};
  CUDA_TRY(ctx, launch_scan(mi, ctx->g_sum.as<uint32_t>(), ctx->g_base.as<uint32_t>(), st, &launches));
  mi.group_base = ctx->g_base.as<uint32_t>();
  mi.out_count = out->count;
  mi.out_depth = reinterpret_cast<float2*>(out->depth);
  mi.out_rgba = reinterpret_cast<float4*>(out->rgba);
  for (int b = 0; b < VDI_N_BUCKETS; ++b) mi.wl[b] = reinterpret_cast<uint32_t*>(gc);  // never written: wl_cap = 0
  mi.wl_count = gc->wl_count[0];
  mi.wl_cap = 0;
  mi.scratch_used = &gc->scratch_used;
  mi.records_in = &gc->records_in;
  mi.fallback_groups = &gc->fallback_groups;
  mi.err = &gc->err;
  CUDA_TRY(ctx, launch_fast(mi, st, &launches));
  return VDI_OK;
}

vdi_status vdi_composite_fullrep(vdi_ctx* ctx, const vdi_full_view* local, const uint32_t* pe_ids, uint32_t n_local,
                                 vdi_full_view* so) {
  if (vdi_status s = check_ctx(ctx)) return s;
  const vdi_config& cf = ctx->cfg;
  const uint32_t G = cf.n_ranks, me = cf.rank, n = cf.n_pes, W = cf.width, K = cf.k_in;
  if (!so || !so->count || !so->depth || !so->rgba) return fail(VDI_ERR_INVALID_ARG, "strip_out is NULL");
  if (so->row_begin != ctx->row0 || so->row_end != ctx->row1)
    return fail(VDI_ERR_CAPACITY, "strip_out rows do not match this rank's strip");
  std::vector<int> slot(n, -1);
  uint32_t expect = 0;
  for (uint32_t s = 0; s < n; ++s)
    if (vdi_pe_home(n, G, s) == me) ++expect;
  if (n_local != expect) return fail(VDI_ERR_INVALID_ARG, "rank %u homes %u PEs, got %u", me, expect, n_local);
  if (n_local && (!local || !pe_ids)) return fail(VDI_ERR_INVALID_ARG, "local_pes / pe_ids is NULL");
  for (uint32_t l = 0; l < n_local; ++l) {
    const uint32_t pe = pe_ids[l];
    if (pe >= n || vdi_pe_home(n, G, pe) != me || slot[pe] >= 0)
      return fail(VDI_ERR_INVALID_ARG, "pe_id %u not homed on rank %u or duplicated", pe, me);
    const vdi_full_view& v = local[l];
    if (!v.count || !v.depth || !v.rgba || v.row_begin != 0 || v.row_end != cf.height)
      return fail(VDI_ERR_INVALID_ARG, "full sub-VDI of PE %u must cover rows [0, H)", pe);
    if ((reinterpret_cast<uintptr_t>(v.rgba) & 15) || (reinterpret_cast<uintptr_t>(v.depth) & 7))
      return fail(VDI_ERR_INVALID_ARG, "full sub-VDI of PE %u misaligned", pe);
    slot[pe] = (int)l;
  }
  cudaStream_t st = ctx->stream;
  const bool timing = cf.flags & VDI_FLAG_STAGE_TIMING;
  int launches = 0;
  uint64_t sent = 0, recvd = 0;
  const uint64_t Pg = ctx->P;
  if (timing) CUDA_TRY(ctx, cudaEventRecord(ctx->ev[0], st));
  // sources: this strip's rows of every PE's full representation (k_in slots per list)
  std::vector<const uint8_t*> sc(n);
  std::vector<const float*> sd(n), sr(n);
  for (uint32_t s = 0; s < n; ++s) {
    if (slot[s] < 0) continue;
    const vdi_full_view& v = local[slot[s]];
    const size_t o = (size_t)ctx->row0 * W;
    sc[s] = v.count + o;
    sd[s] = v.depth + o * K * 2;
    sr[s] = v.rgba + o * K * 4;
  }
  if (G > 1) {
    // fixed-size all-to-all of the full-representation slices (no size exchange)
    for (uint32_t s = 0; s < n; ++s) {
      if (slot[s] >= 0) continue;
      CUDA_TRY(ctx, ctx->rcount[s].grow(Pg));
      CUDA_TRY(ctx, ctx->rdepth[s].grow(Pg * K * 8));
      CUDA_TRY(ctx, ctx->rrgba[s].grow(Pg * K * 16));
      sc[s] = ctx->rcount[s].as<uint8_t>();
      sd[s] = ctx->rdepth[s].as<float>();
      sr[s] = ctx->rrgba[s].as<float>();
    }
    NCCL_TRY(ctx, ncclGroupStart());
    for (uint32_t g = 0; g < G; ++g) {
      if (g == me) continue;
      const uint32_t a = strip_row(cf.height, G, g), b = strip_row(cf.height, G, g + 1);
      const size_t P2 = (size_t)(b - a) * W, o = (size_t)a * W;
      for (uint32_t s = 0; s < n; ++s) {
        if (slot[s] < 0) continue;
        const vdi_full_view& v = local[slot[s]];
        NCCL_TRY(ctx, ncclSend(v.count + o, P2, ncclUint8, (int)g, ctx->comm, st));
        NCCL_TRY(ctx, ncclSend(v.depth + o * K * 2, P2 * K * 2, ncclFloat32, (int)g, ctx->comm, st));
        NCCL_TRY(ctx, ncclSend(v.rgba + o * K * 4, P2 * K * 4, ncclFloat32, (int)g, ctx->comm, st));
        sent += P2 * (1 + 24ull * K);
      }
      for (uint32_t s = 0; s < n; ++s) {
        if (vdi_pe_home(n, G, s) != g) continue;
        NCCL_TRY(ctx, ncclRecv(ctx->rcount[s].p, Pg, ncclUint8, (int)g, ctx->comm, st));
        NCCL_TRY(ctx, ncclRecv(ctx->rdepth[s].p, Pg * K * 2, ncclFloat32, (int)g, ctx->comm, st));
        NCCL_TRY(ctx, ncclRecv(ctx->rrgba[s].p, Pg * K * 4, ncclFloat32, (int)g, ctx->comm, st));
        recvd += Pg * (1 + 24ull * K);
      }
    }
    NCCL_TRY(ctx, ncclGroupEnd());
  }
  if (timing) CUDA_TRY(ctx, cudaEventRecord(ctx->ev[1], st));
  // compositing from the full representation: each source is compacted to
  // the dense layout (scan of its counts, packed copy of its records), then
  // merged like vdi_composite -- the same lists, so the same image
  const size_t ng = (Pg + 31) / 32;
  MergeParams ms{};
  ms.n_src = (int)n;
  ms.P = (uint32_t)Pg;
  ms.n_groups = (uint32_t)ng;
  for (uint32_t s = 0; s < n; ++s) ms.src[s].count = sc[s];
  CUDA_TRY(ctx, ctx->xsum.grow(((size_t)scan_chunks(ms.P) * n + 8) * 4));
  CUDA_TRY(ctx, ctx->xbase.grow((ng * n + 8) * 4));
  CUDA_TRY(ctx, ctx->xtot.grow(64));
  unsigned long long* dtot = ctx->xtot.as<unsigned long long>();
  if (Pg) {
    CUDA_TRY(ctx, launch_scan(ms, ctx->xsum.as<uint32_t>(), ctx->xbase.as<uint32_t>(), st, &launches));
    CUDA_TRY(ctx, launch_total(ms, ctx->xsum.as<uint32_t>(), dtot, st, &launches));
  } else {
    CUDA_TRY(ctx, cudaMemsetAsync(dtot, 0, 8, st));
  }
  while (ctx->xdense.size() < n) ctx->xdense.emplace_back(new DevBuf());
  MergeParams mp{};
  mp.n_src = (int)n;
  mp.k_out = (int)cf.k_out;
  mp.max_iters = (int)cf.max_iters;
  mp.gamma_max = cf.gamma_max;
  for (uint32_t s = 0; s < n; ++s) {
    DevBuf& xd = *ctx->xdense[s];
    CUDA_TRY(ctx, xd.grow(std::max<uint64_t>(Pg * K, 1) * 24));
    float4* dc = xd.as<float4>();
    float2* dd = reinterpret_cast<float2*>(dc + std::max<uint64_t>(Pg * K, 1));
    CUDA_TRY(ctx, launch_compact(sc[s], reinterpret_cast<const float2*>(sd[s]), reinterpret_cast<const float4*>(sr[s]),
                                 (uint32_t)Pg, (int)K, ctx->xbase.as<uint32_t>() + (size_t)s * ng, dd, dc, st,
                                 &launches));
    mp.src[s] = SrcDesc{sc[s], dd, dc};
  }
  unsigned long long S_here = 0;
  CUDA_TRY(ctx, cudaMemcpyAsync(&S_here, dtot, 8, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(ctx, cudaStreamSynchronize(st));
  if (vdi_status e = merge_lists(ctx, mp, Pg, S_here, so, timing, launches)) return e;
  if (timing) {
    CUDA_TRY(ctx, cudaEventRecord(ctx->ev[2], st));
    ctx->timing_pending = true;
  }
  ctx->have_stats = cf.flags & VDI_FLAG_PIXEL_STATS;
  ctx->last = vdi_counters{};
  ctx->last.bytes_sent = sent;
  ctx->last.bytes_received = recvd;
  ctx->last.kernel_launches = (uint32_t)launches;
  return VDI_OK;
}

vdi_status vdi_gather(vdi_ctx* ctx, const vdi_full_view* strip, vdi_full_view* image) {
  if (vdi_status s = check_ctx(ctx)) return s;
  const vdi_config& cf = ctx->cfg;
  const uint32_t G = cf.n_ranks, me = cf.rank, W = cf.width, k = cf.k_out;
  if (!strip || !strip->count || !strip->depth || !strip->rgba)
    return fail(VDI_ERR_INVALID_ARG, "strip is NULL");
  if (strip->row_begin != ctx->row0 || strip->row_end != ctx->row1)
    return fail(VDI_ERR_CAPACITY, "strip rows do not match this rank");
  const uint32_t R = cf.root;
  const bool root = me == R;
  if (root && (!image || !image->count || !image->depth || !image->rgba || image->row_begin != 0 ||
               image->row_end != cf.height))
    return fail(VDI_ERR_INVALID_ARG, "root image_out must cover rows [0, H)");
  cudaStream_t st = ctx->stream;
  const bool timing = cf.flags & VDI_FLAG_STAGE_TIMING;
  if (timing) CUDA_TRY(ctx, cudaEventRecord(ctx->gev[0], st));
  auto copy_strip = [&](uint32_t row0, const vdi_full_view* src) -> cudaError_t {
    const size_t P = (size_t)(src->row_end - src->row_begin) * W;
    const size_t o = (size_t)row0 * W;
    cudaError_t e = cudaSuccess;
    if (image->count + o != src->count)
      e = cudaMemcpyAsync(image->count + o, src->count, P, cudaMemcpyDeviceToDevice, st);
    if (e == cudaSuccess && image->depth + o * k * 2 != src->depth)
      e = cudaMemcpyAsync(image->depth + o * k * 2, src->depth, P * k * 8, cudaMemcpyDeviceToDevice, st);
    if (e == cudaSuccess && image->rgba + o * k * 4 != src->rgba)
      e = cudaMemcpyAsync(image->rgba + o * k * 4, src->rgba, P * k * 16, cudaMemcpyDeviceToDevice, st);
    return e;
  };
  if (G == 1) {
    CUDA_TRY(ctx, copy_strip(0, strip));
  } else if (!(cf.flags & VDI_FLAG_FULL_GATHER)) {
    // Dense gather: every rank compacts its composited lists
    // (counts + packed records) and the root re-inflates the
    // full representation with the pass-through kernel; the image
    // is bit-identical to the full-representation gather.
    int launches = 0;
    const size_t Pg = ctx->P, ng = (Pg + 31) / 32;
    CUDA_TRY(ctx, ctx->g_sum.grow(((size_t)scan_chunks((uint32_t)std::max<size_t>(Pg, (size_t)cf.width * cf.height)) + 8) * 4));
    CUDA_TRY(ctx, ctx->g_base.grow(((size_t)cf.width * cf.height / 32 + 8) * 4));
    CUDA_TRY(ctx, ctx->g_tot.grow((G + 2) * 8));
    unsigned long long* dtot = ctx->g_tot.as<unsigned long long>();
    MergeParams ms{};
    ms.n_src = 1;
    ms.P = (uint32_t)Pg;
    ms.n_groups = (uint32_t)ng;
    ms.src[0].count = strip->count;
    CUDA_TRY(ctx, launch_scan(ms, ctx->g_sum.as<uint32_t>(), ctx->g_base.as<uint32_t>(), st, &launches));
    CUDA_TRY(ctx, launch_total(ms, ctx->g_sum.as<uint32_t>(), dtot + G, st, &launches));
    NCCL_TRY(ctx, ncclAllGather(dtot + G, dtot, 1, ncclUint64, ctx->comm, st));
    std::vector<unsigned long long> tot(G);
    CUDA_TRY(ctx, cudaMemcpyAsync(tot.data(), dtot, G * 8, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(ctx, cudaStreamSynchronize(st));
    if (!root) {
      const uint64_t T = tot[me];
      CUDA_TRY(ctx, ctx->g_dense.grow(std::max<uint64_t>(T, 1) * 24));
      float4* dc4 = ctx->g_dense.as<float4>();
      float2* dd2 = reinterpret_cast<float2*>(dc4 + std::max<uint64_t>(T, 1));
      CUDA_TRY(ctx, launch_compact(strip->count, reinterpret_cast<const float2*>(strip->depth),
                                   reinterpret_cast<const float4*>(strip->rgba), (uint32_t)Pg, (int)k,
                                   ctx->g_base.as<uint32_t>(), dd2, dc4, st, &launches));
      NCCL_TRY(ctx, ncclGroupStart());
      NCCL_TRY(ctx, ncclSend(strip->count, Pg, ncclUint8, (int)R, ctx->comm, st));
      if (T) {
        NCCL_TRY(ctx, ncclSend(dd2, T * 2, ncclFloat32, (int)R, ctx->comm, st));
        NCCL_TRY(ctx, ncclSend(dc4, T * 4, ncclFloat32, (int)R, ctx->comm, st));
      }
      NCCL_TRY(ctx, ncclGroupEnd());
    } else {
      // receive every other strip: counts at their image rows (the root's own
      // rows stay unused), payloads concatenated in rank order
      const size_t Pimg = (size_t)cf.height * W;
      uint64_t Trem = 0;
      for (uint32_t g = 0; g < G; ++g)
        if (g != R) Trem += tot[g];
      CUDA_TRY(ctx, ctx->g_rcount.grow(Pimg + 64));
      CUDA_TRY(ctx, ctx->g_rpay.grow(std::max<uint64_t>(Trem, 1) * 24 + 64));
      float4* rc4 = ctx->g_rpay.as<float4>();
      float2* rd2 = reinterpret_cast<float2*>(rc4 + std::max<uint64_t>(Trem, 1));
      uint8_t* rcnt = ctx->g_rcount.as<uint8_t>();
      NCCL_TRY(ctx, ncclGroupStart());
      uint64_t off = 0, off_after = 0;
      for (uint32_t g = 0; g < G; ++g) {
        if (g == R) {
          off_after = off;
          continue;
        }
        const uint32_t a = strip_row(cf.height, G, g), b = strip_row(cf.height, G, g + 1);
        NCCL_TRY(ctx, ncclRecv(rcnt + (size_t)a * W, (size_t)(b - a) * W, ncclUint8, (int)g, ctx->comm, st));
        if (tot[g]) {
          NCCL_TRY(ctx, ncclRecv(rd2 + off, tot[g] * 2, ncclFloat32, (int)g, ctx->comm, st));
          NCCL_TRY(ctx, ncclRecv(rc4 + off, tot[g] * 4, ncclFloat32, (int)g, ctx->comm, st));
        }
        off += tot[g];
      }
      NCCL_TRY(ctx, ncclGroupEnd());
      CUDA_TRY(ctx, ctx->g_misc.grow(sizeof(DevCounters) + 256));
      DevCounters* gc = ctx->g_misc.as<DevCounters>();
      CUDA_TRY(ctx, cudaMemsetAsync(gc, 0, sizeof(DevCounters), st));
      // inflate the received rows (already depth-ordered, m <= k_out): one
      // pass-through launch per contiguous row range, [0, root rows) and
      // [after root rows, H)
      auto inflate = [&](uint32_t ra, uint32_t rb, uint64_t poff) -> vdi_status {
        const size_t Pr = (size_t)(rb - ra) * W;
        if (!Pr) return VDI_OK;
        MergeParams mi{};
        mi.n_src = 1;
        mi.k_out = (int)k;
        mi.max_iters = (int)cf.max_iters;
        mi.gamma_max = cf.gamma_max;
        mi.P = (uint32_t)Pr;
        mi.n_groups = (uint32_t)((Pr + 31) / 32);
        mi.g_begin = 0;
        mi.g_end = mi.n_groups;
        mi.src[0] = SrcDesc{rcnt + (size_t)ra * W, rd2 + poff, rc4 + poff};
        CUDA_TRY(ctx, launch_scan(mi, ctx->g_sum.as<uint32_t>(), ctx->g_base.as<uint32_t>(), st, &launches));
        mi.group_base = ctx->g_base.as<uint32_t>();
        mi.out_count = image->count + (size_t)ra * W;
        mi.out_depth = reinterpret_cast<float2*>(image->depth) + (size_t)ra * W * k;
        mi.out_rgba = reinterpret_cast<float4*>(image->rgba) + (size_t)ra * W * k;
        for (int b = 0; b < VDI_N_BUCKETS; ++b) mi.wl[b] = reinterpret_cast<uint32_t*>(gc);  // never written: wl_cap = 0
        mi.wl_count = gc->wl_count[0];
        mi.wl_cap = 0;
        mi.scratch_used = &gc->scratch_used;
        mi.records_in = &gc->records_in;
        mi.fallback_groups = &gc->fallback_groups;
        mi.err = &gc->err;
        CUDA_TRY(ctx, launch_fast(mi, st, &launches));
        return VDI_OK;
      };
      if (vdi_status s = inflate(0, ctx->row0, 0)) return s;
      if (vdi_status s = inflate(ctx->row1, cf.height, off_after)) return s;
      CUDA_TRY(ctx, copy_strip(ctx->row0, strip));
    }
    ctx->last.bytes_gather = 0;
    for (uint32_t g = 0; g < G; ++g)
      if (g != R)
        ctx->last.bytes_gather += (uint64_t)(strip_row(cf.height, G, g + 1) - strip_row(cf.height, G, g)) * W + 24 * tot[g];
    ctx->last.kernel_launches += (uint32_t)launches;
  } else {
    // MPI_Gather of the full-representation strips as grouped send/recv
    NCCL_TRY(ctx, ncclGroupStart());
    if (root) {
      for (uint32_t g = 0; g < G; ++g) {
        if (g == R) continue;
        const uint32_t r0 = strip_row(cf.height, G, g), r1 = strip_row(cf.height, G, g + 1);
        const size_t P = (size_t)(r1 - r0) * W, o = (size_t)r0 * W;
        NCCL_TRY(ctx, ncclRecv(image->count + o, P, ncclUint8, (int)g, ctx->comm, st));
        NCCL_TRY(ctx, ncclRecv(image->depth + o * k * 2, P * k * 2, ncclFloat32, (int)g, ctx->comm, st));
        NCCL_TRY(ctx, ncclRecv(image->rgba + o * k * 4, P * k * 4, ncclFloat32, (int)g, ctx->comm, st));
      }
    } else {
      const size_t P = ctx->P;
      NCCL_TRY(ctx, ncclSend(strip->count, P, ncclUint8, (int)R, ctx->comm, st));
      NCCL_TRY(ctx, ncclSend(strip->depth, P * k * 2, ncclFloat32, (int)R, ctx->comm, st));
      NCCL_TRY(ctx, ncclSend(strip->rgba, P * k * 4, ncclFloat32, (int)R, ctx->comm, st));
    }
    NCCL_TRY(ctx, ncclGroupEnd());
    if (root) CUDA_TRY(ctx, copy_strip(ctx->row0, strip));
    ctx->last.bytes_gather =
        (uint64_t)(cf.height - (strip_row(cf.height, G, R + 1) - strip_row(cf.height, G, R))) * W * (1 + 24ull * k);
  }
  if (timing) {
    CUDA_TRY(ctx, cudaEventRecord(ctx->gev[1], st));
    ctx->gather_timing_pending = true;
  }
  return VDI_OK;
}

// host sub-VDIs -> ctx-owned device copies (H2D on the ctx stream); dv gets device views
// H2D of the host sub-VDIs into input slot `set` (0: the single-frame
// entries; 0/1: the double-buffered frames pipeline), on stream st
static vdi_status upload_host_pes(vdi_ctx* ctx, const vdi_dense_view* local, uint32_t n_local,
                                  std::vector<vdi_dense_view>& dv, int set = 0, cudaStream_t st = nullptr) {
  const vdi_config& cf = ctx->cfg;
  if (n_local && !local) return fail(VDI_ERR_INVALID_ARG, "local_pes is NULL");
  if (n_local > cf.n_pes) return fail(VDI_ERR_INVALID_ARG, "too many local PEs");
  if (!st) st = ctx->stream;
  std::vector<DevBuf>& hcount = set ? ctx->hcount1 : ctx->hcount;
  std::vector<DevBuf>& hoffset = set ? ctx->hoffset1 : ctx->hoffset;
  std::vector<DevBuf>& hdepth = set ? ctx->hdepth1 : ctx->hdepth;
  std::vector<DevBuf>& hrgba = set ? ctx->hrgba1 : ctx->hrgba;
  const size_t P = (size_t)cf.width * cf.height;
  dv.assign(n_local, vdi_dense_view{});
  for (uint32_t l = 0; l < n_local; ++l) {
    const vdi_dense_view& v = local[l];
    if (!v.count || (v.total && (!v.depth || !v.rgba)) || (cf.n_ranks > 1 && !v.offset))
      return fail(VDI_ERR_INVALID_ARG, "host view %u has NULL arrays", l);
  }
  // Host arrays packed in one span (e.g. one pinned arena per frame): ONE
  // copy of the span instead of 3-4 per PE -- many mid-sized H2D copies run
  // the host link at ~80 % of one large copy (profiles/pipeline_probe.py).
  // Device views keep the host arrays' offsets inside the span (alignment
  // mod 256 preserved); a gap-ridden span falls back to per-array copies.
  {
    uintptr_t lo = UINTPTR_MAX, hi = 0;
    size_t sum = 0;
    bool aligned = true;
    auto add = [&](const void* p, size_t n, size_t al) {
      if (!n) return;
      const uintptr_t a = reinterpret_cast<uintptr_t>(p);
      lo = std::min(lo, a);
      hi = std::max(hi, a + n);
      sum += n;
      aligned &= (a % al) == 0;
    };
    for (uint32_t l = 0; l < n_local; ++l) {
      const vdi_dense_view& v = local[l];
      add(v.count, P, 1);
      add(v.depth, v.total * 8, 8);
      add(v.rgba, v.total * 16, 16);
      if (cf.n_ranks > 1) add(v.offset, (P + 1) * 4, 4);
    }
    if (sum && aligned) {
      lo &= ~(uintptr_t)255;
      const size_t span = hi - lo;
      if (span <= sum + std::max<size_t>(sum / 16, (size_t)1 << 20)) {
        DevBuf& ar = ctx->harena[set];
        CUDA_TRY(ctx, ar.grow(span));
        CUDA_TRY(ctx, cudaMemcpyAsync(ar.p, reinterpret_cast<const void*>(lo), span, cudaMemcpyHostToDevice, st));
        uint8_t* base = ar.as<uint8_t>();
        auto dev = [&](const void* p) { return base + (reinterpret_cast<uintptr_t>(p) - lo); };
        for (uint32_t l = 0; l < n_local; ++l) {
          const vdi_dense_view& v = local[l];
          dv[l] = v;
          dv[l].count = dev(v.count);
          dv[l].depth = reinterpret_cast<float*>(v.total ? dev(v.depth) : base);  // base: never read
          dv[l].rgba = reinterpret_cast<float*>(v.total ? dev(v.rgba) : base);
          dv[l].offset = cf.n_ranks > 1 ? reinterpret_cast<uint32_t*>(dev(v.offset)) : nullptr;
        }
        return VDI_OK;
      }
    }
  }
  for (uint32_t l = 0; l < n_local; ++l) {
    const vdi_dense_view& v = local[l];
    CUDA_TRY(ctx, hcount[l].grow(P));
    CUDA_TRY(ctx, hdepth[l].grow(std::max<uint64_t>(v.total, 1) * 8));
    CUDA_TRY(ctx, hrgba[l].grow(std::max<uint64_t>(v.total, 1) * 16));
    CUDA_TRY(ctx, cudaMemcpyAsync(hcount[l].p, v.count, P, cudaMemcpyHostToDevice, st));
    if (v.total) {
      CUDA_TRY(ctx, cudaMemcpyAsync(hdepth[l].p, v.depth, v.total * 8, cudaMemcpyHostToDevice, st));
      CUDA_TRY(ctx, cudaMemcpyAsync(hrgba[l].p, v.rgba, v.total * 16, cudaMemcpyHostToDevice, st));
    }
    dv[l] = v;
    dv[l].count = hcount[l].as<uint8_t>();
    dv[l].depth = hdepth[l].as<float>();
    dv[l].rgba = hrgba[l].as<float>();
    if (cf.n_ranks > 1) {
      CUDA_TRY(ctx, hoffset[l].grow((P + 1) * 4));
      CUDA_TRY(ctx, cudaMemcpyAsync(hoffset[l].p, v.offset, (P + 1) * 4, cudaMemcpyHostToDevice, st));
      dv[l].offset = hoffset[l].as<uint32_t>();
    } else {
      dv[l].offset = nullptr;
    }
  }
  return VDI_OK;
}

// n_ranks > 1: peers pull their strip slices out of this rank's staging
// buffers during their own compositing; a one-byte allreduce on the stream
// after the merge (every rank's pulls precede its merge) keeps the next host
// call from overwriting a slot a peer is still reading
static vdi_status peer_quiesce(vdi_ctx* ctx, cudaStream_t st) {
  if (ctx->cfg.n_ranks <= 1) return VDI_OK;
  CUDA_TRY(ctx, ctx->bounds.grow(16));
  NCCL_TRY(ctx, ncclAllReduce(ctx->bounds.p, ctx->bounds.p, 1, ncclUint8, ncclSum, ctx->comm, st));
  return VDI_OK;
}

vdi_status vdi_composite_host(vdi_ctx* ctx, const vdi_dense_view* local, uint32_t n_local, vdi_full_view* so) {
  if (vdi_status s = check_ctx(ctx)) return s;
  const vdi_config& cf = ctx->cfg;
  if (!so || !so->count || !so->depth || !so->rgba) return fail(VDI_ERR_INVALID_ARG, "strip_out is NULL");
  cudaStream_t st = ctx->stream;
  std::vector<vdi_dense_view> dv;
  if (vdi_status s = upload_host_pes(ctx, local, n_local, dv)) return s;
  const size_t Ps = ctx->P, k = cf.k_out;
  CUDA_TRY(ctx, ctx->hstrip_count.grow(Ps));
  CUDA_TRY(ctx, ctx->hstrip_depth.grow(Ps * k * 8));
  CUDA_TRY(ctx, ctx->hstrip_rgba.grow(Ps * k * 16));
  vdi_full_view ds{ctx->row0, ctx->row1, ctx->hstrip_count.as<uint8_t>(), ctx->hstrip_depth.as<float>(),
                   ctx->hstrip_rgba.as<float>()};
  if (vdi_status s = vdi_composite(ctx, dv.data(), n_local, &ds)) return s;
  if (vdi_status s = peer_quiesce(ctx, st)) return s;
  CUDA_TRY(ctx, cudaMemcpyAsync(so->count, ds.count, Ps, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(ctx, cudaMemcpyAsync(so->depth, ds.depth, Ps * k * 8, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(ctx, cudaMemcpyAsync(so->rgba, ds.rgba, Ps * k * 16, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(ctx, cudaStreamSynchronize(st));
  return VDI_OK;
}

vdi_status vdi_composite_host_dense(vdi_ctx* ctx, const vdi_dense_view* local, uint32_t n_local,
                                    vdi_dense_strip* out) {
  if (vdi_status s = check_ctx(ctx)) return s;
  const vdi_config& cf = ctx->cfg;
  if (!out || !out->count || (out->capacity && (!out->depth || !out->rgba)))
    return fail(VDI_ERR_INVALID_ARG, "out is NULL");
  if (out->row_begin != ctx->row0 || out->row_end != ctx->row1)
    return fail(VDI_ERR_CAPACITY, "out rows do not match this rank's strip");
  cudaStream_t st = ctx->stream;
  std::vector<vdi_dense_view> dv;
  if (vdi_status s = upload_host_pes(ctx, local, n_local, dv)) return s;
  const size_t Ps = ctx->P, k = cf.k_out;
  CUDA_TRY(ctx, ctx->hstrip_count.grow(Ps));
  CUDA_TRY(ctx, ctx->hstrip_depth.grow(Ps * k * 8));
  CUDA_TRY(ctx, ctx->hstrip_rgba.grow(Ps * k * 16));
  vdi_full_view ds{ctx->row0, ctx->row1, ctx->hstrip_count.as<uint8_t>(), ctx->hstrip_depth.as<float>(),
                   ctx->hstrip_rgba.as<float>()};
  if (vdi_status s = vdi_composite(ctx, dv.data(), n_local, &ds)) return s;
  if (vdi_status s = peer_quiesce(ctx, st)) return s;
  // the composited strip in the dense representation:
  // scan of its counts, packed copy of its records, then only those bytes
  // cross PCIe
  int launches = 0;
  const size_t ng = (Ps + 31) / 32;
  CUDA_TRY(ctx, ctx->xsum.grow(((size_t)scan_chunks((uint32_t)std::max<size_t>(Ps, 1)) + 8) * 4));
  CUDA_TRY(ctx, ctx->xbase.grow((ng + 8) * 4));
  CUDA_TRY(ctx, ctx->xtot.grow(64));
  unsigned long long* dtot = ctx->xtot.as<unsigned long long>();
  MergeParams ms{};
  ms.n_src = 1;
  ms.P = (uint32_t)Ps;
  ms.n_groups = (uint32_t)ng;
  ms.src[0].count = ds.count;
  unsigned long long T = 0;
  if (Ps) {
    CUDA_TRY(ctx, launch_scan(ms, ctx->xsum.as<uint32_t>(), ctx->xbase.as<uint32_t>(), st, &launches));
    CUDA_TRY(ctx, launch_total(ms, ctx->xsum.as<uint32_t>(), dtot, st, &launches));
    CUDA_TRY(ctx, cudaMemcpyAsync(&T, dtot, 8, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(ctx, cudaStreamSynchronize(st));
  }
  out->total = T;
  if (T > out->capacity) return fail(VDI_ERR_CAPACITY, "dense strip needs %llu supersegments, capacity %llu", T,
                                     (unsigned long long)out->capacity);
  CUDA_TRY(ctx, ctx->g_dense.grow(std::max<uint64_t>(T, 1) * 24));
  float4* dc4 = ctx->g_dense.as<float4>();
  float2* dd2 = reinterpret_cast<float2*>(dc4 + std::max<uint64_t>(T, 1));
  if (Ps)
    CUDA_TRY(ctx, launch_compact(ds.count, reinterpret_cast<const float2*>(ds.depth),
                                 reinterpret_cast<const float4*>(ds.rgba), (uint32_t)Ps, (int)k,
                                 ctx->xbase.as<uint32_t>(), dd2, dc4, st, &launches));
  CUDA_TRY(ctx, cudaMemcpyAsync(out->count, ds.count, Ps, cudaMemcpyDeviceToHost, st));
  if (T) {
    CUDA_TRY(ctx, cudaMemcpyAsync(out->depth, dd2, T * 8, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(ctx, cudaMemcpyAsync(out->rgba, dc4, T * 16, cudaMemcpyDeviceToHost, st));
  }
  CUDA_TRY(ctx, cudaStreamSynchronize(st));
  ctx->last.kernel_launches += (uint32_t)launches;
  return VDI_OK;
}

#ifndef VDI_E2E_MAPPED
#define VDI_E2E_MAPPED 1  // frame totals stored by the kernel into mapped host memory (else an 8-byte D2H)
#endif
// Pipelined vdi_composite_host_dense over independent frames: frame f's H2D
// (stream pin_st, input slot f&1) overlaps frame f-1's compositing (ctx
// stream) and frame f-2's D2H (stream pout_st, output slot f&1).  Each frame
// is exactly one vdi_composite + dense compaction, as in the single call.
vdi_status vdi_composite_host_dense_frames(vdi_ctx* ctx, uint32_t F, const vdi_dense_view* local, uint32_t n_local,
                                           vdi_dense_strip* outs) {
  if (vdi_status s = check_ctx(ctx)) return s;
  const vdi_config& cf = ctx->cfg;
  if (F == 0) return VDI_OK;
  if (!outs || (n_local && !local)) return fail(VDI_ERR_INVALID_ARG, "outs / local_pes is NULL");
  for (uint32_t f = 0; f < F; ++f) {
    const vdi_dense_strip& o = outs[f];
    if (!o.count || (o.capacity && (!o.depth || !o.rgba))) return fail(VDI_ERR_INVALID_ARG, "outs[%u] is NULL", f);
    if (o.row_begin != ctx->row0 || o.row_end != ctx->row1)
      return fail(VDI_ERR_CAPACITY, "outs[%u] rows do not match this rank's strip", f);
  }
  cudaStream_t st = ctx->stream;
  if (!ctx->pin_st) {
    CUDA_TRY(ctx, cudaStreamCreateWithFlags(&ctx->pin_st, cudaStreamNonBlocking));
    CUDA_TRY(ctx, cudaStreamCreateWithFlags(&ctx->pout_st, cudaStreamNonBlocking));
    for (cudaEvent_t* a : {ctx->pev_in, ctx->pev_used, ctx->pev_tot, ctx->pev_comp, ctx->pev_out})
      for (int i = 0; i < 2; ++i) CUDA_TRY(ctx, cudaEventCreateWithFlags(&a[i], cudaEventDisableTiming));
    CUDA_TRY(ctx, cudaHostAlloc(reinterpret_cast<void**>(&ctx->ptot), 2 * sizeof(unsigned long long),
                                cudaHostAllocMapped));
    CUDA_TRY(ctx, cudaHostGetDevicePointer(reinterpret_cast<void**>(&ctx->ptot_dev), ctx->ptot, 0));
  }
  const size_t Ps = ctx->P, k = cf.k_out, Tmax = std::max<size_t>(Ps * k, 1);  // a strip holds <= Ps*k
  CUDA_TRY(ctx, ctx->hstrip_count.grow(Ps));
  CUDA_TRY(ctx, ctx->hstrip_depth.grow(Ps * k * 8));
  CUDA_TRY(ctx, ctx->hstrip_rgba.grow(Ps * k * 16));
  const size_t ng = (Ps + 31) / 32;
  CUDA_TRY(ctx, ctx->xsum.grow(((size_t)scan_chunks((uint32_t)std::max<size_t>(Ps, 1)) + 8) * 4));
  CUDA_TRY(ctx, ctx->xbase.grow((ng + 8) * 4));
  CUDA_TRY(ctx, ctx->xtot.grow(64));
  for (int i = 0; i < 2; ++i) {
    CUDA_TRY(ctx, ctx->pcount[i].grow(std::max<size_t>(Ps, 1)));
    CUDA_TRY(ctx, ctx->pdense[i].grow(Tmax * 24));
  }
  // the strip's counts go straight to the output slot (read by the D2H);
  // its records to the shared full-representation scratch (read by the compaction)
  vdi_full_view ds{ctx->row0, ctx->row1, nullptr, ctx->hstrip_depth.as<float>(), ctx->hstrip_rgba.as<float>()};
  std::vector<vdi_dense_view> dv[2];
  int launches = 0;
  // H2D of frame f into slot f&1, once the compositing of frame f-2 has read
  // it.  n_ranks > 1: peers pull their strip slices out of this rank's slot
  // during THEIR compositing of f-2, which has ended once this rank's
  // compositing of f-1 is past its size-exchange collective -- so wait for f-1
  auto h2d = [&](uint32_t f) -> vdi_status {
    const int sl = f & 1;
    CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->pin_st, ctx->pev_used[cf.n_ranks > 1 ? sl ^ 1 : sl], 0));
    if (vdi_status s = upload_host_pes(ctx, local + (size_t)f * n_local, n_local, dv[sl], sl, ctx->pin_st)) return s;
    CUDA_TRY(ctx, cudaEventRecord(ctx->pev_in[sl], ctx->pin_st));
    return VDI_OK;
  };
  // composite + dense compaction of frame f into output slot f&1
  auto compute = [&](uint32_t f) -> vdi_status {
    const int sl = f & 1;
    CUDA_TRY(ctx, cudaStreamWaitEvent(st, ctx->pev_out[sl], 0));  // frame f-2's D2H has read the slot
    CUDA_TRY(ctx, cudaStreamWaitEvent(st, ctx->pev_in[sl], 0));
    ds.count = ctx->pcount[sl].as<uint8_t>();
    if (vdi_status s = vdi_composite(ctx, dv[sl].data(), n_local, &ds)) return s;
    CUDA_TRY(ctx, cudaEventRecord(ctx->pev_used[sl], st));
    MergeParams ms{};
    ms.n_src = 1;
    ms.P = (uint32_t)Ps;
    ms.n_groups = (uint32_t)ng;
    ms.src[0].count = ds.count;
    if (Ps) {  // the total is stored by the kernel into mapped host memory (no copy-engine hop)
      CUDA_TRY(ctx, launch_scan(ms, ctx->xsum.as<uint32_t>(), ctx->xbase.as<uint32_t>(), st, &launches));
#if VDI_E2E_MAPPED
      CUDA_TRY(ctx, launch_total(ms, ctx->xsum.as<uint32_t>(), ctx->ptot_dev + sl, st, &launches));
#else
      CUDA_TRY(ctx, launch_total(ms, ctx->xsum.as<uint32_t>(), ctx->xtot.as<unsigned long long>(), st, &launches));
      CUDA_TRY(ctx, cudaMemcpyAsync(ctx->ptot + sl, ctx->xtot.p, 8, cudaMemcpyDeviceToHost, st));
#endif
    } else {
      ctx->ptot[sl] = 0;
    }
    CUDA_TRY(ctx, cudaEventRecord(ctx->pev_tot[sl], st));
    float4* dc4 = ctx->pdense[sl].as<float4>();
    float2* dd2 = reinterpret_cast<float2*>(dc4 + Tmax);
    if (Ps) {
      CUDA_TRY(ctx, launch_compact(ds.count, reinterpret_cast<const float2*>(ds.depth),
                                   reinterpret_cast<const float4*>(ds.rgba), (uint32_t)Ps, (int)k,
                                   ctx->xbase.as<uint32_t>(), dd2, dc4, st, &launches));
    }
    CUDA_TRY(ctx, cudaEventRecord(ctx->pev_comp[sl], st));
    return VDI_OK;
  };
  // D2H of frame f once its total is known on the host
  vdi_status first_err = VDI_OK;
  auto d2h = [&](uint32_t f) -> vdi_status {
    const int sl = f & 1;
    CUDA_TRY(ctx, cudaEventSynchronize(ctx->pev_tot[sl]));
    const unsigned long long T = *static_cast<volatile unsigned long long*>(ctx->ptot + sl);
    vdi_dense_strip& o = outs[f];
    o.total = T;
    CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->pout_st, ctx->pev_comp[sl], 0));
    if (T > o.capacity) {
      if (first_err == VDI_OK)
        first_err = fail(VDI_ERR_CAPACITY, "frame %u: dense strip needs %llu supersegments, capacity %llu", f, T,
                         (unsigned long long)o.capacity);
    } else {
      const float4* dc4 = ctx->pdense[sl].as<float4>();
      const float2* dd2 = reinterpret_cast<const float2*>(dc4 + Tmax);
      CUDA_TRY(ctx, cudaMemcpyAsync(o.count, ctx->pcount[sl].p, Ps, cudaMemcpyDeviceToHost, ctx->pout_st));
      if (T) {
        CUDA_TRY(ctx, cudaMemcpyAsync(o.depth, dd2, T * 8, cudaMemcpyDeviceToHost, ctx->pout_st));
        CUDA_TRY(ctx, cudaMemcpyAsync(o.rgba, dc4, T * 16, cudaMemcpyDeviceToHost, ctx->pout_st));
      }
    }
    CUDA_TRY(ctx, cudaEventRecord(ctx->pev_out[sl], ctx->pout_st));
    return VDI_OK;
  };
  // order: H2D(f+1) is queued before the host waits for frame f's total, and
  // compute(f+1) after D2H(f) is queued (vdi_composite may wait on the host
  // for the size exchange when n_ranks > 1)
  if (vdi_status s = h2d(0)) return s;
  if (vdi_status s = compute(0)) return s;
  for (uint32_t f = 0; f < F; ++f) {
    if (f + 1 < F)
      if (vdi_status s = h2d(f + 1)) return s;
    if (vdi_status s = d2h(f)) return s;
    if (f + 1 < F)
      if (vdi_status s = compute(f + 1)) return s;
  }
  if (vdi_status s = peer_quiesce(ctx, st)) return s;  // the last frames' slots (next call)
  CUDA_TRY(ctx, cudaStreamSynchronize(ctx->pout_st));
  CUDA_TRY(ctx, cudaStreamSynchronize(ctx->pin_st));
  CUDA_TRY(ctx, cudaStreamSynchronize(st));
  ctx->last.kernel_launches += (uint32_t)launches;
  return first_err;
}

vdi_status vdi_pixel_stats(vdi_ctx* ctx, float* gamma, uint16_t* m) {
  if (vdi_status s = check_ctx(ctx)) return s;
  if (!ctx->have_stats) return fail(VDI_ERR_STATE, "VDI_FLAG_PIXEL_STATS was not set for the last composite");
  if (gamma)
    CUDA_TRY(ctx, cudaMemcpyAsync(gamma, ctx->stat_gamma.p, ctx->mP * 4, cudaMemcpyDeviceToDevice, ctx->stream));
  if (m) CUDA_TRY(ctx, cudaMemcpyAsync(m, ctx->stat_m.p, ctx->mP * 2, cudaMemcpyDeviceToDevice, ctx->stream));
  return VDI_OK;
}

vdi_status vdi_get_counters(vdi_ctx* ctx, vdi_counters* out) {
  if (vdi_status s = check_ctx(ctx)) return s;
  if (!out) return fail(VDI_ERR_INVALID_ARG, "out is NULL");
  DevCounters h{};
  if (ctx->dcnt.p) {
    CUDA_TRY(ctx, cudaMemcpyAsync(&h, ctx->dcnt.p, sizeof h, cudaMemcpyDeviceToHost, ctx->stream));
    CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  }
  if (h.err & 1) return fail(VDI_ERR_INTERNAL, "merge work list / scratch / search pool overflow");
  ctx->last.records_in = h.records_in;
  ctx->last.records_search = h.records_search;
  ctx->last.searched_lists = 0;
  ctx->last.general_lists = 0;
  for (int b = 0; b < 4; ++b) ctx->last.bucket_lists[b] = 0;
  for (int c = 0; c < ctx->n_chunks; ++c) {
    ctx->last.general_lists += h.wl_count[c][VDI_BUCKET_GENERAL];
    for (int b = 0; b < VDI_N_BUCKETS; ++b) {
      ctx->last.searched_lists += h.wl_count[c][b];
      if (b < 4) ctx->last.bucket_lists[b] += h.wl_count[c][b];
    }
  }
  ctx->last.fallback_groups = h.fallback_groups;
  if (ctx->timing_pending) {
    CUDA_TRY(ctx, cudaEventElapsedTime(&ctx->last.ms_exchange, ctx->ev[0], ctx->ev[1]));
    CUDA_TRY(ctx, cudaEventElapsedTime(&ctx->last.ms_merge, ctx->ev[1], ctx->ev[2]));
    if (ctx->mP) {
      CUDA_TRY(ctx, cudaEventElapsedTime(&ctx->last.ms_scan, ctx->ev[1], ctx->ev[3]));
      CUDA_TRY(ctx, cudaEventElapsedTime(&ctx->last.ms_fast, ctx->ev[3], ctx->ev[4]));
      CUDA_TRY(ctx, cudaEventElapsedTime(&ctx->last.ms_search, ctx->ev[4], ctx->ev[5]));
    }
    ctx->timing_pending = false;
  }
  if (ctx->frames_timing_pending) {
    CUDA_TRY(ctx, cudaEventElapsedTime(&ctx->last.ms_sizes, ctx->ev[0], ctx->fev[0]));
    CUDA_TRY(ctx, cudaEventElapsedTime(&ctx->last.ms_pull, ctx->fev[0], ctx->fev[1]));
    ctx->frames_timing_pending = false;
  }
  if (ctx->gather_timing_pending) {
    CUDA_TRY(ctx, cudaEventElapsedTime(&ctx->last.ms_gather, ctx->gev[0], ctx->gev[1]));
    ctx->gather_timing_pending = false;
  }
  *out = ctx->last;
  return VDI_OK;
}

}  // extern "C"
