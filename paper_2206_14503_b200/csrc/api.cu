// api.cu — libvdi C ABI (include/vdi.h): context, validation, the Phase-2
// orchestration (strip partition, device-driven exchange, receive-side scan,
// merge) and the gather to the root.
//
// Multi-GPU (n_ranks > 1): every context owns one window
// allocation -- flag words, the receive slots of the strip exchange and the
// root-side gather buffers, each double-buffered -- whose CUDA IPC handle is
// exchanged ONCE at init (NCCL all-gather; VDI_FLAG_LOOPBACK: an in-process
// registry of contexts on one device).  After that no call synchronises the
// host: senders push slices into their peers' windows (comm.cu) and the
// receivers learn that the data landed from block-counted flag words.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <condition_variable>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "comm.h"
#include "internal.h"
#include "render.h"

namespace {
// NVTX range over one public call (profiler timelines; ncu --nvtx filters by it)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};
}  // namespace
#define VDI_NVTX(name) NvtxRange vdi_nvtx_range_(name)

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

// Grow-only device buffer.  A grown buffer's old allocation is NOT freed on
// the spot (cudaFree waits for the whole device, which may be spinning on a
// flag that another context of a loopback group only sets later): it is kept
// until the buffer dies (the context is destroyed).
struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  std::vector<void*> old;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), bytes(o.bytes), old(std::move(o.old)) {
    o.p = nullptr;
    o.bytes = 0;
  }
  ~DevBuf() {
    if (p) cudaFree(p);
    for (void* q : old) cudaFree(q);
  }
  cudaError_t grow(size_t need) {
    if (need <= bytes) return cudaSuccess;
    size_t want = std::max(need, (size_t)256);
    if (p) want = std::max(want, bytes + bytes / 4);  // headroom: regrowth is rare
    void* q = nullptr;
    cudaError_t e = cudaMalloc(&q, want);
    if (e != cudaSuccess) return e;
    if (p) old.push_back(p);
    p = q;
    bytes = want;
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

// device-side counters of one merge
struct DevCounters {
  uint32_t wl_count[VDI_N_BUCKETS];
  uint32_t search_ticket[VDI_N_BUCKETS];
  int err;
  uint32_t pool_next;
  unsigned long long records_in;
  unsigned long long fallback_groups;
  unsigned long long records_search;
  unsigned long long long_used;
  unsigned long long sweep_steps;
};

// VDI_TRACE=1 (debug): timing events around the merge kernels of
// vdi_composite_frames, printed to stderr at the end of the call (one sync)
struct TraceEv {
  const char* what;
  int frame;
  cudaEvent_t ev;
};
static std::vector<TraceEv>& trace_log() {
  static std::vector<TraceEv> v;
  return v;
}
static bool trace_on() {
  static const bool on = getenv("VDI_TRACE") != nullptr;
  return on;
}
static int g_trace_frame = -1;
static int g_trace_rank = 0;
static void trace(const char* what, cudaStream_t st) {
  if (!trace_on() || g_trace_frame < 0) return;
  static std::vector<cudaEvent_t> pool;
  static size_t used = 0;
  auto& log = trace_log();
  if (log.empty()) used = 0;
  if (used == pool.size()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    pool.push_back(e);
  }
  cudaEvent_t e = pool[used++];
  cudaEventRecord(e, st);
  log.push_back(TraceEv{what, g_trace_frame, e});
}
static void trace_dump(cudaStream_t st) {
  auto& log = trace_log();
  if (!trace_on() || log.empty()) return;
  cudaStreamSynchronize(st);
  cudaDeviceSynchronize();
  for (auto& t : log) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, log[0].ev, t.ev);
    fprintf(stderr, "trace r%d f%d %-14s %9.4f\n", g_trace_rank, t.frame, t.what, ms);
  }
  log.clear();
}

inline size_t al256(size_t b) { return (b + 255) & ~(size_t)255; }
constexpr size_t kShortSlotBytes = 40 * 32 * 16 + 40 * 32 * 8 + 64 * 4;  // one short-search pool slot
uint32_t strip_row(uint32_t H, uint32_t G, uint32_t g) { return (uint32_t)((uint64_t)g * H / G); }

// flag words of a window: [kind][rank]
enum { XREADY = 0, XFREE = 1, GREADY = 2, GFREE = 3 };
constexpr size_t kFlagBytes = 4 * VDI_MAX_RANKS * 4;

// Window layout of rank r, computable by every rank from the config:
//   flags | xwin: 2 parities x n_remote(r) receive slots | gwin: 2 parities x gather buffer
struct Layout {
  uint32_t W, H, G, n, k_in, k_out;
  uint32_t rows(uint32_t r) const { return strip_row(H, G, r + 1) - strip_row(H, G, r); }
  uint32_t row0(uint32_t r) const { return strip_row(H, G, r); }
  uint32_t home(uint32_t s) const { return (uint32_t)((uint64_t)s * G / n); }
  uint32_t n_local(uint32_t r) const {
    uint32_t c = 0;
    for (uint32_t s = 0; s < n; ++s) c += home(s) == r;
    return c;
  }
  // receive slot of PE s at rank r: header | count [P_r] | group bases [P_r/32 + 1] |
  // depth [P_r k_in] | rgba [P_r k_in]
  size_t slot_bytes(uint32_t r) const {
    const size_t P = (size_t)rows(r) * W;
    return 256 + al256(P) + al256(((P + 31) / 32 + 1) * 4) + al256(P * k_in * 8) + al256(P * k_in * 16);
  }
  uint32_t slot_index(uint32_t s, uint32_t r) const {  // PEs homed elsewhere, in PE order
    uint32_t j = 0;
    for (uint32_t t = 0; t < s; ++t) j += home(t) != r;
    return j;
  }
  size_t xwin_bytes(uint32_t r) const { return 2 * (size_t)(n - n_local(r)) * slot_bytes(r); }
  size_t x_off(uint32_t r, uint32_t q, uint32_t s) const {
    return kFlagBytes + ((size_t)q * (n - n_local(r)) + slot_index(s, r)) * slot_bytes(r);
  }
  // gather buffer: count [P] | gbase [P/32 + G + 64] | hdr [G] u64 | depth [P k_out] | rgba [P k_out]
  size_t img() const { return (size_t)W * H; }
  size_t gbase_words() const { return img() / 32 + G * 2 + 64; }
  size_t g_count_off() const { return 0; }
  size_t g_gbase_off() const { return al256(img()); }
  size_t g_hdr_off() const { return g_gbase_off() + al256(gbase_words() * 4); }
  size_t g_depth_off() const { return g_hdr_off() + al256((size_t)G * 8); }
  size_t g_rgba_off() const { return g_depth_off() + al256(img() * k_out * 8); }
  size_t gpar_bytes() const { return g_rgba_off() + al256(img() * k_out * 16); }
  size_t g_off(uint32_t r, uint32_t q) const { return kFlagBytes + xwin_bytes(r) + (size_t)q * gpar_bytes(); }
  size_t win_bytes(uint32_t r) const { return g_off(r, 2); }
  // strip starts on 32-list boundaries: the root inflates contiguous rank ranges in one launch
  bool aligned() const {
    for (uint32_t r = 0; r < G; ++r)
      if (((size_t)row0(r) * W) % 32) return false;
    return true;
  }
  // index of rank r's group bases in a gather buffer
  size_t gbase_index(uint32_t r) const {
    if (aligned()) return (size_t)row0(r) * W / 32;
    size_t o = 0;
    for (uint32_t t = 0; t < r; ++t) o += ((size_t)rows(t) * W + 31) / 32 + 1;
    return o;
  }
};

// the arrays of a receive slot of P lists (see Layout::slot_bytes)
struct Slot {
  unsigned long long* hdr;
  uint8_t* count;
  uint32_t* gbase;
  float2* depth;
  float4* rgba;
};
inline Slot slot_at(char* p, size_t P, uint32_t k_in) {
  Slot sl;
  sl.hdr = reinterpret_cast<unsigned long long*>(p);
  p += 256;
  sl.count = reinterpret_cast<uint8_t*>(p);
  p += al256(P);
  sl.gbase = reinterpret_cast<uint32_t*>(p);
  p += al256(((P + 31) / 32 + 1) * 4);
  sl.depth = reinterpret_cast<float2*>(p);
  p += al256(P * k_in * 8);
  sl.rgba = reinterpret_cast<float4*>(p);
  return sl;
}

// VDI_FLAG_LOOPBACK: contexts of one process that form one group, keyed by
// the 128-byte id; members publish their window base pointers here.  The
// ranks of a loopback group are threads of one process sharing a device, and
// kernels that spin on each other must not share a device (nothing guarantees
// they run concurrently): a loopback rank instead waits on the HOST until the
// producer has enqueued its side (an event per (kind, producer, consumer,
// sequence)), makes its stream wait on that event, and then only CHECKS the
// flag words the device path would have spun on (a check kernel counts
// shortfalls; vdi_get_counters reports them).
struct LoopGroup {
  std::vector<char*> base;
  std::mutex mu;
  std::condition_variable cv;
  std::map<std::tuple<int, uint32_t, uint32_t, uint32_t>, cudaEvent_t> posted;
  ~LoopGroup() {
    for (auto& kv : posted) cudaEventDestroy(kv.second);
  }
};
std::mutex g_loop_mu;
std::map<std::string, std::shared_ptr<LoopGroup>> g_loop;

}  // namespace

struct vdi_ctx {
  vdi_config cfg{};
  Layout lay{};
  cudaStream_t stream = nullptr;
  int device = 0;
  ncclComm_t comm = nullptr;
  bool poisoned = false;
  uint32_t row0 = 0, row1 = 0;
  uint64_t P = 0;   // lists in this rank's strip
  uint64_t mP = 0;  // lists of the last merge
  // window and peers (n_ranks > 1)
  DevBuf win;
  std::vector<char*> peer;  // window base of every rank (own included)
  bool peers_ready = false;
  std::string loop_key;
  std::shared_ptr<LoopGroup> grp;  // VDI_FLAG_LOOPBACK
  std::vector<void*> ipc_opened;
  uint32_t xcalls = 0;               // exchange calls so far (epoch)
  std::vector<uint32_t> gcalls_to;   // gathers to each root so far
  DevBuf bnd, srcbase, segbuf, ccnt, gsum, gbase_loc;
  DevBuf gsum_x, gbase_x;                // exchange: scan of the local PEs' counts (2 parities)
  cudaEvent_t xev_bounds[2] = {}, xev_merged[2] = {};
  cudaStream_t xst = nullptr;            // vdi_composite_frames: the push stream
  cudaStream_t xpst = nullptr;           // push stream of the current call (null: the ctx stream)
  int xpar = 0;                          // parity of the exchange buffers of the current call
  // merge scratch; the work lists, counters and search pools come in two
  // parities (frames in flight: frame f's search overlaps frame f+1's pass-through)
  DevBuf group_sum, group_base, stat_gamma, stat_m, stat_margin;
  struct MScratch {
    DevBuf wl, slots, dcnt, scratch, srch, lpool;
  } ms[2];
  int mpar = 0;                   // parity of the current merge
  int last_mpar = 0;              // parity of the last merge (counters)
  cudaStream_t msst = nullptr;    // search stream of the current merge (null: the ctx stream)
  uint32_t* long_hint = nullptr;      // pinned, mapped host word: a recent frame had > kSerialLong long lists
  uint32_t* long_hint_dptr = nullptr;  // its device alias
  DevBuf long_hint_mirror;             // device copy of the last value written
  cudaStream_t sst = nullptr;     // vdi_composite_frames: the search stream
  cudaEvent_t mev_fast[2] = {}, mev_done[2] = {};
  DevBuf g_misc;  // inflate counters
  // vdi_composite_fullrep: per-source dense scratch of the compaction + its scan
  std::vector<std::unique_ptr<DevBuf>> xdense;
  DevBuf xsum, xbase, xtot;
  // generator outputs per pe
  std::vector<GenOut> gen;
  DevBuf gen_tmp;
  void* cub_tmp = nullptr;
  size_t cub_tmp_bytes = 0;
  // host e2e staging: two input slots, per-slot dense outputs, copy streams and slot events
  std::vector<DevBuf> hcount[2], hdepth[2], hrgba[2];
  DevBuf harena[2];
  DevBuf hstrip_count, hstrip_depth, hstrip_rgba;
  DevBuf pcount[2], pdense[2], g_dense;
  cudaStream_t pin_st = nullptr, pout_st = nullptr;
  cudaEvent_t pev_in[2] = {}, pev_used[2] = {}, pev_tot[2] = {}, pev_comp[2] = {}, pev_out[2] = {};
  unsigned long long* ptot = nullptr;      // pinned, mapped host [2]: frame totals written by the kernel
  unsigned long long* ptot_dev = nullptr;  // its device alias
  // counters
  vdi_counters last{};
  bool have_stats = false;
  int last_gather_root = -1;
  uint32_t last_gather_parity = 0;
  cudaEvent_t ev[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
  bool timing_pending = false;
  bool gather_timing_pending = false;
  cudaEvent_t gev[2] = {nullptr, nullptr};
  cudaEvent_t pev_t[2] = {nullptr, nullptr};  // STAGE_TIMING: around the exchange push kernel
  bool push_timing_pending = false;
  // vdi_composite_frames: the root's inflate stream and the non-root strips
  cudaStream_t gst = nullptr;
  cudaStream_t gsst = nullptr;  // the non-root strips' gather sends (beside the next frame's search)
  cudaEvent_t sev_merged[2] = {};
  cudaEvent_t gev_in = nullptr, gev_out = nullptr;
  static constexpr int kStripBufs = 4;  // non-root strips in flight (frame f reuses frame f-4's)
  DevBuf fs_count[kStripBufs], fs_depth[kStripBufs], fs_rgba[kStripBufs];
  cudaEvent_t fsev[kStripBufs] = {};  // strip buffer read by its gather send
  ~vdi_ctx() {
    if (sst) {
      cudaStreamSynchronize(sst);
      cudaStreamDestroy(sst);
    }
    for (int i = 0; i < 2; ++i) {
      if (mev_fast[i]) cudaEventDestroy(mev_fast[i]);
      if (mev_done[i]) cudaEventDestroy(mev_done[i]);
    }
    if (xst) {
      cudaStreamSynchronize(xst);
      cudaStreamDestroy(xst);
    }
    for (int i = 0; i < 2; ++i) {
      if (xev_bounds[i]) cudaEventDestroy(xev_bounds[i]);
      if (xev_merged[i]) cudaEventDestroy(xev_merged[i]);
    }
    if (gsst) {
      cudaStreamSynchronize(gsst);
      cudaStreamDestroy(gsst);
    }
    for (int i = 0; i < kStripBufs; ++i)
      if (fsev[i]) cudaEventDestroy(fsev[i]);
    for (int i = 0; i < 2; ++i) {
      if (sev_merged[i]) cudaEventDestroy(sev_merged[i]);
      if (pev_t[i]) cudaEventDestroy(pev_t[i]);
    }
    if (gst) {
      cudaStreamSynchronize(gst);
      cudaStreamDestroy(gst);
    }
    if (gev_in) cudaEventDestroy(gev_in);
    if (gev_out) cudaEventDestroy(gev_out);
    if (pin_st) cudaStreamSynchronize(pin_st);
    if (pout_st) cudaStreamSynchronize(pout_st);
    if (pin_st) cudaStreamDestroy(pin_st);
    if (pout_st) cudaStreamDestroy(pout_st);
    for (cudaEvent_t* a : {pev_in, pev_used, pev_tot, pev_comp, pev_out})
      for (int i = 0; i < 2; ++i)
        if (a[i]) cudaEventDestroy(a[i]);
    if (ptot) cudaFreeHost(ptot);
    if (long_hint) cudaFreeHost(long_hint);
    if (cub_tmp) cudaFree(cub_tmp);
    for (auto& e : ev)
      if (e) cudaEventDestroy(e);
    for (auto& e : gev)
      if (e) cudaEventDestroy(e);
    // local teardown: drain our stream, then abort (not finalize) the
    // communicator so destroying contexts never waits on other ranks
    cudaStreamSynchronize(stream);
    for (void* p : ipc_opened) cudaIpcCloseMemHandle(p);
    if (!loop_key.empty()) {
      std::lock_guard<std::mutex> lk(g_loop_mu);
      auto it = g_loop.find(loop_key);
      if (it != g_loop.end()) {
        {
          std::lock_guard<std::mutex> lk2(it->second->mu);
          it->second->base[cfg.rank] = nullptr;
        }
        bool any = false;
        for (char* b : it->second->base) any |= b != nullptr;
        if (!any) g_loop.erase(it);
      }
    }
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

vdi_status check_ctx(vdi_ctx* ctx) {
  if (!ctx) return fail(VDI_ERR_INVALID_ARG, "ctx is NULL");
  if (ctx->poisoned) return fail(VDI_ERR_STATE, "context poisoned by an earlier CUDA/NCCL error");
  return VDI_OK;
}

uint32_t* flag_at(char* base, int kind, uint32_t r) {
  return reinterpret_cast<uint32_t*>(base) + kind * VDI_MAX_RANKS + r;
}

// peers' window bases (n_ranks > 1): loopback contexts look each other up
vdi_status resolve_peers(vdi_ctx* ctx) {
  if (ctx->peers_ready) return VDI_OK;
  if (ctx->loop_key.empty()) return fail(VDI_ERR_STATE, "peer windows were not exchanged");
  std::lock_guard<std::mutex> lk(g_loop_mu);
  auto it = g_loop.find(ctx->loop_key);
  if (it == g_loop.end()) return fail(VDI_ERR_STATE, "loopback group vanished");
  std::lock_guard<std::mutex> lk2(it->second->mu);
  for (uint32_t r = 0; r < ctx->cfg.n_ranks; ++r)
    if (!it->second->base[r]) return fail(VDI_ERR_STATE, "loopback group incomplete: rank %u not initialised", r);
  ctx->peer = it->second->base;
  ctx->grp = it->second;
  ctx->peers_ready = true;
  return VDI_OK;
}

}  // namespace

// Merge of P lists whose sources are set in mp.src[0..n_pes) (receive-side
// scan, pass-through + classification, gamma search, general path;
// PAPER.md:166-185) into the full representation `so` (P lists).  S_est sizes
// the search pools (a list that finds no pool room takes the general path,
// so an estimate never changes a result); m_max bounds a list's records.
// Buffers of a merge of P lists (grow-only; S_est sizes the search pools,
// m_max the general path's per-thread scratch)
static vdi_status reserve_merge(vdi_ctx* ctx, uint64_t P, uint64_t S_est, uint32_t m_max, int b = 0) {
  const vdi_config& cf = ctx->cfg;
  vdi_ctx::MScratch& sc = ctx->ms[b];
  const uint32_t n = cf.n_pes, k = cf.k_out;
  const size_t ng = (P + 31) / 32;
  CUDA_TRY(ctx, ctx->group_sum.grow((size_t)scan_chunks((uint32_t)P) * n * 4 + 64));
  CUDA_TRY(ctx, ctx->group_base.grow(ng * n * 4 + 64));
  CUDA_TRY(ctx, sc.wl.grow(((size_t)std::max<uint64_t>(P, 1) * (3 + n) * VDI_N_BUCKETS + 64) * 4));
  CUDA_TRY(ctx, sc.slots.grow((2 * ng + 64) * 4));
  CUDA_TRY(ctx, sc.dcnt.grow(sizeof(DevCounters)));
  if (cf.flags & VDI_FLAG_PIXEL_STATS) {
    CUDA_TRY(ctx, ctx->stat_gamma.grow(P * 4 + 64));
    CUDA_TRY(ctx, ctx->stat_m.grow(P * 2 + 64));
    CUDA_TRY(ctx, ctx->stat_margin.grow(P * 4 + 64));
  }
  CUDA_TRY(ctx, sc.scratch.grow((size_t)general_threads(m_max) * 4 * std::max<uint32_t>(m_max, 1) * sizeof(Rec)));
  // short-list search pool: a list in bucket 0/1 has m > k_out samples, so at
  // most S / (k_out + 1) such lists exist; + one partial batch per bucket
  // (at most 2 GB: lists that find no slot take the general path)
  const uint64_t pool_cap =
      std::min<uint64_t>(std::min<uint64_t>((S_est / (k + 1) + 31) / 32 + 4, ng + 4), (2ull << 30) / kShortSlotBytes);
  CUDA_TRY(ctx, sc.srch.grow(pool_cap * kShortSlotBytes + 256));
  // long-list search: warp-private slots (independent of S)
  size_t lslot = 0;
  const uint32_t lw = long_warps(m_max, &lslot);
  CUDA_TRY(ctx, sc.lpool.grow((size_t)lw * lslot));
  CUDA_TRY(ctx, ctx->g_misc.grow(sizeof(DevCounters) + 256));
  return VDI_OK;
}

// Merge of P lists whose sources are set in mp.src[0..n_pes) (receive-side
// scan, pass-through + classification, gamma search, general path;
// PAPER.md:166-185) into the full representation `so` (P lists).  S_est sizes
// the search pools (a list that finds no pool room takes the general path,
// so an estimate never changes a result); m_max bounds a list's records.
static vdi_status merge_lists(vdi_ctx* ctx, MergeParams& mp, uint64_t P, uint64_t S_est, uint32_t m_max,
                              vdi_full_view* so, bool timing, int& launches_ref) {
  const vdi_config& cf = ctx->cfg;
  const uint32_t n = cf.n_pes, k = cf.k_out;
  cudaStream_t st = ctx->stream;
  const int b = ctx->mpar;
  cudaStream_t sst = ctx->msst ? ctx->msst : st;  // the search kernels' stream
  vdi_ctx::MScratch& sc = ctx->ms[b];
  ctx->last_mpar = b;
  int launches = 0;
  mp.P = (uint32_t)P;
  mp.n_groups = (uint32_t)((P + 31) / 32);
  mp.g_begin = 0;
  mp.g_end = mp.n_groups;
  ctx->mP = P;
  const size_t ng = mp.n_groups;
  if (vdi_status s = reserve_merge(ctx, P, S_est, m_max, b)) return s;
  const bool stats = cf.flags & VDI_FLAG_PIXEL_STATS;
  // pass-through -> search kernels -> general path.  One VDI: one stream
  // (within a VDI the search needs the pass-through's work lists; measured,
  // profiles/README.md: overlapping them on a second stream runs the
  // latency-bound search ~2x slower beside the HBM-bound pass-through).
  // Frames in flight (vdi_composite_frames): the search kernels of this VDI
  // run on a second stream beside the next VDI's pass-through, with their own
  // parity of work lists, counters and pools (this parity's previous search
  // must be done first).
  if (sst != st) {
    CUDA_TRY(ctx, cudaStreamWaitEvent(st, ctx->mev_done[b], 0));
    // a long search that fills the GPU for many waves does not gain from the
    // next VDI's pass-through beside it, it loses (C5: 18 % slower search,
    // profiles/README.md): when a recent frame of this context had more than
    // kSerialLong long lists, this pass-through also waits for the previous
    // VDI's search.  The hint is a mapped host word that the long-search kernel
    // rewrites only when its answer changes; a stale value only changes the
    // schedule, never a result.
    if (!ctx->long_hint) {
      CUDA_TRY(ctx, cudaHostAlloc(reinterpret_cast<void**>(&ctx->long_hint), sizeof(uint32_t), cudaHostAllocMapped));
      CUDA_TRY(ctx, cudaHostGetDevicePointer(reinterpret_cast<void**>(&ctx->long_hint_dptr), ctx->long_hint, 0));
      *ctx->long_hint = 0;
      CUDA_TRY(ctx, ctx->long_hint_mirror.grow(sizeof(uint32_t)));
      CUDA_TRY(ctx, cudaMemsetAsync(ctx->long_hint_mirror.p, 0, sizeof(uint32_t), st));
    }
    if (*static_cast<volatile uint32_t*>(ctx->long_hint)) CUDA_TRY(ctx, cudaStreamWaitEvent(st, ctx->mev_done[b ^ 1], 0));
    mp.long_hint = ctx->long_hint_dptr;
    mp.long_hint_dev = ctx->long_hint_mirror.as<uint32_t>();
  }
  mp.wl_cap = (uint32_t)std::max<uint64_t>(P, 1);
  mp.gen_threads = general_threads(m_max);
  mp.gen_stride = 4 * std::max<uint32_t>(m_max, 1);
  const uint64_t pool_cap = std::min<uint64_t>((sc.srch.bytes - 256) / kShortSlotBytes, ng + 4);
  {
    char* q = sc.srch.as<char>();
    mp.pool_rgba = reinterpret_cast<float4*>(q);
    q += pool_cap * 40 * 32 * 16;
    mp.pool_depth = reinterpret_cast<float2*>(q);
    q += pool_cap * 40 * 32 * 8;
    mp.pool_gap = reinterpret_cast<uint32_t*>(q);
    mp.pool_cap = (uint32_t)pool_cap;
  }
  mp.long_pool = sc.lpool.as<char>();
  mp.long_warps = long_warps(m_max, &mp.long_slot);
  mp.long_maxm = std::min<uint32_t>(std::max<uint32_t>(m_max, 41), 1024);
  DevCounters* dc = sc.dcnt.as<DevCounters>();
  CUDA_TRY(ctx, cudaMemsetAsync(dc, 0, sizeof(DevCounters), st));
  mp.group_base = ctx->group_base.as<uint32_t>();
  mp.out_count = so->count;
  mp.out_depth = reinterpret_cast<float2*>(so->depth);
  mp.out_rgba = reinterpret_cast<float4*>(so->rgba);
  mp.fallback_groups = &dc->fallback_groups;
  mp.pool_next = &dc->pool_next;
  mp.scratch = sc.scratch.as<Rec>();
  mp.stat_gamma = stats ? ctx->stat_gamma.as<float>() : nullptr;
  mp.stat_m = stats ? ctx->stat_m.as<uint16_t>() : nullptr;
  mp.stat_margin = stats ? ctx->stat_margin.as<float>() : nullptr;
  mp.records_in = &dc->records_in;
  mp.records_search = &dc->records_search;
  mp.sweep_steps = stats ? &dc->sweep_steps : nullptr;
  mp.err = &dc->err;
  mp.validate = (cf.flags & VDI_FLAG_VALIDATE) ? 1 : 0;
  uint32_t* slp = sc.slots.as<uint32_t>();
  mp.batch_slot[0] = slp;
  mp.batch_slot[1] = slp + ng + 32;
  uint32_t* wlp = sc.wl.as<uint32_t>();
  for (int b = 0; b < VDI_N_BUCKETS; ++b) mp.wl[b] = wlp + (size_t)b * mp.wl_cap * (3 + n);
  mp.wl_count = dc->wl_count;
  mp.search_ticket = dc->search_ticket;
  if (P) {
    bool scan = false;  // some source has neither an offset array nor group bases: receive-side scan
    for (uint32_t s = 0; s < n; ++s) scan |= !mp.src[s].offset && !mp.src[s].gbase;
    if (scan)
      CUDA_TRY(ctx, launch_scan(mp, ctx->group_sum.as<uint32_t>(), ctx->group_base.as<uint32_t>(), st, &launches));
    if (timing) CUDA_TRY(ctx, cudaEventRecord(ctx->ev[3], st));
    // pass-through (writes every slot of the strip) -> search kernels -> general path
    trace("fast_start", st);
    CUDA_TRY(ctx, launch_fast(mp, st, &launches));
    trace("fast_end", st);
    if (timing) CUDA_TRY(ctx, cudaEventRecord(ctx->ev[4], st));
    if (sst != st) {
      CUDA_TRY(ctx, cudaEventRecord(ctx->mev_fast[b], st));
      CUDA_TRY(ctx, cudaStreamWaitEvent(sst, ctx->mev_fast[b], 0));
    }
    trace("search_start", sst);
    CUDA_TRY(ctx, launch_search(mp, sst, &launches));
    trace("search_end", sst);
    if (timing) CUDA_TRY(ctx, cudaEventRecord(ctx->ev[5], sst));
    CUDA_TRY(ctx, launch_general(mp, sst, &launches));
    trace("general_end", sst);
    if (stats) CUDA_TRY(ctx, launch_margins(mp, sst, &launches));
  }
  launches_ref += launches;
  return VDI_OK;
}

// Pass-through launch that re-inflates packed, depth-ordered lists (m <= k)
// into the full representation (the root side of the dense gather, and
// vdi_dense_to_full): one source, group bases given.
static vdi_status inflate(vdi_ctx* ctx, const uint8_t* count, const float2* depth, const float4* rgba,
                          const uint32_t* group_base, uint64_t P, uint32_t k, uint8_t* oc, float2* od, float4* orgba,
                          int& launches, cudaStream_t st = nullptr) {
  if (!st) st = ctx->stream;
  if (!P) return VDI_OK;
  CUDA_TRY(ctx, ctx->g_misc.grow(sizeof(DevCounters) + 256));
  DevCounters* gc = ctx->g_misc.as<DevCounters>();
  CUDA_TRY(ctx, cudaMemsetAsync(gc, 0, sizeof(DevCounters), st));
  MergeParams mi{};
  mi.n_src = 1;
  mi.k_out = (int)k;
  mi.max_iters = (int)ctx->cfg.max_iters;
  mi.gamma_max = ctx->cfg.gamma_max;
  mi.P = (uint32_t)P;
  mi.n_groups = (uint32_t)((P + 31) / 32);
  mi.g_begin = 0;
  mi.g_end = mi.n_groups;
  mi.src[0] = SrcDesc{count, depth, rgba, nullptr};
  mi.group_base = group_base;
  mi.out_count = oc;
  mi.out_depth = od;
  mi.out_rgba = orgba;
  for (int b = 0; b < VDI_N_BUCKETS; ++b) mi.wl[b] = reinterpret_cast<uint32_t*>(gc);  // never written: wl_cap = 0
  mi.wl_count = gc->wl_count;
  mi.wl_cap = 0;
  mi.records_in = &gc->records_in;
  mi.fallback_groups = &gc->fallback_groups;
  mi.err = &gc->err;
  CUDA_TRY(ctx, launch_fast(mi, st, &launches));
  return VDI_OK;
}

extern "C" {

const char* vdi_version(void) { return "libvdi 0.2 (sm_100a)"; }

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
  if (cfg->n_ranks < 1 || cfg->n_ranks > VDI_MAX_RANKS || cfg->rank >= cfg->n_ranks)
    return fail(VDI_ERR_INVALID_ARG, "bad rank/n_ranks (n_ranks must be in 1..%d)", VDI_MAX_RANKS);
  if (cfg->root >= cfg->n_ranks) return fail(VDI_ERR_INVALID_ARG, "root %u >= n_ranks %u", cfg->root, cfg->n_ranks);
  if (cfg->n_ranks > cfg->height) return fail(VDI_ERR_INVALID_ARG, "more ranks than image rows");
  if (cfg->n_ranks > 1 && !cfg->nccl_unique_id) return fail(VDI_ERR_INVALID_ARG, "nccl_unique_id required");
  if ((uint64_t)cfg->width * cfg->height > (1ull << 31)) return fail(VDI_ERR_INVALID_ARG, "image too large");
  if ((uint64_t)cfg->width * cfg->height * std::max(cfg->k_in, cfg->k_out) >= (1ull << 32))
    return fail(VDI_ERR_INVALID_ARG, "W*H*k must be < 2^32 (u32 record indices)");
  vdi_ctx* ctx = new vdi_ctx();
  ctx->cfg = *cfg;
  if (!ctx->cfg.max_iters) ctx->cfg.max_iters = 16;
  if (!(ctx->cfg.gamma_max > 0.0f)) ctx->cfg.gamma_max = 2.0f;
  ctx->cfg.nccl_unique_id = nullptr;
  ctx->stream = static_cast<cudaStream_t>(cfg->cuda_stream);
  ctx->lay = Layout{cfg->width, cfg->height, cfg->n_ranks, cfg->n_pes, cfg->k_in, cfg->k_out};
  cudaError_t e = cudaGetDevice(&ctx->device);
  if (e != cudaSuccess) {
    delete ctx;
    return fail(VDI_ERR_CUDA, "cudaGetDevice: %s", cudaGetErrorString(e));
  }
  ctx->row0 = strip_row(cfg->height, cfg->n_ranks, cfg->rank);
  ctx->row1 = strip_row(cfg->height, cfg->n_ranks, cfg->rank + 1);
  ctx->P = (uint64_t)(ctx->row1 - ctx->row0) * cfg->width;
  ctx->gen.resize(cfg->n_pes);
  ctx->gcalls_to.assign(cfg->n_ranks, 0);
  for (auto& ev : ctx->ev) cudaEventCreate(&ev);
  for (auto& ev : ctx->gev) cudaEventCreate(&ev);
  if (cfg->n_ranks > 1) {
    const uint32_t G = cfg->n_ranks, me = cfg->rank;
    // the window: flags | exchange receive slots | gather buffers (zeroed flags)
    e = ctx->win.grow(ctx->lay.win_bytes(me));
    if (e == cudaSuccess) e = cudaMemset(ctx->win.p, 0, kFlagBytes);
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      delete ctx;
      return fail(e == cudaErrorMemoryAllocation ? VDI_ERR_OUT_OF_MEMORY : VDI_ERR_CUDA, "window (%zu B): %s",
                  ctx->lay.win_bytes(me), cudaGetErrorString(e));
    }
    if (cfg->flags & VDI_FLAG_LOOPBACK) {
      // every kernel loaded up front: with lazy loading, a later first launch
      // could wait for a device on which another context's wait kernel spins
      static std::once_flag once;
      std::call_once(once, [] {
        preload_merge();
        preload_comm();
        preload_render();
      });
      ctx->loop_key.assign(reinterpret_cast<const char*>(cfg->nccl_unique_id), 128);
      std::lock_guard<std::mutex> lk(g_loop_mu);
      std::shared_ptr<LoopGroup>& grp = g_loop[ctx->loop_key];
      if (!grp) grp = std::make_shared<LoopGroup>();
      std::lock_guard<std::mutex> lk2(grp->mu);
      if (grp->base.empty()) grp->base.assign(G, nullptr);
      if (grp->base.size() != G || grp->base[me]) {
        ctx->loop_key.clear();
        delete ctx;
        return fail(VDI_ERR_INVALID_ARG, "loopback group: rank %u registered twice or n_ranks differs", me);
      }
      grp->base[me] = ctx->win.as<char>();
    } else {
      ncclUniqueId id;
      memcpy(&id, cfg->nccl_unique_id, sizeof id);
      ncclResult_t r = ncclCommInitRank(&ctx->comm, (int)G, id, (int)me);
      if (r != ncclSuccess) {
        ctx->comm = nullptr;
        delete ctx;
        return fail(VDI_ERR_NCCL, "ncclCommInitRank: %s", ncclGetErrorString(r));
      }
      // one all-gather of the windows' IPC handles (the only host round trip
      // of the multi-GPU path; calls never synchronise the host afterwards)
      cudaIpcMemHandle_t mine;
      std::vector<cudaIpcMemHandle_t> all(G);
      DevBuf hb;
      e = cudaIpcGetMemHandle(&mine, ctx->win.p);
      if (e == cudaSuccess) e = hb.grow((size_t)G * sizeof mine * 2);
      if (e == cudaSuccess) e = cudaMemcpy(hb.as<char>() + (size_t)G * sizeof mine, &mine, sizeof mine,
                                           cudaMemcpyHostToDevice);
      if (e != cudaSuccess) {
        delete ctx;
        return fail(VDI_ERR_CUDA, "window IPC handle: %s", cudaGetErrorString(e));
      }
      r = ncclAllGather(hb.as<char>() + (size_t)G * sizeof mine, hb.p, sizeof mine, ncclUint8, ctx->comm, ctx->stream);
      if (r == ncclSuccess) e = cudaStreamSynchronize(ctx->stream);
      if (r == ncclSuccess && e == cudaSuccess)
        e = cudaMemcpy(all.data(), hb.p, (size_t)G * sizeof mine, cudaMemcpyDeviceToHost);
      if (r != ncclSuccess || e != cudaSuccess) {
        delete ctx;
        return fail(r != ncclSuccess ? VDI_ERR_NCCL : VDI_ERR_CUDA, "window handle exchange: %s",
                    r != ncclSuccess ? ncclGetErrorString(r) : cudaGetErrorString(e));
      }
      ctx->peer.assign(G, nullptr);
      for (uint32_t g = 0; g < G; ++g) {
        if (g == me) {
          ctx->peer[g] = ctx->win.as<char>();
          continue;
        }
        void* b = nullptr;
        e = cudaIpcOpenMemHandle(&b, all[g], cudaIpcMemLazyEnablePeerAccess);
        if (e != cudaSuccess) {
          delete ctx;
          return fail(VDI_ERR_CUDA, "cudaIpcOpenMemHandle(rank %u): %s", g, cudaGetErrorString(e));
        }
        ctx->ipc_opened.push_back(b);
        ctx->peer[g] = static_cast<char*>(b);
      }
      ctx->peers_ready = true;
    }
  }
  if (cfg->n_ranks > 1) {
    // the fixed-size buffers of the exchange, the merge and the gather are
    // reserved now, so that calls do not allocate in the steady state
    const Layout& L = ctx->lay;
    const uint32_t G = cfg->n_ranks, nl = L.n_local(cfg->rank);
    const uint64_t Pimg = (uint64_t)cfg->width * cfg->height;
    const uint64_t ngs = (ctx->P + 31) / 32;
    vdi_status s = VDI_OK;
    cudaError_t e2 = cudaSuccess;
    for (auto [b, need] : std::initializer_list<std::pair<DevBuf*, size_t>>{
             {&ctx->ccnt, 64},
             {&ctx->srcbase, 2 * VDI_MAX_SRC * 4 + 64},
             {&ctx->bnd, (size_t)std::max<uint32_t>(nl, 1) * (G + 1) * 8 + 64},
             {&ctx->segbuf, (size_t)2 * VDI_MAX_SRC * VDI_MAX_RANKS * sizeof(PushSeg)},
             {&ctx->gsum, ((size_t)scan_chunks((uint32_t)ctx->P) + 8) * 4 + 64},
             {&ctx->gbase_loc, (ngs + 8) * 4 + 64},
             {&ctx->gsum_x, (size_t)scan_chunks((uint32_t)Pimg) * std::max<uint32_t>(nl, 1) * 4 + 64},
             {&ctx->gbase_x, 2 * ((Pimg + 31) / 32) * std::max<uint32_t>(nl, 1) * 4 + 64}})
      if (e2 == cudaSuccess) e2 = b->grow(need);
    for (int i = 0; i < 2 && e2 == cudaSuccess; ++i) {
      e2 = cudaEventCreateWithFlags(&ctx->xev_bounds[i], cudaEventDisableTiming);
      if (e2 == cudaSuccess) e2 = cudaEventCreateWithFlags(&ctx->xev_merged[i], cudaEventDisableTiming);
    }
    if (e2 == cudaSuccess)
      s = reserve_merge(ctx, ctx->P, std::min<uint64_t>((uint64_t)cfg->n_pes * ctx->P * cfg->k_in, (uint64_t)cfg->n_pes * ctx->P * 2),
                        cfg->n_pes * cfg->k_in);
    if (e2 == cudaSuccess) e2 = cudaMemset(ctx->ccnt.p, 0, 64);  // [2]: loopback check shortfalls (never reset)
    if (e2 != cudaSuccess || s != VDI_OK) {
      delete ctx;
      return e2 != cudaSuccess ? fail(VDI_ERR_OUT_OF_MEMORY, "reserve: %s", cudaGetErrorString(e2)) : s;
    }
  }
  *out = ctx;
  return VDI_OK;
}

void vdi_composite_destroy(vdi_ctx* ctx) { delete ctx; }

// ---------------------------------------------------------------------------
// Phase 1 (SUPPORT)
// ---------------------------------------------------------------------------
static vdi_status generate(vdi_ctx* ctx, const vdi_volume_desc* vol, const vdi_tf_desc* tf, const vdi_camera* cam,
                           const vdi_decomp_desc* dec, uint32_t pe_id, vdi_dense_view* out, bool limit) {
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
  gp.limit = limit ? 1 : 0;

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

vdi_status vdi_generate_subvdi(vdi_ctx* ctx, const vdi_volume_desc* vol, const vdi_tf_desc* tf,
                               const vdi_camera* cam, const vdi_decomp_desc* dec, uint32_t pe_id,
                               vdi_dense_view* out) {
  VDI_NVTX("vdi_generate_subvdi");
  return generate(ctx, vol, tf, cam, dec, pe_id, out, false);
}

vdi_status vdi_generate_limit(vdi_ctx* ctx, const vdi_volume_desc* vol, const vdi_tf_desc* tf, const vdi_camera* cam,
                              const vdi_decomp_desc* dec, uint32_t pe_id, vdi_dense_view* out) {
  VDI_NVTX("vdi_generate_limit");
  return generate(ctx, vol, tf, cam, dec, pe_id, out, true);
}

// ---------------------------------------------------------------------------
// Phase 2: the hot path
// ---------------------------------------------------------------------------
// local_pes -> slot[s] = index in local[] of PE s homed here, -1 elsewhere
static vdi_status check_local(vdi_ctx* ctx, const vdi_dense_view* local, uint32_t n_local, std::vector<int>& slot) {
  const vdi_config& cf = ctx->cfg;
  const uint32_t G = cf.n_ranks, me = cf.rank, n = cf.n_pes;
  slot.assign(n, -1);
  const uint32_t expect = ctx->lay.n_local(me);
  if (n_local != expect) return fail(VDI_ERR_INVALID_ARG, "rank %u homes %u PEs, got %u", me, expect, n_local);
  if (n_local && !local) return fail(VDI_ERR_INVALID_ARG, "local_pes is NULL");
  for (uint32_t l = 0; l < n_local; ++l) {
    const vdi_dense_view& v = local[l];
    if (v.pe_id >= n || vdi_pe_home(n, G, v.pe_id) != me || slot[v.pe_id] >= 0)
      return fail(VDI_ERR_INVALID_ARG, "pe_id %u not homed on rank %u or duplicated", v.pe_id, me);
    if (!v.count || (v.total && (!v.depth || !v.rgba)))
      return fail(VDI_ERR_INVALID_ARG, "dense view of PE %u has NULL arrays", v.pe_id);
    if ((reinterpret_cast<uintptr_t>(v.rgba) & 15) || (reinterpret_cast<uintptr_t>(v.depth) & 7))
      return fail(VDI_ERR_INVALID_ARG, "dense view of PE %u: depth/rgba misaligned", v.pe_id);
    slot[v.pe_id] = (int)l;
  }
  return VDI_OK;
}

// loopback: publish "this rank's side of (kind, seq) is enqueued" to each consumer
static vdi_status loop_post(vdi_ctx* ctx, int kind, const std::vector<uint32_t>& consumers, uint32_t seq,
                            cudaStream_t st) {
  for (uint32_t c : consumers) {
    cudaEvent_t ev;
    CUDA_TRY(ctx, cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    CUDA_TRY(ctx, cudaEventRecord(ev, st));
    std::lock_guard<std::mutex> lk(ctx->grp->mu);
    ctx->grp->posted[std::make_tuple(kind, ctx->cfg.rank, c, seq)] = ev;
  }
  ctx->grp->cv.notify_all();
  return VDI_OK;
}

// A wait of the device path: each entry = (peer rank, flag target, sequence).
// Multi-GPU: one-CTA spin kernel until the flag words reach their targets.
// Loopback: the host waits until each peer has posted (kind, seq), the
// stream waits on the posted event, and a check kernel verifies the flags.
struct WaitOn {
  uint32_t rank, target, seq;
};
static vdi_status wait_flags(vdi_ctx* ctx, int kind, const std::vector<WaitOn>& who, cudaStream_t st = nullptr) {
  if (!st) st = ctx->stream;
  WaitArgs w{};
  for (const WaitOn& x : who) {
    w.addr[w.n] = flag_at(ctx->peer[ctx->cfg.rank], kind, x.rank);
    w.target[w.n] = x.target;
    ++w.n;
  }
  if (!ctx->grp) {
    CUDA_TRY(ctx, launch_wait(w, st));
    return VDI_OK;
  }
  for (const WaitOn& x : who) {
    cudaEvent_t ev;
    {
      std::unique_lock<std::mutex> lk(ctx->grp->mu);
      const auto key = std::make_tuple(kind, x.rank, ctx->cfg.rank, x.seq);
      ctx->grp->cv.wait(lk, [&] { return ctx->grp->posted.count(key) > 0; });
      ev = ctx->grp->posted[key];
      ctx->grp->posted.erase(key);
    }
    CUDA_TRY(ctx, cudaStreamWaitEvent(st, ev, 0));
    CUDA_TRY(ctx, cudaEventDestroy(ev));
  }
  CUDA_TRY(ctx, launch_check(w, ctx->ccnt.as<unsigned long long>() + 2, st));
  return VDI_OK;
}

// release store of `value` into flag word (kind, me) of each listed peer
// (loopback: and post (kind, seq) to them)
static vdi_status signal_peers(vdi_ctx* ctx, int kind, const std::vector<uint32_t>& peers, uint32_t value,
                               cudaStream_t st = nullptr, uint32_t seq = 0) {
  if (!st) st = ctx->stream;
  SignalArgs s{};
  for (uint32_t r : peers) {
    s.addr[s.n] = flag_at(ctx->peer[r], kind, ctx->cfg.rank);
    s.value[s.n] = value;
    ++s.n;
  }
  CUDA_TRY(ctx, launch_signal(s, st));
  if (ctx->grp) return loop_post(ctx, kind, peers, seq, st);
  return VDI_OK;
}

// Exchange (a2-a5), sending half: the strip bounds of this
// rank's PEs (on the device) and the push of every (local PE, strip g != me)
// slice -- counts, the 32-list group bases of the slice (so the receiver
// needs no scan; strips starting on 32-list boundaries) and the packed
// records -- into g's window, once g has released the slot of the same
// parity.  dense: `local` are dense views (slices [offset[row_g W],
// offset[row_{g+1} W]) found on the device); full (vdi_composite_fullrep):
// `flocal` are full representations (fixed-size slices).  Runs on stream pst;
// the device arrays the merge will read (local group bases / strip starts)
// are double-buffered by `par` and ready at event ctx->xev_bounds[par].
// Returns the call's epoch in *epoch.
static vdi_status exchange_push(vdi_ctx* ctx, const vdi_dense_view* local, const vdi_full_view* flocal,
                                uint32_t n_local, const uint32_t* full_ids, int& launches, cudaStream_t pst, int par,
                                uint32_t* epoch) {
  const vdi_config& cf = ctx->cfg;
  const Layout& L = ctx->lay;
  const uint32_t G = cf.n_ranks, me = cf.rank, n = cf.n_pes, W = cf.width, K = cf.k_in;
  if (vdi_status s = resolve_peers(ctx)) return s;
  const uint32_t e = ++ctx->xcalls, q = e & 1;
  *epoch = e;
  const uint64_t Pimg = (uint64_t)W * cf.height;
  const uint32_t ngimg = (uint32_t)((Pimg + 31) / 32);
  const bool aligned = L.aligned();
  trace("push_begin", pst);
  CUDA_TRY(ctx, cudaMemsetAsync(ctx->ccnt.p, 0, 8, pst));
  CUDA_TRY(ctx, cudaMemsetAsync(ctx->srcbase.as<uint32_t>() + (size_t)par * VDI_MAX_SRC, 0, (size_t)n * 4, pst));
  unsigned long long* bnd = ctx->bnd.as<unsigned long long>();
  const uint32_t* gb32 = nullptr;  // the local PEs' 32-list group bases from the image start (no offset arrays)
  if (!flocal && n_local) {
    // a2: strip bounds of the local PEs on the device
    BoundsArgs ba{};
    bool all_off = true;
    for (uint32_t l = 0; l < n_local; ++l) all_off &= local[l].offset != nullptr;
    if (!all_off) {  // scan of the counts (no offset arrays, e.g. the host entry points)
      MergeParams ms{};
      ms.n_src = (int)n_local;
      ms.P = (uint32_t)Pimg;
      ms.n_groups = ngimg;
      for (uint32_t l = 0; l < n_local; ++l) ms.src[l].count = local[l].count;
      uint32_t* gbx = ctx->gbase_x.as<uint32_t>() + (size_t)par * n_local * ngimg;
      CUDA_TRY(ctx, launch_scan(ms, ctx->gsum_x.as<uint32_t>(), gbx, pst, &launches));
      ba.gbase = gbx;
      gb32 = gbx;
    }
    for (uint32_t l = 0; l < n_local; ++l) {
      ba.offset[l] = local[l].offset;
      ba.count[l] = local[l].count;
      ba.total[l] = local[l].total;
      ba.pe[l] = local[l].pe_id;
    }
    for (uint32_t g = 0; g <= G; ++g) ba.rows[g] = strip_row(cf.height, G, g);
    ba.n_groups = ngimg;
    ba.W = W;
    ba.n_local = (int)n_local;
    ba.G = (int)G;
    ba.bnd = bnd;
    // the merge reads its own strip of the local PEs in place: src_base = bnd[l][me]
    ba.srcbase = ctx->srcbase.as<uint32_t>() + (size_t)par * VDI_MAX_SRC;
    ba.me = (int)me;
    CUDA_TRY(ctx, launch_bounds(ba, pst));
    ++launches;
  }
  CUDA_TRY(ctx, cudaEventRecord(ctx->xev_bounds[par], pst));
  std::vector<uint32_t> dests;
  for (uint32_t g = 0; g < G; ++g)
    if (g != me && n_local) dests.push_back(g);
  // (loopback: the receiver's merge of the previous call, posted as seq e - 1)
  if (n_local && e > (ctx->grp ? 1u : 2u)) {
    std::vector<WaitOn> wt;
    for (uint32_t g : dests) wt.push_back({g, e - 2, e - 1});
    if (vdi_status s = wait_flags(ctx, XFREE, wt, pst)) return s;
    ++launches;
  }
  trace("push_free", pst);
  std::vector<PushSeg> segs;
  for (uint32_t l = 0; l < n_local; ++l) {
    const uint32_t pe = flocal ? full_ids[l] : local[l].pe_id;
    for (uint32_t g : dests) {
      const uint32_t a = strip_row(cf.height, G, g), b = strip_row(cf.height, G, g + 1);
      const size_t Pg = (size_t)(b - a) * W;
      const Slot sl = slot_at(ctx->peer[g] + L.x_off(g, q, pe), Pg, K);
      PushSeg sg{};
      if (flocal) {
        const vdi_full_view& v = flocal[l];
        sg.src_count = v.count + (size_t)a * W;
        sg.src_depth = reinterpret_cast<const float2*>(v.depth);
        sg.src_rgba = reinterpret_cast<const float4*>(v.rgba);
        sg.rec0 = (unsigned long long)a * W * K;
        sg.nrec = (unsigned long long)Pg * K;
      } else {
        const vdi_dense_view& v = local[l];
        sg.src_count = v.count + (size_t)a * W;
        sg.src_depth = reinterpret_cast<const float2*>(v.depth);
        sg.src_rgba = reinterpret_cast<const float4*>(v.rgba);
        sg.bnd = bnd + (size_t)l * (G + 1) + g;
        if (aligned) {  // the slice's group bases, relative to its first record
          sg.src_offset = v.offset ? v.offset + (size_t)a * W : nullptr;
          sg.src_gb32 = v.offset ? nullptr : gb32 + (size_t)l * ngimg + (size_t)a * W / 32;
          sg.n_groups = (uint32_t)((Pg + 31) / 32);
          sg.dst_gbase = sl.gbase;
        }
      }
      sg.n_count = Pg;
      sg.cap_rec = (unsigned long long)Pg * K;
      sg.src_total = flocal ? (unsigned long long)cf.width * cf.height * K : local[l].total;
      sg.dst_hdr = sl.hdr;
      sg.dst_count = sl.count;
      sg.dst_depth = sl.depth;
      sg.dst_rgba = sl.rgba;
      sg.bytes = ctx->ccnt.as<unsigned long long>();
      sg.flag = flag_at(ctx->peer[g], XREADY, me);
      segs.push_back(sg);
    }
  }
  if (!segs.empty()) {
    PushSeg* dsegs = ctx->segbuf.as<PushSeg>() + (size_t)par * VDI_MAX_SRC * VDI_MAX_RANKS;
    CUDA_TRY(ctx, cudaMemcpyAsync(dsegs, segs.data(), segs.size() * sizeof(PushSeg), cudaMemcpyHostToDevice, pst));
    const bool ptime = cf.flags & VDI_FLAG_STAGE_TIMING;
    if (ptime) {
      if (!ctx->pev_t[0])
        for (int i = 0; i < 2; ++i) CUDA_TRY(ctx, cudaEventCreate(&ctx->pev_t[i]));
      CUDA_TRY(ctx, cudaEventRecord(ctx->pev_t[0], pst));
    }
    CUDA_TRY(ctx, launch_push(dsegs, (uint32_t)segs.size(), push_blocks(n_local, G), pst));
    ++launches;
    if (ptime) {
      CUDA_TRY(ctx, cudaEventRecord(ctx->pev_t[1], pst));
      ctx->push_timing_pending = true;
    }
    trace("push_end", pst);
    if (ctx->grp)
      if (vdi_status s = loop_post(ctx, XREADY, dests, e, pst)) return s;
  }
  return VDI_OK;
}

// Exchange, receiving half (stream = the ctx stream): wait until every
// sender's slices of epoch e have landed, then point the merge's sources at
// the own PEs (read in place) and the receive slots.  With 32-list aligned
// strips every source comes with its group bases (offsets, the sender's
// pushed bases, or the local scan) and the receive-side scan is skipped.
static vdi_status exchange_recv(vdi_ctx* ctx, const vdi_dense_view* local, const vdi_full_view* flocal,
                                const std::vector<int>& slot, uint32_t e, int par, MergeParams& mp, int& launches) {
  const vdi_config& cf = ctx->cfg;
  const Layout& L = ctx->lay;
  const uint32_t G = cf.n_ranks, me = cf.rank, n = cf.n_pes, W = cf.width, K = cf.k_in;
  const uint32_t q = e & 1;
  const uint64_t Pimg = (uint64_t)W * cf.height;
  const uint32_t ngimg = (uint32_t)((Pimg + 31) / 32);
  const bool direct = !flocal && L.aligned();
  CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->stream, ctx->xev_bounds[par], 0));
  std::vector<WaitOn> wt;
  for (uint32_t s = 0; s < G; ++s)
    if (s != me && L.n_local(s)) {
      const uint32_t nl = L.n_local(s);
      wt.push_back({s, e * nl * push_blocks(nl, G), e});
    }
  trace("recv_wait", ctx->stream);
  if (!wt.empty()) {
    if (vdi_status st = wait_flags(ctx, XREADY, wt)) return st;
    ++launches;
  }
  trace("recv_ready", ctx->stream);
  const size_t Pm = ctx->P;
  uint32_t l_of[VDI_MAX_SRC];
  for (uint32_t s = 0; s < n; ++s) l_of[s] = slot[s] >= 0 ? (uint32_t)slot[s] : 0u;
  for (uint32_t s = 0; s < n; ++s) {
    if (slot[s] >= 0) {
      if (flocal) {
        const vdi_full_view& v = flocal[slot[s]];
        const size_t o = (size_t)ctx->row0 * W;
        mp.src[s] = SrcDesc{v.count + o, reinterpret_cast<const float2*>(v.depth) + o * K,
                            reinterpret_cast<const float4*>(v.rgba) + o * K, nullptr, nullptr};
      } else {
        const vdi_dense_view& v = local[slot[s]];
        const size_t o = (size_t)ctx->row0 * W;
        mp.src[s] = SrcDesc{v.count + o, reinterpret_cast<const float2*>(v.depth),
                            reinterpret_cast<const float4*>(v.rgba), nullptr, nullptr, v.total};
        if (direct) {
          if (v.offset) mp.src[s].offset = v.offset + o;  // absolute record indices
          else mp.src[s].gbase = ctx->gbase_x.as<uint32_t>() + ((size_t)par * L.n_local(me) + l_of[s]) * ngimg + o / 32;
        }
      }
    } else {
      const Slot sl = slot_at(ctx->peer[me] + L.x_off(me, q, s), Pm, K);
      mp.src[s] = SrcDesc{sl.count, sl.depth, sl.rgba, nullptr, direct ? sl.gbase : nullptr,
                          (unsigned long long)Pm * K};
    }
  }
  mp.src_base = flocal ? nullptr : ctx->srcbase.as<uint32_t>() + (size_t)par * VDI_MAX_SRC;
  return VDI_OK;
}

// after the merge: the senders may reuse this call's slots (XFREE)
static vdi_status release_slots(vdi_ctx* ctx, int& launches, cudaStream_t st = nullptr) {
  std::vector<uint32_t> senders;
  for (uint32_t g = 0; g < ctx->cfg.n_ranks; ++g)
    if (g != ctx->cfg.rank && ctx->lay.n_local(g)) senders.push_back(g);
  if (senders.empty()) return VDI_OK;
  if (vdi_status s = signal_peers(ctx, XFREE, senders, ctx->xcalls, st, ctx->xcalls)) return s;
  ++launches;
  return VDI_OK;
}

vdi_status vdi_composite(vdi_ctx* ctx, const vdi_dense_view* local, uint32_t n_local, vdi_full_view* so) {
  VDI_NVTX("vdi_composite");
  if (vdi_status s = check_ctx(ctx)) return s;
  const vdi_config& cf = ctx->cfg;
  const uint32_t G = cf.n_ranks, n = cf.n_pes, k = cf.k_out;
  if (!so || !so->count || !so->depth || !so->rgba) return fail(VDI_ERR_INVALID_ARG, "strip_out is NULL");
  if (so->row_begin != ctx->row0 || so->row_end != ctx->row1)
    return fail(VDI_ERR_CAPACITY, "strip_out rows [%u,%u) != this rank's strip [%u,%u)", so->row_begin,
                so->row_end, ctx->row0, ctx->row1);
  if ((reinterpret_cast<uintptr_t>(so->rgba) & 15) || (reinterpret_cast<uintptr_t>(so->depth) & 7))
    return fail(VDI_ERR_INVALID_ARG, "strip_out depth/rgba must be 8/16-byte aligned");
  std::vector<int> slot;
  if (vdi_status s = check_local(ctx, local, n_local, slot)) return s;
  cudaStream_t st = ctx->stream;
  if (cf.flags & VDI_FLAG_VALIDATE) {  // debug: check the inputs on the device, one host sync
    CUDA_TRY(ctx, ctx->gen_tmp.grow(16));
    int* derr = ctx->gen_tmp.as<int>();
    CUDA_TRY(ctx, cudaMemsetAsync(derr, 0, 4, st));
    for (uint32_t l = 0; l < n_local; ++l)
      CUDA_TRY(ctx, launch_validate(local[l].count, local[l].offset, reinterpret_cast<const float2*>(local[l].depth),
                                    reinterpret_cast<const float4*>(local[l].rgba), cf.width * cf.height,
                                    (int)cf.k_in, local[l].total, derr, st));
    int herr = 0;
    CUDA_TRY(ctx, cudaMemcpyAsync(&herr, derr, 4, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(ctx, cudaStreamSynchronize(st));
    if (herr)
      return fail(VDI_ERR_INVALID_ARG, "VDI_FLAG_VALIDATE: invalid input (%s%s%s%s%s)", herr & 1 ? "count > k_in; " : "",
                  herr & 2 ? "offsets are not the exclusive scan of count / total; " : "",
                  herr & 4 ? "t_front >= t_back; " : "", herr & 8 ? "alpha outside [0, 1]; " : "",
                  herr & 16 ? "records not front-to-back and disjoint within a list" : "");
  }
  const bool timing = cf.flags & VDI_FLAG_STAGE_TIMING;
  int launches = 0;
  if (timing) CUDA_TRY(ctx, cudaEventRecord(ctx->ev[0], st));
  MergeParams mp{};
  mp.n_src = (int)n;
  mp.k_out = (int)k;
  mp.max_iters = (int)cf.max_iters;
  mp.gamma_max = cf.gamma_max;
  uint64_t S_loc = 0;
  for (uint32_t l = 0; l < n_local; ++l) S_loc += local[l].total;
  uint64_t S_est;
  if (G == 1) {
    // every source is whole and local: when all carry their offset arrays
    // (Fig. 2) the group bases are read from them and the
    // receive-side scan is skipped
    bool all_off = true;
    for (uint32_t s = 0; s < n; ++s) all_off &= local[slot[s]].offset != nullptr;
    for (uint32_t s = 0; s < n; ++s) {
      const vdi_dense_view& v = local[slot[s]];
      mp.src[s] = SrcDesc{v.count, reinterpret_cast<const float2*>(v.depth), reinterpret_cast<const float4*>(v.rgba),
                          all_off ? v.offset : nullptr, nullptr, v.total};
    }
    S_est = S_loc;
  } else {
    uint32_t e = 0;
    if (vdi_status s = exchange_push(ctx, local, nullptr, n_local, nullptr, launches, ctx->xpst ? ctx->xpst : st,
                                     ctx->xpar, &e))
      return s;
    if (vdi_status s = exchange_recv(ctx, local, nullptr, slot, e, ctx->xpar, mp, launches)) return s;
    // the strip's records are known only on the device: size the pools for
    // twice this rank's share of the whole VDI (estimated from the local PEs)
    const uint64_t cap = (uint64_t)n * ctx->P * cf.k_in;
    S_est = n_local ? std::min<uint64_t>(cap, 2 * S_loc * n / n_local / G + 4096) : std::min<uint64_t>(cap, ctx->P * 8);
  }
  if (timing) CUDA_TRY(ctx, cudaEventRecord(ctx->ev[1], st));
  if (vdi_status s = merge_lists(ctx, mp, ctx->P, S_est, n * cf.k_in, so, timing, launches)) return s;
  cudaStream_t sst = ctx->msst ? ctx->msst : st;  // where the merge ends
  if (G > 1) {
    CUDA_TRY(ctx, cudaEventRecord(ctx->xev_merged[ctx->xpar], sst));  // the exchange buffers of this parity are read
    if (vdi_status s = release_slots(ctx, launches, sst)) return s;
  }
  if (timing) {
    CUDA_TRY(ctx, cudaEventRecord(ctx->ev[2], sst));
    ctx->timing_pending = true;
  }
  ctx->have_stats = cf.flags & VDI_FLAG_PIXEL_STATS;
  ctx->last = vdi_counters{};
  ctx->last.kernel_launches = (uint32_t)launches;
  return VDI_OK;
}

vdi_status vdi_dense_to_full(vdi_ctx* ctx, const vdi_dense_view* in, vdi_full_view* out) {
  VDI_NVTX("vdi_dense_to_full");
  if (vdi_status s = check_ctx(ctx)) return s;
  const vdi_config& cf = ctx->cfg;
  if (!in || !out || !in->count || (in->total && (!in->depth || !in->rgba)))
    return fail(VDI_ERR_INVALID_ARG, "in/out is NULL");
  if (!out->count || !out->depth || !out->rgba || out->row_begin != 0 || out->row_end != cf.height)
    return fail(VDI_ERR_INVALID_ARG, "out must cover rows [0, H)");
  if ((reinterpret_cast<uintptr_t>(out->rgba) & 15) || (reinterpret_cast<uintptr_t>(out->depth) & 7) ||
      (reinterpret_cast<uintptr_t>(in->rgba) & 15) || (reinterpret_cast<uintptr_t>(in->depth) & 7))
    return fail(VDI_ERR_INVALID_ARG, "depth/rgba misaligned");
  const size_t P = (size_t)cf.width * cf.height;
  int launches = 0;
  MergeParams ms{};
  ms.n_src = 1;
  ms.P = (uint32_t)P;
  ms.n_groups = (uint32_t)((P + 31) / 32);
  ms.src[0].count = in->count;
  CUDA_TRY(ctx, ctx->gsum.grow(((size_t)scan_chunks((uint32_t)P) + 8) * 4));
  CUDA_TRY(ctx, ctx->gbase_loc.grow((P / 32 + 8) * 4));
  CUDA_TRY(ctx, launch_scan(ms, ctx->gsum.as<uint32_t>(), ctx->gbase_loc.as<uint32_t>(), ctx->stream, &launches));
  // k_in slots per list: every list passes through verbatim (m <= k_in)
  return inflate(ctx, in->count, reinterpret_cast<const float2*>(in->depth), reinterpret_cast<const float4*>(in->rgba),
                 ctx->gbase_loc.as<uint32_t>(), P, cf.k_in, out->count, reinterpret_cast<float2*>(out->depth),
                 reinterpret_cast<float4*>(out->rgba), launches);
}

vdi_status vdi_composite_fullrep(vdi_ctx* ctx, const vdi_full_view* local, const uint32_t* pe_ids, uint32_t n_local,
                                 vdi_full_view* so) {
  VDI_NVTX("vdi_composite_fullrep");
  if (vdi_status s = check_ctx(ctx)) return s;
  const vdi_config& cf = ctx->cfg;
  const uint32_t G = cf.n_ranks, me = cf.rank, n = cf.n_pes, K = cf.k_in;
  if (!so || !so->count || !so->depth || !so->rgba) return fail(VDI_ERR_INVALID_ARG, "strip_out is NULL");
  if (so->row_begin != ctx->row0 || so->row_end != ctx->row1)
    return fail(VDI_ERR_CAPACITY, "strip_out rows do not match this rank's strip");
  std::vector<int> slot(n, -1);
  if (n_local != ctx->lay.n_local(me))
    return fail(VDI_ERR_INVALID_ARG, "rank %u homes %u PEs, got %u", me, ctx->lay.n_local(me), n_local);
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
  const uint64_t Pg = ctx->P;
  if (timing) CUDA_TRY(ctx, cudaEventRecord(ctx->ev[0], st));
  MergeParams mx{};
  if (G > 1) {
    // fixed-size slices of the full representation (no size exchange): pushed
    // into the same window slots as the dense exchange
    uint32_t e = 0;
    if (vdi_status s = exchange_push(ctx, nullptr, local, n_local, pe_ids, launches, st, 0, &e)) return s;
    if (vdi_status s = exchange_recv(ctx, nullptr, local, slot, e, 0, mx, launches)) return s;
  } else {
    for (uint32_t s = 0; s < n; ++s) {
      const vdi_full_view& v = local[slot[s]];
      mx.src[s] = SrcDesc{v.count, reinterpret_cast<const float2*>(v.depth), reinterpret_cast<const float4*>(v.rgba),
                          nullptr};
    }
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
  for (uint32_t s = 0; s < n; ++s) ms.src[s].count = mx.src[s].count;
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
    CUDA_TRY(ctx, launch_compact(mx.src[s].count, mx.src[s].depth, mx.src[s].rgba, (uint32_t)Pg, (int)K,
                                 ctx->xbase.as<uint32_t>() + (size_t)s * ng, dd, dc, st, &launches));
    mp.src[s] = SrcDesc{mx.src[s].count, dd, dc, nullptr};
  }
  unsigned long long S_here = 0;  // the paper's full pipeline: one size read-back before the merge
  CUDA_TRY(ctx, cudaMemcpyAsync(&S_here, dtot, 8, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(ctx, cudaStreamSynchronize(st));
  if (vdi_status e = merge_lists(ctx, mp, Pg, S_here, n * K, so, timing, launches)) return e;
  if (G > 1) {
    CUDA_TRY(ctx, cudaEventRecord(ctx->xev_merged[0], st));
    if (vdi_status s = release_slots(ctx, launches)) return s;
  }
  if (timing) {
    CUDA_TRY(ctx, cudaEventRecord(ctx->ev[2], st));
    ctx->timing_pending = true;
  }
  ctx->have_stats = cf.flags & VDI_FLAG_PIXEL_STATS;
  ctx->last = vdi_counters{};
  ctx->last.kernel_launches = (uint32_t)launches;
  return VDI_OK;
}

// Gather (a11), non-root side: compaction of the composited
// strip straight into root R's window (stream st), gather sequence number j
static vdi_status gather_send(vdi_ctx* ctx, const vdi_full_view* strip, uint32_t R, uint32_t j, cudaStream_t st,
                              int& launches) {
  const Layout& L = ctx->lay;
  const uint32_t me = ctx->cfg.rank, W = ctx->cfg.width, k = ctx->cfg.k_out;
  char* gp = ctx->peer[R] + L.g_off(R, j & 1);
  trace("gsend_begin", st);
  CUDA_TRY(ctx, cudaMemsetAsync(ctx->ccnt.as<unsigned long long>() + 1, 0, 8, st));
  if (j > (ctx->grp ? 1u : 2u)) {  // the root has inflated this buffer's previous contents
    if (vdi_status s = wait_flags(ctx, GFREE, {{R, j - 2, j - 1}}, st)) return s;
    ++launches;
  }
  trace("gsend_free", st);
  const uint32_t P = (uint32_t)ctx->P, ng = (P + 31) / 32;
  MergeParams ms{};
  ms.n_src = 1;
  ms.P = P;
  ms.n_groups = ng;
  ms.src[0].count = strip->count;
  CUDA_TRY(ctx, launch_scan(ms, ctx->gsum.as<uint32_t>(), ctx->gbase_loc.as<uint32_t>(), st, &launches));
  CompactPushArgs a{};
  a.count = strip->count;
  a.depth = reinterpret_cast<const float2*>(strip->depth);
  a.rgba = reinterpret_cast<const float4*>(strip->rgba);
  a.P = P;
  a.k = (int)k;
  a.group_base = ctx->gbase_loc.as<uint32_t>();
  a.region = (uint32_t)((size_t)ctx->row0 * W * k);
  a.region_cap = (unsigned long long)P * k;
  a.dst_count = reinterpret_cast<uint8_t*>(gp + L.g_count_off()) + (size_t)ctx->row0 * W;
  a.dst_gbase = reinterpret_cast<uint32_t*>(gp + L.g_gbase_off()) + L.gbase_index(me);
  a.dst_depth = reinterpret_cast<float2*>(gp + L.g_depth_off());
  a.dst_rgba = reinterpret_cast<float4*>(gp + L.g_rgba_off());
  a.total_out = reinterpret_cast<unsigned long long*>(gp + L.g_hdr_off()) + me;
  a.bytes = ctx->ccnt.as<unsigned long long>() + 1;
  a.flag = flag_at(ctx->peer[R], GREADY, me);
  CUDA_TRY(ctx, launch_compact_push(a, compact_push_blocks(P), st));
  ++launches;
  trace("gsend_end", st);
  if (ctx->grp) return loop_post(ctx, GREADY, {R}, j, st);
  return VDI_OK;
}

// Gather, root side (this rank is R): wait until every other rank's
// compaction j has landed, re-inflate their rows of `image` with the
// pass-through kernel, release the buffer (stream st)
static vdi_status gather_recv(vdi_ctx* ctx, vdi_full_view* image, uint32_t j, cudaStream_t st, int& launches) {
  const Layout& L = ctx->lay;
  const uint32_t G = ctx->cfg.n_ranks, R = ctx->cfg.rank, W = ctx->cfg.width, k = ctx->cfg.k_out;
  char* gp = ctx->peer[R] + L.g_off(R, j & 1);
  std::vector<WaitOn> wt;
  for (uint32_t g = 0; g < G; ++g)
    if (g != R) wt.push_back({g, j * compact_push_blocks(L.rows(g) * W), j});
  trace("grecv_wait", st);
  if (vdi_status s = wait_flags(ctx, GREADY, wt, st)) return s;
  ++launches;
  trace("grecv_ready", st);
  const uint8_t* gc = reinterpret_cast<const uint8_t*>(gp + L.g_count_off());
  const uint32_t* gb = reinterpret_cast<const uint32_t*>(gp + L.g_gbase_off());
  const float2* gd = reinterpret_cast<const float2*>(gp + L.g_depth_off());
  const float4* gr = reinterpret_cast<const float4*>(gp + L.g_rgba_off());
  auto infl = [&](size_t p0, size_t P, const uint32_t* gbp) -> vdi_status {
    return inflate(ctx, gc + p0, gd, gr, gbp, P, k, image->count + p0, reinterpret_cast<float2*>(image->depth) + p0 * k,
                   reinterpret_cast<float4*>(image->rgba) + p0 * k, launches, st);
  };
  if (L.aligned()) {  // the rows before and after the root's own strip: one launch each
    const size_t a0 = 0, a1 = (size_t)ctx->row0 * W, b0 = (size_t)ctx->row1 * W, b1 = L.img();
    if (vdi_status s = infl(a0, a1 - a0, gb + a0 / 32)) return s;
    if (vdi_status s = infl(b0, b1 - b0, gb + b0 / 32)) return s;
  } else {
    for (uint32_t g = 0; g < G; ++g)
      if (g != R)
        if (vdi_status s = infl((size_t)L.row0(g) * W, (size_t)L.rows(g) * W, gb + L.gbase_index(g))) return s;
  }
  std::vector<uint32_t> others;
  for (uint32_t g = 0; g < G; ++g)
    if (g != R) others.push_back(g);
  trace("grecv_inflated", st);
  if (vdi_status s = signal_peers(ctx, GFREE, others, j, st, j)) return s;
  ++launches;
  return VDI_OK;
}

// Gather (a11) of the composited strips onto rank R
static vdi_status gather_to(vdi_ctx* ctx, const vdi_full_view* strip, vdi_full_view* image, uint32_t R) {
  if (vdi_status s = check_ctx(ctx)) return s;
  const vdi_config& cf = ctx->cfg;
  const uint32_t G = cf.n_ranks, me = cf.rank, W = cf.width, k = cf.k_out;
  if (!strip || !strip->count || !strip->depth || !strip->rgba) return fail(VDI_ERR_INVALID_ARG, "strip is NULL");
  if (strip->row_begin != ctx->row0 || strip->row_end != ctx->row1)
    return fail(VDI_ERR_CAPACITY, "strip rows do not match this rank");
  if (R >= G) return fail(VDI_ERR_INVALID_ARG, "root %u >= n_ranks %u", R, G);
  const bool root = me == R;
  if (root && (!image || !image->count || !image->depth || !image->rgba || image->row_begin != 0 ||
               image->row_end != cf.height))
    return fail(VDI_ERR_INVALID_ARG, "root image_out must cover rows [0, H)");
  if (root && ((reinterpret_cast<uintptr_t>(image->rgba) & 15) || (reinterpret_cast<uintptr_t>(image->depth) & 7)))
    return fail(VDI_ERR_INVALID_ARG, "image_out depth/rgba must be 8/16-byte aligned");
  cudaStream_t st = ctx->stream;
  const bool timing = cf.flags & VDI_FLAG_STAGE_TIMING;
  if (timing) CUDA_TRY(ctx, cudaEventRecord(ctx->gev[0], st));
  auto copy_own = [&]() -> cudaError_t {
    const size_t P = ctx->P, o = (size_t)ctx->row0 * W;
    cudaError_t e = cudaSuccess;
    if (image->count + o != strip->count) e = cudaMemcpyAsync(image->count + o, strip->count, P, cudaMemcpyDeviceToDevice, st);
    if (e == cudaSuccess && image->depth + o * k * 2 != strip->depth)
      e = cudaMemcpyAsync(image->depth + o * k * 2, strip->depth, P * k * 8, cudaMemcpyDeviceToDevice, st);
    if (e == cudaSuccess && image->rgba + o * k * 4 != strip->rgba)
      e = cudaMemcpyAsync(image->rgba + o * k * 4, strip->rgba, P * k * 16, cudaMemcpyDeviceToDevice, st);
    return e;
  };
  int launches = 0;
  if (G == 1) {
    CUDA_TRY(ctx, copy_own());
  } else {
    // Dense gather: each rank compacts its composited lists
    // (counts + packed records) straight into the root's
    // window; the root re-inflates the full representation
    // with the pass-through kernel -- the image is bit-identical to gathering
    // the full representation
    if (vdi_status s = resolve_peers(ctx)) return s;
    const uint32_t j = ++ctx->gcalls_to[R];
    if (!root) {
      if (vdi_status s = gather_send(ctx, strip, R, j, st, launches)) return s;
    } else {
      if (vdi_status s = gather_recv(ctx, image, j, st, launches)) return s;
      CUDA_TRY(ctx, copy_own());
    }
    ctx->last_gather_root = (int)R;
    ctx->last_gather_parity = j & 1;
  }
  ctx->last.kernel_launches += (uint32_t)launches;
  if (timing) {
    CUDA_TRY(ctx, cudaEventRecord(ctx->gev[1], st));
    ctx->gather_timing_pending = true;
  }
  return VDI_OK;
}

vdi_status vdi_gather(vdi_ctx* ctx, const vdi_full_view* strip, vdi_full_view* image) {
  VDI_NVTX("vdi_gather");
  if (vdi_status s = check_ctx(ctx)) return s;
  return gather_to(ctx, strip, image, ctx->cfg.root);
}

vdi_status vdi_gather_root(vdi_ctx* ctx, uint32_t root, const vdi_full_view* strip, vdi_full_view* image) {
  VDI_NVTX("vdi_gather_root");
  return gather_to(ctx, strip, image, root);
}

// Frames in flight through strip mode: frame f =
// vdi_composite + vdi_gather onto roots[f], but the root merges its strip
// straight into the rows of images[f] and re-inflates the other rows on a
// second stream, so that its exchange and merge of frame f+1 do not wait for
// its inflate of frame f (and neither do the other ranks, whose next slices
// it pushes right after its merge).  Non-root strips: four ctx-owned buffers, each compacted to the root on its own stream.
vdi_status vdi_composite_frames(vdi_ctx* ctx, uint32_t F, const vdi_dense_view* local, uint32_t n_local,
                                vdi_full_view* images, const uint32_t* roots) {
  VDI_NVTX("vdi_composite_frames");
  if (vdi_status s = check_ctx(ctx)) return s;
  const vdi_config& cf = ctx->cfg;
  const uint32_t G = cf.n_ranks, me = cf.rank, W = cf.width, H = cf.height, k = cf.k_out;
  if (!F) return VDI_OK;
  if (!images || (n_local && !local)) return fail(VDI_ERR_INVALID_ARG, "images / local_pes is NULL");
  for (uint32_t f = 0; f < F; ++f) {
    const uint32_t R = roots ? roots[f] : cf.root;
    if (R >= G) return fail(VDI_ERR_INVALID_ARG, "roots[%u] = %u >= n_ranks", f, R);
    if (R != me) continue;
    const vdi_full_view& im = images[f];
    if (!im.count || !im.depth || !im.rgba || im.row_begin != 0 || im.row_end != H)
      return fail(VDI_ERR_INVALID_ARG, "images[%u] (root %u) must cover rows [0, H)", f, R);
    if ((reinterpret_cast<uintptr_t>(im.rgba) & 15) || (reinterpret_cast<uintptr_t>(im.depth) & 7))
      return fail(VDI_ERR_INVALID_ARG, "images[%u]: depth/rgba must be 8/16-byte aligned", f);
  }
  cudaStream_t st = ctx->stream;
  const size_t P = ctx->P, o = (size_t)ctx->row0 * W;
  if (G > 1)
    if (vdi_status s = resolve_peers(ctx)) return s;
  // frame f's search kernels run on the search stream beside frame f+1's
  // pass-through (not with VDI_FLAG_PIXEL_STATS: the statistics arrays are single)
  const bool overlap = !(cf.flags & VDI_FLAG_PIXEL_STATS);
  if (!ctx->sst) {
    CUDA_TRY(ctx, cudaStreamCreateWithFlags(&ctx->sst, cudaStreamNonBlocking));
    CUDA_TRY(ctx, cudaStreamCreateWithFlags(&ctx->xst, cudaStreamNonBlocking));
    CUDA_TRY(ctx, cudaStreamCreateWithFlags(&ctx->gst, cudaStreamNonBlocking));
    CUDA_TRY(ctx, cudaStreamCreateWithFlags(&ctx->gsst, cudaStreamNonBlocking));
    for (int i = 0; i < 2; ++i) CUDA_TRY(ctx, cudaEventCreateWithFlags(&ctx->sev_merged[i], cudaEventDisableTiming));
    for (int i = 0; i < vdi_ctx::kStripBufs; ++i)
      CUDA_TRY(ctx, cudaEventCreateWithFlags(&ctx->fsev[i], cudaEventDisableTiming));
    CUDA_TRY(ctx, cudaEventCreateWithFlags(&ctx->gev_in, cudaEventDisableTiming));
    CUDA_TRY(ctx, cudaEventCreateWithFlags(&ctx->gev_out, cudaEventDisableTiming));
    for (int i = 0; i < 2; ++i) {
      CUDA_TRY(ctx, cudaEventCreateWithFlags(&ctx->mev_fast[i], cudaEventDisableTiming));
      CUDA_TRY(ctx, cudaEventCreateWithFlags(&ctx->mev_done[i], cudaEventDisableTiming));
    }
  }
  if (G > 1)
    for (uint32_t i = 0; i < std::min<uint32_t>(F, vdi_ctx::kStripBufs); ++i) {
      CUDA_TRY(ctx, ctx->fs_count[i].grow(P));
      CUDA_TRY(ctx, ctx->fs_depth[i].grow(P * k * 8));
      CUDA_TRY(ctx, ctx->fs_rgba[i].grow(P * k * 16));
    }
  // the side streams start once the caller's stream has reached this call
  CUDA_TRY(ctx, cudaEventRecord(ctx->gev_in, st));
  for (cudaStream_t x : {ctx->gst, ctx->gsst, ctx->xst, ctx->sst}) CUDA_TRY(ctx, cudaStreamWaitEvent(x, ctx->gev_in, 0));
  int launches = 0;
  vdi_status err = VDI_OK;
  for (uint32_t f = 0; f < F && err == VDI_OK; ++f) {
    const uint32_t R = roots ? roots[f] : cf.root;
    const int b = (int)(f & 1);
    vdi_full_view so;
    if (G == 1) {
      so = vdi_full_view{0, H, images[f].count, images[f].depth, images[f].rgba};
    } else if (R == me) {  // the root's strip is its image rows
      so = vdi_full_view{ctx->row0, ctx->row1, images[f].count + o, images[f].depth + o * k * 2,
                         images[f].rgba + o * k * 4};
    } else {  // a ctx-owned strip buffer; frame f - kStripBufs's gather send must have read it
      const int sb = (int)(f % vdi_ctx::kStripBufs);
      so = vdi_full_view{ctx->row0, ctx->row1, ctx->fs_count[sb].as<uint8_t>(), ctx->fs_depth[sb].as<float>(),
                         ctx->fs_rgba[sb].as<float>()};
      if (f >= (uint32_t)vdi_ctx::kStripBufs) CUDA_TRY(ctx, cudaStreamWaitEvent(st, ctx->fsev[sb], 0));
    }
    // frame f's push runs on the push stream beside frame f-1's merge; its
    // double-buffered exchange arrays wait for the merge of frame f-2
    ctx->mpar = b;
    ctx->msst = overlap ? ctx->sst : nullptr;
    if (G > 1) {
      ctx->xpst = ctx->xst;
      ctx->xpar = b;
      if (f >= 2) err = cudaStreamWaitEvent(ctx->xst, ctx->xev_merged[b], 0) == cudaSuccess ? VDI_OK : VDI_ERR_CUDA;
    }
    g_trace_frame = (int)f;
    if (err == VDI_OK) err = vdi_composite(ctx, local + (size_t)f * n_local, n_local, &so);
    ctx->xpst = nullptr;
    ctx->xpar = 0;
    ctx->mpar = 0;
    ctx->msst = nullptr;
    if (err != VDI_OK) break;
    launches += ctx->last.kernel_launches;
    cudaStream_t es = overlap ? ctx->sst : st;  // the stream the frame's merge ends on
    if (G > 1) {
      const uint32_t j = ++ctx->gcalls_to[R];
      if (R != me) {  // the compaction on its own stream: the next frame's search does not wait for it
        CUDA_TRY(ctx, cudaEventRecord(ctx->sev_merged[b], es));
        CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->gsst, ctx->sev_merged[b], 0));
        err = gather_send(ctx, &so, R, j, ctx->gsst, launches);
        if (err == VDI_OK) CUDA_TRY(ctx, cudaEventRecord(ctx->fsev[f % vdi_ctx::kStripBufs], ctx->gsst));
      } else {
        err = gather_recv(ctx, &images[f], j, ctx->gst, launches);
      }
      ctx->last_gather_root = (int)R;
      ctx->last_gather_parity = j & 1;
    }
    g_trace_frame = -1;
    // this parity's merge scratch is free again
    if (err == VDI_OK && overlap) CUDA_TRY(ctx, cudaEventRecord(ctx->mev_done[b], es));
  }
  if (err != VDI_OK) return err;
  // the call ends on the caller's stream once the side streams have too
  for (cudaStream_t x : {ctx->gst, ctx->gsst, ctx->xst, ctx->sst}) {
    CUDA_TRY(ctx, cudaEventRecord(ctx->gev_out, x));
    CUDA_TRY(ctx, cudaStreamWaitEvent(st, ctx->gev_out, 0));
  }
  ctx->last.kernel_launches = (uint32_t)launches;
  g_trace_rank = (int)me;
  trace_dump(st);
  return VDI_OK;
}

// H2D of the host sub-VDIs into input slot `set` (0/1: the double-buffered
// frames pipeline) on stream st; dv gets device views (no offset arrays: the
// strip bounds / group bases are scanned from the counts on the device)
static vdi_status upload_host_pes(vdi_ctx* ctx, const vdi_dense_view* local, uint32_t n_local,
                                  std::vector<vdi_dense_view>& dv, int set, cudaStream_t st) {
  const vdi_config& cf = ctx->cfg;
  if (n_local && !local) return fail(VDI_ERR_INVALID_ARG, "local_pes is NULL");
  if (n_local > cf.n_pes) return fail(VDI_ERR_INVALID_ARG, "too many local PEs");
  const size_t P = (size_t)cf.width * cf.height;
  dv.assign(n_local, vdi_dense_view{});
  for (uint32_t l = 0; l < n_local; ++l) {
    const vdi_dense_view& v = local[l];
    if (!v.count || (v.total && (!v.depth || !v.rgba))) return fail(VDI_ERR_INVALID_ARG, "host view %u has NULL arrays", l);
  }
  if (cf.flags & VDI_FLAG_HOST_SPAN) {
    // the caller promises that the arrays of a call lie in one host
    // allocation (e.g. a pinned arena): ONE copy of their span instead of
    // 3 per PE (many mid-sized H2D copies run the host link at ~80 % of one
    // large copy, profiles/pipeline_probe.py); device views keep the arrays'
    // offsets inside the span (alignment mod 256 preserved)
    uintptr_t lo = UINTPTR_MAX, hi = 0;
    bool aligned = true;
    auto add = [&](const void* p, size_t nb, size_t al) {
      if (!nb) return;
      const uintptr_t a = reinterpret_cast<uintptr_t>(p);
      lo = std::min(lo, a);
      hi = std::max(hi, a + nb);
      aligned &= (a % al) == 0;
    };
    for (uint32_t l = 0; l < n_local; ++l) {
      add(local[l].count, P, 1);
      add(local[l].depth, local[l].total * 8, 8);
      add(local[l].rgba, local[l].total * 16, 16);
    }
    if (!aligned) return fail(VDI_ERR_INVALID_ARG, "VDI_FLAG_HOST_SPAN: depth/rgba must be 8/16-byte aligned");
    if (hi > lo) {
      lo &= ~(uintptr_t)255;
      const size_t span = hi - lo;
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
        dv[l].offset = nullptr;
      }
      return VDI_OK;
    }
  }
  ctx->hcount[set].resize(std::max<size_t>(ctx->hcount[set].size(), n_local));
  ctx->hdepth[set].resize(std::max<size_t>(ctx->hdepth[set].size(), n_local));
  ctx->hrgba[set].resize(std::max<size_t>(ctx->hrgba[set].size(), n_local));
  for (uint32_t l = 0; l < n_local; ++l) {
    const vdi_dense_view& v = local[l];
    DevBuf &hc = ctx->hcount[set][l], &hd = ctx->hdepth[set][l], &hr = ctx->hrgba[set][l];
    CUDA_TRY(ctx, hc.grow(P));
    CUDA_TRY(ctx, hd.grow(std::max<uint64_t>(v.total, 1) * 8));
    CUDA_TRY(ctx, hr.grow(std::max<uint64_t>(v.total, 1) * 16));
    CUDA_TRY(ctx, cudaMemcpyAsync(hc.p, v.count, P, cudaMemcpyHostToDevice, st));
    if (v.total) {
      CUDA_TRY(ctx, cudaMemcpyAsync(hd.p, v.depth, v.total * 8, cudaMemcpyHostToDevice, st));
      CUDA_TRY(ctx, cudaMemcpyAsync(hr.p, v.rgba, v.total * 16, cudaMemcpyHostToDevice, st));
    }
    dv[l] = v;
    dv[l].count = hc.as<uint8_t>();
    dv[l].depth = hd.as<float>();
    dv[l].rgba = hr.as<float>();
    dv[l].offset = nullptr;
  }
  return VDI_OK;
}

vdi_status vdi_composite_host(vdi_ctx* ctx, const vdi_dense_view* local, uint32_t n_local, vdi_full_view* so) {
  VDI_NVTX("vdi_composite_host");
  if (vdi_status s = check_ctx(ctx)) return s;
  const vdi_config& cf = ctx->cfg;
  if (!so || !so->count || !so->depth || !so->rgba) return fail(VDI_ERR_INVALID_ARG, "strip_out is NULL");
  if (so->row_begin != ctx->row0 || so->row_end != ctx->row1)
    return fail(VDI_ERR_CAPACITY, "strip_out rows do not match this rank's strip");
  cudaStream_t st = ctx->stream;
  std::vector<vdi_dense_view> dv;
  if (vdi_status s = upload_host_pes(ctx, local, n_local, dv, 0, st)) return s;
  const size_t Ps = ctx->P, k = cf.k_out;
  CUDA_TRY(ctx, ctx->hstrip_count.grow(Ps));
  CUDA_TRY(ctx, ctx->hstrip_depth.grow(Ps * k * 8));
  CUDA_TRY(ctx, ctx->hstrip_rgba.grow(Ps * k * 16));
  vdi_full_view ds{ctx->row0, ctx->row1, ctx->hstrip_count.as<uint8_t>(), ctx->hstrip_depth.as<float>(),
                   ctx->hstrip_rgba.as<float>()};
  if (vdi_status s = vdi_composite(ctx, dv.data(), n_local, &ds)) return s;
  CUDA_TRY(ctx, cudaMemcpyAsync(so->count, ds.count, Ps, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(ctx, cudaMemcpyAsync(so->depth, ds.depth, Ps * k * 8, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(ctx, cudaMemcpyAsync(so->rgba, ds.rgba, Ps * k * 16, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(ctx, cudaStreamSynchronize(st));
  return VDI_OK;
}

// composited strip (device, full representation) -> dense representation in
// `pc` (counts) / dd2, dc4 (packed records); total into *tot (device)
static vdi_status compact_strip(vdi_ctx* ctx, const vdi_full_view& ds, unsigned long long* tot, float2* dd2,
                                float4* dc4, bool do_compact, int& launches) {
  const size_t Ps = ctx->P, ng = (Ps + 31) / 32;
  cudaStream_t st = ctx->stream;
  CUDA_TRY(ctx, ctx->xsum.grow(((size_t)scan_chunks((uint32_t)std::max<size_t>(Ps, 1)) + 8) * 4));
  CUDA_TRY(ctx, ctx->xbase.grow((ng + 8) * 4));
  MergeParams ms{};
  ms.n_src = 1;
  ms.P = (uint32_t)Ps;
  ms.n_groups = (uint32_t)ng;
  ms.src[0].count = ds.count;
  if (!Ps) {
    CUDA_TRY(ctx, cudaMemsetAsync(tot, 0, 8, st));
    return VDI_OK;
  }
  CUDA_TRY(ctx, launch_scan(ms, ctx->xsum.as<uint32_t>(), ctx->xbase.as<uint32_t>(), st, &launches));
  CUDA_TRY(ctx, launch_total(ms, ctx->xsum.as<uint32_t>(), tot, st, &launches));
  if (do_compact)
    CUDA_TRY(ctx, launch_compact(ds.count, reinterpret_cast<const float2*>(ds.depth),
                                 reinterpret_cast<const float4*>(ds.rgba), (uint32_t)Ps, (int)ctx->cfg.k_out,
                                 ctx->xbase.as<uint32_t>(), dd2, dc4, st, &launches));
  return VDI_OK;
}

vdi_status vdi_composite_host_dense(vdi_ctx* ctx, const vdi_dense_view* local, uint32_t n_local,
                                    vdi_dense_strip* out) {
  VDI_NVTX("vdi_composite_host_dense");
  if (vdi_status s = check_ctx(ctx)) return s;
  const vdi_config& cf = ctx->cfg;
  if (!out || !out->count || (out->capacity && (!out->depth || !out->rgba)))
    return fail(VDI_ERR_INVALID_ARG, "out is NULL");
  if (out->row_begin != ctx->row0 || out->row_end != ctx->row1)
    return fail(VDI_ERR_CAPACITY, "out rows do not match this rank's strip");
  cudaStream_t st = ctx->stream;
  std::vector<vdi_dense_view> dv;
  if (vdi_status s = upload_host_pes(ctx, local, n_local, dv, 0, st)) return s;
  const size_t Ps = ctx->P, k = cf.k_out;
  CUDA_TRY(ctx, ctx->hstrip_count.grow(Ps));
  CUDA_TRY(ctx, ctx->hstrip_depth.grow(Ps * k * 8));
  CUDA_TRY(ctx, ctx->hstrip_rgba.grow(Ps * k * 16));
  vdi_full_view ds{ctx->row0, ctx->row1, ctx->hstrip_count.as<uint8_t>(), ctx->hstrip_depth.as<float>(),
                   ctx->hstrip_rgba.as<float>()};
  if (vdi_status s = vdi_composite(ctx, dv.data(), n_local, &ds)) return s;
  // the composited strip in the dense representation:
  // scan of its counts, packed copy of its records, then only those bytes
  // cross PCIe
  int launches = 0;
  CUDA_TRY(ctx, ctx->xtot.grow(64));
  unsigned long long T = 0;
  if (vdi_status s = compact_strip(ctx, ds, ctx->xtot.as<unsigned long long>(), nullptr, nullptr, false, launches))
    return s;
  CUDA_TRY(ctx, cudaMemcpyAsync(&T, ctx->xtot.p, 8, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(ctx, cudaStreamSynchronize(st));
  out->total = T;
  if (T > out->capacity)
    return fail(VDI_ERR_CAPACITY, "dense strip needs %llu supersegments, capacity %llu", T,
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

// Pipelined vdi_composite_host_dense over independent frames: frame f's H2D
// (stream pin_st, input slot f&1) overlaps frame f-1's compositing (ctx
// stream) and frame f-2's D2H (stream pout_st, output slot f&1).  Each frame
// is exactly one vdi_composite + dense compaction, as in the single call.
vdi_status vdi_composite_host_dense_frames(vdi_ctx* ctx, uint32_t F, const vdi_dense_view* local, uint32_t n_local,
                                           vdi_dense_strip* outs) {
  VDI_NVTX("vdi_composite_host_dense_frames");
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
    // the first frames wait on these before any slot was used
    for (int i = 0; i < 2; ++i) {
      CUDA_TRY(ctx, cudaEventRecord(ctx->pev_used[i], st));
      CUDA_TRY(ctx, cudaEventRecord(ctx->pev_out[i], st));
    }
  }
  const size_t Ps = ctx->P, k = cf.k_out, Tmax = std::max<size_t>(Ps * k, 1);  // a strip holds <= Ps*k
  CUDA_TRY(ctx, ctx->hstrip_depth.grow(Ps * k * 8));
  CUDA_TRY(ctx, ctx->hstrip_rgba.grow(Ps * k * 16));
  for (int i = 0; i < 2; ++i) {
    CUDA_TRY(ctx, ctx->pcount[i].grow(std::max<size_t>(Ps, 1)));
    CUDA_TRY(ctx, ctx->pdense[i].grow(Tmax * 24));
  }
  // the strip's counts go straight to the output slot (read by the D2H);
  // its records to the shared full-representation scratch (read by the compaction)
  vdi_full_view ds{ctx->row0, ctx->row1, nullptr, ctx->hstrip_depth.as<float>(), ctx->hstrip_rgba.as<float>()};
  std::vector<vdi_dense_view> dv[2];
  int launches = 0;
  // H2D of frame f into slot f&1 once the compositing of frame f-2 has read it
  // (at n_ranks > 1 only this rank reads its input slots: the exchange pushes
  // from them inside that compositing)
  auto h2d = [&](uint32_t f) -> vdi_status {
    const int sl = f & 1;
    CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->pin_st, ctx->pev_used[sl], 0));
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
    float4* dc4 = ctx->pdense[sl].as<float4>();
    float2* dd2 = reinterpret_cast<float2*>(dc4 + Tmax);
    // the total is stored by the kernel into mapped host memory (no copy-engine hop)
    if (vdi_status s = compact_strip(ctx, ds, ctx->ptot_dev + sl, dd2, dc4, true, launches)) return s;
    CUDA_TRY(ctx, cudaEventRecord(ctx->pev_tot[sl], st));
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
  // order: H2D(f+1) is queued before the host waits for frame f's total
  if (vdi_status s = h2d(0)) return s;
  if (vdi_status s = compute(0)) return s;
  for (uint32_t f = 0; f < F; ++f) {
    if (f + 1 < F)
      if (vdi_status s = h2d(f + 1)) return s;
    if (f + 1 < F)
      if (vdi_status s = compute(f + 1)) return s;
    if (vdi_status s = d2h(f)) return s;
  }
  CUDA_TRY(ctx, cudaStreamSynchronize(ctx->pout_st));
  CUDA_TRY(ctx, cudaStreamSynchronize(ctx->pin_st));
  CUDA_TRY(ctx, cudaStreamSynchronize(st));
  ctx->last.kernel_launches += (uint32_t)launches;
  return first_err;
}

// ---------------------------------------------------------------------------
// The limit case and the renderers
// ---------------------------------------------------------------------------
vdi_status vdi_composite_image(vdi_ctx* ctx, const vdi_dense_view* local, uint32_t n_local, float* strip_rgba) {
  VDI_NVTX("vdi_composite_image");
  if (vdi_status s = check_ctx(ctx)) return s;
  const vdi_config& cf = ctx->cfg;
  const uint32_t G = cf.n_ranks, n = cf.n_pes;
  if (!strip_rgba || (reinterpret_cast<uintptr_t>(strip_rgba) & 15))
    return fail(VDI_ERR_INVALID_ARG, "strip_rgba is NULL or not 16-byte aligned");
  std::vector<int> slot;
  if (vdi_status s = check_local(ctx, local, n_local, slot)) return s;
  cudaStream_t st = ctx->stream;
  int launches = 0;
  MergeParams mp{};
  mp.n_src = (int)n;
  mp.P = (uint32_t)ctx->P;
  mp.n_groups = (uint32_t)((ctx->P + 31) / 32);
  if (G == 1) {
    for (uint32_t s = 0; s < n; ++s) {
      const vdi_dense_view& v = local[slot[s]];
      mp.src[s] = SrcDesc{v.count, reinterpret_cast<const float2*>(v.depth), reinterpret_cast<const float4*>(v.rgba),
                          v.offset, nullptr};
    }
  } else {
    uint32_t e = 0;
    if (vdi_status s = exchange_push(ctx, local, nullptr, n_local, nullptr, launches, st, 0, &e)) return s;
    if (vdi_status s = exchange_recv(ctx, local, nullptr, slot, e, 0, mp, launches)) return s;
  }
  bool scan = false;
  for (uint32_t s = 0; s < n; ++s) scan |= !mp.src[s].offset && !mp.src[s].gbase;
  CUDA_TRY(ctx, ctx->group_sum.grow((size_t)scan_chunks(mp.P) * n * 4 + 64));
  CUDA_TRY(ctx, ctx->group_base.grow((size_t)mp.n_groups * n * 4 + 64));
  mp.group_base = ctx->group_base.as<uint32_t>();
  if (scan && mp.P)
    CUDA_TRY(ctx, launch_scan(mp, ctx->group_sum.as<uint32_t>(), ctx->group_base.as<uint32_t>(), st, &launches));
  CUDA_TRY(ctx, launch_image(mp, reinterpret_cast<float4*>(strip_rgba), st));
  ++launches;
  if (G > 1) {
    CUDA_TRY(ctx, cudaEventRecord(ctx->xev_merged[0], st));
    if (vdi_status s = release_slots(ctx, launches)) return s;
  }
  ctx->last = vdi_counters{};
  ctx->last.kernel_launches = (uint32_t)launches;
  return VDI_OK;
}

vdi_status vdi_gather_image(vdi_ctx* ctx, const float* strip_rgba, float* image_rgba) {
  VDI_NVTX("vdi_gather_image");
  if (vdi_status s = check_ctx(ctx)) return s;
  const vdi_config& cf = ctx->cfg;
  const Layout& L = ctx->lay;
  const uint32_t G = cf.n_ranks, me = cf.rank, W = cf.width, R = cf.root;
  if (!strip_rgba) return fail(VDI_ERR_INVALID_ARG, "strip_rgba is NULL");
  if (me == R && !image_rgba) return fail(VDI_ERR_INVALID_ARG, "image_rgba is NULL on the root");
  cudaStream_t st = ctx->stream;
  const size_t o = (size_t)ctx->row0 * W;
  int launches = 0;
  if (G == 1) {
    if (image_rgba != strip_rgba)
      CUDA_TRY(ctx, cudaMemcpyAsync(image_rgba, strip_rgba, ctx->P * 16, cudaMemcpyDeviceToDevice, st));
    return VDI_OK;
  }
  if (vdi_status s = resolve_peers(ctx)) return s;
  const uint32_t j = ++ctx->gcalls_to[R];
  char* gp = ctx->peer[R] + L.g_off(R, j & 1);
  float4* win = reinterpret_cast<float4*>(gp + L.g_rgba_off());  // the rows of the image, W*H float4
  if (me != R) {
    if (j > (ctx->grp ? 1u : 2u)) {
      if (vdi_status s = wait_flags(ctx, GFREE, {{R, j - 2, j - 1}}, st)) return s;
      ++launches;
    }
    CUDA_TRY(ctx, launch_rows_push(reinterpret_cast<const float4*>(strip_rgba), win + o, (uint32_t)ctx->P,
                                   compact_push_blocks((uint32_t)ctx->P), flag_at(ctx->peer[R], GREADY, me), st));
    ++launches;
    if (ctx->grp)
      if (vdi_status s = loop_post(ctx, GREADY, {R}, j, st)) return s;
  } else {
    std::vector<WaitOn> wt;
    std::vector<uint32_t> others;
    for (uint32_t g = 0; g < G; ++g)
      if (g != R) {
        wt.push_back({g, j * compact_push_blocks(L.rows(g) * W), j});
        others.push_back(g);
      }
    if (vdi_status s = wait_flags(ctx, GREADY, wt, st)) return s;
    ++launches;
    const size_t a1 = o, b0 = (size_t)ctx->row1 * W, img = L.img();
    float4* im = reinterpret_cast<float4*>(image_rgba);
    if (a1) CUDA_TRY(ctx, cudaMemcpyAsync(im, win, a1 * 16, cudaMemcpyDeviceToDevice, st));
    if (img > b0) CUDA_TRY(ctx, cudaMemcpyAsync(im + b0, win + b0, (img - b0) * 16, cudaMemcpyDeviceToDevice, st));
    if (image_rgba + o * 4 != strip_rgba)
      CUDA_TRY(ctx, cudaMemcpyAsync(im + o, strip_rgba, ctx->P * 16, cudaMemcpyDeviceToDevice, st));
    if (vdi_status s = signal_peers(ctx, GFREE, others, j, st, j)) return s;
    ++launches;
  }
  ctx->last.kernel_launches += (uint32_t)launches;
  return VDI_OK;
}

vdi_status vdi_render_generation_view(vdi_ctx* ctx, const vdi_full_view* vdi, float* out_rgba) {
  VDI_NVTX("vdi_render_generation_view");
  if (vdi_status s = check_ctx(ctx)) return s;
  if (!vdi || !vdi->count || !vdi->rgba || !out_rgba || vdi->row_end < vdi->row_begin)
    return fail(VDI_ERR_INVALID_ARG, "vdi / out_rgba is NULL");
  if ((reinterpret_cast<uintptr_t>(vdi->rgba) | reinterpret_cast<uintptr_t>(out_rgba)) & 15)
    return fail(VDI_ERR_INVALID_ARG, "rgba arrays must be 16-byte aligned");
  const uint32_t P = (vdi->row_end - vdi->row_begin) * ctx->cfg.width;
  CUDA_TRY(ctx, launch_gen_view(vdi->count, reinterpret_cast<const float4*>(vdi->rgba), P, (int)ctx->cfg.k_out,
                                reinterpret_cast<float4*>(out_rgba), ctx->stream));
  return VDI_OK;
}

static CamF camf(const vdi_camera& c) {
  CamF f;
  for (int a = 0; a < 3; ++a) {
    f.eye[a] = c.eye[a];
    f.fwd[a] = c.fwd[a];
    f.right[a] = c.right[a];
    f.up[a] = c.up[a];
  }
  f.tan_x = c.tan_x;
  f.tan_y = c.tan_y;
  return f;
}

vdi_status vdi_render_novel_view(vdi_ctx* ctx, const vdi_full_view* vdi, const vdi_camera* gen_cam,
                                 const vdi_camera* view_cam, const uint32_t dims[3], uint32_t w_out, uint32_t h_out,
                                 float* out_rgba) {
  VDI_NVTX("vdi_render_novel_view");
  if (vdi_status s = check_ctx(ctx)) return s;
  const vdi_config& cf = ctx->cfg;
  if (!vdi || !vdi->count || !vdi->depth || !vdi->rgba || !gen_cam || !view_cam || !dims || !out_rgba)
    return fail(VDI_ERR_INVALID_ARG, "NULL argument");
  if (vdi->row_begin != 0 || vdi->row_end != cf.height) return fail(VDI_ERR_INVALID_ARG, "vdi must cover rows [0, H)");
  if (!w_out || !h_out || !dims[0] || !dims[1] || !dims[2]) return fail(VDI_ERR_INVALID_ARG, "empty image or volume");
  if ((reinterpret_cast<uintptr_t>(vdi->rgba) | reinterpret_cast<uintptr_t>(out_rgba)) & 15)
    return fail(VDI_ERR_INVALID_ARG, "rgba arrays must be 16-byte aligned");
  NovelParams np{};
  np.count = vdi->count;
  np.depth = reinterpret_cast<const float2*>(vdi->depth);
  np.rgba = reinterpret_cast<const float4*>(vdi->rgba);
  np.W = cf.width;
  np.H = cf.height;
  np.k = (int)cf.k_out;
  np.gen = camf(*gen_cam);
  np.view = camf(*view_cam);
  const uint32_t md = std::max(dims[0], std::max(dims[1], dims[2]));
  for (int a = 0; a < 3; ++a) np.half[a] = (float)dims[a] / (2.0f * (float)md);
  np.dt = 1.0f / (float)md;
  np.W_out = w_out;
  np.H_out = h_out;
  np.out = reinterpret_cast<float4*>(out_rgba);
  CUDA_TRY(ctx, launch_novel_view(np, ctx->stream));
  return VDI_OK;
}

vdi_status vdi_render_dvr(vdi_ctx* ctx, const vdi_volume_desc* vol, const vdi_tf_desc* tf, const vdi_camera* cam,
                          uint32_t w_out, uint32_t h_out, float* out_rgba) {
  VDI_NVTX("vdi_render_dvr");
  if (vdi_status s = check_ctx(ctx)) return s;
  if (!vol || !tf || !cam || !out_rgba || !vol->voxels || !tf->table) return fail(VDI_ERR_INVALID_ARG, "NULL argument");
  if (vol->bytes_per_voxel != 1 && vol->bytes_per_voxel != 2)
    return fail(VDI_ERR_INVALID_ARG, "bytes_per_voxel must be 1 or 2");
  if (!w_out || !h_out || !vol->dims[0] || !vol->dims[1] || !vol->dims[2])
    return fail(VDI_ERR_INVALID_ARG, "empty image or volume");
  if (reinterpret_cast<uintptr_t>(out_rgba) & 15) return fail(VDI_ERR_INVALID_ARG, "out_rgba must be 16-byte aligned");
  GenParams gp{};
  gp.vox = vol->voxels;
  gp.bytes = (int)vol->bytes_per_voxel;
  for (int a = 0; a < 3; ++a) {
    gp.dims[a] = (int)vol->dims[a];
    gp.eye[a] = cam->eye[a];
    gp.fwd[a] = cam->fwd[a];
    gp.right[a] = cam->right[a];
    gp.up[a] = cam->up[a];
  }
  gp.tf = reinterpret_cast<const float4*>(tf->table);
  gp.tan_x = cam->tan_x;
  gp.tan_y = cam->tan_y;
  gp.W = (int)w_out;
  gp.H = (int)h_out;
  CUDA_TRY(ctx, launch_dvr(gp, reinterpret_cast<float4*>(out_rgba), ctx->stream));
  return VDI_OK;
}

vdi_status vdi_pixel_stats(vdi_ctx* ctx, float* gamma, float* min_margin, uint16_t* m) {
  if (vdi_status s = check_ctx(ctx)) return s;
  if (!ctx->have_stats) return fail(VDI_ERR_STATE, "VDI_FLAG_PIXEL_STATS was not set for the last composite");
  if (gamma)
    CUDA_TRY(ctx, cudaMemcpyAsync(gamma, ctx->stat_gamma.p, ctx->mP * 4, cudaMemcpyDeviceToDevice, ctx->stream));
  if (min_margin)
    CUDA_TRY(ctx, cudaMemcpyAsync(min_margin, ctx->stat_margin.p, ctx->mP * 4, cudaMemcpyDeviceToDevice, ctx->stream));
  if (m) CUDA_TRY(ctx, cudaMemcpyAsync(m, ctx->stat_m.p, ctx->mP * 2, cudaMemcpyDeviceToDevice, ctx->stream));
  return VDI_OK;
}

vdi_status vdi_get_counters(vdi_ctx* ctx, vdi_counters* out) {
  if (vdi_status s = check_ctx(ctx)) return s;
  if (!out) return fail(VDI_ERR_INVALID_ARG, "out is NULL");
  const vdi_config& cf = ctx->cfg;
  const Layout& L = ctx->lay;
  DevCounters h{};
  if (ctx->ms[ctx->last_mpar].dcnt.p)
    CUDA_TRY(ctx, cudaMemcpyAsync(&h, ctx->ms[ctx->last_mpar].dcnt.p, sizeof h, cudaMemcpyDeviceToHost, ctx->stream));
  unsigned long long cc[3] = {0, 0, 0};
  if (ctx->ccnt.p) CUDA_TRY(ctx, cudaMemcpyAsync(cc, ctx->ccnt.p, 24, cudaMemcpyDeviceToHost, ctx->stream));
  // records received in the last exchange (slot headers) and, at the root,
  // in the last gather (region headers)
  const uint32_t G = cf.n_ranks, me = cf.rank;
  std::vector<unsigned long long> xh, gh;
  if (G > 1 && ctx->xcalls) {
    const uint32_t q = ctx->xcalls & 1;
    for (uint32_t s = 0; s < cf.n_pes; ++s)
      if (L.home(s) != me) {
        xh.push_back(0);
        CUDA_TRY(ctx, cudaMemcpyAsync(&xh.back(), ctx->peer[me] + L.x_off(me, q, s), 8, cudaMemcpyDeviceToHost,
                                      ctx->stream));
      }
  }
  if (G > 1 && ctx->last_gather_root == (int)me) {
    gh.assign(G, 0);
    CUDA_TRY(ctx, cudaMemcpyAsync(gh.data(), ctx->peer[me] + L.g_off(me, ctx->last_gather_parity) + L.g_hdr_off(),
                                  (size_t)G * 8, cudaMemcpyDeviceToHost, ctx->stream));
  }
  CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  if (h.err & 1) return fail(VDI_ERR_INTERNAL, "merge work-list overflow");
  if (cc[2]) return fail(VDI_ERR_INTERNAL, "loopback: %llu flag words short of their targets", cc[2]);
  ctx->last.records_in = h.records_in;
  ctx->last.records_search = h.records_search;
  ctx->last.searched_lists = 0;
  for (int b = 0; b < VDI_N_BUCKETS; ++b) ctx->last.searched_lists += h.wl_count[b];
  for (int b = 0; b < 4; ++b) ctx->last.bucket_lists[b] = h.wl_count[b];
  ctx->last.general_lists = h.wl_count[VDI_BUCKET_GENERAL];
  ctx->last.fallback_groups = h.fallback_groups;
  ctx->last.sweep_steps = h.sweep_steps;
  ctx->last.bytes_sent = cc[0];
  ctx->last.bytes_received = 0;
  for (unsigned long long t : xh) ctx->last.bytes_received += ctx->P + 24ull * t;
  if (ctx->last_gather_root == (int)me && G > 1) {
    ctx->last.bytes_gather = 0;
    for (uint32_t g = 0; g < G; ++g)
      if (g != me) {
        const uint64_t Pg = (uint64_t)L.rows(g) * cf.width;
        ctx->last.bytes_gather += Pg + 4 * ((Pg + 31) / 32) + 24ull * gh[g];
      }
  } else {
    ctx->last.bytes_gather = cc[1];
  }
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
  if (ctx->gather_timing_pending) {
    CUDA_TRY(ctx, cudaEventElapsedTime(&ctx->last.ms_gather, ctx->gev[0], ctx->gev[1]));
    ctx->gather_timing_pending = false;
  }
  if (ctx->push_timing_pending) {
    CUDA_TRY(ctx, cudaEventElapsedTime(&ctx->last.ms_push, ctx->pev_t[0], ctx->pev_t[1]));
    ctx->push_timing_pending = false;
  }
  *out = ctx->last;
  return VDI_OK;
}

}  // extern "C"
