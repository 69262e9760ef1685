/*
 * vdi.h — C ABI of libvdi: B200-native sort-last parallel compositing of
 * Volumetric Depth Images (arXiv 2206.14503).
 *
 * Citations "PAPER.md:N" are lines of the paper text; readings Qn / Gn are
 * listed in DESIGN.md §2.  All device pointers are CUDA global-memory
 * pointers on the calling process's current device; all work is enqueued on
 * vdi_config.cuda_stream.  No C++ or torch types cross this boundary.
 *
 * Error behaviour: every call returns a vdi_status; no exception crosses the
 * ABI.  vdi_last_error() gives the detail text.  After a CUDA or NCCL error a
 * context is poisoned: later calls return VDI_ERR_STATE; destroy it.
 * Threading: a context is single-threaded; separate contexts are independent.
 */
#ifndef VDI_H_
#define VDI_H_

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#pragma GCC visibility push(default) /* the library is built with -fvisibility=hidden */
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  VDI_OK = 0,
  VDI_ERR_INVALID_ARG = 1,   /* bad pointer / size / config value */
  VDI_ERR_OUT_OF_MEMORY = 2, /* cudaMalloc failed */
  VDI_ERR_CUDA = 3,          /* CUDA runtime error (context poisoned) */
  VDI_ERR_NCCL = 4,          /* NCCL error (context poisoned) */
  VDI_ERR_STATE = 5,         /* context poisoned or call out of order */
  VDI_ERR_CAPACITY = 6,      /* caller buffer too small, or a ray needs > k supersegments (Q20) */
  VDI_ERR_INTERNAL = 7
} vdi_status;

/* vdi_config.flags */
#define VDI_FLAG_PIXEL_STATS 0x1u  /* keep per-list gamma*, tie margin and m of the last composite (vdi_pixel_stats) */
#define VDI_FLAG_VALIDATE 0x2u     /* vdi_composite checks its inputs on the device first (count <= k_in, offsets =
                                      exclusive scan of count, tf < tb, 0 <= alpha <= 1, a list's records
                                      front-to-back and disjoint) and returns VDI_ERR_INVALID_ARG naming the
                                      violation; costs one host synchronisation per call */
#define VDI_FLAG_STAGE_TIMING 0x4u /* record CUDA-event times of the exchange / merge / gather stages */
#define VDI_FLAG_LOOPBACK 0x10u    /* n_ranks > 1 contexts in ONE process (any devices, e.g. all on one GPU):
                                      nccl_unique_id is only the group's key, the windows are exchanged
                                      in-process instead of by NCCL + CUDA IPC; the device path is the same */
#define VDI_FLAG_HOST_SPAN 0x20u   /* _host entries: the caller promises that the host arrays of one call lie
                                      in ONE allocation (e.g. a pinned arena); libvdi then copies the span
                                      [lowest array start, highest array end) with one host->device copy,
                                      gap bytes included (default: one copy per array) */

typedef struct vdi_ctx vdi_ctx; /* opaque */

/* Compositing configuration.  All ranks pass identical values except `rank`.
 * PEs (processing elements) are the sources of sub-VDIs; PE s
 * is homed on rank floor(s * n_ranks / n_pes) ("block manner").
 * Rank g composites image rows [floor(g H / G), floor((g+1) H / G)) with
 * G = n_ranks (direct send; Q13).
 * n_ranks > 1: vdi_composite_init allocates this rank's window (flag words,
 * two parities of receive slots for the strip slices of every PE homed
 * elsewhere -- rows*W*(1 + 24 k_in) bytes each -- and two parities of a
 * root-side gather buffer of W*H*(1 + 24 k_out) bytes) and exchanges its
 * CUDA IPC handle with all ranks (one NCCL all-gather, collective; with
 * VDI_FLAG_LOOPBACK an in-process registry).  After init no call
 * synchronises the host. */
typedef struct {
  uint32_t width, height;  /* image = N_lists = w h lists */
  uint32_t k_in;           /* per-PE budget of the sub-VDIs, 1..255 */
  uint32_t k_out;          /* budget of the composited lists, 1..255 (N_s) */
  uint32_t n_pes;          /* number of PEs (sources), >= 1 */
  uint32_t n_ranks, rank;  /* GPUs (one process per GPU; 1..64) and this context's index */
  uint32_t root;           /* rank that receives the gathered image of vdi_gather (Q14: 0) */
  uint32_t max_iters;      /* bisection iterations I; 0 -> 16 (Q5) */
  float gamma_max;         /* upper end of the gamma search; 0 -> 2.0 (Q5) */
  uint32_t flags;          /* VDI_FLAG_* */
  const uint8_t* nccl_unique_id; /* 128 bytes from vdi_get_unique_id on rank 0; required iff n_ranks > 1
                                    (VDI_FLAG_LOOPBACK: any 128 bytes shared by the group's contexts) */
  void* cuda_stream;             /* cudaStream_t (borrowed); NULL = legacy default stream */
} vdi_config;

/* Dense sub-VDI of one PE (Fig. 2): per-list counts, their
 * exclusive prefix sum, and the packed supersegments of all lists in list
 * (row-major pixel) order, front-to-back within a list.  A supersegment is
 * 24 B: depth (t_front, t_back) world-space distance along the
 * unit ray (Q10) and accumulated premultiplied RGBA (Q7).
 * Memory: device, caller-owned (borrowed until the stream passes the call),
 * except when returned by vdi_generate_subvdi (ctx-owned). */
typedef struct {
  uint32_t pe_id;
  uint64_t total;         /* S_s = number of supersegments */
  const uint8_t* count;   /* [W*H], each <= k_in */
  const uint32_t* offset; /* [W*H + 1] exclusive scan of count (offset[W*H] == total) */
  const float* depth;     /* [total][2]  (t_front, t_back) */
  const float* rgba;      /* [total][4]  premultiplied, accumulated over [t_front, t_back] */
} vdi_dense_view;

/* Full-resolution representation of image rows [row_begin, row_end)
 * (PAPER.md:111, :185): k_out slots per list, unused slots all-zero (Q16).
 * Layout is list-major, slot fastest: element (y, x, j) at
 * ((y - row_begin) * W + x) * k_out + j.  Caller-owned device memory. */
typedef struct {
  uint32_t row_begin, row_end;
  uint8_t* count; /* [rows*W] */
  float* depth;   /* [rows*W][k_out][2] */
  float* rgba;    /* [rows*W][k_out][4] */
} vdi_full_view;

/* Scene description for the reference raycaster that produces sub-VDIs
 * (Phase 1; SUPPORT, untimed).  World box: longest side 1,
 * centred at the origin; voxel i covers continuous coordinate [i, i+1). */
typedef struct {
  const void* voxels;       /* device, x-fastest [dz][dy][dx] */
  uint32_t bytes_per_voxel; /* 1 (u8, /255) or 2 (u16, /65535) */
  uint32_t dims[3];
} vdi_volume_desc;

typedef struct {
  const float* table; /* device [256][4] RGBA, non-premultiplied, linear interpolation */
} vdi_tf_desc;

typedef struct {
  float eye[3], fwd[3], right[3], up[3]; /* orthonormal basis, world units */
  float tan_x, tan_y;                    /* tan(vfov/2)*aspect, tan(vfov/2) */
} vdi_camera;

/* Axis-aligned brick grid; brick (bx,by,bz) covers voxels [xb[bx], xb[bx+1])
 * x [yb[by], yb[by+1]) x [zb[bz], zb[bz+1]) (half-open) and belongs to PE
 * owner[(bz*gy + by)*gx + bx].  Host memory, copied by the call.  Unions of
 * bricks may be non-convex. */
typedef struct {
  uint32_t grid[3]; /* gx, gy, gz; product <= 4096 */
  const int32_t* xb;
  const int32_t* yb;
  const int32_t* zb;
  const int32_t* owner;
} vdi_decomp_desc;

/* ---- lifecycle ---------------------------------------------------------- */
const char* vdi_version(void);
const char* vdi_status_string(vdi_status s);
const char* vdi_last_error(const vdi_ctx* ctx); /* NULL-safe; thread-local text of the last failed call */

/* 128-byte NCCL unique id for vdi_config.nccl_unique_id (call on rank 0,
 * broadcast to the other ranks out of band, e.g. torch.distributed). */
vdi_status vdi_get_unique_id(uint8_t out[128]);

/* Validates cfg (VDI_ERR_INVALID_ARG), binds the current CUDA device, and for
 * n_ranks > 1 allocates the window and exchanges it (collective over all
 * ranks: NCCL communicator + all-gather of CUDA IPC handles; VDI_FLAG_LOOPBACK:
 * registration in the process, the group is complete once all n_ranks
 * contexts exist -- calls before that return VDI_ERR_STATE).
 * VDI_ERR_OUT_OF_MEMORY if the window does not fit. */
vdi_status vdi_composite_init(const vdi_config* cfg, vdi_ctx** out);
void vdi_composite_destroy(vdi_ctx* ctx); /* NULL-safe; waits for the ctx's stream, frees ctx-owned memory; local
                                             (no collective) -- destroy a group's contexts only once no rank
                                             has calls in flight (peers write into this window) */

/* ---- Phase 1 (SUPPORT): sub-VDI of PE pe_id --------------------------------
 * Two passes per ray: pass 1 finds gamma and the count it
 * generates (gamma = 0 if count(0) <= k_in, else the bisection of
 * PAPER.md:100-101, reading G1), an exclusive scan gives the offsets, pass 2
 * writes each list at its offset.  Samples lie on the global grid
 * t_i = t_in + (i+0.5)/max(dims) (one voxel, Q18); a sample owned by another
 * PE forces the open supersegment to end.  The output is
 * ctx-owned and valid until the next call with the same pe_id or destroy;
 * synchronises the stream once (to size the payload).
 * VDI_ERR_CAPACITY: some ray needs more than k_in supersegments (Q20). */
vdi_status vdi_generate_subvdi(vdi_ctx* ctx, const vdi_volume_desc* vol, const vdi_tf_desc* tf,
                               const vdi_camera* cam, const vdi_decomp_desc* decomp, uint32_t pe_id,
                               vdi_dense_view* out);

/* Limit case: the sub-VDI of PE pe_id with a
 * single S~ per sub-domain intersection -- the sweep of vdi_generate_subvdi
 * at gamma = infinity, so only leaving the PE's domain ends a supersegment
 * (PAPER.md:196).  k_in must cover the most domain intervals with content on
 * a ray (VDI_ERR_CAPACITY otherwise).  Output as vdi_generate_subvdi. */
vdi_status vdi_generate_limit(vdi_ctx* ctx, const vdi_volume_desc* vol, const vdi_tf_desc* tf,
                              const vdi_camera* cam, const vdi_decomp_desc* decomp, uint32_t pe_id,
                              vdi_dense_view* out);

/* ---- Phase 2: the hot path -------------------------------------------------
 * Parallel compositing of the sub-VDIs, collective over
 * all ranks (n_ranks == 1: local):
 *   a2  strip bounds: each rank finds, ON THE DEVICE, where every strip g
 *       starts in each of its PEs' payloads (offset[row_g W], or a scan of
 *       the counts when a view has no offset array);
 *   a3/a4 exchange: each rank pushes, for every local PE and
 *       every other strip g, the count slice and the packed payload slice
 *       into rank g's window over NVLink (one kernel, plain stores into CUDA
 *       IPC mappings); every block then bumps a counter word at g, and rank
 *       g proceeds once the counter of each sender reaches its block count
 *       for this call -- sizes never cross the host;
 *   a5  receive-side scan of every source's count slice (Q17);
 *   a6-a10 per list: depth ordering, overlap subdivision
 *       (Eq. 2 generalised, Q12), verbatim pass-through when m <= k_out (Q9),
 *       otherwise the per-ray gamma bisection over the sub-supersegments
 *        and the final greedy sweep, written in the full
 *       representation.
 * local_pes: the n_local sub-VDIs homed on this rank, any order, each with a
 * distinct pe_id; device memory (any allocation: only this rank reads it).
 * Offset arrays are optional: with one rank, when every view carries its
 * offsets they supply the group bases and the receive-side scan is skipped
 * (they must then be the exclusive scan of count).  strip_out: caller-owned,
 * rows of this rank's strip (VDI_ERR_CAPACITY if the row range does not
 * match).  Never synchronises the host; the inputs are free once the stream
 * passes the call (only this rank reads them).  The receive slots are
 * double-buffered: a sender waits (on the device) until the receiver has
 * merged the call before last. */
vdi_status vdi_composite(vdi_ctx* ctx, const vdi_dense_view* local_pes, uint32_t n_local,
                         vdi_full_view* strip_out);

/* The full-representation variant of the compositing (Fig. 6
 * "full"): every local PE's sub-VDI is given in the full
 * representation (rows [0, H), k_in slots per list, unused slots zero,
 * PAPER.md:111), the strips are exchanged as fixed-size slices (pushed into
 * the same window slots, P_g (1 + 24 k_in) bytes per PE and strip), and each
 * source is compacted to the dense layout on the receiver before the same
 * merge as vdi_composite -- so the image is identical.  pe_ids[l] names the
 * PE of local_pes[l].  Collective; synchronises the host once (the record
 * total of the compaction sizes the merge, as in the paper's pipeline). */
vdi_status vdi_composite_fullrep(vdi_ctx* ctx, const vdi_full_view* local_pes, const uint32_t* pe_ids,
                                 uint32_t n_local, vdi_full_view* strip_out);

/* Dense -> full representation of one sub-VDI:
 * out (rows [0, H), k_in slots per list) receives each list's records in its
 * first count slots and zeros elsewhere.  Local (no collective). */
vdi_status vdi_dense_to_full(vdi_ctx* ctx, const vdi_dense_view* in, vdi_full_view* out);

/* Same as vdi_composite with HOST buffers (the end-to-end entry point):
 * copies the local sub-VDIs host->device (pinned memory recommended),
 * composites, and copies the strip back device->host into strip_out.
 * Pointers in local_pes / strip_out are host pointers.  Synchronises.
 * Host inputs of every _host entry: count, depth and rgba are copied (offset
 * arrays are ignored: the device re-derives what it needs from the counts),
 * one copy per array, or one copy of their span with VDI_FLAG_HOST_SPAN. */
vdi_status vdi_composite_host(vdi_ctx* ctx, const vdi_dense_view* local_pes, uint32_t n_local,
                              vdi_full_view* strip_out);

/* Composited strip in the dense representation: per-list
 * counts and the packed supersegments, list-major, slots in depth order. */
typedef struct {
  uint32_t row_begin, row_end; /* must be this rank's strip */
  uint64_t capacity;           /* supersegments depth/rgba can hold */
  uint64_t total;              /* out: supersegments written (set even on VDI_ERR_CAPACITY) */
  uint8_t* count;              /* [rows*W] */
  float* depth;                /* [capacity][2] */
  float* rgba;                 /* [capacity][4] */
} vdi_dense_strip;

/* vdi_composite_host with the result returned in the dense representation:
 * host sub-VDIs -> device -> composite -> compaction on the device -> only
 * the counts and the packed supersegments cross back to the host buffers of
 * out (vdi_dense_to_full re-inflates on a device when the full
 * representation is needed).  VDI_ERR_CAPACITY if out->capacity < total.
 * Synchronises. */
vdi_status vdi_composite_host_dense(vdi_ctx* ctx, const vdi_dense_view* local_pes, uint32_t n_local,
                                    vdi_dense_strip* out);

/* vdi_composite_host_dense over n_frames independent frames (the serving
 * loop: a new set of host sub-VDIs per frame), pipelined: frame f's
 * host->device copies overlap frame f-1's compositing and frame f-2's
 * device->host copies (two copy streams, double-buffered device inputs and
 * dense outputs).  local_pes is frame-major [n_frames][n_local] (host
 * pointers, read until the call returns); outs[n_frames] as for
 * vdi_composite_host_dense (host buffers; one buffer may serve several
 * frames only if the caller accepts that the last frame wins).  Each frame's
 * result is identical to a vdi_composite_host_dense call on its inputs
 * (PAPER.md:113-115, :164-185).  Device scratch: two input slots and two
 * output slots of the strip's full capacity (rows*W*k_out*24 B each), grow-only.
 * VDI_ERR_CAPACITY (after every frame ran) if a frame's total exceeds its
 * outs[f].capacity; outs[f].total is set for every frame.  Synchronises. */
vdi_status vdi_composite_host_dense_frames(vdi_ctx* ctx, uint32_t n_frames, const vdi_dense_view* local_pes,
                                           uint32_t n_local, vdi_dense_strip* outs);

/* Gather (a11) of the composited strips onto vdi_config.root (PAPER.md:185
 * MPI_Gather; Q14): image_out (rows [0, H), root only; ignored elsewhere)
 * receives every rank's strip at its rows.  Each non-root rank compacts its
 * strip to counts + packed records (the dense representation,
 * PAPER.md:113-115) straight into the root's window over NVLink and bumps a
 * counter word there; the root waits for every rank's blocks, re-inflates the
 * full representation with the pass-through kernel and copies its own strip
 * (none if strip aliases the image rows).  The image is identical to gathering
 * the full representation.  Never synchronises the host; the root's gather
 * buffer is double-buffered (a rank waits on the device until the root has
 * inflated the gather before last).  n_ranks == 1: copies the strip if the
 * buffers differ. */
vdi_status vdi_gather(vdi_ctx* ctx, const vdi_full_view* strip, vdi_full_view* image_out);

/* vdi_gather onto rank `root` instead of vdi_config.root (e.g. a root that
 * rotates over consecutive frames so that no GPU re-inflates every image);
 * all ranks pass the same root. */
vdi_status vdi_gather_root(vdi_ctx* ctx, uint32_t root, const vdi_full_view* strip, vdi_full_view* image_out);

/* Frames in flight through strip mode: n_frames VDIs,
 * each composited in strips on every rank (vdi_composite) and gathered onto
 * roots[f] (vdi_gather_root; roots == NULL: vdi_config.root for all).  The
 * root of a frame merges its own strip straight into the rows of images[f]
 * and re-inflates the other ranks' rows on a second, ctx-owned stream, so its
 * exchange and merge of frame f+1 -- and through them every other rank's --
 * overlap its inflate of frame f.  Each image equals vdi_composite +
 * vdi_gather of that frame bit for bit.  local_pes: [n_frames][n_local]
 * (frame-major) dense views homed on this rank; images[n_frames]: full
 * representations of rows [0, H), read only for the frames this rank is the
 * root of (others may be zeroed structs); distinct buffers per frame (frames
 * overlap: frame f's search kernels run on a third ctx-owned stream beside
 * frame f+1's pass-through, with two parities of merge scratch; not with
 * VDI_FLAG_PIXEL_STATS; a frame whose long-list search fills the GPU for many
 * waves -- more than 600 000 lists with m > 40 in a recent frame, noted by the
 * long-search kernel in a mapped host word -- runs without the next
 * pass-through beside it).  The call is complete when the caller's stream
 * passes it; never synchronises the host.  ctx-owned scratch (n_ranks > 1):
 * four non-root strips (rows*W*(1 + 24 k_out) bytes each); a second set of
 * merge scratch.
 * n_ranks == 1: frames in flight on one GPU, images[f] written whole. */
vdi_status vdi_composite_frames(vdi_ctx* ctx, uint32_t n_frames, const vdi_dense_view* local_pes,
                                uint32_t n_local, vdi_full_view* images, const uint32_t* roots);

/* ---- limit case and rendering ------------------------------ */
/* The limit case of the compositing: the exchange of
 * vdi_composite, then every list's S~ are placed in depth order
 * and over-composited along the list, giving the plain
 * volume-rendered image of this rank's strip -- DVR on a non-convex domain
 * decomposition without synchronisation between PEs.  With limit sub-VDIs
 * (vdi_generate_limit) the image equals direct volume rendering up to fp32
 * rounding.  Overlapping records are composited in (t_front, PE id) order
 * without subdivision.  strip_rgba: device [rows*W][4] premultiplied,
 * 16-byte aligned.  Collective (n_ranks > 1); never synchronises the host. */
vdi_status vdi_composite_image(vdi_ctx* ctx, const vdi_dense_view* local_pes, uint32_t n_local, float* strip_rgba);

/* Gather of the strips of vdi_composite_image onto vdi_config.root:
 * image_rgba (root only, device [H*W][4]) receives every strip at its rows
 * (pushed into the root's window over NVLink).  Collective. */
vdi_status vdi_gather_image(vdi_ctx* ctx, const float* strip_rgba, float* image_rgba);

/* A VDI rendered from its generation viewpoint: the over of each list's
 * supersegments front to back -- the exact image by associativity of over
 * (PAPER.md:77).  vdi: any rows (device, k_out slots); out_rgba: device
 * [rows*W][4] premultiplied, 16-byte aligned.  Local. */
vdi_status vdi_render_generation_view(vdi_ctx* ctx, const vdi_full_view* vdi, float* out_rgba);

/* A full VDI (rows [0, H), k_out slots, generated with camera gen_cam)
 * rendered from camera view_cam at w_out x h_out: rays
 * through the new pixel centres are marched through the volume's world box
 * (dims, longest side 1) one voxel per step; each sample is projected into
 * gen_cam, the supersegment of the nearest list containing its depth along
 * that list's ray contributes opacity 1 - (1 - a)^(dt / L) (L its length;
 * Eq. 2) and colour scaled alike, over-composited front to
 * back.  out_rgba: device [h_out*w_out][4] premultiplied.  Local. */
vdi_status vdi_render_novel_view(vdi_ctx* ctx, const vdi_full_view* vdi, const vdi_camera* gen_cam,
                                 const vdi_camera* view_cam, const uint32_t dims[3], uint32_t w_out, uint32_t h_out,
                                 float* out_rgba);

/* Ground truth for the quality evaluation: direct volume
 * rendering of the whole volume with camera cam at w_out x h_out -- the
 * over of every sample of the global grid (the generator's sampling, Q18,
 * Q19), fp32, no early termination (Q21).  out_rgba: device [h_out*w_out][4]. */
vdi_status vdi_render_dvr(vdi_ctx* ctx, const vdi_volume_desc* vol, const vdi_tf_desc* tf, const vdi_camera* cam,
                          uint32_t w_out, uint32_t h_out, float* out_rgba);

/* ---- introspection ---------------------------------------------------------- */
/* Per-list gamma* (0 for pass-through), tie margin and m (samples after
 * sort/subdivision) of this rank's strip for the last composite; device
 * pointers [rows*W], each may be NULL.  The tie margin is the minimum over the
 * executed comparisons of the bisection and the final sweep of
 * |sqrt(D^2) - gamma| (double; +inf when no comparison ran) -- lists whose
 * margin is < 1e-6 are the "ties" of the parity bar.  Requires
 * VDI_FLAG_PIXEL_STATS (a replay kernel per composite computes the margins). */
vdi_status vdi_pixel_stats(vdi_ctx* ctx, float* gamma, float* min_margin, uint16_t* m);

/* Counters of the last vdi_composite / vdi_gather on this rank (synchronises the stream). */
typedef struct {
  uint64_t records_in;      /* sum over local strip lists of m before subdivision (supersegments merged) */
  uint64_t records_search;  /* the part of records_in that belongs to lists needing the gamma search / general path */
  uint64_t searched_lists;  /* lists that needed the gamma search or subdivision */
  uint64_t bytes_sent;      /* exchange bytes this rank pushed to other ranks (counts + records) */
  uint64_t bytes_received;  /* exchange bytes other ranks pushed into this rank's window */
  uint32_t kernel_launches; /* libvdi kernels launched by the call */
  float ms_exchange, ms_merge, ms_gather; /* VDI_FLAG_STAGE_TIMING, else 0 */
  uint64_t bucket_lists[4];  /* lists sent to the search buckets m <= 32, <= 40, <= 64, > 64 */
  uint64_t general_lists;    /* lists sent to the general path (overlaps, alpha == 0, no search-pool room) */
  uint64_t bytes_gather;     /* last vdi_gather: bytes that crossed into the root (root) / pushed (others) */
  uint64_t fallback_groups;  /* 32-list groups written with plain stores (tail group / unaligned output) */
  float ms_scan, ms_fast, ms_search; /* VDI_FLAG_STAGE_TIMING: receive scan, pass-through kernel, search kernels */
  uint64_t sweep_steps;      /* VDI_FLAG_PIXEL_STATS: sample-steps of the plain bisection procedure (every count
                                sweep to its early exit + the final sweep) over the searched lists -- the
                                algorithmic work of the search (the kernels' memoised bisection skips some) */
  float ms_push;             /* VDI_FLAG_STAGE_TIMING, n_ranks > 1: the exchange push kernel alone (CUDA events on
                                the push stream): bytes_sent / ms_push is this rank's NVLink egress rate */
} vdi_counters;
vdi_status vdi_get_counters(vdi_ctx* ctx, vdi_counters* out);

/* ---- host-only helpers (no GPU needed) --------------------------------------- */
/* Rows [*row_begin, *row_end) of strip g of G (Q13). */
vdi_status vdi_strip_rows(uint32_t height, uint32_t n_ranks, uint32_t g, uint32_t* row_begin,
                          uint32_t* row_end);
/* Home rank of PE pe: floor(pe * n_ranks / n_pes). */
uint32_t vdi_pe_home(uint32_t n_pes, uint32_t n_ranks, uint32_t pe);
/* Bytes of a full-representation view of `rows` rows: rows*W*(1 + 24*k). */
uint64_t vdi_full_bytes(uint32_t width, uint32_t rows, uint32_t k);

#ifdef __cplusplus
}
#endif

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif
#endif /* VDI_H_ */
