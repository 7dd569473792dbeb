/* gml.h -- C ABI of the B200-native GMLake allocation engine (libgml.so).
 *
 * GMLake (arXiv 2401.08156) keeps a primitive pool of pBlocks (PAPER.md
 * §3.2) and a stitched pool of sBlocks (L343-350) and serves each
 * request through BestFit (Algorithm 1) and the S1-S5 strategy
 * (§4.1); small requests (< 2 MB) use PyTorch's BFC splitting
 * (L322). This library exposes:
 *
 *   gml_replay  -- batched replay of allocation traces through that engine
 *                  (and through the BFC baselines), one warp per
 *                  (trace, policy) on sm_100a. Returns per-event block
 *                  assignments and per-(trace, policy) statistics from which
 *                  utilisation / fragmentation (§5.1) follow.
 *   gml_malloc / gml_free / gml_stats
 *               -- a live allocator over the CUDA VMM driver API (Alloc =
 *                  cuMemCreate on 2 MiB granules + map, Stitch =
 *                  cuMemAddressReserve + cuMemMap + cuMemSetAccess onto the
 *                  members' chunks, L306-327, L381-387) running the same
 *                  policy code on the host.
 *
 * Conventions: all calls return gml_status; no C++ exception crosses the ABI;
 * no pointer is retained after a call returns (replay) or after gml_destroy
 * (live allocator). All integers are little-endian.
 */
#ifndef GML_H
#define GML_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  GML_OK = 0,
  GML_ERR_INVALID = 1,          /* bad argument or malformed trace            */
  GML_ERR_OOM = 2,              /* S5 / BFC cannot grow        */
  GML_ERR_CUDA = 3,             /* a CUDA runtime / driver call failed         */
  GML_ERR_TABLE_OVERFLOW = 4,   /* internal: a replay table was too small;
                                   gml_replay re-runs the unit with larger
                                   tables, callers never see it in stats      */
  GML_ERR_UNSUPPORTED = 5       /* e.g. no VMM support on the device           */
} gml_status;

typedef enum {
  GML_POLICY_BFC_TORCH = 0,     /* PyTorch 2.x caching allocator rules (L111-125, L624) */
  GML_POLICY_BFC_EXACT = 1,     /* BFC, segment = rounded request    */
  GML_POLICY_GMLAKE = 2         /* GMLake (§3-§4)                               */
} gml_policy_kind;

/* Switches for readings the paper leaves open. */
enum {
  GML_F_S1_PBLOCK_FIRST = 1,    /* D5: scan pPool before sPool in S1              */
  GML_F_NO_COMPANION = 2,       /* D11: no [F, R] companion sBlock on Split       */
  GML_F_SPLIT_INVALIDATES = 4,  /* D12: Split deletes sBlocks over the parent     */
  GML_F_REMAINDER_RULE = 8,     /* D8: split only if remainder >= limit           */
  GML_F_LIMIT_GATES_REQUEST = 16 /* D8': requests < frag limit take the small path
                                   (PAPER.md L571 read for the request, L322);
                                   set in the default GMLake policy V2          */
};

typedef struct {                /* 56 bytes, POD */
  uint32_t kind;                /* gml_policy_kind                                      */
  uint32_t flags;               /* GML_F_*                                               */
  uint64_t capacity_bytes;      /* device memory the policy may reserve (80 GiB: L589)  */
  uint64_t chunk_bytes;         /* physical chunk / granule, 2 MiB (L319); mult. of 512  */
  uint64_t small_threshold_bytes; /* raw < this -> BFC small path (L322), 2 MiB         */
  uint64_t frag_limit_bytes;    /* fragmentation limit (L569-572), 128 MiB               */
  uint32_t spool_max_entries;   /* StitchFree count cap (L563-567), 4096                 */
  uint32_t _pad;                /* must be 0                                              */
  uint64_t spool_max_inactive_bytes; /* StitchFree byte cap on inactive sBlocks           */
} gml_policy;

typedef struct {                /* 272 bytes, all integers */
  uint64_t peak_active_bytes;   /* max over events of bytes bound to live tensors (L631) */
  uint64_t peak_reserved_bytes; /* max of chunks*chunk + BFC segments (L632)             */
  uint64_t peak_requested_bytes;/* max of sum of raw request bytes                        */
  uint64_t peak_active_vmm_bytes, peak_reserved_vmm_bytes; /* VMM path only              */
  uint64_t final_active_bytes, final_reserved_bytes;
  uint64_t n_events;            /* trace length                                          */
  uint64_t n_events_done;       /* events replayed before termination                    */
  int64_t oom_event;            /* index of the OOM event, -1 if none                    */
  uint32_t status;              /* GML_OK or GML_ERR_OOM (or GML_ERR_INVALID)            */
  uint32_t _p;                  /* 0                                                      */
  uint64_t state_count[7];      /* S1..S5, small/BFC cache hit, small/BFC new segment    */
  uint64_t n_split, n_stitch, n_companion, n_alloc, n_evict, n_seg_alloc, n_seg_release;
  uint64_t vmm_calls[7];        /* modelled VMM calls (L273): reserve, create, map,
                                   set_access, unmap, addr_free, release                 */
  uint32_t max_pblocks, max_sblocks, max_live_handles, max_bfc_blocks;
} gml_stats_t;

/* Packed event (u64): bit 63 = free; bits 40..62 = slot; bits 0..39 = raw
 * bytes (malloc) or 0 (free).
 *
 * Assignment record (u64 per event and policy): bits 0..31 block ordinal
 * (BFC: offset in 512-byte units); bits 32..33 kind (0 pBlock, 1 sBlock,
 * 2 BFC block); bits 34..36 state (1..5 = S1..S5, 6 = BFC cache hit,
 * 7 = BFC new segment, 0 = free); bits 40..63 BFC segment ordinal. A free
 * records the block it unbinds. The terminating OOM event records state 5 and
 * ordinal 0xFFFFFFFF; later events record 0. */

typedef struct gml_replay_caps {  /* per-(trace, policy) table capacities (hints) */
  uint32_t pblocks, sblocks, intervals, bfc_blocks;
} gml_replay_caps;

typedef struct {
  const uint64_t* events;       /* DEVICE: all traces back to back (packed events)       */
  const uint64_t* trace_offsets;/* DEVICE: n_traces + 1 event offsets                     */
  uint32_t n_traces, n_policies;
  const gml_policy* policies;   /* HOST: n_policies entries                               */
  uint64_t* assignments;        /* DEVICE: [n_policies][total_events], or NULL            */
  gml_stats_t* stats;           /* DEVICE: [n_traces][n_policies]                          */
  void* stream;                 /* cudaStream_t; NULL = default stream                    */
  gml_replay_caps* caps;        /* HOST, optional: [n_traces][n_policies] hints, updated
                                   on return with capacities that sufficed               */
  uint64_t* timeline;           /* DEVICE, optional: [n_policies][total_events][2] =
                                   (active, reserved) bytes after each event (the
                                   terminating event's state included; 0 after it):
                                   the fig:trace series, PAPER.md L766-791         */
} gml_trace_batch;

/* Host-side trace check: every free names a live slot, every
 * malloc slot is free, sizes > 0, free words carry size 0. host_events is a
 * HOST pointer to n events; *max_slots receives 1 + the largest slot.
 * Returns GML_ERR_INVALID (and *max_slots = index of the bad event) on a
 * malformed trace. */
gml_status gml_trace_validate(const uint64_t* host_events, uint64_t n, uint32_t* max_slots);

/* Replay every (trace, policy) pair of the batch on the GPU. The call is
 * stream-ordered on b->stream and returns after the stream has completed the
 * replay (it reads back per-unit status to re-run units whose tables
 * overflowed). Per-trace OOM is reported in stats[t][p].status, not as a call
 * failure. Traces must be valid (gml_trace_validate); a malformed trace ends
 * its units with status GML_ERR_INVALID. Internally a GMLake unit may replay
 * its VMM path and its small path concurrently (two-path units, see
 * gml_last_split_count); every output is identical to the one-warp replay. */
gml_status gml_replay(const gml_trace_batch* b);

/* Number of kernel launches the last gml_replay on this thread issued, and
 * the device time (CUDA events on b->stream) of its K1 replay launches. */
uint32_t gml_last_launch_count(void);
float gml_last_kernel_ms(void);

/* Split units of the last gml_replay on this thread (diagnostic): in the
 * latency placement (fewer than 4 units per SM, no timeline) a GMLake unit
 * replays its VMM path and its small path on two warps of one CTA, which
 * take the same decisions as one warp while neither path fails a capacity
 * check (the paths share only the capacity).
 * Returns the number of units that completed split; *serial_reruns (if not
 * NULL) receives the number of split units the single-warp replay re-ran
 * (an OOM or segment release in a path, the paths' reserved bytes summing
 * over capacity, or an invalid trace). */
uint32_t gml_last_split_count(uint32_t* serial_reruns);

/* Host-side metrics. utilization = peak active / peak
 * reserved, 1.0 for (0, 0); fragmentation = 1 - utilization. */
double gml_utilization(const gml_stats_t* s);
double gml_fragmentation(const gml_stats_t* s);

/* ---- live allocator over the CUDA VMM driver API ---- */
typedef struct gml_allocator gml_allocator;

/* Create an allocator on `device` with policy *p (kind must be GMLAKE; the
 * chunk must be a multiple of the device's VMM granularity). */
gml_status gml_create(int device, const gml_policy* p, gml_allocator** out);
/* Allocate `bytes`; *out_ptr = device VA valid until gml_free/gml_destroy,
 * NULL on error. GML_ERR_OOM in state S5: the capacity check failed, or a
 * driver allocation (cuMemCreate / cuMemMap / cudaMalloc) failed -- "If the
 * Alloc function call fails, GMLake immediately reports an OOM" (PAPER.md
 * L528); nothing is committed and the allocator stays usable.
 * GML_ERR_TABLE_OVERFLOW: a host table is full (nothing committed). Never
 * blocks on the device. */
gml_status gml_malloc(gml_allocator* a, size_t bytes, void** out_ptr);
/* Release a pointer returned by gml_malloc (GML_ERR_INVALID if unknown);
 * the block is reusable at once (single-stream semantics, D24). */
gml_status gml_free(gml_allocator* a, void* ptr);
/* The stream the allocator's work is ordered on (cudaStream_t; default NULL =
 * the legacy default stream). StitchFree unmaps an
 * evicted sBlock's VA only after an event recorded on this stream at the
 * eviction has completed (no device-wide synchronisation). */
gml_status gml_set_stream(gml_allocator* a, void* stream);
/* Drive the live allocator with a packed trace (HOST pointer, n events,
 * the gml_trace_batch event encoding): each malloc / free is issued as
 * gml_malloc / gml_free. Optional outputs (host, n entries): records[i] =
 * the assignment record of event i (gml_replay's encoding, so live, replay
 * and oracle decisions compare event by event), ns[i] = host time of the
 * call (steady_clock ns). Stops at the first failing call and returns its
 * status (records[i] = the S5 record on OOM); *n_done = events completed.
 * Blocks still live at the end are freed (after the last timed call). */
gml_status gml_live_trace(gml_allocator* a, const uint64_t* events, uint64_t n, uint64_t* records, uint64_t* ns,
                          uint64_t* n_done);
/* The same trace as plain cudaMalloc / cudaFree calls on `device` (the
 * latency baseline of Table 1 / C5); ns and n_done as above. */
gml_status gml_cudamalloc_trace(int device, const uint64_t* events, uint64_t n, uint64_t* ns, uint64_t* n_done);
/* Statistics of the live allocator, same record as a replay. */
gml_status gml_stats(const gml_allocator* a, gml_stats_t* out);
/* Actual driver calls issued so far, same order as gml_stats_t.vmm_calls. */
gml_status gml_driver_calls(const gml_allocator* a, uint64_t out[7]);
/* GML_ERR_INVALID if live allocations remain (nothing is released then). */
gml_status gml_destroy(gml_allocator* a);

/* ---- PyTorch pluggable-allocator backend (the paper's
 * deployment mode: "integrate it into the caching allocator of PyTorch",
 * PAPER.md L578, drop-in for tensor (de)allocation, L470-473) ----
 * Signatures are the ones torch.cuda.memory.CUDAPluggableAllocator calls.
 * One live allocator per device, created on the device's first request with
 * the policy set by gml_torch_configure (default: GMLake V2, capacity = the
 * device's free memory at creation minus 1 % (>= 256 MiB) of headroom,
 * rounded down to the chunk). Calls are serialised by
 * a mutex. gml_torch_malloc returns NULL on OOM (S5) or error (size 0 ->
 * NULL); gml_torch_free ignores NULL. Streams: the stream of a device's first
 * request is its main stream (gml_set_stream). A request on another stream
 * first makes that stream wait for the main stream's work so far, and a free
 * on another stream makes the main stream wait for that stream's work so far
 * (event record + cudaStreamWaitEvent, no host synchronisation): every block
 * handed out is then ordered after all work on the blocks freed before it,
 * whatever stream used them. */
void* gml_torch_malloc(ptrdiff_t size, int device, void* stream);
void gml_torch_free(void* ptr, ptrdiff_t size, int device, void* stream);
/* Policy for allocators created after the call (HOST pointer, copied).
 * GML_ERR_INVALID if an allocator already exists for any device. */
gml_status gml_torch_configure(const gml_policy* p);
/* Statistics of the allocator of `device` (GML_ERR_INVALID if none yet). */
gml_status gml_torch_stats(int device, gml_stats_t* out);

/* ---- VMM API latency probe (Table 1 / fig:virtual,
 * PAPER.md L207-274, re-measured on this device) ----
 * One allocation of `bytes` built from `bytes / chunk` physical chunks,
 * `reps` times; host wall time (steady_clock) per API in microseconds,
 * median over reps, into out_us[10]:
 *   [0] cudaMalloc(bytes)          [1] cudaFree
 *   [2] cuMemAddressReserve        [3] sum of cuMemCreate (one per chunk)
 *   [4] sum of cuMemMap (per chunk)
 *   [5] sum of cuMemSetAccess, one call per chunk (the paper's Table 1)
 *   [6] one cuMemSetAccess over the whole range (what gml_malloc issues)
 *   [7] teardown: cuMemUnmap + cuMemRelease per chunk + cuMemAddressFree
 *   [8] VMM total as in Table 1 = [2]+[3]+[4]+[5]
 *   [9] VMM total as gml_malloc's Alloc = [2]+[3]+[4]+[6]
 * bytes must be a multiple of chunk, chunk a multiple of the device's VMM
 * granularity. GML_ERR_UNSUPPORTED without VMM support. */
gml_status gml_vmm_profile(int device, uint64_t bytes, uint64_t chunk, int reps, double* out_us);

/* K2: streaming read+write kernel over n bytes at src -> dst (device
 * pointers, 16-byte aligned), `iters` times on `stream`; *ms = device time of
 * one pass (the mean over the iters passes). */
gml_status gml_stream_copy(const void* src, void* dst, size_t n, int iters, void* stream, float* ms);

const char* gml_status_string(gml_status s);

#ifdef __cplusplus
}
#endif
#endif /* GML_H */
