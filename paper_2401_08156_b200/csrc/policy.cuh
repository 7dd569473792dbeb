// policy.cuh -- the GMLake allocation engine, written once for the executors
// ("groups" of cooperating threads that own one replay):
//
//   * DeviceWarp: the 32 lanes of one warp own one (trace, policy) replay on
//     sm_100a; scans stride words / 16-byte vectors over the lanes and finish
//     with __reduce_min_sync / ballots (the "warp-level argmin/ballot best-fit
//     search" of the north star).
//   * HostWarp: width 1, for the live allocator (gml_malloc / gml_free), so
//     the live path and the replay take identical decisions.
//   * (tests/engine_sim.cpp adds a 32-thread CPU emulation of a warp that runs
//     this same code, to check the lane-parallel logic without a GPU.)
//
// Every thread of a group holds the same scalar state and takes the same
// (uniform) decisions; table writes are done by the leader (or by distinct
// lanes on distinct words, with shared-memory atomics where words can be
// shared) and published with sync(). The method (§3.3 Algorithm 1
// L390-452, §4.1) is walked in the paper's order; readings D1..D30
// are listed in DESIGN.md. The engine never reads the oracle (oracle/), and
// the oracle never reads this file.
//
// Data layout per replay ("arena", SoA, u32 unless noted; in shared memory
// when it fits, else in global memory -- see Lay<C> below). Activity (D18,
// "if even one pBlock is active, all corresponding sBlocks
// are labeled as active"): a pBlock is active iff a live tensor owns it (PIN
// bit clear), an sBlock iff some chunk inside its intervals is owned (BM).
//   bitmap   BM: 1 bit per chunk, set = owned by a live tensor; BMS: 1 bit
//            per BM word, set whenever the word may be non-zero (set on every
//            bind, cleared lazily by the test that finds the word zero), so
//            binds and frees are fire-and-forget atomics and a range test
//            reads the two edge words and the summary words of the interior.
//   pPool    the paper's sorted set (L337-339) as PE = 16-byte entries
//            {ordinal, size, row, -} ascending in (size << 32 | ordinal); pool order (size desc, ordinal
//            asc, D4) is size groups from the top, positions ascending inside
//            a group. PIN holds one bit per sorted POSITION: set = that
//            pBlock is inactive, so "first inactive pBlock of size b" (S1),
//            "smallest eligible inactive size > b" (S2) and the greedy walk
//            (S3) are find-first-set over PIN words, 32 words (1024 blocks)
//            per ballot. Rows: PN granules, PLO first chunk, PNEXT address
//            successor, PPOS sorted position. Rows are never deleted: Split
//            rewrites the parent's row as the front piece F and appends R.
//   sPool    SE sorted set (L344) of entries {ordinal, size, row, witness}
//            + rows SN (granules, 0 = free row), SORD, SLAST (LRU key), SBORN
//            (free-row link), SIVO / SIVN (interval list). The
//            witness is a chunk of the sBlock seen owned: while it stays owned
//            the sBlock is active (one bitmap load skips the interval test);
//            NONE32 records "last tested inactive".
//   ivs      IVROW (first member row), IVLO, IVN: chunk intervals of sBlocks,
//            double-buffered for compaction. A member row stays the row of
//            the pBlock at IVLO forever (Split keeps F in P's row), so PNEXT
//            walks from IVROW cover the interval.
//   handles  u64 per slot: kind (2 b) | row (22 b) | raw bytes (40 b).
//   BFC      BSIZE / BOFF (512-byte units), BSEG, BPREV, BNEXT, BPF (free-list
//            index | ALLOC | POOL1 flags); one free-list array FLR / FLS / FLA
//            shared by the two pools (pool 0 from the bottom, pool 1 from the
//            top), so best-fit scans read one size word per free block.
#pragma once
#include <stdint.h>

#if !defined(__CUDACC__)
#include <vector_types.h>
#endif

#include "gml.h"

#if defined(__CUDACC__)
#define GML_HD __host__ __device__ __forceinline__
#define GML_HDI __host__ __device__
#define GML_NOINL __host__ __device__ __noinline__
#else
#define GML_HD inline
#define GML_HDI
#define GML_NOINL inline
#endif

// cold engine paths (Split, Stitch, Alloc): inlined (GML_HD) or out of line
// (GML_COLD_NOINL: the engine object then lives in local memory across the
// call, but the kernel's code and register allocation shrink)
#if defined(GML_COLD_NOINL)
#define GML_COLD GML_NOINL
#else
#define GML_COLD GML_HD
#endif

// Free-list initialisation. The BFC best-fit scan reads the free lists in
// 16-byte vectors of 4 entries and masks off the entries outside the pool,
// some of which may never have been written. 2 (product) = no zeroing: the
// masked reads are harmless; 1 = the lists are zeroed at init (the build
// compute-sanitizer initcheck runs on, tools/gpu_sanitize.sh); 0 = a pool
// zeroes the rest of a vector group when it first grows into it. Measured
// on C4 (same box, ms per step): 2 -> 236-240, 1 -> 246-249, 0 -> 259-266
// (any code on the push path perturbs the whole kernel's allocation).
#ifndef GML_FL_ZERO
#define GML_FL_ZERO 2
#endif

#ifndef GML_SHIFT_U
#define GML_SHIFT_U 4   // sorted-set shift: entries per lane per round
#endif

#if defined(GML_PHASE_PROF) && defined(__CUDA_ARCH__)
// per-phase cycle counters kept in registers (constant k only) and written
// out by finish(): no memory traffic on the unit's chain
#define GML_PROF_ON 1
#define GML_T0(v) long long v = clock64()
#define GML_T1(k, v) pacc[k] += (unsigned long long)(clock64() - v)
#else
#define GML_T0(v)
#define GML_T1(k, v)
#endif

// host-only operation counters (tools/host_counts.cpp; never in product builds)
#if defined(GML_HOST_COUNT) && !defined(__CUDA_ARCH__)
extern unsigned long long gml_hc[32];
#define GML_HC(k, v) (gml_hc[k] += (unsigned long long)(v))
#else
#define GML_HC(k, v)
#endif

namespace gml {

constexpr uint32_t NONE32 = 0xFFFFFFFFu;
constexpr uint64_t MASK40 = (1ull << 40) - 1;

GML_HD uint32_t ctz32(uint32_t m) {
#if defined(__CUDA_ARCH__)
  return (uint32_t)(__ffs(m) - 1);
#else
  return (uint32_t)__builtin_ctz(m);
#endif
}
GML_HD uint32_t popc32(uint32_t m) {
#if defined(__CUDA_ARCH__)
  return (uint32_t)__popc(m);
#else
  return (uint32_t)__builtin_popcount(m);
#endif
}
GML_HD uint32_t clz32(uint32_t m) {
#if defined(__CUDA_ARCH__)
  return (uint32_t)__clz(m);
#else
  return (uint32_t)__builtin_clz(m);
#endif
}

struct KeyRow {           // result of an argmin: key (~0 = none) and its row
  uint64_t key;
  uint32_t row;
};

// ---------------------------------------------------------------- executors
struct DeviceWarp {
  using ctr_t = uint32_t;    // per-replay event counters (a trace has < 2^32 events)
  // the replay executor: each handle table is sized from its trace's max
  // slot (K0), so no event's slot is out of range, and the kernel stops a
  // unit on overflow after the step, so step() need not test either
  static constexpr bool kReplay = true;
  GML_HD uint32_t lane() const {
#if defined(__CUDA_ARCH__)
    return threadIdx.x & 31u;
#else
    return 0;
#endif
  }
  GML_HD uint32_t width() const { return 32; }
  GML_HD bool leader() const { return lane() == 0; }
  GML_HD void sync() const {
#if defined(__CUDA_ARCH__)
    __syncwarp();
#endif
  }
  GML_HD uint32_t ballot(bool p) const {
#if defined(__CUDA_ARCH__)
    return __ballot_sync(0xFFFFFFFFu, p);
#else
    return p;
#endif
  }
  GML_HD uint32_t shfl(uint32_t v, uint32_t s) const {
#if defined(__CUDA_ARCH__)
    return __shfl_sync(0xFFFFFFFFu, v, s);
#else
    (void)s;
    return v;
#endif
  }
  GML_HD uint32_t wmin(uint32_t v) const {
#if defined(__CUDA_ARCH__)
    return __reduce_min_sync(0xFFFFFFFFu, v);
#else
    return v;
#endif
  }
  GML_HD uint32_t match_any(uint32_t v) const {   // lanes holding the same value
#if defined(__CUDA_ARCH__)
    return __match_any_sync(0xFFFFFFFFu, v);
#else
    (void)v;
    return 1u;
#endif
  }
  GML_HD uint64_t add_u64(uint64_t v) const {
#if defined(__CUDA_ARCH__)
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
#endif
    return v;
  }
  // warp sum of u32 values, exact in 64 bits (two 16-bit halves, REDUX)
  GML_HD uint64_t sum_u32(uint32_t v) const {
#if defined(__CUDA_ARCH__)
    const uint32_t lo = __reduce_add_sync(0xFFFFFFFFu, v & 0xFFFFu), hi = __reduce_add_sync(0xFFFFFFFFu, v >> 16);
    return ((uint64_t)hi << 16) + lo;
#else
    return v;
#endif
  }
  GML_HD uint64_t bcast64(uint64_t v) const {   // lane 0's value
#if defined(__CUDA_ARCH__)
    const uint32_t lo = __shfl_sync(0xFFFFFFFFu, (uint32_t)v, 0), hi = __shfl_sync(0xFFFFFFFFu, (uint32_t)(v >> 32), 0);
    return ((uint64_t)hi << 32) | lo;
#else
    return v;
#endif
  }
  GML_HD uint32_t aadd(uint32_t* p, uint32_t v) const {
#if defined(__CUDA_ARCH__)
    return atomicAdd(p, v);
#else
    uint32_t o = *p; *p = o + v; return o;
#endif
  }
  // shared-memory / global atomics on u32 words (return the old value)
  GML_HD uint32_t aor(uint32_t* p, uint32_t v) const {
#if defined(__CUDA_ARCH__)
    return atomicOr(p, v);
#else
    uint32_t o = *p; *p = o | v; return o;
#endif
  }
  GML_HD uint32_t aand(uint32_t* p, uint32_t v) const {
#if defined(__CUDA_ARCH__)
    return atomicAnd(p, v);
#else
    uint32_t o = *p; *p = o & v; return o;
#endif
  }
};

struct HostWarp {
  using ctr_t = uint64_t;    // the live allocator runs for the life of a process
  static constexpr bool kReplay = false;
  GML_HD uint32_t lane() const { return 0; }
  GML_HD uint32_t width() const { return 1; }
  GML_HD bool leader() const { return true; }
  GML_HD void sync() const {}
  GML_HD uint32_t ballot(bool p) const { return p ? 1u : 0u; }
  GML_HD uint32_t shfl(uint32_t v, uint32_t) const { return v; }
  GML_HD uint32_t wmin(uint32_t v) const { return v; }
  GML_HD uint32_t match_any(uint32_t) const { return 1u; }
  GML_HD uint64_t add_u64(uint64_t v) const { return v; }
  GML_HD uint64_t bcast64(uint64_t v) const { return v; }
  GML_HD uint64_t sum_u32(uint32_t v) const { return v; }
  GML_HD uint32_t aadd(uint32_t* p, uint32_t v) const { uint32_t o = *p; *p = o + v; return o; }
  GML_HD uint32_t aor(uint32_t* p, uint32_t v) const { uint32_t o = *p; *p = o | v; return o; }
  GML_HD uint32_t aand(uint32_t* p, uint32_t v) const { uint32_t o = *p; *p = o & v; return o; }
};

// Driver-call hooks: the live allocator turns decisions into VMM calls; the
// replay kernel ignores them.
// on_alloc / on_stitch / on_bfc_segment run BEFORE the engine commits the
// new block and may fail (kCanFail): the engine then takes the S5 path ("If
// the Alloc function call fails, GMLake immediately reports an OOM",
// PAPER.md L528) with its tables consistent.
struct NoHooks {
  static constexpr bool kCanFail = false;
  GML_HD bool on_alloc(uint32_t, uint32_t, uint32_t) { return true; }
  GML_HD void on_split(uint32_t, uint32_t, uint32_t, uint32_t) {}
  GML_HD bool on_stitch(uint32_t, const uint32_t*, const uint32_t*, uint32_t) { return true; }
  GML_HD void on_evict(uint32_t) {}
  GML_HD bool on_bfc_segment(uint32_t, uint64_t) { return true; }
  GML_HD void on_bfc_release(uint32_t) {}
};

// ------------------------------------------------------------- table sizes
// Table capacities are compile-time per kernel instance ("size class"), so
// every table offset is an immediate and the engine keeps one base pointer;
// only the bitmap length (capacity / chunk) and the handle table (max slot)
// are runtime. The host picks the smallest class that fits each unit and
// moves a unit to the next class when a table overflows (D30).
// The BFC family (P = S = IV = 4: no pools) replays only BFC policies (the
// host never puts a GMLake unit in it), so its kernels compile without the
// VMM path: VMM = false removes vmm_malloc and its state from the instance.
// A GMLake class with B = 4 (no BFC rows: the VMM path of a split or path
// unit) compiles without the small path: SMALL = false removes bfc_malloc /
// bfc_free / bfc_release from the instance.
template <uint32_t P_, uint32_t S_, uint32_t IV_, uint32_t B_>
struct Cfg {
  static constexpr uint32_t P = P_, S = S_, IV = IV_, B = B_, CB = P_ + 4;
  static constexpr bool VMM = P_ > 4;
  static constexpr bool SMALL = B_ > 4;
};

GML_HD constexpr uint32_t round4(uint32_t x) { return (x + 3u) & ~3u; }

constexpr uint32_t BMS_WORDS = 128;          // summary words: bitmap <= 4096 words = 131072 chunks
constexpr uint64_t kMaxChunks = 32ull * 32 * BMS_WORDS;   // 256 GiB of 2 MiB chunks

template <class C>
struct Lay {                                  // offsets in u32 words from the arena base
  static constexpr uint32_t PINW = round4((C::P + 31) / 32);
  static constexpr uint32_t CACHE = 128;     // entries per size -> run-start cache
  static constexpr uint32_t STATS = 0;        // gml_stats_t, 68 words
  // sorted-set entries are 16-byte records {ordinal, size, row, witness}:
  // the u64 (size << 32 | ordinal) key is their first 8 bytes
  static constexpr uint32_t PE = 68;
  static constexpr uint32_t PN = PE + 4 * C::P, PLO = PN + C::P, PNEXT = PLO + C::P, PPOS = PNEXT + C::P;
  static constexpr uint32_t PCNT = PPOS + C::P;   // live sBlocks containing the pBlock (row)
  static constexpr uint32_t PIN = PCNT + C::P;
  static constexpr uint32_t PCACHE = PIN + PINW, SCACHE = PCACHE + 2 * CACHE;   // u64 size -> start caches
  static constexpr uint32_t MCACHE = SCACHE + 2 * CACHE;   // u64 size -> sPool S1 miss at epoch
  static constexpr uint32_t SE = MCACHE + 2 * CACHE;
  static constexpr uint32_t SN = SE + 4 * C::S, SORD = SN + C::S, SLAST = SORD + C::S, SBORN = SLAST + C::S,
                            SIVO = SBORN + C::S, SIVN = SIVO + C::S, SPND = SIVN + C::S, PSTK = SPND + C::S;
  static constexpr uint32_t IVROW = PSTK + C::S, IVLO = IVROW + 2 * C::IV, IVN = IVLO + 2 * C::IV;
  static constexpr uint32_t BSIZE = IVN + 2 * C::IV, BOFF = BSIZE + C::B, BSEG = BOFF + C::B,
                            BPREV = BSEG + C::B, BNEXT = BPREV + C::B, BPF = BNEXT + C::B;
  static constexpr uint32_t FLA = BPF + C::B, FLR = FLA + 2 * C::B, FLS = FLR + C::B;   // FLA: u64 address
  static constexpr uint32_t CB = FLS + C::B;
  static constexpr uint32_t BMS = CB + round4(C::CB);
  static constexpr uint32_t BM = BMS + BMS_WORDS;
  static_assert(C::P % 4 == 0 && C::S % 4 == 0 && C::IV % 4 == 0 && C::B % 4 == 0, "16-byte rows");
  static_assert(PCACHE % 4 == 0 && PE % 4 == 0 && SE % 4 == 0 && FLS % 4 == 0, "aligned u64 / vector tables");
  GML_HD static uint32_t h_off(uint32_t bm_words) { return BM + round4(bm_words); }   // u64 handle table
  GML_HD static uint64_t bytes(uint32_t bm_words, uint32_t h) { return 4ull * h_off(bm_words) + 8ull * h; }
};

struct RtCaps {
  uint32_t bm_words;   // ceil((capacity chunks + 1) / 32) <= 32 * BMS_WORDS
  uint32_t h;          // handle slots
};

// overflow bits (internal; reported through gml_stats_t._p, cleared by host)
enum : uint32_t { OV_P = 1, OV_S = 2, OV_IV = 4, OV_H = 8, OV_B = 16, OV_CB = 32 };

// BPF flags (low 30 bits: free-list index of a free block)
enum : uint32_t { BF_ALLOC = 0x80000000u, BF_POOL1 = 0x40000000u, BF_IDX = 0x3FFFFFFFu };
enum : int { ST_S1 = 1, ST_S2 = 2, ST_S3 = 3, ST_S4 = 4, ST_S5 = 5, ST_HIT = 6, ST_NEWSEG = 7 };
enum : uint32_t { HK_P = 0, HK_S = 1, HK_B = 2, HK_EMPTY = 3 };
enum { V_RESERVE, V_CREATE, V_MAP, V_ACCESS, V_UNMAP, V_ADDR_FREE, V_RELEASE };

constexpr uint64_t BFC_SMALL_SIZE = 1ull << 20;        // PyTorch kSmallSize (D21)
constexpr uint64_t BFC_SMALL_BUFFER = 2ull << 20;      // kSmallBuffer
constexpr uint64_t BFC_MIN_LARGE_ALLOC = 10ull << 20;  // kMinLargeAlloc
constexpr uint64_t BFC_LARGE_BUFFER = 20ull << 20;     // kLargeBuffer
constexpr uint64_t BFC_ROUND_LARGE = 2ull << 20;       // kRoundLarge

GML_HD uint64_t rec_of(uint32_t ord, uint32_t kind, uint32_t state) {
  return (uint64_t)ord | ((uint64_t)kind << 32) | ((uint64_t)state << 34);
}
GML_HD uint64_t rec_oom() { return 0xFFFFFFFFull | ((uint64_t)ST_S5 << 34); }

// ------------------------------------------------------------------ engine
// kFuse: S1 binds a proven sBlock from the intervals its proof left in the
// lanes (measured: faster with shared-memory arenas, slower with global ones)
// kPinS: the PIN words live in a separate (shared-memory) region given to
// init (persistent path units, whose arenas are in global memory: the pPool
// searches' PIN loads were their largest stall site); kBmS: the chunk bitmap
// (summary + words) follows them there
template <class W, class C, class HK = NoHooks, bool kFuse = true, bool kPinS = false, bool kBmS = false>
struct Engine {
  using L = Lay<C>;
  // An instance without the small path (the VMM path of a split or path
  // unit) leaves the requested-bytes, live-handle and active peaks (total and
  // VMM) to the unit's ledger and merge (split_kernel.cuh): it does not keep them.
  static constexpr bool kOwnPeaks = C::SMALL;
  W w;
  HK* hooks;
  // policy
  uint32_t kind, flags;
  uint64_t capacity, G, small_thr, vm_thr, limit_bytes, spool_max_inactive;
  uint32_t spool_max, elig_n, gshift;
  // tables: one base pointer, compile-time offsets (Lay<C>)
  uint32_t* A;
  uint64_t* H;          // handle table (runtime offset)
  uint32_t h_cap, bm_words;
  unsigned long long* prof = nullptr;   // GML_PHASE_PROF debug counters (output)
#if defined(GML_PROF_ON)
  unsigned long long pacc[16];
#endif
  // scalar state (identical in every thread of the group)
  uint32_t Cn, next_p, next_s, n_p, last_p, s_hw, s_count, s_freerow, iv_base, iv_hw;
  uint32_t pstk_n;      // sBlocks bound with their members' PIN bits deferred (lazy PIN, pin_flush)
  uint32_t sep;         // sPool epoch: bumped by every free that can make an sBlock inactive (miss cache)
  uint32_t b_hw, b_freerow, b_live, fl_n0, fl_n1, next_seg;
  uint64_t T, serial, active, requested, active_vmm, seg_bytes, s_bytes, s_bound, live;   // serial: mallocs (live allocator)
  uint32_t overflow, status;
  uint32_t born_row;    // sBlock row created earlier in this malloc (D17: not a count-cap victim)
  bool hk_fail;         // a driver hook failed (live allocator): the malloc is an S5
  bool sfb_clean;       // no VMM-path free since the last byte-cap check (stitch_free_bytes)
  // peaks kept in registers
  uint64_t pk_active, pk_reserved, pk_requested, pk_active_vmm, pk_reserved_vmm;
  uint32_t mx_p, mx_s, mx_h, mx_b;
  uint32_t live_iv, mx_iv;   // live sBlock intervals (sizing hint only)
  typename W::ctr_t sc[7];   // S1..S5, BFC hit, BFC new segment (registers: every malloc counts one;
                             // only constant indices, so the array stays in registers)

  // -------------------------------------------------------------- set-up
  uint32_t* pin_ext = nullptr;   // kPinS: the PIN words [, kBmS: then the bitmap summary and words]
  GML_HD uint32_t* pin() const {
    if constexpr (kPinS) return pin_ext;
    else return A + L::PIN;
  }
  GML_HD uint32_t* bms() const {
    if constexpr (kBmS) return pin_ext + L::PINW;
    else return A + L::BMS;
  }
  GML_HD uint32_t* bm() const { return bms() + BMS_WORDS; }
  GML_HDI void init(const gml_policy& pol, const RtCaps& c, uint8_t* arena, HK* hk, uint32_t* pin_words = nullptr) {
    pin_ext = pin_words;
    hooks = hk;
    kind = pol.kind;
    flags = pol.flags;
    capacity = pol.capacity_bytes;
    G = pol.chunk_bytes;
    small_thr = pol.small_threshold_bytes;
    limit_bytes = pol.frag_limit_bytes;
    // requests below vm_thr take the small path: < 2 MiB (D1) and,
    // under D8' (LIMIT_GATES_REQUEST), below the fragmentation limit
    vm_thr = small_thr;
    if ((flags & GML_F_LIMIT_GATES_REQUEST) && limit_bytes > vm_thr) vm_thr = limit_bytes;
    spool_max = pol.spool_max_entries;
    spool_max_inactive = pol.spool_max_inactive_bytes;
    // eligible (D8) iff n * G >= limit  <=>  n >= ceil(limit / G)
    uint64_t e = (limit_bytes + G - 1) / G;
    elig_n = e > 0x7FFFFFFFull ? 0x7FFFFFFFu : (uint32_t)e;
    gshift = 0xFF;
    for (uint32_t k = 0; k < 64; ++k)
      if ((1ull << k) == G) gshift = k;
    A = reinterpret_cast<uint32_t*>(arena);
    H = reinterpret_cast<uint64_t*>(A + L::h_off(c.bm_words));
    h_cap = c.h;
    bm_words = c.bm_words;
    Cn = next_p = next_s = n_p = s_hw = s_count = 0;
    last_p = NONE32;
    s_freerow = NONE32;
    iv_base = 0; iv_hw = 0;
    pstk_n = 0;
    sep = 0;
    b_hw = b_live = fl_n0 = fl_n1 = next_seg = 0;
    b_freerow = NONE32;
    T = serial = active = requested = active_vmm = seg_bytes = s_bytes = s_bound = live = 0;
    overflow = 0; status = GML_OK;
    born_row = NONE32;
    hk_fail = false;
    sfb_clean = false;
    pk_active = pk_reserved = pk_requested = pk_active_vmm = pk_reserved_vmm = 0;
    mx_p = mx_s = mx_h = mx_b = 0;
    live_iv = mx_iv = 0;
    for (int i = 0; i < 7; ++i) sc[i] = 0;
#if defined(GML_PROF_ON)
    for (int i = 0; i < 16; ++i) pacc[i] = 0;
#endif
    // zero stats, PIN, caches, bitmap; mark every handle slot empty
    uint32_t* sw = A + L::STATS;
    for (uint32_t i = w.lane(); i < sizeof(gml_stats_t) / 4; i += w.width()) sw[i] = 0;
    for (uint32_t i = w.lane(); i < L::PINW; i += w.width()) pin()[i] = 0;
    for (uint32_t i = w.lane(); i < BMS_WORDS + c.bm_words; i += w.width()) bms()[i] = 0;
    for (uint32_t i = w.lane(); i < 6 * L::CACHE; i += w.width()) A[L::PCACHE + i] = 0;
    for (uint32_t i = w.lane(); i < c.h; i += w.width()) H[i] = (uint64_t)HK_EMPTY << 62;
#if GML_FL_ZERO == 1
    for (uint32_t i = w.lane(); i < 4 * C::B; i += w.width()) A[L::FLA + i] = 0;   // FLA (2B), FLR, FLS
#endif
    w.sync();
  }

  GML_HD uint64_t reserved_vmm() const { return (uint64_t)Cn * G; }
  GML_HD uint64_t reserved() const { return reserved_vmm() + seg_bytes; }
  GML_HD gml_stats_t* S() const { return reinterpret_cast<gml_stats_t*>(A + L::STATS); }
  GML_HD void cnt(uint64_t& f, uint64_t v = 1) { if (w.leader()) f += v; }
  GML_HD uint4* pe() const { return reinterpret_cast<uint4*>(A + L::PE); }
  GML_HD uint4* se() const { return reinterpret_cast<uint4*>(A + L::SE); }
  GML_HD const uint64_t* pkeys() const { return reinterpret_cast<const uint64_t*>(A + L::PE); }   // stride 2
  GML_HD const uint64_t* skeys() const { return reinterpret_cast<const uint64_t*>(A + L::SE); }   // stride 2
  GML_HD static uint4 entry(uint32_t ord, uint32_t size, uint32_t row, uint32_t wit) {
    uint4 e;
    e.x = ord; e.y = size; e.z = row; e.w = wit;
    return e;
  }
  GML_HD static uint64_t skey(uint32_t size, uint32_t ord) { return ((uint64_t)size << 32) | ord; }

  GML_HD static uint32_t word_mask(uint32_t wd, uint32_t lo, uint32_t hi) {   // bits of [lo, hi] in word wd
    uint32_t m = 0xFFFFFFFFu;
    if (wd == (lo >> 5)) m &= 0xFFFFFFFFu << (lo & 31);
    if (wd == (hi >> 5)) m &= 0xFFFFFFFFu >> (31 - (hi & 31));
    return m;
  }

  // ------------------------------------------------------------ bitmap
  // set / clear the chunks of word wd selected by m (atomics: lanes working
  // on neighbouring intervals may share a word); a set also sets the summary
  // bit, a clear leaves it (bm_first clears it when it finds the word zero)
  GML_HD void bm_word(uint32_t wd, uint32_t m, bool on) {
    if (on) {
      w.aor(&bm()[wd], m);
      w.aor(&bms()[wd >> 5], 1u << (wd & 31));
    } else {
      w.aand(&bm()[wd], ~m);
    }
  }
  // chunks [lo, lo+n): words spread over the lanes
  GML_HD void bm_range_par(uint32_t lo, uint32_t n, bool on) {
    const uint32_t hi = lo + n - 1, a = lo >> 5, z = hi >> 5;
    GML_HC(18, z - a + 1); GML_HC(19, 1);
    for (uint32_t wd = a + w.lane(); wd <= z; wd += w.width()) bm_word(wd, word_mask(wd, lo, hi), on);
  }
  // chunks [lo, lo+n) by the calling thread alone
  GML_HD void bm_range_seq(uint32_t lo, uint32_t n, bool on) {
    const uint32_t hi = lo + n - 1, a = lo >> 5, z = hi >> 5;
    GML_HC(16, z - a + 1); GML_HC(17, 1); GML_HC(20 + (z - a < 8 ? z - a : 8), 1);
    for (uint32_t wd = a; wd <= z; ++wd) bm_word(wd, word_mask(wd, lo, hi), on);
  }
  GML_HD bool bm_bit(uint32_t c) const { return (bm()[c >> 5] >> (c & 31)) & 1u; }
  // single thread: some owned chunk of [lo, lo+n), NONE32 if none; interior
  // words are found through the summary level (a summary bit whose word is
  // zero is cleared on the way: no bind runs concurrently with a test)
  GML_HD uint32_t bm_first(uint32_t lo, uint32_t n) {
    const uint32_t hi = lo + n - 1, a = lo >> 5, z = hi >> 5;
    uint32_t v = bm()[a] & word_mask(a, lo, hi);
    if (v) return (a << 5) + ctz32(v);
    if (z == a) return NONE32;
    v = bm()[z] & word_mask(z, lo, hi);
    if (v) return (z << 5) + ctz32(v);
    if (z - a < 2) return NONE32;
    const uint32_t x = a + 1, y = z - 1;        // interior words [x, y]
    for (uint32_t sw = x >> 5; sw <= (y >> 5); ++sw) {
      for (uint32_t s = bms()[sw] & word_mask(sw, x, y); s; s &= s - 1) {
        const uint32_t wd = (sw << 5) + ctz32(s);
        const uint32_t v = bm()[wd];
        if (v) return (wd << 5) + ctz32(v);
        w.aand(&bms()[sw], ~(1u << (wd & 31)));
      }
    }
    return NONE32;
  }
  // Single thread: is the sBlock of sPool entry e at position pos inactive
  // (D18)? The witness answers
  // "active" while it stays owned; otherwise the intervals are tested and the
  // entry's witness is refreshed (or set to NONE32: tested inactive).
  GML_HD bool s_inactive_at(uint32_t pos, const uint4& e) {
    const uint32_t wt = e.w;
    if (wt != NONE32 && bm_bit(wt)) return false;
    const uint32_t r = e.z, o = A[L::SIVO + r], k = A[L::SIVN + r];
    for (uint32_t i = 0; i < k; ++i) {
      const uint32_t c = bm_first(A[L::IVLO + o + i], A[L::IVN + o + i]);
      if (c != NONE32) { se()[pos].w = c; return false; }
    }
    if (wt != NONE32) se()[pos].w = NONE32;
    return true;
  }

  // uniform (the whole warp): an owned chunk of sBlock r, NONE32 if it is
  // inactive; lanes test one interval each
  // keep (optional): this lane's interval of the first 32 (lane i <->
  // interval i) and its first member row, so that binding a proven-inactive
  // sBlock (S1) does not reload them
  struct IvLane { uint32_t k, lo, n, row; };
  GML_HD uint32_t s_proof(uint32_t r, IvLane* keep = nullptr) {
    const uint32_t o = A[L::SIVO + r], k = A[L::SIVN + r];
    for (uint32_t i0 = 0; i0 < k; i0 += w.width()) {
      const uint32_t i = i0 + w.lane();
      uint32_t c = NONE32, lo = 0, n = 0;
      if (i < k) { lo = A[L::IVLO + o + i]; n = A[L::IVN + o + i]; c = bm_first(lo, n); }
      if (keep && i0 == 0) { keep->k = k; keep->lo = lo; keep->n = n; keep->row = i < k ? A[L::IVROW + o + i] : 0u; }
      const uint32_t m = w.ballot(c != NONE32);
      if (m) return w.shfl(c, ctz32(m));
    }
    return NONE32;
  }

  // uniform: every member pBlock row of sBlock s, in interval order
  template <class F>
  GML_HD void s_members(uint32_t s, F&& f) {
    const uint32_t o = A[L::SIVO + s], k = A[L::SIVN + s];
    for (uint32_t i = 0; i < k; ++i) {
      uint32_t r = A[L::IVROW + o + i];
      for (uint32_t left = A[L::IVN + o + i]; left;) {
        const uint32_t nx = A[L::PNEXT + r], pn = A[L::PN + r];
        f(r);
        left -= pn;
        r = nx;
      }
    }
  }

  // --------------------------------------------------------- sorted sets
  // W-ary search (W lanes test W pivots per step): first index with
  // a[ST * i] >= x (ST = 2: keys of 16-byte entries)
  template <uint32_t ST = 2>
  GML_HD uint32_t lower_bound(const uint64_t* a, uint32_t n, uint64_t x) {
    if (w.width() == 1) {                       // host: plain binary search
      uint32_t lo = 0, hi = n;
      while (lo < hi) {
        uint32_t mid = lo + (hi - lo) / 2;
        if (a[ST * mid] < x) lo = mid + 1; else hi = mid;
      }
      return lo;
    }
    const uint32_t WD = w.width();
    uint32_t lo = 0, hi = n;                    // answer in [lo, hi]
    while (hi - lo > WD) {
      const uint32_t len = hi - lo;
      const uint32_t i = w.lane();
      const uint32_t piv = lo + (uint32_t)(((uint64_t)len * (i + 1)) / WD) - 1;
      const uint32_t m = w.ballot(a[ST * piv] >= x);
      if (!m) return hi;
      const uint32_t j = ctz32(m);
      uint32_t nlo = lo + (uint32_t)(((uint64_t)len * j) / WD);
      hi = lo + (uint32_t)(((uint64_t)len * (j + 1)) / WD) - 1;
      lo = nlo;
    }
    const uint32_t k = lo + w.lane();
    const uint32_t m = w.ballot(k < hi && a[ST * k] >= x);
    return m ? lo + ctz32(m) : hi;
  }
  // Sorted-set shifts: 4 entries per lane per round (the 4 loads of a lane
  // are independent, so a round of 4 x width entries costs about one load's
  // latency); with ppos the moved pBlocks' positions follow. Out of line on
  // the device (static: no `this`, so the engine's registers stay put) --
  // inlined, the unrolled body inflates every kernel's register allocation.
  template <bool kPos>
  GML_NOINL static void shift_up(W w, uint4* a, uint32_t* ppos, uint32_t lo, uint32_t n) {   // a[lo,n) -> a[lo+1,n+1)
    constexpr int U = GML_SHIFT_U;
    const int32_t WD = (int32_t)w.width(), CH = U * WD;
    GML_HC(11, n - lo); GML_HC(15, 1);
    for (int32_t top = (int32_t)n - 1; top >= (int32_t)lo; top -= CH) {
      uint4 v[U];
      int32_t idx[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        idx[u] = top - (int32_t)w.lane() - u * WD;
        if (idx[u] >= (int32_t)lo) v[u] = a[idx[u]];
      }
      w.sync();
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (idx[u] >= (int32_t)lo) {
          a[idx[u] + 1] = v[u];
          if (kPos) ppos[v[u].z] = (uint32_t)idx[u] + 1;
        }
      w.sync();
    }
  }
  template <bool kPos>
  GML_NOINL static void shift_down(W w, uint4* a, uint32_t* ppos, uint32_t pos, uint32_t n) {   // a[pos+1,n) -> a[pos,n-1)
    constexpr int U = GML_SHIFT_U;
    const uint32_t WD = w.width(), CH = U * WD;
    GML_HC(11, n - pos); GML_HC(15, 1);
    for (uint32_t base = pos; base + 1 < n; base += CH) {
      uint4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t i = base + w.lane() + u * WD;
        if (i + 1 < n) v[u] = a[i + 1];
      }
      w.sync();
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t i = base + w.lane() + u * WD;
        if (i + 1 < n) {
          a[i] = v[u];
          if (kPos) ppos[v[u].z] = i;
        }
      }
      w.sync();
    }
  }

  // sPool sorted set: insert entry e / erase the entry with key k
  GML_HD void s_insert(const uint4& e) {
    const uint32_t n = s_count;
    const uint32_t pos = lower_bound(skeys(), n, skey(e.y, e.x));
    uint4* a = se();
    shift_up<false>(w, a, nullptr, pos, n);
    cache_clear(L::SCACHE);
    if (w.leader()) a[pos] = e;
    w.sync();
  }
  GML_HD void s_erase(uint64_t k) {
    const uint32_t n = s_count;
    const uint32_t pos = lower_bound(skeys(), n, k);   // present by construction
    shift_down<false>(w, se(), nullptr, pos, n);
    cache_clear(L::SCACHE);
    w.sync();
  }

  // ---- run-start caches: size b -> lower_bound(keys, skey(b, 0)), valid
  // until the next insert / erase of that sorted set (which clears it). In
  // steady state (only S1) every lookup hits.
  GML_HD uint32_t run_start(uint32_t cache, const uint64_t* key, uint32_t n, uint32_t b) {
    uint64_t* c = reinterpret_cast<uint64_t*>(A + cache);
    const uint32_t h = b & (L::CACHE - 1);
    const uint64_t e = c[h];
    if ((uint32_t)e == b + 1) return (uint32_t)(e >> 32);
    const uint32_t x = lower_bound(key, n, skey(b, 0));
    w.sync();
    if (w.leader()) c[h] = ((uint64_t)x << 32) | (b + 1);
    w.sync();
    return x;
  }
  GML_HD void cache_clear(uint32_t cache) {
    uint4* c = reinterpret_cast<uint4*>(A + cache);
    uint4 z;
    z.x = z.y = z.z = z.w = 0;
    for (uint32_t i = w.lane(); i < L::CACHE / 2; i += w.width()) c[i] = z;
  }
  GML_HD uint32_t p_start(uint32_t b) { return run_start(L::PCACHE, pkeys(), n_p, b); }
  GML_HD uint32_t s_start(uint32_t b) { return run_start(L::SCACHE, skeys(), s_count, b); }

  // ---- pPool: sorted set + PPOS + PIN (inactive bit per position) ----
  // first set PIN bit at a position >= x (positions >= n_p are never set)
  GML_HD uint32_t pin_first(uint32_t x) {
    const uint32_t nw = (n_p + 31) >> 5, x0 = x >> 5;
    for (uint32_t w0 = x0; w0 < nw; w0 += w.width()) {
      const uint32_t wd = w0 + w.lane();
      uint32_t v = wd < nw ? pin()[wd] : 0u;
      if (wd == x0) v &= 0xFFFFFFFFu << (x & 31);
      const uint32_t m = w.ballot(v != 0);
      if (m) {
        const uint32_t l = ctz32(m);
        return ((w0 + l) << 5) + ctz32(w.shfl(v, l));
      }
    }
    return NONE32;
  }
  // last set PIN bit in [lo, hi); NONE32 if none
  GML_HD uint32_t pin_last(uint32_t lo, uint32_t hi) {
    if (hi <= lo) return NONE32;
    const int32_t wlo = (int32_t)(lo >> 5), whi = (int32_t)((hi - 1) >> 5);
    for (int32_t w0 = whi; w0 >= wlo; w0 -= (int32_t)w.width()) {
      const int32_t wd = w0 - (int32_t)w.lane();
      uint32_t v = wd >= wlo ? pin()[wd] & word_mask((uint32_t)wd, lo, hi - 1) : 0u;
      const uint32_t m = w.ballot(v != 0);
      if (m) {
        const uint32_t l = ctz32(m);
        return ((uint32_t)(w0 - (int32_t)l) << 5) + 31 - clz32(w.shfl(v, l));
      }
    }
    return NONE32;
  }
  GML_HD void pin_set(uint32_t r, bool inactive) {   // one lane
    const uint32_t pos = A[L::PPOS + r];
    if (inactive) w.aor(&pin()[pos >> 5], 1u << (pos & 31));
    else w.aand(&pin()[pos >> 5], ~(1u << (pos & 31)));
  }
  // insert key k (row r, inactive) at its place among n_p entries
  GML_HD void p_insert(uint64_t k, uint32_t r) {
    const uint32_t n = n_p;
    const uint32_t pos = lower_bound(pkeys(), n, k);
    uint4* a = pe();
    shift_up<true>(w, a, A + L::PPOS, pos, n);
    const int32_t WD = (int32_t)w.width();
    // PIN bits [pos, n) move up by one; bit pos = 1 (inactive)
    const int32_t wp = (int32_t)(pos >> 5), wt = (int32_t)(n >> 5);
    for (int32_t top = wt; top >= wp; top -= WD) {
      const int32_t wd = top - (int32_t)w.lane();
      const bool on = wd >= wp;
      uint32_t nv = 0;
      if (on) {
        const uint32_t v = pin()[wd];
        const uint32_t below = wd > wp ? pin()[wd - 1] >> 31 : 0u;
        const uint32_t sh = (v << 1) | below;
        if (wd == wp) {
          const uint32_t bb = pos & 31, low = (1u << bb) - 1u;
          nv = (v & low) | (sh & ~low) | (1u << bb);
        } else {
          nv = sh;
        }
      }
      w.sync();
      if (on) pin()[wd] = nv;
      w.sync();
    }
    cache_clear(L::PCACHE);
    if (w.leader()) { a[pos] = entry((uint32_t)k, (uint32_t)(k >> 32), r, 0); A[L::PPOS + r] = pos; }
    w.sync();
  }
  // erase the entry at position pos (of n_p entries)
  GML_HD void p_erase_at(uint32_t pos) {
    const uint32_t n = n_p;
    shift_down<true>(w, pe(), A + L::PPOS, pos, n);
    const uint32_t WD = w.width();
    // PIN bits (pos, n) move down by one; bit n-1 becomes 0
    const uint32_t wp = pos >> 5, wl = (n - 1) >> 5;
    for (uint32_t bot = wp; bot <= wl; bot += WD) {
      const uint32_t wd = bot + w.lane();
      const bool on = wd <= wl;
      uint32_t nv = 0;
      if (on) {
        const uint32_t v = pin()[wd];
        const uint32_t above = wd < wl ? (pin()[wd + 1] & 1u) : 0u;
        const uint32_t sh = (v >> 1) | (above << 31);
        if (wd == wp) {
          const uint32_t low = (1u << (pos & 31)) - 1u;
          nv = (v & low) | (sh & ~low);
        } else {
          nv = sh;
        }
      }
      w.sync();
      if (on) pin()[wd] = nv;
      w.sync();
    }
    cache_clear(L::PCACHE);
    w.sync();
  }

  // --------------------------------------------------------- sPool rows
  GML_HD void s_evict(uint32_t r) {   // StitchFree of one sBlock
    s_members(r, [&](uint32_t m) {
      if (w.leader()) A[L::PCNT + m] -= 1u;
    });
    w.sync();
    const uint32_t sn = A[L::SN + r];
    s_bytes -= (uint64_t)sn * G;
    live_iv -= A[L::SIVN + r];
    s_erase(skey(sn, A[L::SORD + r]));
    w.sync();
    if (w.leader()) {
      A[L::SN + r] = 0;
      A[L::SBORN + r] = s_freerow;     // free-row link
    }
    s_freerow = r;
    s_count--;
    cnt(S()->n_evict);
    cnt(S()->vmm_calls[V_UNMAP]);
    cnt(S()->vmm_calls[V_ADDR_FREE]);
    if (w.leader()) hooks->on_evict(r);
    w.sync();
  }

  // argmin of last_use over inactive live sBlocks (optionally excluding the
  // ones born in this malloc); NONE32 if none. last_use values are unique.
  GML_HD uint32_t s_lru(bool exclude_born) {
    uint32_t best = NONE32, row = NONE32;
    GML_HC(14, 1);
    for (uint32_t p = w.lane(); p < s_count; p += w.width()) {
      const uint4 e = se()[p];
      if (exclude_born && e.z == born_row) continue;   // (a malloc creates at most one sBlock before its last)
      const uint32_t lu = A[L::SLAST + e.z];
      if (lu < best && s_inactive_at(p, e)) { best = lu; row = e.z; }
    }
    w.sync();   // the lanes' witness rewrites (s_inactive_at) precede any later read of the entries
    const uint32_t g = w.wmin(best);
    if (g == NONE32) return NONE32;
    return w.shfl(row, ctz32(w.ballot(best == g)));
  }

  // D17(ii): at VMM-path malloc entry, release LRU inactive sBlocks while the
  // inactive ones hold more than the byte cap. Two
  // upper bounds settle most calls without testing every sBlock: bound
  // sBlocks are active (s_bytes - s_bound), and an sBlock whose witness
  // chunk is still owned is active, one whose last full test found nothing
  // is counted as inactive untested. Only if that bound exceeds the cap are
  // the untested ones tested, giving the exact figure.
  //
  // After any check the inactive bytes are <= the cap, and only a VMM-path
  // free can raise them (a malloc binds, and its stitches are bound at once
  // or overlap the block it binds): with no such free since the last check,
  // the check is skipped (sfb_clean).
  GML_HD void stitch_free_bytes() {
    if (sfb_clean) return;
    sfb_clean = true;
    if (s_bytes - s_bound <= spool_max_inactive) return;
    // bound 2: witness bits only (an entry whose witness is not owned counts
    // as inactive, untested); 4 entries per lane per round, loads independent;
    // granules per lane fit u32 (S <= 65536 entries of < 2^17 granules / 32)
    {
      uint32_t g = 0;
      const uint32_t WD = w.width();
      for (uint32_t p0 = 0; p0 < s_count; p0 += 4 * WD) {
        uint4 e[4];
        bool on[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint32_t p = p0 + w.lane() + u * WD;
          on[u] = p < s_count;
          if (on[u]) e[u] = se()[p];
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (on[u] && (e[u].w == NONE32 || !bm_bit(e[u].w))) g += e[u].y;
      }
      if (w.sum_u32(g) * G <= spool_max_inactive) return;
    }
    uint64_t part = 0;
    // bound 3: entries with a stale witness are tested (and re-witnessed)
    for (uint32_t p = w.lane(); p < s_count; p += w.width()) {
      const uint4 e = se()[p];
      if (e.w == NONE32 || (!bm_bit(e.w) && s_inactive_at(p, e))) part += (uint64_t)e.y * G;
    }
    if (w.add_u64(part) <= spool_max_inactive) return;
    part = 0;
    for (uint32_t p = w.lane(); p < s_count; p += w.width()) {
      const uint4 e = se()[p];
      if (s_inactive_at(p, e)) part += (uint64_t)e.y * G;
    }
    uint64_t inact = w.add_u64(part);
    w.sync();
    while (inact > spool_max_inactive) {
      uint32_t v = s_lru(false);
      if (v == NONE32) break;
      inact -= (uint64_t)A[L::SN + v] * G;
      s_evict(v);
    }
  }

  // interval arena: double-buffered; compaction copies live lists to the
  // other half (rows keep their identity).
  GML_HD bool iv_reserve(uint32_t k) {
    if (iv_hw + k <= C::IV) return true;
    GML_HC(12, 1); GML_HC(13, s_hw);
    uint32_t dst = iv_base ^ C::IV;   // other half
    uint32_t pos = 0;
    for (uint32_t r = 0; r < s_hw; ++r) {
      if (A[L::SN + r] == 0) continue;
      uint32_t o = A[L::SIVO + r], n = A[L::SIVN + r];
      for (uint32_t i = w.lane(); i < n; i += w.width()) {
        A[L::IVROW + dst + pos + i] = A[L::IVROW + o + i];
        A[L::IVLO + dst + pos + i] = A[L::IVLO + o + i];
        A[L::IVN + dst + pos + i] = A[L::IVN + o + i];
      }
      w.sync();
      if (w.leader()) A[L::SIVO + r] = dst + pos;
      pos += n;
    }
    w.sync();
    iv_base = dst;
    iv_hw = pos;
    if (iv_hw + k > C::IV) { overflow |= OV_IV; return false; }
    return true;
  }

  // Stitch of the pBlock rows rows[0..k): a new sBlock
  // over their chunks, no new physical memory. Count cap (D17(i)): evict
  // LRU inactive sBlocks not born in this malloc while at the cap; a
  // companion that finds no room is skipped. Returns the row or NONE32.
  GML_HD uint32_t stitch(const uint32_t* rows, uint32_t k, bool companion) {   // (phase-timed in GML_PHASE_PROF builds)
    GML_T0(t);
    const uint32_t r = stitch_impl(rows, k, companion);
    GML_T1(13, t);
    return r;
  }
  GML_COLD uint32_t stitch_impl(const uint32_t* rows, uint32_t k, bool companion) {
    while (s_count >= spool_max) {
      uint32_t v = s_lru(true);
      if (v == NONE32) break;
      s_evict(v);
    }
    if (companion && s_count >= spool_max) return NONE32;
    if (!iv_reserve(k)) return NONE32;   // (may compact: before a new row exists)
    uint32_t r;
    if (s_freerow != NONE32) {
      r = s_freerow;
      s_freerow = A[L::SBORN + r];
    } else {
      if (s_hw >= C::S) { overflow |= OV_S; return NONE32; }
      r = s_hw++;
    }
    const uint32_t o = iv_base + iv_hw;
    uint32_t tot = 0;
    for (uint32_t i = 0; i < k; ++i) tot += A[L::PN + rows[i]];
    for (uint32_t i = w.lane(); i < k; i += w.width()) {
      uint32_t m = rows[i];
      A[L::IVROW + o + i] = m;
      A[L::IVLO + o + i] = A[L::PLO + m];
      A[L::IVN + o + i] = A[L::PN + m];
      A[L::PCNT + m] += 1u;   // (members are distinct rows)
    }
    const uint32_t niv = k;   // one interval per member: s_own spreads members over lanes
                              // (merging adjacent members measured slower: serial member walks)
    iv_hw += niv;
    live_iv += niv;
    if (live_iv > mx_iv) mx_iv = live_iv;
    lru_tick();
    born_row = r;
    w.sync();
    if (w.leader()) {
      A[L::SN + r] = tot; A[L::SORD + r] = next_s; A[L::SLAST + r] = (uint32_t)T;
      A[L::SIVO + r] = o; A[L::SIVN + r] = niv; A[L::SPND + r] = 0u;
    }
    w.sync();
    // witness: the first member's first chunk, owned right after (the stitch
    // or, for a companion, its front piece is bound next)
    s_insert(entry(next_s, tot, r, A[L::PLO + rows[0]]));
    next_s++;
    s_count++;
    if (s_count > mx_s) mx_s = s_count;   // (no sBlock is released later in the same malloc)
    s_bytes += (uint64_t)tot * G;
    cnt(S()->n_stitch);
    if (companion) cnt(S()->n_companion);
    cnt(S()->vmm_calls[V_RESERVE]);
    cnt(S()->vmm_calls[V_MAP], tot);
    cnt(S()->vmm_calls[V_ACCESS], tot);
    w.sync();
    bool hok = true;
    if (w.leader()) hok = hooks->on_stitch(r, A + L::IVLO + o, A + L::IVN + o, niv);
    if (HK::kCanFail && !hok) {   // no mapping: the sBlock goes again
      s_evict(r);
      hk_fail = true;
      return NONE32;
    }
    return r;
  }

  // LRU clock (D17): SLAST holds the low 32 bits of T. A replayed trace has
  // < 2^32 events; the live allocator renumbers the keys of its live sBlocks
  // (order kept) before the 32-bit stamps could wrap.
  GML_HD void lru_tick() {
    if constexpr (!W::kReplay) {
      if (T >= 0xFFFFFF00ull) lru_renumber();
    }
    T++;
  }
  // width-1 executor only (live allocator), once per ~4e9 touches: the i-th
  // smallest key becomes i; since the i-th smallest old key is >= i, the
  // keys not yet renumbered are exactly those > k
  GML_HD void lru_renumber() {
    uint32_t k = 0;
    for (;;) {
      uint32_t best = NONE32, br = NONE32;
      for (uint32_t r = 0; r < s_hw; ++r)
        if (A[L::SN + r] && A[L::SLAST + r] > k && A[L::SLAST + r] < best) {
          best = A[L::SLAST + r];
          br = r;
        }
      if (br == NONE32) break;
      A[L::SLAST + br] = ++k;
    }
    T = k;
  }

  // Split: P -> F (first n chunks, keeps P's row, new
  // ordinal) + R (new row); no memory is created (D10). P is inactive.
  GML_HD uint32_t split(uint32_t P, uint32_t n) {   // (phase-timed in GML_PHASE_PROF builds)
    GML_T0(t);
    const uint32_t r = split_impl(P, n);
    GML_T1(12, t);
    return r;
  }
  GML_COLD uint32_t split_impl(uint32_t P, uint32_t n) {
    if (n_p >= C::P) { overflow |= OV_P; return NONE32; }
    const uint32_t lo = A[L::PLO + P], pnn = A[L::PN + P], nx = A[L::PNEXT + P];
    p_erase_at(A[L::PPOS + P]);
    n_p--;
    const uint32_t R = n_p + 1;                   // row count before the erase
    p_insert(skey(n, next_p), P);
    n_p++;
    if (w.leader()) {
      A[L::PN + P] = n; A[L::PNEXT + P] = R; A[L::PCNT + R] = A[L::PCNT + P];   // (R is inside every sBlock over P)
      A[L::PLO + R] = lo + n; A[L::PN + R] = pnn - n; A[L::PNEXT + R] = nx;
    }
    w.sync();
    p_insert(skey(pnn - n, next_p + 1), R);
    n_p++;
    if (n_p > mx_p) mx_p = n_p;
    if (last_p == P) last_p = R;
    next_p += 2;
    cnt(S()->n_split);
    cnt(S()->vmm_calls[V_RESERVE], 2);
    cnt(S()->vmm_calls[V_MAP], pnn);
    cnt(S()->vmm_calls[V_ACCESS], pnn);
    cnt(S()->vmm_calls[V_UNMAP]);
    cnt(S()->vmm_calls[V_ADDR_FREE]);
    w.sync();
    if (w.leader()) hooks->on_split(P, R, lo, n);
    if (flags & GML_F_SPLIT_INVALIDATES) {   // D12 variant: drop sBlocks over P
      for (uint32_t r = 0; r < s_hw; ++r) {  // uniform walk (rare path)
        if (!A[L::SN + r]) continue;
        uint32_t o = A[L::SIVO + r], k = A[L::SIVN + r];
        bool hit = false;
        for (uint32_t i = 0; i < k; ++i)
          if (A[L::IVLO + o + i] < lo + pnn && lo < A[L::IVLO + o + i] + A[L::IVN + o + i]) hit = true;
        if (hit) s_evict(r);
      }
    }
    return R;
  }

  // Alloc: the only source of new chunks.
  GML_HD uint32_t alloc(uint32_t n) {   // (phase-timed in GML_PHASE_PROF builds)
    GML_T0(t);
    const uint32_t r = alloc_impl(n);
    GML_T1(14, t);
    return r;
  }
  GML_COLD uint32_t alloc_impl(uint32_t n) {
    if (n_p >= C::P) { overflow |= OV_P; return NONE32; }
    const uint32_t r = n_p;
    bool hok = true;
    if (w.leader()) hok = hooks->on_alloc(r, Cn, n);
    if (HK::kCanFail && !hok) { hk_fail = true; return NONE32; }   // nothing committed
    if (w.leader()) {
      A[L::PLO + r] = Cn; A[L::PN + r] = n; A[L::PNEXT + r] = NONE32; A[L::PCNT + r] = 0u;
      if (last_p != NONE32) A[L::PNEXT + last_p] = r;
    }
    w.sync();
    p_insert(skey(n, next_p), r);
    n_p++;
    last_p = r;
    next_p++;
    Cn += n;
    if (n_p > mx_p) mx_p = n_p;
    sample_growth();
    cnt(S()->n_alloc);
    cnt(S()->vmm_calls[V_RESERVE]);
    cnt(S()->vmm_calls[V_CREATE], n);
    cnt(S()->vmm_calls[V_MAP], n);
    cnt(S()->vmm_calls[V_ACCESS], n);
    w.sync();
    return r;
  }

  GML_HD void bind_p(uint32_t slot, uint32_t r, uint64_t raw) {
    const uint32_t n = A[L::PN + r];
    bm_range_par(A[L::PLO + r], n, true);
    if (w.leader()) {
      pin_set(r, false);
      H[slot] = ((uint64_t)HK_P << 62) | ((uint64_t)r << 40) | raw;
    }
    const uint64_t by = (uint64_t)n * G;
    active += by; active_vmm += by;
    if constexpr (kOwnPeaks) requested += raw;
    w.sync();
  }
  // Lazy PIN for sBlocks. Binding an sBlock owns its chunks in the bitmap at
  // once (sBlock activity, D18, reads only the bitmap) but defers clearing
  // its member pBlocks' PIN bits: the row is marked pending (SPND) and
  // pushed on a stack (PSTK). PIN is read only by the pPool searches of a
  // malloc whose sPool S1 scan missed (S1 pPool, S2, S3), which first flush
  // the pending rows (pin_flush). A pending sBlock freed before any flush
  // only releases its chunks: its members' PIN bits were never cleared
  // (C2 V3: 78 % of sBlock binds end before a pPool search).
  //
  // own (on) or release every chunk of sBlock s and, if pin, flip the PIN
  // bits of the pBlocks inside its intervals: one lane per interval
  // returns (in the leader) the first chunk of the first interval
  GML_HD uint32_t s_own(uint32_t s, bool on, bool pin = true) {
    const uint32_t o = A[L::SIVO + s], k = A[L::SIVN + s];
    uint32_t first = NONE32;
    GML_HC(5, 1); GML_HC(6, k);
    for (uint32_t i = w.lane(); i < k; i += w.width()) {
      const uint32_t lo = A[L::IVLO + o + i], n = A[L::IVN + o + i];
      uint32_t r = A[L::IVROW + o + i];
      if (i == 0) first = lo;
      bm_range_seq(lo, n, on);
      if (pin)
        for (uint32_t left = n; left;) {
          const uint32_t pn = A[L::PN + r], nx = A[L::PNEXT + r];
          pin_set(r, !on);
          GML_HC(7, 1);
          left -= pn;
          r = nx;
        }
    }
    w.sync();
    return first;
  }
  // own the chunks of a proven sBlock from the intervals its proof left in
  // the lanes (<= 32 intervals); its PIN bits are deferred (lazy PIN)
  GML_HD uint32_t s_own_kept(const IvLane& kv) {
    if (w.lane() < kv.k) bm_range_seq(kv.lo, kv.n, true);
    const uint32_t first = w.shfl(kv.lo, 0);
    w.sync();
    return first;
  }
  // A free that releases chunks some live sBlock contains (an sBlock, or a
  // pBlock whose containment count PCNT is non-zero) may make sBlocks
  // inactive: it opens a new sPool epoch (the S1 miss cache, below) and
  // re-arms the byte-cap check (stitch_free_bytes). A free of a pBlock no
  // sBlock contains changes no sBlock's activity (D18): it does neither.
  GML_HD void spool_touched() {
    sfb_clean = false;
    if (++sep == 0) cache_clear(L::MCACHE);   // (epoch wrap: forget every cached miss)
  }

  // mark bound sBlock r pending (its members' PIN bits not yet cleared)
  GML_HD void pin_defer(uint32_t r) {
    if (pstk_n >= C::S) pin_flush();   // (stack full: flush first)
    if (w.leader()) {
      A[L::SPND + r] = 1u;
      A[L::PSTK + pstk_n] = r;
    }
    pstk_n++;
  }
  // clear the PIN bits of the members of every pending bound sBlock: lanes
  // over the stack (an entry whose sBlock was freed meanwhile, or repeated,
  // finds SPND clear)
  GML_HD void pin_flush() {
    for (uint32_t i = w.lane(); i < pstk_n; i += w.width()) {
      const uint32_t s = A[L::PSTK + i];
      if (!A[L::SPND + s]) continue;
      A[L::SPND + s] = 0u;
      const uint32_t o = A[L::SIVO + s], k = A[L::SIVN + s];
      for (uint32_t j = 0; j < k; ++j) {
        uint32_t r = A[L::IVROW + o + j];
        for (uint32_t left = A[L::IVN + o + j]; left;) {
          const uint32_t pn = A[L::PN + r], nx = A[L::PNEXT + r];
          pin_set(r, false);
          left -= pn;
          r = nx;
        }
      }
    }
    pstk_n = 0;
    w.sync();
  }
  // kv (optional): the sBlock's intervals as its proof left them; sn: its size
  GML_HD void bind_s(uint32_t slot, uint32_t r, uint64_t raw, uint32_t pos = NONE32, const IvLane* kv = nullptr,
                     uint32_t sn = 0) {
    const uint32_t first = (kv && kv->k <= w.width()) ? s_own_kept(*kv) : s_own(r, true, false);
    pin_defer(r);   // (measured: deferring only S1 reuses, not fresh S3/S4 stitches, gains nothing)
    if (w.leader()) {
      H[slot] = ((uint64_t)HK_S << 62) | ((uint64_t)r << 40) | raw;
      if (pos != NONE32) se()[pos].w = first;   // its own first chunk: owned now
    }
    const uint64_t by = (uint64_t)(kv ? sn : A[L::SN + r]) * G;
    active += by; active_vmm += by; s_bound += by;
    if constexpr (kOwnPeaks) requested += raw;
    w.sync();
  }

  // --------------------------------------------------------------- BFC
  // One free-list array for both pools: pool 0 at [0, fl_n0), pool 1 at
  // [B - fl_n1, B); BPF[row] holds a free block's index.
  GML_HD uint32_t fl_lo(uint32_t pool) const { return pool ? C::B - fl_n1 : 0u; }
  GML_HD uint32_t fl_hi(uint32_t pool) const { return pool ? C::B : fl_n0; }
  GML_HD uint64_t* fla() const { return reinterpret_cast<uint64_t*>(A + L::FLA); }
  // a slot for a new entry of `pool` (GML_FL_ZERO == 0: when a pool grows
  // into a vector group, the group's other entries, outside both pools, are
  // zeroed by the leader)
  GML_HD uint32_t fl_grow(uint32_t pool) {
    const uint32_t k = pool ? C::B - 1 - fl_n1 : fl_n0;
    if (pool) fl_n1++; else fl_n0++;
#if GML_FL_ZERO == 0
    if (w.leader() && (k & 3) == (pool ? 3u : 0u)) {
      const uint32_t a = pool ? ((k >= 3 && k - 3 > fl_n0) ? k - 3 : fl_n0) : k + 1;
      const uint32_t z = pool ? k : (k + 4 < C::B - fl_n1 ? k + 4 : C::B - fl_n1);
      for (uint32_t i = a; i < z; ++i) {
        A[L::FLS + i] = 0; A[L::FLR + i] = 0; fla()[i] = 0;
      }
    }
#endif
    return k;
  }
  GML_HD void fl_push(uint32_t pool, uint32_t r, uint32_t size, uint64_t addr) {
    const uint32_t k = fl_grow(pool);
    if (w.leader()) {
      A[L::FLR + k] = r; A[L::FLS + k] = size; fla()[k] = addr;
      A[L::BPF + r] = k | (pool ? BF_POOL1 : 0u);
    }
  }
  // remove entry k (the last entry of the pool moves into it)
  GML_HD void fl_remove_at(uint32_t pool, uint32_t k) {
    const uint32_t last = pool ? C::B - fl_n1 : fl_n0 - 1;
    const uint32_t lr = A[L::FLR + last], ls = A[L::FLS + last];
    const uint64_t la = fla()[last];
    w.sync();
    if (w.leader() && k != last) {
      A[L::FLR + k] = lr; A[L::FLS + k] = ls; fla()[k] = la;
      A[L::BPF + lr] = k | (pool ? BF_POOL1 : 0u);
    }
    if (pool) fl_n1--; else fl_n0--;
    w.sync();
  }
  // link: the free-row list successor of b_freerow, if the caller loaded
  // it already (before any write; the caller syncs before rewriting the row)
  GML_HD uint32_t b_newrow(uint32_t link = NONE32, bool have_link = false) {
    uint32_t r;
    if (b_freerow != NONE32) {
      r = b_freerow;
      if (have_link) {
        b_freerow = link;
      } else {
        b_freerow = A[L::BNEXT + r];
        w.sync();   // every lane has read the link before the leader rewrites the row
      }
    } else if (b_hw < C::B) {
      r = b_hw++;
    } else {
      overflow |= OV_B;
      return NONE32;
    }
    b_live++;
    if (b_live > mx_b) mx_b = b_live;
    return r;
  }
  GML_HD void b_delrow(uint32_t r) {
    if (w.leader()) A[L::BNEXT + r] = b_freerow;
    b_freerow = r;
    b_live--;
  }

  // release every fully free segment (PyTorch release_cached_blocks on the
  // OOM path); uniform sequential walk of the free lists (rare path).
  GML_HD void bfc_release() {
    for (uint32_t pool = 0; pool < 2; ++pool) {
      uint32_t k = fl_lo(pool);
      while (k < fl_hi(pool)) {
        uint32_t r = A[L::FLR + k];
        if (A[L::BPREV + r] == NONE32 && A[L::BNEXT + r] == NONE32) {
          seg_bytes -= (uint64_t)A[L::BSIZE + r] * 512;
          cnt(S()->n_seg_release);
          if (w.leader()) hooks->on_bfc_release(A[L::BSEG + r]);
          if (pool) {                 // pool 1 shrinks from the bottom: move its lowest entry into k
            const uint32_t first = C::B - fl_n1;
            const uint32_t fr = A[L::FLR + first], fs = A[L::FLS + first];
            const uint64_t fa = fla()[first];
            w.sync();
            if (w.leader() && k != first) { A[L::FLR + k] = fr; A[L::FLS + k] = fs; fla()[k] = fa; A[L::BPF + fr] = k | BF_POOL1; }
            fl_n1--;
            w.sync();
            if (k == first) ++k;        // (the entry at k is gone; k is now below the pool)
          } else {
            fl_remove_at(0, k);
          }
          b_delrow(r);
          w.sync();
        } else {
          ++k;
        }
      }
    }
  }

  GML_HD uint64_t bfc_segment_size(uint64_t r, bool exact) const {
    if (exact) return r;
    if (r <= BFC_SMALL_SIZE) return BFC_SMALL_BUFFER;
    if (r < BFC_MIN_LARGE_ALLOC) return BFC_LARGE_BUFFER;
    return (r + BFC_ROUND_LARGE - 1) / BFC_ROUND_LARGE * BFC_ROUND_LARGE;
  }

  // BFC malloc (PAPER.md L116-122 ops 1-2). false on OOM.
  GML_HD bool bfc_malloc(uint32_t slot, uint64_t raw, uint64_t& rec) {
    const bool exact = kind == GML_POLICY_BFC_EXACT;
    const uint64_t r = raw < 512 ? 512 : (raw + 511) / 512 * 512;
    const uint32_t ru = (uint32_t)(r / 512);
    const uint32_t pool = exact ? 0 : (r <= BFC_SMALL_SIZE ? 0 : 1);
    const uint32_t pflag = pool ? BF_POOL1 : 0u;
    const uint32_t frn = b_freerow != NONE32 ? A[L::BNEXT + b_freerow] : NONE32;   // for a split after a hit
    // op 1: best fit = min (size, segment, offset) among free blocks >= r
    // (PyTorch orders by (size, address), D21-D23): one pass over 16-byte
    // vectors of sizes and addresses, branch-free per lane, then an argmin
    // over the warp.
    const uint32_t lo = fl_lo(pool), hi = fl_hi(pool);
    uint32_t bs = NONE32, bk = NONE32, br = NONE32;
    GML_HC(9, 1); GML_HC(10, hi - lo);
    uint64_t ba = ~0ull;
    for (uint32_t q = (lo >> 2) + w.lane(); q < ((hi + 3) >> 2); q += w.width()) {
      const uint4 z = reinterpret_cast<const uint4*>(A + L::FLS)[q];
      const uint4 rr = reinterpret_cast<const uint4*>(A + L::FLR)[q];   // rows ride along (off the chain)
      const ulonglong2 a01 = reinterpret_cast<const ulonglong2*>(A + L::FLA)[2 * q];
      const ulonglong2 a23 = reinterpret_cast<const ulonglong2*>(A + L::FLA)[2 * q + 1];
      const uint32_t zz[4] = {z.x, z.y, z.z, z.w};
      const uint64_t aa[4] = {a01.x, a01.y, a23.x, a23.y};
      const uint32_t rw[4] = {rr.x, rr.y, rr.z, rr.w};
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const uint32_t k = 4 * q + i;
        const bool ok = k >= lo && k < hi && zz[i] >= ru && (zz[i] < bs || (zz[i] == bs && aa[i] < ba));
        bs = ok ? zz[i] : bs;
        ba = ok ? aa[i] : ba;
        bk = ok ? k : bk;
        br = ok ? rw[i] : br;
      }
    }
    uint32_t row, k = NONE32, size, off, seg;
    int state;
    const uint32_t gs = w.wmin(bs);
    if (gs != NONE32) {
      // the lane holding the smallest size; if several lanes tie on it, the
      // one with the lowest address (64-bit min in two reductions)
      const uint32_t tie = w.ballot(bs == gs);
      uint32_t src = ctz32(tie);
      if (tie & (tie - 1)) {
        const uint64_t ca = bs == gs ? ba : ~0ull;
        const uint32_t ahi = w.wmin((uint32_t)(ca >> 32));
        const uint32_t alo = w.wmin((uint32_t)(ca >> 32) == ahi ? (uint32_t)ca : NONE32);
        src = ctz32(w.ballot(bs == gs && ba == (((uint64_t)ahi << 32) | alo)));
      }
      k = w.shfl(bk, src);
      seg = w.shfl((uint32_t)(ba >> 32), src);
      off = w.shfl((uint32_t)ba, src);
      row = w.shfl(br, src);
      size = gs;
      state = ST_HIT;
    } else {
      uint64_t ss = bfc_segment_size(r, exact);
      if (reserved_vmm() + seg_bytes + ss > capacity) {
        bfc_release();
        if (reserved_vmm() + seg_bytes + ss > capacity) { rec = rec_oom(); sc[ST_S5 - 1]++; return false; }
      }
      // the rows this malloc needs (segment + split remainder) must exist
      // before anything is committed
      const uint32_t need = 1u + ((ss - r) >= ((exact || pool == 0) ? 512ull : BFC_SMALL_SIZE + 1) ? 1u : 0u);
      if (b_live + need > C::B) { overflow |= OV_B; return false; }
      bool hok = true;
      if (w.leader()) hok = hooks->on_bfc_segment(next_seg, ss);
      if (HK::kCanFail && !hok) {   // the device allocation failed: release cached segments, retry once
        bfc_release();
        if (w.leader()) hok = hooks->on_bfc_segment(next_seg, ss);
        if (!hok) { hk_fail = true; return false; }
      }
      row = b_newrow();
      seg = next_seg++;
      size = (uint32_t)(ss / 512); off = 0;
      if (w.leader()) {
        A[L::BSIZE + row] = size; A[L::BOFF + row] = 0; A[L::BSEG + row] = seg;
        A[L::BPREV + row] = NONE32; A[L::BNEXT + row] = NONE32;
      }
      seg_bytes += ss;
      sample_growth();
      cnt(S()->n_seg_alloc);
      state = ST_NEWSEG;
      w.sync();
    }
    // op 2: split, front allocated, remainder stays in the pool (it takes
    // the chosen block's free-list entry)
    const uint64_t rem = (uint64_t)(size - ru) * 512;
    const bool do_split = (exact || pool == 0) ? rem >= 512 : rem > BFC_SMALL_SIZE;
    if (do_split) {
      const uint32_t rest = b_newrow(frn, state == ST_HIT);
      if (rest == NONE32) return false;
      const uint32_t nx = A[L::BNEXT + row];
      if (k == NONE32) {                        // new segment: the rest is pushed
        k = fl_grow(pool);
      }
      w.sync();
      if (w.leader()) {
        A[L::BSIZE + rest] = size - ru; A[L::BOFF + rest] = off + ru; A[L::BSEG + rest] = seg;
        A[L::BPREV + rest] = row; A[L::BNEXT + rest] = nx;
        if (nx != NONE32) A[L::BPREV + nx] = rest;
        A[L::BNEXT + row] = rest; A[L::BSIZE + row] = ru;
        A[L::FLR + k] = rest; A[L::FLS + k] = size - ru; fla()[k] = ((uint64_t)seg << 32) | (off + ru);
        A[L::BPF + rest] = k | pflag;
      }
    } else if (k != NONE32) {
      fl_remove_at(pool, k);
    }
    if (w.leader()) {
      A[L::BPF + row] = BF_ALLOC | pflag;
      H[slot] = ((uint64_t)HK_B << 62) | ((uint64_t)row << 40) | raw;
    }
    const uint32_t asz = do_split ? ru : size;
    active += (uint64_t)asz * 512; requested += raw;
    if (state == ST_HIT) sc[ST_HIT - 1]++; else sc[ST_NEWSEG - 1]++;
    rec = (uint64_t)off | ((uint64_t)HK_B << 32) | ((uint64_t)state << 34) | ((uint64_t)seg << 40);
    w.sync();
    return true;
  }

  // BFC free + merge (PAPER.md L123-125 ops 3-4): the merged block keeps a
  // free-list entry of one of its parts.
  GML_HD void bfc_free(uint32_t row) {
    const uint32_t f = A[L::BPF + row];
    const uint32_t pool = (f & BF_POOL1) ? 1 : 0, pflag = f & BF_POOL1;
    const uint32_t p = A[L::BPREV + row], n = A[L::BNEXT + row], size = A[L::BSIZE + row];
    const uint64_t addr = ((uint64_t)A[L::BSEG + row] << 32) | A[L::BOFF + row];
    // the neighbours' flags, sizes and links in one round of loads
    const uint32_t pf = p != NONE32 ? A[L::BPF + p] : BF_ALLOC;
    const uint32_t nf = n != NONE32 ? A[L::BPF + n] : BF_ALLOC;
    const uint32_t ps = p != NONE32 ? A[L::BSIZE + p] : 0u;
    const uint32_t ns = n != NONE32 ? A[L::BSIZE + n] : 0u, nn = n != NONE32 ? A[L::BNEXT + n] : NONE32;
    const bool mp = !(pf & BF_ALLOC), mn = !(nf & BF_ALLOC);
    w.sync();
    if (!mp && !mn) {
      fl_push(pool, row, size, addr);
    } else if (mp && !mn) {                     // prev absorbs row
      if (w.leader()) {
        A[L::BSIZE + p] = ps + size; A[L::BNEXT + p] = n;
        if (n != NONE32) A[L::BPREV + n] = p;
        A[L::FLS + (pf & BF_IDX)] = ps + size;
      }
      b_delrow(row);
    } else if (!mp && mn) {                     // row absorbs next, takes its entry
      const uint32_t kn = nf & BF_IDX;
      if (w.leader()) {
        A[L::BSIZE + row] = size + ns; A[L::BNEXT + row] = nn;
        if (nn != NONE32) A[L::BPREV + nn] = row;
        A[L::FLR + kn] = row; A[L::FLS + kn] = size + ns; fla()[kn] = addr; A[L::BPF + row] = kn | pflag;
      }
      w.sync();
      b_delrow(n);
    } else {                                    // prev absorbs row and next
      const uint32_t kp = pf & BF_IDX;
      if (w.leader()) {
        A[L::BSIZE + p] = ps + size + ns; A[L::BNEXT + p] = nn;
        if (nn != NONE32) A[L::BPREV + nn] = p;
        A[L::FLS + kp] = ps + size + ns;
      }
      w.sync();
      fl_remove_at(pool, nf & BF_IDX);          // (may move p's entry; it carries the new size)
      b_delrow(row);
      w.sync();
      b_delrow(n);
    }
    w.sync();
  }

  // ------------------------------------------------------------ GMLake
  // GMLake malloc: Algorithm 1 + S1-S5
  GML_HD bool vmm_malloc(uint32_t slot, uint64_t raw, uint64_t& rec) {
    const uint32_t b = (uint32_t)(gshift < 64 ? (raw + G - 1) >> gshift : (raw + G - 1) / G);   // D2
    GML_T0(ta);
    stitch_free_bytes();                                                                         // D17(ii)
    GML_T1(4, ta);
    GML_T0(tb);
    const bool rr = flags & GML_F_REMAINDER_RULE;
    const bool pfirst = flags & GML_F_S1_PBLOCK_FIRST;
    const uint4* const pa = pe();
    // ---- S1 on pPool: the first inactive position at or after the start
    // of the size-b run; a hit iff it still has size b (Alg. 1 L2-4; D4, D5)
    // (computed after the sPool scan misses, unless S1_PBLOCK_FIRST: in the
    // steady state most S1 hits are sBlocks)
    uint32_t s1p_row = NONE32, s1p_ord = NONE32;
    auto s1_ppool = [&]() {
      if (pstk_n) pin_flush();   // PIN exact from here on in this malloc (lazy PIN)
      const uint32_t x = pin_first(p_start(b));
      if (x != NONE32) {
        const uint4 ex = pa[x];
        if (ex.y == b) { s1p_row = ex.z; s1p_ord = ex.x; }
      }
    };
    if (pfirst) s1_ppool();
    GML_T1(5, tb);
    GML_T0(tc);
    // ---- S1 on sPool (sPool first unless S1_PBLOCK_FIRST, D5): the size-b
    // run in ordinal order, one candidate per lane ----
    // S1 miss cache: a scan of size b that found no inactive sBlock stays
    // valid while the sPool epoch is unchanged (no free since has released
    // chunks of any sBlock, and a new sBlock is active when created)
    uint64_t* const mcache = reinterpret_cast<uint64_t*>(A + L::MCACHE);
    const uint64_t mkey = ((uint64_t)sep << 32) | (uint64_t)(b + 1u);
    if (!(pfirst && s1p_row != NONE32) && mcache[b & (L::CACHE - 1)] != mkey) {
      uint32_t srow = NONE32, sord = NONE32, spos = NONE32;
      IvLane kv;
      GML_T0(tss);
      const uint32_t s0 = s_start(b);
      GML_HC(8, 1);
      GML_T1(9, tss);
      GML_T0(tsl);
      for (uint32_t base = s0; base < s_count; base += w.width()) {
#if defined(GML_PHASE_PROF) && defined(__CUDA_ARCH__)
        pacc[11] += 1;
#endif
        const uint32_t k = base + w.lane();
        uint4 e = entry(0, 0, 0, 0);
        if (k < s_count) e = se()[k];
        const bool in = k < s_count && e.y == b;
        // one witness load per candidate; the candidates whose witness is
        // not owned are then proven, in order, by the whole warp (lanes over
        // the sBlock's intervals): the first one proven inactive is the hit
        const bool known_active = in && e.w != NONE32 && bm_bit(e.w);
        uint32_t todo = w.ballot(in && !known_active);
        const uint32_t mo = w.ballot(!in);
        GML_HC(0, 1); GML_HC(1, in); GML_HC(2, in && !known_active);
        while (todo) {
          const uint32_t j = ctz32(todo);
          GML_HC(3, 1); GML_HC(4, A[L::SIVN + w.shfl(e.z, j)]);
          const uint32_t c = s_proof(w.shfl(e.z, j), kFuse ? &kv : nullptr);
          if (c == NONE32) {
            srow = w.shfl(e.z, j); sord = w.shfl(e.x, j); spos = base + j;
            break;
          }
          w.sync();   // every lane's read of this round's entries precedes the rewrite
          if (w.leader()) se()[base + j].w = c;   // active: a fresh witness
          todo &= todo - 1;
        }
        if (srow != NONE32 || mo) break;
      }
      GML_T1(10, tsl);
      GML_T1(6, tc);
      if (srow != NONE32) {
        GML_T0(td);
        if (kFuse) bind_s(slot, srow, raw, spos, &kv, b);
        else bind_s(slot, srow, raw, spos);
        GML_T1(7, td);
        lru_tick();
        if (w.leader()) A[L::SLAST + srow] = (uint32_t)T;
        rec = rec_of(sord, HK_S, ST_S1);
        sc[ST_S1 - 1]++;
        w.sync();
        return true;
      }
      w.sync();
      if (w.leader()) mcache[b & (L::CACHE - 1)] = mkey;   // a miss at this epoch
    }
    if (!pfirst) {
      GML_T0(tp);
      s1_ppool();
      GML_T1(5, tp);
    }
    if (s1p_row != NONE32) {
      GML_T0(te);
      bind_p(slot, s1p_row, raw);
      GML_T1(8, te);
      rec = rec_of(s1p_ord, HK_P, ST_S1);
      sc[ST_S1 - 1]++;
      w.sync();
      return true;
    }
    // ---- Alg. 1 L6-8: the replace-loop keeps the smallest size >= bSize,
    // ties -> the last in pool order = highest ordinal (D6); candidates are
    // inactive pBlocks, eligible (size >= limit, D8) unless REMAINDER_RULE.
    GML_T0(tq);
    uint32_t s2_row = NONE32, s2_ord = 0, s2_n = 0;
    {
      const uint32_t from = (rr || elig_n <= b + 1) ? b + 1 : elig_n;
      const uint32_t c1 = pin_first(p_start(from));
      if (c1 != NONE32) {
        s2_n = pa[c1].y;
        const uint32_t e = p_start(s2_n + 1);                         // end of the size group
        const uint32_t x = pin_last(c1, e);                           // last inactive in the group
        const uint4 ex = pa[x];
        s2_row = ex.z;
        s2_ord = ex.x;
      }
    }
    GML_T1(15, tq);
    if (s2_row != NONE32) {
      // ---- S2: split, companion stitch, assign the front ----
      uint32_t P = s2_row;
      if (rr && (uint64_t)(s2_n - b) * G < limit_bytes) {
        bind_p(slot, P, raw);
        rec = rec_of(s2_ord, HK_P, ST_S2);
      } else {
        uint32_t R = split(P, b);
        if (R == NONE32) return false;
        if (!(flags & GML_F_NO_COMPANION)) {
          uint32_t prr[2] = {P, R};
          stitch(prr, 2, true);
          if (overflow) return false;
        }
        bind_p(slot, P, raw);
        rec = rec_of(next_p - 2, HK_P, ST_S2);   // F's ordinal
      }
      sc[ST_S2 - 1]++;
      w.sync();
      return true;
    }
    // ---- Alg. 1 L9-10: greedy largest-first accumulation over eligible
    // inactive pBlocks (all < b now): size groups from the top, ordinals
    // ascending in a group, taking just enough blocks to reach b.
    GML_T0(tg);
    uint32_t k = 0;
    uint64_t CBsize = 0;
    {
      const uint32_t lo_idx = p_start(elig_n);
      uint32_t cur = p_start(b);
      while (CBsize < b && cur > lo_idx) {
        const uint32_t gsz = pa[cur - 1].y;
        uint32_t gs = p_start(gsz);
        if (gs < lo_idx) gs = lo_idx;
        uint64_t need = (b - CBsize + gsz - 1) / gsz;
        for (uint32_t x = gs; need;) {
          const uint32_t p = pin_first(x);
          if (p == NONE32 || p >= cur) break;
          if (k + 2 > C::CB) { overflow |= OV_CB; return false; }
          if (w.leader()) A[L::CB + k] = pa[p].z;
          k++;
          need--;
          CBsize += gsz;
          x = p + 1;
        }
        cur = gs;
      }
    }
    w.sync();
    GML_T1(15, tg);
    if (CBsize >= b) {
      // ---- S3: split the last candidate (D14), stitch ----
      if (CBsize > b) {
        uint32_t last = A[L::CB + k - 1];
        uint32_t lastn = A[L::PN + last];
        uint32_t n = (uint32_t)(b - (CBsize - lastn));
        if (!(rr && (uint64_t)(lastn - n) * G < limit_bytes)) {
          uint32_t R = split(last, n);
          if (R == NONE32) return false;
          if (!(flags & GML_F_NO_COMPANION)) {
            uint32_t prr[2] = {last, R};
            stitch(prr, 2, true);
            if (overflow) return false;
          }
        }
      }
      uint32_t s = stitch(A + L::CB, k, false);
      if (s == NONE32) return false;
      bind_s(slot, s, raw);
      rec = rec_of(A[L::SORD + s], HK_S, ST_S3);
      sc[ST_S3 - 1]++;
      w.sync();
      return true;
    }
    // ---- S4: Alloc the shortfall (D15) ----
    uint32_t shortfall = (uint32_t)(b - CBsize);
    // D16: before Alloc fails, the small path returns its fully free cached
    // segments (PyTorch's release on a failed device allocation)
    if constexpr (C::SMALL) {
      if (reserved() + (uint64_t)shortfall * G > capacity && seg_bytes) bfc_release();
    }
    if (reserved() + (uint64_t)shortfall * G > capacity) {
      rec = rec_oom();                                               // S5 (L528, D16)
      sc[ST_S5 - 1]++;
      return false;
    }
    uint32_t p = alloc(shortfall);
    if (p == NONE32) return false;
    if (k == 0) {
      bind_p(slot, p, raw);
      rec = rec_of(next_p - 1, HK_P, ST_S4);
    } else {
      if (w.leader()) A[L::CB + k] = p;
      w.sync();
      uint32_t s = stitch(A + L::CB, k + 1, false);
      if (s == NONE32) return false;
      bind_s(slot, s, raw);
      rec = rec_of(A[L::SORD + s], HK_S, ST_S4);
    }
    sc[ST_S4 - 1]++;
    w.sync();
    return true;
  }

  // ordinal of pBlock row r (its sorted key's low word)
  GML_HD uint32_t p_ord(uint32_t r) const { return pe()[A[L::PPOS + r]].x; }

  // Update: unbind, no release, no merge (D19).
  GML_HD uint64_t do_free(uint32_t slot, uint64_t hv) {
    const uint32_t hk = (uint32_t)(hv >> 62);
    const uint32_t row = (uint32_t)((hv >> 40) & 0x3FFFFF);
    const uint64_t raw = hv & MASK40;
    uint64_t by, rec;
    if (C::VMM && hk == HK_P) {   // (a BFC-family instance only ever holds BFC handles)
      const uint32_t n = A[L::PN + row];
      by = (uint64_t)n * G;
      rec = rec_of(p_ord(row), HK_P, 0);
      const bool contained = A[L::PCNT + row] != 0u;
      bm_range_par(A[L::PLO + row], n, false);
      if (w.leader()) pin_set(row, true);
      active_vmm -= by;
      if (contained) spool_touched();
    } else if (C::VMM && hk == HK_S) {
      by = (uint64_t)A[L::SN + row] * G;
      rec = rec_of(A[L::SORD + row], HK_S, 0);
      const bool pend = A[L::SPND + row] != 0u;    // (PIN bits never cleared: nothing to restore)
      w.sync();
      if (pend && w.leader()) A[L::SPND + row] = 0u;
      s_own(row, false, !pend);
      active_vmm -= by;
      s_bound -= by;
      spool_touched();
    } else if constexpr (C::SMALL) {
      by = (uint64_t)A[L::BSIZE + row] * 512;
      rec = (uint64_t)A[L::BOFF + row] | ((uint64_t)HK_B << 32) | ((uint64_t)A[L::BSEG + row] << 40);
      bfc_free(row);
    } else {   // (an instance without the small path only ever holds VMM handles)
      by = 0;
      rec = 0;
    }
    active -= by;
    if constexpr (kOwnPeaks) {
      requested -= raw;
      live--;
    }
    if (w.leader()) H[slot] = (uint64_t)HK_EMPTY << 62;
    w.sync();
    return rec;
  }

  // The run of frees that starts at the lowest lane of m (the unit's
  // window events still to replay; mall: the window's mallocs, of any
  // path): m's events before the next malloc. 0 if the lowest is a malloc.
  GML_HD static uint32_t free_run_mask(uint32_t m, uint32_t mall) {
    const uint32_t low = m & (0u - m);
    const uint32_t stop = mall & ~(low - 1u);
    return m & (stop ? (stop & (0u - stop)) - 1u : 0xFFFFFFFFu);
  }

  // A run of consecutive VMM-path frees (no malloc between them) unbinds
  // disjoint blocks (Update: each clears its own chunks
  // and PIN bits), so the unbinds commute and the run is done at once: lane
  // l holds event l of the run (`run`: the lanes in it), unbinds a pBlock
  // itself, and the intervals of all the run's sBlocks are spread over the
  // lanes (a lane finds its interval's owner by a binary search over the
  // lanes' interval-count prefix). The chain is about one free's instead of
  // one per free. Returns false with nothing changed when a lane's event is
  // not the free of a live VMM-path block or two lanes free one slot (the
  // caller then steps the events one by one, which handles BFC frees and
  // reports INVALID). Lane l receives its event's record.
  GML_HD bool free_run(uint32_t run, uint64_t ev, uint64_t& rec) {
    if constexpr (!C::VMM) {
      return false;
    } else {
      const uint32_t ln = w.lane();
      const bool on = (run >> ln) & 1u;
      const uint32_t slot = (uint32_t)((ev >> 40) & 0x7FFFFFu);
      const uint64_t hv = on ? H[slot] : 0;
      const uint32_t hk = (uint32_t)(hv >> 62);
      const uint32_t dup = w.match_any(on ? slot : (0x80000000u | ln));
      if (w.ballot(on && ((hk != HK_P && hk != HK_S) || (ev & MASK40) || (dup & (dup - 1))))) return false;
      w.sync();   // every lane has read its handle before any rewrite
      GML_T0(t0);
      const uint32_t row = (uint32_t)((hv >> 40) & 0x3FFFFF);
      uint32_t nch = 0, k = 0, o = 0, pd = 0;
      bool touch = false;
      if (on) {
        if (hk == HK_P) {
          nch = A[L::PN + row];
          rec = rec_of(p_ord(row), HK_P, 0);
          touch = A[L::PCNT + row] != 0u;
          bm_range_seq(A[L::PLO + row], nch, false);
          pin_set(row, true);
        } else {
          touch = true;
          nch = A[L::SN + row];
          rec = rec_of(A[L::SORD + row], HK_S, 0);
          k = A[L::SIVN + row];
          o = A[L::SIVO + row];
          pd = A[L::SPND + row];   // pending (lazy PIN): only the chunks to release
          if (pd) A[L::SPND + row] = 0u;
        }
        H[slot] = (uint64_t)HK_EMPTY << 62;
      }
      // inclusive prefix of the interval counts over the lanes
      uint32_t e = k;
      for (uint32_t d = 1; d < w.width(); d <<= 1) {
        const uint32_t x = w.shfl(e, ln >= d ? ln - d : ln);
        if (ln >= d) e += x;
      }
      const uint32_t K = w.shfl(e, w.width() - 1);
      for (uint32_t i0 = 0; i0 < K; i0 += w.width()) {
        const uint32_t i = i0 + ln;
        uint32_t pos = 0;                                   // first lane whose prefix end exceeds i
        for (uint32_t st = w.width() >> 1; st; st >>= 1) {
          const uint32_t x = w.shfl(e, pos + st - 1);
          if (x <= i) pos += st;
        }
        const uint32_t ow = pos < w.width() ? pos : 0;
        const uint32_t oe = w.shfl(e, ow), ok = w.shfl(k, ow), oo = w.shfl(o, ow), opd = w.shfl(pd, ow);
        if (i < K) {
          const uint32_t ix = oo + (i - (oe - ok));
          const uint32_t lo = A[L::IVLO + ix], n = A[L::IVN + ix];
          uint32_t r = A[L::IVROW + ix];
          bm_range_seq(lo, n, false);
          if (!opd)
            for (uint32_t left = n; left;) {
              const uint32_t pn = A[L::PN + r], nx = A[L::PNEXT + r];
              pin_set(r, true);
              left -= pn;
              r = nx;
            }
        }
      }
      const uint64_t tot = w.sum_u32(nch) * G, tot_s = w.sum_u32(hk == HK_S ? nch : 0u) * G;
      if constexpr (kOwnPeaks) {
        const uint64_t raw = on ? (hv & MASK40) : 0;
        requested -= w.sum_u32((uint32_t)raw) + (w.sum_u32((uint32_t)(raw >> 32)) << 32);
        live -= popc32(run);
      }
      active -= tot;
      active_vmm -= tot;
      s_bound -= tot_s;
      if (w.ballot(touch)) spool_touched();
      w.sync();
      GML_T1(0, t0);
      return true;
    }
  }

  // One event. Returns the assignment record; sets `status` (OOM / INVALID)
  // or `overflow` when the replay must stop.
  GML_HD uint64_t step(uint64_t ev) {
    bool is_free = ev >> 63;
    uint32_t slot = (uint32_t)((ev >> 40) & 0x7FFFFFu);
    uint64_t raw = ev & MASK40;
    if (!W::kReplay && slot >= h_cap) { overflow |= OV_H; return 0; }
    uint64_t hv = H[slot];
    bool empty = (hv >> 62) == HK_EMPTY;
    uint64_t rec = 0;
    w.sync();   // every lane has read H[slot] before the leader may rewrite it
    if (is_free) {
      if (empty || raw) { status = GML_ERR_INVALID; return 0; }
      GML_T0(t0);
      uint64_t fr = do_free(slot, hv);
      if ((hv >> 62) == HK_B) { GML_T1(1, t0); } else { GML_T1(0, t0); }
      return fr;
    }
    if (!empty || raw == 0) { status = GML_ERR_INVALID; return 0; }
    if constexpr (!W::kReplay) serial++;
    born_row = NONE32;
    GML_T0(t1);
    bool vm = C::VMM && (!C::SMALL || (kind == GML_POLICY_GMLAKE && raw >= vm_thr));
    bool ok;
    if constexpr (C::SMALL) ok = vm ? vmm_malloc(slot, raw, rec) : bfc_malloc(slot, raw, rec);
    else ok = vmm_malloc(slot, raw, rec);
    if (vm) { GML_T1(2, t1); } else { GML_T1(3, t1); }
    if (!W::kReplay && overflow) return 0;   // (the replay kernel stops on E.overflow after the step)
    if (!ok) {
      if (!W::kReplay && hk_fail) {   // a failed driver allocation is the paper's S5 (L528)
        hk_fail = false;
        rec = rec_oom();
        sc[ST_S5 - 1]++;
      }
      status = GML_ERR_OOM;
      return rec;
    }
    if constexpr (kOwnPeaks) live++;
    sample(vm);   // peaks only grow on a completed malloc (a free lowers every sum)
    return rec;
  }

  // peaks after the event: active, reserved and requested
  // bytes and the table maxima can only grow during a malloc, so sampling
  // after each completed malloc equals sampling after every event. Reserved
  // bytes and table sizes are sampled where they grow instead (Alloc, a new
  // BFC segment, Split, Stitch, a new BFC row): nothing later in the same
  // malloc lowers them, so the maxima are the same.
  GML_HD void sample(bool vm) {
    if constexpr (kOwnPeaks) {   // (without the small path: the ledger's, from the path's active series)
      if (active > pk_active) pk_active = active;
      if (requested > pk_requested) pk_requested = requested;
      if (live > mx_h) mx_h = (uint32_t)live;
      if (vm && active_vmm > pk_active_vmm) pk_active_vmm = active_vmm;
    }
  }
  GML_HD void sample_growth() {
    const uint64_t rs = reserved();
    if (rs > pk_reserved) pk_reserved = rs;
    if (reserved_vmm() > pk_reserved_vmm) pk_reserved_vmm = reserved_vmm();
  }

  // write the register-held fields of the stats record (leader)
  GML_HD void finish(uint64_t n_events, uint64_t n_done, int64_t oom_event) {
    w.sync();
    if (w.leader()) {
      for (int i = 0; i < 7; ++i) S()->state_count[i] = sc[i];
      S()->peak_active_bytes = pk_active;
      S()->peak_reserved_bytes = pk_reserved;
      S()->peak_requested_bytes = pk_requested;
      S()->peak_active_vmm_bytes = pk_active_vmm;
      S()->peak_reserved_vmm_bytes = pk_reserved_vmm;
      S()->final_active_bytes = active;
      S()->final_reserved_bytes = reserved();
      S()->n_events = n_events;
      S()->n_events_done = n_done;
      S()->oom_event = oom_event;
      S()->status = status;
      S()->_p = overflow;
      S()->max_pblocks = mx_p;
      S()->max_sblocks = mx_s;
      S()->max_live_handles = mx_h;
      S()->max_bfc_blocks = mx_b;
#if defined(GML_PROF_ON)
      if (prof)
        for (int i = 0; i < 16; ++i) prof[i] = pacc[i];
#endif
    }
    w.sync();
  }
};

}  // namespace gml
