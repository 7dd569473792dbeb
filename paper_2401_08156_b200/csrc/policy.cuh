// policy.cuh -- the GMLake allocation engine, written once for three
// executors ("groups" of cooperating threads that own one replay):
//
//   * DeviceWarp: the 32 lanes of one warp own one (trace, policy) replay on
//     sm_100a; table scans stride 16-byte vectors of rows over the lanes and
//     finish with __reduce_{min,max}_sync / ballots (the "warp-level
//     argmin/ballot best-fit search" of the north star).
//   * DeviceCta<NW>: NW warps own one replay (latency mode for batches too
//     small to fill the GPU): per-warp reductions, then one shared-memory
//     exchange and one named barrier.
//   * HostWarp: width 1, for the live allocator (gml_malloc / gml_free), so
//     the live path and the replay take identical decisions.
//
// Every thread of a group holds the same scalar state and takes the same
// (uniform) decisions; table writes are done by the leader and published with
// sync(). The method (§3.3 Algorithm 1, §4.1) is
// walked in the paper's order; readings D1..D30 are listed in DESIGN.md. The
// engine never reads the oracle (oracle/), and the oracle never reads this
// file.
//
// Data layout per replay ("arena", SoA, u32 unless noted; in shared memory
// when it fits, else in global memory):
//   bitmap   1 bit per chunk: chunk owned by a live tensor (D18); an sBlock is
//            inactive iff its chunk intervals hold no set bit.
//   pPool    p_key = granules | ACT (bit 31: the pBlock is active), p_ord,
//            p_lo (first chunk), p_next (address successor). Rows are never
//            deleted: Split rewrites the parent's row as the front piece F and
//            appends R, so rows are 0..n_p-1 and |pPool| = n_p. S1 on pPool is
//            one 16-byte load + one compare per 4 rows.
//   sPool    s_n (granules, 0 = free row), s_ord, s_last (LRU key), s_born
//            (malloc serial / free-row link), s_ivo / s_ivn (interval list).
//   ivs      iv_row (first member row), iv_lo, iv_n: chunk intervals of
//            sBlocks, double-buffered for compaction. A member row stays the
//            row of the pBlock at iv_lo forever (Split keeps F in P's row), so
//            p_next walks from iv_row cover the interval.
//   handles  u64 per slot: kind (2 b) | row (22 b) | raw bytes (40 b).
//   BFC      b_size / b_off (512-byte units), b_seg, b_prev, b_next, b_flags,
//            b_pos; per-pool free lists (fl_row, fl_sz) so best-fit scans read
//            one size word per free block only.
#pragma once
#include <stdint.h>

#include "gml.h"

#if defined(__CUDACC__)
#define GML_HD __host__ __device__ __forceinline__
#define GML_HDI __host__ __device__
#else
#define GML_HD inline
#define GML_HDI
#endif

#if defined(GML_PHASE_PROF) && defined(__CUDA_ARCH__)
#define GML_T0(v) long long v = clock64()
#define GML_T1(k, v) \
  if (prof && w.leader()) prof[k] += (unsigned long long)(clock64() - v)
#else
#define GML_T0(v)
#define GML_T1(k, v)
#endif

namespace gml {

constexpr uint32_t NONE32 = 0xFFFFFFFFu;
constexpr uint64_t MASK40 = (1ull << 40) - 1;
constexpr uint32_t ACT = 0x80000000u;

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

struct KeyRow {           // result of an argmin: key (~0 = none) and its row
  uint64_t key;
  uint32_t row;
};

// ---------------------------------------------------------------- executors
struct DeviceWarp {
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
  GML_HD uint32_t wmin(uint32_t v) const {
#if defined(__CUDA_ARCH__)
    return __reduce_min_sync(0xFFFFFFFFu, v);
#else
    return v;
#endif
  }
  GML_HD uint32_t wballot(bool p) const {
#if defined(__CUDA_ARCH__)
    return __ballot_sync(0xFFFFFFFFu, p);
#else
    return p;
#endif
  }
  GML_HD uint32_t wshfl(uint32_t v, uint32_t s) const {
#if defined(__CUDA_ARCH__)
    return __shfl_sync(0xFFFFFFFFu, v, s);
#else
    (void)s;
    return v;
#endif
  }
  // argmin over the warp of a 64-bit key (keys unique unless ~0)
  GML_HD KeyRow argmin(uint64_t key, uint32_t row) const {
    uint32_t hi = wmin((uint32_t)(key >> 32));
    uint32_t lo = wmin(((uint32_t)(key >> 32) == hi) ? (uint32_t)key : NONE32);
    uint64_t g = ((uint64_t)hi << 32) | lo;
    if (g == ~0ull) return KeyRow{g, NONE32};
    uint32_t m = wballot(key == g);
    return KeyRow{g, wshfl(row, ctz32(m))};
  }
  GML_HD uint64_t add_u64(uint64_t v) const {
#if defined(__CUDA_ARCH__)
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
#endif
    return v;
  }
  // lowest thread index whose predicate holds, NONE32 if none
  GML_HD uint32_t first_true(bool p) const {
    uint32_t m = wballot(p);
    return m ? ctz32(m) : NONE32;
  }
  // number of true predicates on lower thread indices; *total = all of them
  GML_HD uint32_t rank_true(bool p, uint32_t* total) const {
    uint32_t m = wballot(p);
    *total = popc32(m);
    return popc32(m & ((1u << lane()) - 1u));
  }
};

// NW warps of one CTA own one replay (latency mode). Cross-warp reductions:
// warp-level reduce, one shared-memory exchange, one CTA barrier; the scratch
// is double-buffered so consecutive reductions need no second barrier.
template <int NW>
struct DeviceCta {
  uint64_t* scratch;   // 2 buffers x NW x (key, row), in shared memory
  uint32_t phase;
  GML_HD uint32_t lane() const {
#if defined(__CUDA_ARCH__)
    return threadIdx.x;
#else
    return 0;
#endif
  }
  GML_HD uint32_t width() const { return 32 * NW; }
  GML_HD bool leader() const { return lane() == 0; }
  GML_HD void sync() const {
#if defined(__CUDA_ARCH__)
    __syncthreads();
#endif
  }
  GML_HD KeyRow argmin(uint64_t key, uint32_t row) {
#if defined(__CUDA_ARCH__)
    DeviceWarp w;
    KeyRow k = w.argmin(key, row);
    uint64_t* s = scratch + phase * 2 * NW;
    phase ^= 1u;
    const uint32_t wi = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) { s[2 * wi] = k.key; s[2 * wi + 1] = k.row; }
    __syncthreads();
    KeyRow best{~0ull, NONE32};
#pragma unroll
    for (int i = 0; i < NW; ++i) {
      uint64_t kk = s[2 * i];
      if (kk < best.key) { best.key = kk; best.row = (uint32_t)s[2 * i + 1]; }
    }
    return best;
#else
    return KeyRow{key, row};
#endif
  }
  GML_HD uint64_t add_u64(uint64_t v) {
#if defined(__CUDA_ARCH__)
    DeviceWarp w;
    v = w.add_u64(v);
    uint64_t* s = scratch + phase * 2 * NW;
    phase ^= 1u;
    if ((threadIdx.x & 31) == 0) s[2 * (threadIdx.x >> 5)] = v;
    __syncthreads();
    uint64_t t = 0;
#pragma unroll
    for (int i = 0; i < NW; ++i) t += s[2 * i];
    return t;
#else
    return v;
#endif
  }
  GML_HD uint32_t first_true(bool p) {
#if defined(__CUDA_ARCH__)
    uint32_t m = __ballot_sync(0xFFFFFFFFu, p);
    uint64_t* s = scratch + phase * 2 * NW;
    phase ^= 1u;
    const uint32_t wi = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) s[2 * wi] = m ? 32 * wi + ctz32(m) : NONE32;
    __syncthreads();
    uint32_t best = NONE32;
#pragma unroll
    for (int i = 0; i < NW; ++i) best = (uint32_t)s[2 * i] < best ? (uint32_t)s[2 * i] : best;
    return best;
#else
    return p ? 0 : NONE32;
#endif
  }
  GML_HD uint32_t rank_true(bool p, uint32_t* total) {
#if defined(__CUDA_ARCH__)
    uint32_t m = __ballot_sync(0xFFFFFFFFu, p);
    uint64_t* s = scratch + phase * 2 * NW;
    phase ^= 1u;
    const uint32_t wi = threadIdx.x >> 5, ln = threadIdx.x & 31;
    if (ln == 0) s[2 * wi] = popc32(m);
    __syncthreads();
    uint32_t before = 0, tot = 0;
#pragma unroll
    for (int i = 0; i < NW; ++i) {
      uint32_t c = (uint32_t)s[2 * i];
      if (i < (int)wi) before += c;
      tot += c;
    }
    *total = tot;
    return before + popc32(m & ((1u << ln) - 1u));
#else
    *total = p;
    return 0;
#endif
  }
};

struct HostWarp {
  GML_HD uint32_t lane() const { return 0; }
  GML_HD uint32_t width() const { return 1; }
  GML_HD bool leader() const { return true; }
  GML_HD void sync() const {}
  GML_HD KeyRow argmin(uint64_t key, uint32_t row) const { return KeyRow{key, key == ~0ull ? NONE32 : row}; }
  GML_HD uint64_t add_u64(uint64_t v) const { return v; }
  GML_HD uint32_t first_true(bool p) const { return p ? 0 : NONE32; }
  GML_HD uint32_t rank_true(bool p, uint32_t* total) const { *total = p; return 0; }
};

// Driver-call hooks: the live allocator turns decisions into VMM calls; the
// replay kernel ignores them.
struct NoHooks {
  GML_HD void on_alloc(uint32_t, uint32_t, uint32_t) {}
  GML_HD void on_split(uint32_t, uint32_t, uint32_t, uint32_t) {}
  GML_HD void on_stitch(uint32_t, const uint32_t*, const uint32_t*, uint32_t) {}
  GML_HD void on_evict(uint32_t) {}
  GML_HD void on_bfc_segment(uint32_t, uint64_t) {}
  GML_HD void on_bfc_release(uint32_t) {}
};

// ------------------------------------------------------------- table sizes
// Table capacities are compile-time per kernel instance ("size class"), so
// every table offset is an immediate and the engine keeps one base pointer;
// only the bitmap length (capacity / chunk) and the handle table (max slot)
// are runtime. The host picks the smallest class that fits each unit and
// moves a unit to the next class when a table overflows (D30).
template <uint32_t P_, uint32_t S_, uint32_t IV_, uint32_t B_>
struct Cfg {
  static constexpr uint32_t P = P_, S = S_, IV = IV_, B = B_, CB = P_ + 4;
};

GML_HD constexpr uint32_t round4(uint32_t x) { return (x + 3u) & ~3u; }

constexpr uint32_t BMS_WORDS = 128;          // summary words: bitmap <= 4096 words = 131072 chunks

template <class C>
struct Lay {                                  // offsets in u32 words from the arena base
  static constexpr uint32_t STATS = 0;        // gml_stats_t, 68 words
  static constexpr uint32_t PKEY = 68, PORD = PKEY + C::P, PLO = PORD + C::P, PNEXT = PLO + C::P;
  static constexpr uint32_t SN = PNEXT + C::P, SORD = SN + C::S, SLAST = SORD + C::S, SBORN = SLAST + C::S,
                            SIVO = SBORN + C::S, SIVN = SIVO + C::S;
  static constexpr uint32_t IVROW = SIVN + C::S, IVLO = IVROW + 2 * C::IV, IVN = IVLO + 2 * C::IV;
  static constexpr uint32_t BSIZE = IVN + 2 * C::IV, BOFF = BSIZE + C::B, BSEG = BOFF + C::B,
                            BPREV = BSEG + C::B, BNEXT = BPREV + C::B, BFLAGS = BNEXT + C::B, BPOS = BFLAGS + C::B;
  static constexpr uint32_t FL0 = BPOS + C::B, FL0SZ = FL0 + C::B, FL1 = FL0SZ + C::B, FL1SZ = FL1 + C::B;
  static constexpr uint32_t CB = FL1SZ + C::B;
  // the pools as sorted sets: (size << 32 | ordinal)
  // keys ascending, with their rows
  static constexpr uint32_t PSK = CB + C::CB, PSR = PSK + 2 * C::P;
  static constexpr uint32_t SSK = PSR + C::P, SSR = SSK + 2 * C::S;
  static constexpr uint32_t BMS = SSR + C::S;
  static constexpr uint32_t BM = BMS + BMS_WORDS;
  static_assert(C::P % 4 == 0 && C::S % 4 == 0 && C::IV % 4 == 0 && C::B % 4 == 0, "16-byte rows");
  GML_HD static uint32_t h_off(uint32_t bm_words) { return BM + round4(bm_words); }
  GML_HD static uint64_t bytes(uint32_t bm_words, uint32_t h) { return 4ull * h_off(bm_words) + 8ull * h; }
};

struct RtCaps {
  uint32_t bm_words;   // ceil(capacity chunks / 32) <= 32 * BMS_WORDS
  uint32_t h;          // handle slots
};

// overflow bits (internal; reported through gml_stats_t._p, cleared by host)
enum : uint32_t { OV_P = 1, OV_S = 2, OV_IV = 4, OV_H = 8, OV_B = 16, OV_CB = 32 };

enum : uint32_t { BF_ALLOC = 1, BF_POOL1 = 2 };
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
template <class W, class C, class HK = NoHooks>
struct Engine {
  using L = Lay<C>;
  W w;
  HK* hooks;
  // policy
  uint32_t kind, flags;
  uint64_t capacity, G, small_thr, limit_bytes, spool_max_inactive;
  uint32_t spool_max, elig_n, gshift;
  // tables: one base pointer, compile-time offsets (Lay<C>)
  uint32_t* A;
  uint64_t* H;          // handle table (runtime offset)
  uint32_t h_cap, bm_words;
  unsigned long long* prof = nullptr;   // GML_PHASE_PROF debug counters
  // scalar state (identical in every thread of the group)
  uint32_t Cn, next_p, next_s, n_p, last_p, s_hw, s_count, s_freerow, iv_base, iv_hw;
  uint32_t b_hw, b_freerow, b_live, fl_n0, fl_n1, next_seg;
  uint64_t T, serial, active, requested, active_vmm, seg_bytes, s_bytes, live;
  uint32_t overflow, status;
  // peaks kept in registers
  uint64_t pk_active, pk_reserved, pk_requested, pk_active_vmm, pk_reserved_vmm;
  uint32_t mx_p, mx_s, mx_h, mx_b;

  // -------------------------------------------------------------- set-up
  GML_HDI void init(const gml_policy& pol, const RtCaps& c, uint8_t* arena, HK* hk) {
    hooks = hk;
    kind = pol.kind;
    flags = pol.flags;
    capacity = pol.capacity_bytes;
    G = pol.chunk_bytes;
    small_thr = pol.small_threshold_bytes;
    limit_bytes = pol.frag_limit_bytes;
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
    b_hw = b_live = fl_n0 = fl_n1 = next_seg = 0;
    b_freerow = NONE32;
    T = serial = active = requested = active_vmm = seg_bytes = s_bytes = live = 0;
    overflow = 0; status = GML_OK;
    pk_active = pk_reserved = pk_requested = pk_active_vmm = pk_reserved_vmm = 0;
    mx_p = mx_s = mx_h = mx_b = 0;
    // zero stats, bitmap; mark every handle slot empty
    uint32_t* sw = A + L::STATS;
    for (uint32_t i = w.lane(); i < sizeof(gml_stats_t) / 4; i += w.width()) sw[i] = 0;
    for (uint32_t i = w.lane(); i < BMS_WORDS + c.bm_words; i += w.width()) A[L::BMS + i] = 0;
    for (uint32_t i = w.lane(); i < c.h; i += w.width()) H[i] = (uint64_t)HK_EMPTY << 62;
    w.sync();
  }

  GML_HD uint64_t reserved_vmm() const { return (uint64_t)Cn * G; }
  GML_HD uint64_t reserved() const { return reserved_vmm() + seg_bytes; }
  GML_HD gml_stats_t* S() const { return reinterpret_cast<gml_stats_t*>(A + L::STATS); }
  GML_HD void cnt(uint64_t& f, uint64_t v = 1) { if (w.leader()) f += v; }
  GML_HD uint32_t pn(uint32_t r) const { return A[L::PKEY + r] & ~ACT; }

  // ------------------------------------------------------------ bitmap
  // Two levels: bm has one bit per chunk; bms one bit per bm word (word is
  // non-zero), so a range test touches at most the two edge words and the
  // summary words of the interior.
  GML_HD static void or32(uint32_t* a, uint32_t v) {
#if defined(__CUDA_ARCH__)
    atomicOr(a, v);
#else
    *a |= v;
#endif
  }
  GML_HD static void and32(uint32_t* a, uint32_t v) {
#if defined(__CUDA_ARCH__)
    atomicAnd(a, v);
#else
    *a &= v;
#endif
  }
  // set / clear chunks [lo, lo+n): threads own distinct words
  GML_HD void bm_write(uint32_t lo, uint32_t n, bool v) {
    if (n == 0) return;
    uint32_t a = lo >> 5, z = (lo + n - 1) >> 5;
    for (uint32_t wd = a + w.lane(); wd <= z; wd += w.width()) {
      uint32_t m = 0xFFFFFFFFu;
      if (wd == a) m &= 0xFFFFFFFFu << (lo & 31);
      if (wd == z) m &= 0xFFFFFFFFu >> (31 - ((lo + n - 1) & 31));
      uint32_t x = v ? (A[L::BM + wd] | m) : (A[L::BM + wd] & ~m);
      A[L::BM + wd] = x;
      if (x) or32(&A[L::BMS + (wd >> 5)], 1u << (wd & 31));
      else and32(&A[L::BMS + (wd >> 5)], ~(1u << (wd & 31)));
    }
    w.sync();   // the next interval may share a word
  }
  // bits [x, y] (inclusive) of word array `b` any set?
  GML_HD static bool any_bits(const uint32_t* b, uint32_t x, uint32_t y) {
    uint32_t a = x >> 5, z = y >> 5;
    for (uint32_t wd = a; wd <= z; ++wd) {
      uint32_t m = 0xFFFFFFFFu;
      if (wd == a) m &= 0xFFFFFFFFu << (x & 31);
      if (wd == z) m &= 0xFFFFFFFFu >> (31 - (y & 31));
      if (b[wd] & m) return true;
    }
    return false;
  }
  // single-thread test: any chunk of [lo, lo+n) owned?
  GML_HD bool bm_any1(uint32_t lo, uint32_t n) const {
    uint32_t hi = lo + n - 1;
    uint32_t a = lo >> 5, z = hi >> 5;
    if (z - a < 2) return any_bits(A + L::BM, lo, hi);
    if (A[L::BM + a] & (0xFFFFFFFFu << (lo & 31))) return true;
    if (A[L::BM + z] & (0xFFFFFFFFu >> (31 - (hi & 31)))) return true;
    return any_bits(A + L::BMS, a + 1, z - 1);
  }
  GML_HD bool s_inactive1(uint32_t r) const {   // single thread
    uint32_t o = A[L::SIVO + r], k = A[L::SIVN + r];
    for (uint32_t i = 0; i < k; ++i)
      if (bm_any1(A[L::IVLO + o + i], A[L::IVN + o + i])) return false;
    return true;
  }
  // flip the ACT bit of every pBlock inside the intervals of sBlock s (leader
  // walks p_next from each interval's first row)
  GML_HD void s_mark(uint32_t s, bool on) {
    if (w.leader()) {
      uint32_t o = A[L::SIVO + s], k = A[L::SIVN + s];
      for (uint32_t i = 0; i < k; ++i) {
        uint32_t r = A[L::IVROW + o + i], left = A[L::IVN + o + i];
        while (left) {
          uint32_t key = A[L::PKEY + r];
          A[L::PKEY + r] = on ? (key | ACT) : (key & ~ACT);
          left -= key & ~ACT;
          r = A[L::PNEXT + r];
        }
      }
    }
  }

  // --------------------------------------------------------- sorted sets
  // The pools are kept as the paper's sorted sets:
  // arrays of (size << 32 | ordinal) keys, ascending, with their rows. Pool
  // order (size desc, ordinal asc; D4) is walked over size groups from the
  // top, ordinals ascending inside a group. Search is WD-ary (WD threads test
  // WD pivots per step); insert / erase shift the tail by WD entries per step.
  GML_HD uint64_t* psk() const { return reinterpret_cast<uint64_t*>(A + L::PSK); }
  GML_HD uint64_t* ssk() const { return reinterpret_cast<uint64_t*>(A + L::SSK); }

  GML_HD uint32_t lower_bound(const uint64_t* a, uint32_t n, uint64_t x) {
    if (w.width() == 1) {                       // host: plain binary search
      uint32_t lo = 0, hi = n;
      while (lo < hi) {
        uint32_t mid = lo + (hi - lo) / 2;
        if (a[mid] < x) lo = mid + 1; else hi = mid;
      }
      return lo;
    }
    const uint32_t WD = w.width();
    uint32_t lo = 0, hi = n;                    // answer in [lo, hi]
    while (hi - lo > WD) {
      const uint32_t len = hi - lo;
      const uint32_t i = w.lane();
      const uint32_t piv = lo + (uint32_t)(((uint64_t)len * (i + 1)) / WD) - 1;
      uint32_t j = w.first_true(a[piv] >= x);
      if (j == NONE32) return hi;
      uint32_t nlo = lo + (uint32_t)(((uint64_t)len * j) / WD);
      hi = lo + (uint32_t)(((uint64_t)len * (j + 1)) / WD) - 1;
      lo = nlo;
    }
    const uint32_t k = lo + w.lane();
    uint32_t j = w.first_true(k < hi && a[k] >= x);
    return j == NONE32 ? hi : lo + j;
  }
  GML_HD void sorted_insert(uint64_t* key, uint32_t* row, uint32_t n, uint64_t k, uint32_t r) {
    const uint32_t pos = lower_bound(key, n, k);
    const int32_t WD = (int32_t)w.width();
    for (int32_t base = (int32_t)n - 1; base >= (int32_t)pos; base -= WD) {
      const int32_t i = base - (int32_t)w.lane();
      const bool on = i >= (int32_t)pos;
      uint64_t kk = 0;
      uint32_t rr = 0;
      if (on) { kk = key[i]; rr = row[i]; }
      w.sync();
      if (on) { key[i + 1] = kk; row[i + 1] = rr; }
      w.sync();
    }
    if (w.leader()) { key[pos] = k; row[pos] = r; }
    w.sync();
  }
  GML_HD void sorted_erase(uint64_t* key, uint32_t* row, uint32_t n, uint64_t k) {
    const uint32_t pos = lower_bound(key, n, k);   // present by construction
    const uint32_t WD = w.width();
    for (uint32_t base = pos; base + 1 < n; base += WD) {
      const uint32_t i = base + w.lane();
      const bool on = i + 1 < n;
      uint64_t kk = 0;
      uint32_t rr = 0;
      if (on) { kk = key[i + 1]; rr = row[i + 1]; }
      w.sync();
      if (on) { key[i] = kk; row[i] = rr; }
      w.sync();
    }
  }
  GML_HD static uint64_t skey(uint32_t size, uint32_t ord) { return ((uint64_t)size << 32) | ord; }

  // --------------------------------------------------------- sPool rows
  GML_HD void s_evict(uint32_t r) {   // StitchFree of one sBlock
    s_bytes -= (uint64_t)A[L::SN + r] * G;
    sorted_erase(ssk(), A + L::SSR, s_count, skey(A[L::SN + r], A[L::SORD + r]));
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
    for (uint32_t r = w.lane(); r < s_hw; r += w.width()) {
      if (A[L::SN + r] == 0) continue;
      if (exclude_born && A[L::SBORN + r] == (uint32_t)serial) continue;
      uint32_t lu = A[L::SLAST + r];
      if (lu < best && s_inactive1(r)) { best = lu; row = r; }
    }
    KeyRow k = w.argmin(best == NONE32 ? ~0ull : (uint64_t)best, row);
    return k.row;
  }

  // D17(ii): at VMM-path malloc entry, release LRU inactive sBlocks while the
  // inactive ones hold more than the byte cap.
  GML_HD void stitch_free_bytes() {
    if (s_bytes <= spool_max_inactive) return;   // inactive bytes <= all bytes
    uint64_t part = 0;
    for (uint32_t r = w.lane(); r < s_hw; r += w.width())
      if (A[L::SN + r] && s_inactive1(r)) part += (uint64_t)A[L::SN + r] * G;
    uint64_t inact = w.add_u64(part);
    while (inact > spool_max_inactive) {
      uint32_t v = s_lru(false);
      inact -= (uint64_t)A[L::SN + v] * G;
      s_evict(v);
    }
  }

  // interval arena: double-buffered; compaction copies live lists to the
  // other half (rows keep their identity).
  GML_HD bool iv_reserve(uint32_t k) {
    if (iv_hw + k <= C::IV) return true;
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
  GML_HD uint32_t stitch(const uint32_t* rows, uint32_t k, bool companion) {
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
    uint32_t o = iv_base + iv_hw;
    uint32_t tot = 0;
    for (uint32_t i = 0; i < k; ++i) tot += pn(rows[i]);
    for (uint32_t i = w.lane(); i < k; i += w.width()) {
      uint32_t m = rows[i];
      A[L::IVROW + o + i] = m;
      A[L::IVLO + o + i] = A[L::PLO + m];
      A[L::IVN + o + i] = pn(m);
    }
    iv_hw += k;
    T++;
    w.sync();
    if (w.leader()) {
      A[L::SN + r] = tot; A[L::SORD + r] = next_s; A[L::SLAST + r] = (uint32_t)T; A[L::SBORN + r] = (uint32_t)serial;
      A[L::SIVO + r] = o; A[L::SIVN + r] = k;
    }
    w.sync();
    sorted_insert(ssk(), A + L::SSR, s_count, skey(tot, next_s), r);
    next_s++;
    s_count++;
    s_bytes += (uint64_t)tot * G;
    cnt(S()->n_stitch);
    if (companion) cnt(S()->n_companion);
    cnt(S()->vmm_calls[V_RESERVE]);
    cnt(S()->vmm_calls[V_MAP], tot);
    cnt(S()->vmm_calls[V_ACCESS], tot);
    w.sync();
    if (w.leader()) hooks->on_stitch(r, A + L::IVLO + o, A + L::IVN + o, k);
    return r;
  }

  // Split: P -> F (first n chunks, keeps P's row, new
  // ordinal) + R (new row); no memory is created (D10). P is inactive.
  GML_HD uint32_t split(uint32_t P, uint32_t n) {
    if (n_p >= C::P) { overflow |= OV_P; return NONE32; }
    uint32_t lo = A[L::PLO + P], pnn = pn(P), nx = A[L::PNEXT + P];
    sorted_erase(psk(), A + L::PSR, n_p, skey(pnn, A[L::PORD + P]));
    sorted_insert(psk(), A + L::PSR, n_p - 1, skey(n, next_p), P);
    sorted_insert(psk(), A + L::PSR, n_p, skey(pnn - n, next_p + 1), n_p);
    uint32_t R = n_p++;
    w.sync();
    if (w.leader()) {
      A[L::PORD + P] = next_p; A[L::PKEY + P] = n; A[L::PNEXT + P] = R;
      A[L::PORD + R] = next_p + 1; A[L::PLO + R] = lo + n; A[L::PKEY + R] = pnn - n; A[L::PNEXT + R] = nx;
    }
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
  GML_HD uint32_t alloc(uint32_t n) {
    if (n_p >= C::P) { overflow |= OV_P; return NONE32; }
    sorted_insert(psk(), A + L::PSR, n_p, skey(n, next_p), n_p);
    uint32_t r = n_p++;
    if (w.leader()) {
      A[L::PORD + r] = next_p; A[L::PLO + r] = Cn; A[L::PKEY + r] = n; A[L::PNEXT + r] = NONE32;
      if (last_p != NONE32) A[L::PNEXT + last_p] = r;
      hooks->on_alloc(r, Cn, n);
    }
    last_p = r;
    next_p++;
    Cn += n;
    cnt(S()->n_alloc);
    cnt(S()->vmm_calls[V_RESERVE]);
    cnt(S()->vmm_calls[V_CREATE], n);
    cnt(S()->vmm_calls[V_MAP], n);
    cnt(S()->vmm_calls[V_ACCESS], n);
    w.sync();
    return r;
  }

  GML_HD void bind_p(uint32_t slot, uint32_t r, uint64_t raw) {
    uint32_t n = pn(r);
    bm_write(A[L::PLO + r], n, true);
    if (w.leader()) {
      A[L::PKEY + r] = n | ACT;
      H[slot] = ((uint64_t)HK_P << 62) | ((uint64_t)r << 40) | raw;
    }
    uint64_t by = (uint64_t)n * G;
    active += by; active_vmm += by; requested += raw;
    w.sync();
  }
  GML_HD void bind_s(uint32_t slot, uint32_t r, uint64_t raw) {
    uint32_t o = A[L::SIVO + r], k = A[L::SIVN + r];
    for (uint32_t i = 0; i < k; ++i) bm_write(A[L::IVLO + o + i], A[L::IVN + o + i], true);
    s_mark(r, true);
    if (w.leader()) H[slot] = ((uint64_t)HK_S << 62) | ((uint64_t)r << 40) | raw;
    uint64_t by = (uint64_t)A[L::SN + r] * G;
    active += by; active_vmm += by; requested += raw;
    w.sync();
  }

  // --------------------------------------------------------------- BFC
  // (no member arrays indexed by a runtime pool: they would force the engine
  // into local memory)
  GML_HD uint32_t* flr(uint32_t pool) const { return A + (pool ? L::FL1 : L::FL0); }
  GML_HD uint32_t* fls(uint32_t pool) const { return A + (pool ? L::FL1SZ : L::FL0SZ); }
  GML_HD uint32_t fln(uint32_t pool) const { return pool ? fl_n1 : fl_n0; }
  GML_HD void fln_add(uint32_t pool, int d) { if (pool) fl_n1 += d; else fl_n0 += d; }
  GML_HD void fl_push(uint32_t pool, uint32_t r, uint32_t size) {
    uint32_t k = fln(pool);
    fln_add(pool, 1);
    if (w.leader()) { flr(pool)[k] = r; fls(pool)[k] = size; A[L::BPOS + r] = k; }
  }
  GML_HD void fl_remove(uint32_t pool, uint32_t r) {
    uint32_t k = A[L::BPOS + r];
    uint32_t last = fln(pool) - 1;
    uint32_t lr = flr(pool)[last], ls = fls(pool)[last];
    w.sync();
    if (w.leader()) { flr(pool)[k] = lr; fls(pool)[k] = ls; A[L::BPOS + lr] = k; }
    fln_add(pool, -1);
    w.sync();
  }
  GML_HD uint32_t b_newrow() {
    uint32_t r;
    if (b_freerow != NONE32) { r = b_freerow; b_freerow = A[L::BNEXT + r]; }
    else if (b_hw < C::B) r = b_hw++;
    else { overflow |= OV_B; return NONE32; }
    b_live++;
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
      uint32_t k = 0;
      while (k < fln(pool)) {
        uint32_t r = flr(pool)[k];
        if (A[L::BPREV + r] == NONE32 && A[L::BNEXT + r] == NONE32) {
          seg_bytes -= (uint64_t)A[L::BSIZE + r] * 512;
          cnt(S()->n_seg_release);
          if (w.leader()) hooks->on_bfc_release(A[L::BSEG + r]);
          fl_remove(pool, r);
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
    bool exact = kind == GML_POLICY_BFC_EXACT;
    uint64_t r = raw < 512 ? 512 : (raw + 511) / 512 * 512;
    uint32_t ru = (uint32_t)(r / 512);
    uint32_t pool = exact ? 0 : (r <= BFC_SMALL_SIZE ? 0 : 1);
    // op 1: best fit = min (size, segment, offset) among free blocks >= r
    // (PyTorch orders by (size, address), D21-D23): one pass, the address is
    // loaded only for blocks that tie or beat the lane's best size.
    const uint32_t nf = fln(pool);
    const uint32_t* fz = fls(pool);
    const uint32_t* fr = flr(pool);
    uint32_t bs = NONE32, brow = NONE32;
    uint64_t ba = ~0ull;
    for (uint32_t q = w.lane(); q < (nf + 3) / 4; q += w.width()) {
      uint4 z = reinterpret_cast<const uint4*>(fz)[q];
      uint32_t zz[4] = {z.x, z.y, z.z, z.w};
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        if (4 * q + i < nf && zz[i] >= ru && zz[i] <= bs) {
          const uint32_t rr = fr[4 * q + i];
          const uint64_t ad = ((uint64_t)A[L::BSEG + rr] << 32) | A[L::BOFF + rr];
          if (zz[i] < bs || ad < ba) { bs = zz[i]; ba = ad; brow = rr; }
        }
      }
    }
    KeyRow gs = w.argmin(bs == NONE32 ? ~0ull : (uint64_t)bs, 0);
    uint32_t row;
    int state;
    if (gs.key != ~0ull) {
      row = w.argmin(bs == (uint32_t)gs.key ? ba : ~0ull, brow).row;
      fl_remove(pool, row);
      state = ST_HIT;
    } else {
      uint64_t ss = bfc_segment_size(r, exact);
      if (reserved_vmm() + seg_bytes + ss > capacity) {
        bfc_release();
        if (reserved_vmm() + seg_bytes + ss > capacity) { rec = rec_oom(); cnt(S()->state_count[ST_S5 - 1]); return false; }
      }
      row = b_newrow();
      if (row == NONE32) return false;
      uint32_t seg = next_seg++;
      if (w.leader()) {
        A[L::BSIZE + row] = (uint32_t)(ss / 512); A[L::BOFF + row] = 0; A[L::BSEG + row] = seg;
        A[L::BPREV + row] = NONE32; A[L::BNEXT + row] = NONE32; A[L::BFLAGS + row] = pool ? BF_POOL1 : 0;
        hooks->on_bfc_segment(seg, ss);
      }
      seg_bytes += ss;
      cnt(S()->n_seg_alloc);
      state = ST_NEWSEG;
      w.sync();
    }
    // op 2: split, front allocated, remainder stays in the pool
    uint32_t size = A[L::BSIZE + row];
    uint64_t rem = (uint64_t)(size - ru) * 512;
    bool do_split = (exact || pool == 0) ? rem >= 512 : rem > BFC_SMALL_SIZE;
    if (do_split) {
      uint32_t rest = b_newrow();
      if (rest == NONE32) return false;
      uint32_t nx = A[L::BNEXT + row];
      if (w.leader()) {
        A[L::BSIZE + rest] = size - ru; A[L::BOFF + rest] = A[L::BOFF + row] + ru; A[L::BSEG + rest] = A[L::BSEG + row];
        A[L::BPREV + rest] = row; A[L::BNEXT + rest] = nx; A[L::BFLAGS + rest] = A[L::BFLAGS + row] & BF_POOL1;
        if (nx != NONE32) A[L::BPREV + nx] = rest;
        A[L::BNEXT + row] = rest; A[L::BSIZE + row] = ru;
      }
      w.sync();
      fl_push(pool, rest, size - ru);
      w.sync();
    }
    if (w.leader()) {
      A[L::BFLAGS + row] |= BF_ALLOC;
      H[slot] = ((uint64_t)HK_B << 62) | ((uint64_t)row << 40) | raw;
    }
    uint64_t by = (uint64_t)A[L::BSIZE + row] * 512;
    active += by; requested += raw;
    cnt(S()->state_count[state - 1]);
    rec = (uint64_t)A[L::BOFF + row] | ((uint64_t)HK_B << 32) | ((uint64_t)state << 34) | ((uint64_t)A[L::BSEG + row] << 40);
    w.sync();
    return true;
  }

  // BFC free + merge (PAPER.md L123-125 ops 3-4)
  GML_HD void bfc_free(uint32_t row) {
    uint32_t pool = (A[L::BFLAGS + row] & BF_POOL1) ? 1 : 0;
    w.sync();
    if (w.leader()) A[L::BFLAGS + row] &= ~BF_ALLOC;
    w.sync();
    uint32_t p = A[L::BPREV + row];
    if (p != NONE32 && !(A[L::BFLAGS + p] & BF_ALLOC)) {
      fl_remove(pool, p);
      uint32_t nx = A[L::BNEXT + row];
      if (w.leader()) {
        A[L::BSIZE + p] += A[L::BSIZE + row];
        A[L::BNEXT + p] = nx;
        if (nx != NONE32) A[L::BPREV + nx] = p;
      }
      w.sync();
      b_delrow(row);
      w.sync();
      row = p;
    }
    uint32_t n = A[L::BNEXT + row];
    if (n != NONE32 && !(A[L::BFLAGS + n] & BF_ALLOC)) {
      fl_remove(pool, n);
      uint32_t nn = A[L::BNEXT + n];
      if (w.leader()) {
        A[L::BSIZE + row] += A[L::BSIZE + n];
        A[L::BNEXT + row] = nn;
        if (nn != NONE32) A[L::BPREV + nn] = row;
      }
      w.sync();
      b_delrow(n);
      w.sync();
    }
    fl_push(pool, row, A[L::BSIZE + row]);
    w.sync();
  }

  // ------------------------------------------------------------ GMLake
  // GMLake malloc: Algorithm 1 + S1-S5
  GML_HD bool vmm_malloc(uint32_t slot, uint64_t raw, uint64_t& rec) {
    uint32_t b = (uint32_t)(gshift < 64 ? (raw + G - 1) >> gshift : (raw + G - 1) / G);   // D2
    GML_T0(ta);
    stitch_free_bytes();                                                                   // D17(ii)
    GML_T1(4, ta);
    GML_T0(tb);
    bool rr = flags & GML_F_REMAINDER_RULE;
    bool pfirst = flags & GML_F_S1_PBLOCK_FIRST;
    const uint32_t WD = w.width();
    uint64_t* const pk = psk();
    const uint32_t* const pr = A + L::PSR;
    // ---- S1 on pPool: the run of size-b keys, first inactive one in ordinal
    // order (Alg. 1 L2-4; D4, D5). An inactive pBlock's p_key is its size.
    uint32_t s1p_row = NONE32, s1p_ord = NONE32;
    const uint32_t run = lower_bound(pk, n_p, skey(b, 0));
    for (uint32_t base = run; base < n_p; base += WD) {
      const uint32_t k = base + w.lane();
      const bool in = k < n_p && (uint32_t)(pk[k] >> 32) == b;
      const bool hit = in && A[L::PKEY + pr[in ? k : 0]] == b;
      const uint32_t j = w.first_true(hit);
      if (j != NONE32) { s1p_row = pr[base + j]; s1p_ord = (uint32_t)pk[base + j]; break; }
      if (w.first_true(!in) != NONE32) break;
    }
    GML_T1(5, tb);
    GML_T0(tc);
    // ---- S1 on sPool (sPool first unless S1_PBLOCK_FIRST, D5) ----
    if (!(pfirst && s1p_row != NONE32)) {
      const uint64_t* sk = ssk();
      const uint32_t* sr = A + L::SSR;
      uint32_t srow = NONE32, sord = NONE32;
      for (uint32_t base = lower_bound(sk, s_count, skey(b, 0)); base < s_count; base += WD) {
        const uint32_t k = base + w.lane();
        const bool in = k < s_count && (uint32_t)(sk[k] >> 32) == b;
        const bool hit = in && s_inactive1(sr[k]);
        const uint32_t j = w.first_true(hit);
        if (j != NONE32) { srow = sr[base + j]; sord = (uint32_t)sk[base + j]; break; }
        if (w.first_true(!in) != NONE32) break;
      }
      GML_T1(6, tc);
      if (srow != NONE32) {
        GML_T0(td);
        bind_s(slot, srow, raw);
        GML_T1(7, td);
        T++;
        if (w.leader()) A[L::SLAST + srow] = (uint32_t)T;
        rec = rec_of(sord, HK_S, ST_S1);
        cnt(S()->state_count[ST_S1 - 1]);
        w.sync();
        return true;
      }
    }
    if (s1p_row != NONE32) {
      GML_T0(te);
      bind_p(slot, s1p_row, raw);
      GML_T1(8, te);
      rec = rec_of(s1p_ord, HK_P, ST_S1);
      cnt(S()->state_count[ST_S1 - 1]);
      w.sync();
      return true;
    }
    // ---- Alg. 1 L6-8: the replace-loop keeps the smallest size >= bSize,
    // ties -> the last in pool order = highest ordinal (D6); candidates are
    // inactive pBlocks, eligible (size >= limit, D8) unless REMAINDER_RULE.
    uint32_t s2_row = NONE32, s2_ord = 0, s2_n = 0;
    {
      const uint32_t from = (rr || elig_n <= b + 1) ? b + 1 : elig_n;
      uint32_t c1 = NONE32;
      for (uint32_t base = lower_bound(pk, n_p, skey(from, 0)); base < n_p; base += WD) {
        const uint32_t k = base + w.lane();
        const bool hit = k < n_p && A[L::PKEY + pr[k < n_p ? k : 0]] < ACT;
        const uint32_t j = w.first_true(hit);
        if (j != NONE32) { c1 = base + j; break; }
      }
      if (c1 != NONE32) {
        s2_n = (uint32_t)(pk[c1] >> 32);
        const uint32_t e = lower_bound(pk, n_p, skey(s2_n + 1, 0));   // end of the size group
        for (int32_t top = (int32_t)e - 1;; top -= (int32_t)WD) {      // last inactive in the group
          const int32_t k = top - (int32_t)w.lane();
          const bool hit = k >= (int32_t)c1 && A[L::PKEY + pr[k >= (int32_t)c1 ? k : c1]] < ACT;
          const uint32_t j = w.first_true(hit);
          if (j != NONE32) { s2_row = pr[top - j]; s2_ord = (uint32_t)pk[top - j]; break; }
        }
      }
    }
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
        rec = rec_of(A[L::PORD + P], HK_P, ST_S2);
      }
      cnt(S()->state_count[ST_S2 - 1]);
      w.sync();
      return true;
    }
    // ---- Alg. 1 L9-10: greedy largest-first accumulation over eligible
    // inactive pBlocks (all < b now): size groups from the top, ordinals
    // ascending in a group, taking just enough blocks to reach b.
    uint32_t k = 0;
    uint64_t CBsize = 0;
    {
      const uint32_t lo_idx = lower_bound(pk, n_p, skey(elig_n, 0));
      uint32_t cur = lower_bound(pk, n_p, skey(b, 0));
      while (CBsize < b && cur > lo_idx) {
        const uint32_t gsz = (uint32_t)(pk[cur - 1] >> 32);
        uint32_t gs = lower_bound(pk, n_p, skey(gsz, 0));
        if (gs < lo_idx) gs = lo_idx;
        uint64_t need = (b - CBsize + gsz - 1) / gsz;
        for (uint32_t base = gs; base < cur && need; base += WD) {
          const uint32_t kk = base + w.lane();
          const bool hit = kk < cur && A[L::PKEY + pr[kk < cur ? kk : gs]] < ACT;
          uint32_t total;
          const uint32_t rk = w.rank_true(hit, &total);
          const uint32_t take = total < need ? total : (uint32_t)need;
          if (k + take + 2 > C::CB) { overflow |= OV_CB; return false; }
          if (hit && rk < take) A[L::CB + k + rk] = pr[kk];
          k += take;
          need -= take;
          CBsize += (uint64_t)take * gsz;
          w.sync();
        }
        cur = gs;
      }
    }
    w.sync();
    if (CBsize >= b) {
      // ---- S3: split the last candidate (D14), stitch ----
      if (CBsize > b) {
        uint32_t last = A[L::CB + k - 1];
        uint32_t lastn = pn(last);
        uint32_t n = (uint32_t)(b - (CBsize - lastn));
        if (!(rr && (uint64_t)(lastn - n) * G < limit_bytes)) {
          uint32_t R = split(last, n);
          if (R == NONE32) return false;
          if (!(flags & GML_F_NO_COMPANION)) {
            uint32_t pr[2] = {last, R};
            stitch(pr, 2, true);
            if (overflow) return false;
          }
        }
      }
      uint32_t s = stitch(A + L::CB, k, false);
      if (s == NONE32) return false;
      bind_s(slot, s, raw);
      rec = rec_of(A[L::SORD + s], HK_S, ST_S3);
      cnt(S()->state_count[ST_S3 - 1]);
      w.sync();
      return true;
    }
    // ---- S4: Alloc the shortfall (D15) ----
    uint32_t shortfall = (uint32_t)(b - CBsize);
    if (reserved() + (uint64_t)shortfall * G > capacity) {
      rec = rec_oom();                                               // S5 (L528, D16)
      cnt(S()->state_count[ST_S5 - 1]);
      return false;
    }
    uint32_t p = alloc(shortfall);
    if (p == NONE32) return false;
    if (k == 0) {
      bind_p(slot, p, raw);
      rec = rec_of(A[L::PORD + p], HK_P, ST_S4);
    } else {
      if (w.leader()) A[L::CB + k] = p;
      w.sync();
      uint32_t s = stitch(A + L::CB, k + 1, false);
      if (s == NONE32) return false;
      bind_s(slot, s, raw);
      rec = rec_of(A[L::SORD + s], HK_S, ST_S4);
    }
    cnt(S()->state_count[ST_S4 - 1]);
    w.sync();
    return true;
  }

  // Update: unbind, no release, no merge (D19).
  GML_HD uint64_t do_free(uint32_t slot, uint64_t hv) {
    uint32_t hk = (uint32_t)(hv >> 62);
    uint32_t row = (uint32_t)((hv >> 40) & 0x3FFFFF);
    uint64_t raw = hv & MASK40;
    uint64_t by, rec;
    if (hk == HK_P) {
      uint32_t n = pn(row);
      by = (uint64_t)n * G;
      bm_write(A[L::PLO + row], n, false);
      if (w.leader()) A[L::PKEY + row] = n;
      rec = rec_of(A[L::PORD + row], HK_P, 0);
      active_vmm -= by;
    } else if (hk == HK_S) {
      by = (uint64_t)A[L::SN + row] * G;
      uint32_t o = A[L::SIVO + row], k = A[L::SIVN + row];
      for (uint32_t i = 0; i < k; ++i) bm_write(A[L::IVLO + o + i], A[L::IVN + o + i], false);
      s_mark(row, false);
      rec = rec_of(A[L::SORD + row], HK_S, 0);
      active_vmm -= by;
    } else {
      by = (uint64_t)A[L::BSIZE + row] * 512;
      rec = (uint64_t)A[L::BOFF + row] | ((uint64_t)HK_B << 32) | ((uint64_t)A[L::BSEG + row] << 40);
      bfc_free(row);
    }
    active -= by;
    requested -= raw;
    live--;
    w.sync();
    if (w.leader()) H[slot] = (uint64_t)HK_EMPTY << 62;
    w.sync();
    return rec;
  }

  // One event. Returns the assignment record; sets `status` (OOM / INVALID)
  // or `overflow` when the replay must stop.
  GML_HD uint64_t step(uint64_t ev) {
    bool is_free = ev >> 63;
    uint32_t slot = (uint32_t)((ev >> 40) & 0x7FFFFFu);
    uint64_t raw = ev & MASK40;
    if (slot >= h_cap) { overflow |= OV_H; return 0; }
    uint64_t hv = H[slot];
    bool empty = (hv >> 62) == HK_EMPTY;
    uint64_t rec = 0;
    if (is_free) {
      if (empty || raw) { status = GML_ERR_INVALID; return 0; }
      GML_T0(t0);
      uint64_t fr = do_free(slot, hv);
      GML_T1((hv >> 62) == HK_B ? 1 : 0, t0);
      return fr;
    }
    if (!empty || raw == 0) { status = GML_ERR_INVALID; return 0; }
    serial++;
    GML_T0(t1);
    bool vm = kind == GML_POLICY_GMLAKE && raw >= small_thr;
    bool ok = vm ? vmm_malloc(slot, raw, rec) : bfc_malloc(slot, raw, rec);
    GML_T1(vm ? 2 : 3, t1);
    if (overflow) return 0;
    if (!ok) { status = GML_ERR_OOM; return rec; }
    live++;
    return rec;
  }

  GML_HD void sample() {
    if (active > pk_active) pk_active = active;
    uint64_t rs = reserved();
    if (rs > pk_reserved) pk_reserved = rs;
    if (requested > pk_requested) pk_requested = requested;
    if (active_vmm > pk_active_vmm) pk_active_vmm = active_vmm;
    if (reserved_vmm() > pk_reserved_vmm) pk_reserved_vmm = reserved_vmm();
    if (live > mx_h) mx_h = (uint32_t)live;
    if (n_p > mx_p) mx_p = n_p;
    if (s_count > mx_s) mx_s = s_count;
    if (b_live > mx_b) mx_b = b_live;
  }

  // write the register-held fields of the stats record (leader)
  GML_HD void finish(uint64_t n_events, uint64_t n_done, int64_t oom_event) {
    w.sync();
    if (w.leader()) {
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
    }
    w.sync();
  }
};

}  // namespace gml
