// policy.cuh -- the GMLake allocation engine, written once for two executors:
//
//   * DeviceWarp: the 32 lanes of one warp own one (trace, policy) replay on
//     sm_100a; table scans stride the rows over the lanes and finish with
//     __reduce_{min,max}_sync / ballots (the "warp-level argmin/ballot
//     best-fit search" of the north star); mutations are written by lane 0
//     after every lane took the same (uniform) decision.
//   * HostWarp: width 1, for the live allocator (gml_malloc/gml_free), so the
//     live path and the replay take identical decisions.
//
// The method (§3.3 Algorithm 1, §4.1) is walked in
// the paper's order; readings D1..D30 are listed in DESIGN.md. The engine
// never reads the oracle (oracle/), and the oracle never reads this file.
//
// Data layout per replay ("arena", SoA, u32 unless noted; in shared memory
// when it fits, else in global memory):
//   bitmap   1 bit per chunk: chunk owned by a live tensor (D18)  -- the
//            "active" state of pBlocks; an sBlock is inactive iff its chunk
//            intervals hold no set bit.
//   pPool    p_n (granules), p_ord, p_lo (first chunk); rows never deleted
//            (Split rewrites the parent's row as the front piece F and appends
//            R), so rows are 0..n_p-1 and |pPool| = n_p.
//   sPool    s_n (0 = free row), s_ord, s_last (LRU key), s_born (malloc
//            serial), s_ivo / s_ivn (interval list in the interval arena).
//   ivs      iv_lo / iv_n: chunk intervals of sBlocks, double-buffered for
//            compaction.
//   handles  u64 per slot: kind (2 b) | row (22 b) | raw bytes (40 b).
//   BFC      b_size / b_off (512-byte units), b_seg, b_prev, b_next, b_flags,
//            b_pos; free-block lists per pool (pool 0 from the bottom, pool 1
//            from the top of one array) so best-fit scans touch free blocks
//            only.
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

namespace gml {

constexpr uint32_t NONE32 = 0xFFFFFFFFu;
constexpr uint64_t MASK40 = (1ull << 40) - 1;

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
  GML_HD uint32_t min_u32(uint32_t v) const {
#if defined(__CUDA_ARCH__)
    return __reduce_min_sync(0xFFFFFFFFu, v);
#else
    return v;
#endif
  }
  GML_HD uint32_t max_u32(uint32_t v) const {
#if defined(__CUDA_ARCH__)
    return __reduce_max_sync(0xFFFFFFFFu, v);
#else
    return v;
#endif
  }
  GML_HD uint32_t add_u32(uint32_t v) const {
#if defined(__CUDA_ARCH__)
    return __reduce_add_sync(0xFFFFFFFFu, v);
#else
    return v;
#endif
  }
  GML_HD uint32_t ballot(bool p) const {
#if defined(__CUDA_ARCH__)
    return __ballot_sync(0xFFFFFFFFu, p);
#else
    return p ? 1u : 0u;
#endif
  }
  GML_HD uint32_t bcast(uint32_t v, uint32_t src) const {
#if defined(__CUDA_ARCH__)
    return __shfl_sync(0xFFFFFFFFu, v, src);
#else
    (void)src;
    return v;
#endif
  }
  GML_HD uint64_t min_u64(uint64_t v) const {
    uint32_t hi = min_u32((uint32_t)(v >> 32));
    uint32_t lo = min_u32(((uint32_t)(v >> 32) == hi) ? (uint32_t)v : NONE32);
    return ((uint64_t)hi << 32) | lo;
  }
  GML_HD uint64_t add_u64(uint64_t v) const {
#if defined(__CUDA_ARCH__)
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
#endif
    return v;
  }
};

struct HostWarp {
  GML_HD uint32_t lane() const { return 0; }
  GML_HD uint32_t width() const { return 1; }
  GML_HD bool leader() const { return true; }
  GML_HD void sync() const {}
  GML_HD uint32_t min_u32(uint32_t v) const { return v; }
  GML_HD uint32_t max_u32(uint32_t v) const { return v; }
  GML_HD uint32_t add_u32(uint32_t v) const { return v; }
  GML_HD uint32_t ballot(bool p) const { return p ? 1u : 0u; }
  GML_HD uint32_t bcast(uint32_t v, uint32_t) const { return v; }
  GML_HD uint64_t min_u64(uint64_t v) const { return v; }
  GML_HD uint64_t add_u64(uint64_t v) const { return v; }
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
struct Caps {
  uint32_t bm_words;    // ceil(capacity chunks / 32)
  uint32_t p, s, iv, h, b, cb;
};

// Arena layout: byte offsets of every table for a given Caps.
struct Layout {
  uint64_t o_stats, o_bm, o_pn, o_pord, o_plo, o_sn, o_sord, o_slast, o_sborn, o_sivo, o_sivn,
      o_ivlo, o_ivn, o_h, o_bsize, o_boff, o_bseg, o_bprev, o_bnext, o_bflags, o_bpos, o_fl, o_cb,
      bytes;
  GML_HD static Layout make(const Caps& c) {
    Layout L{};
    uint64_t o = 0;
    auto take = [&](uint64_t n) { uint64_t r = o; o += (n + 15) & ~15ull; return r; };
    L.o_stats = take(sizeof(gml_stats_t));
    L.o_h = take(8ull * c.h);
    L.o_bm = take(4ull * c.bm_words);
    L.o_pn = take(4ull * c.p); L.o_pord = take(4ull * c.p); L.o_plo = take(4ull * c.p);
    L.o_sn = take(4ull * c.s); L.o_sord = take(4ull * c.s); L.o_slast = take(4ull * c.s);
    L.o_sborn = take(4ull * c.s); L.o_sivo = take(4ull * c.s); L.o_sivn = take(4ull * c.s);
    L.o_ivlo = take(4ull * 2 * c.iv); L.o_ivn = take(4ull * 2 * c.iv);
    L.o_bsize = take(4ull * c.b); L.o_boff = take(4ull * c.b); L.o_bseg = take(4ull * c.b);
    L.o_bprev = take(4ull * c.b); L.o_bnext = take(4ull * c.b); L.o_bflags = take(4ull * c.b);
    L.o_bpos = take(4ull * c.b); L.o_fl = take(4ull * c.b);
    L.o_cb = take(4ull * c.cb);
    L.bytes = o;
    return L;
  }
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

GML_HD uint32_t ctz32(uint32_t m) {
#if defined(__CUDA_ARCH__)
  return (uint32_t)(__ffs(m) - 1);
#else
  return (uint32_t)__builtin_ctz(m);
#endif
}

GML_HD uint64_t rec_of(uint32_t ord, uint32_t kind, uint32_t state) {
  return (uint64_t)ord | ((uint64_t)kind << 32) | ((uint64_t)state << 34);
}
GML_HD uint64_t rec_oom() { return 0xFFFFFFFFull | ((uint64_t)ST_S5 << 34); }

// ------------------------------------------------------------------ engine
template <class W, class H = NoHooks>
struct Engine {
  W w;
  H* hooks;
  // policy
  uint32_t kind, flags;
  uint64_t capacity, G, small_thr, limit_bytes, spool_max_inactive;
  uint32_t spool_max, elig_n;
  // tables
  Caps cap;
  gml_stats_t* st;
  uint64_t* h;
  uint32_t *bm, *p_n, *p_ord, *p_lo, *s_n, *s_ord, *s_last, *s_born, *s_ivo, *s_ivn, *iv_lo, *iv_n;
  uint32_t *b_size, *b_off, *b_seg, *b_prev, *b_next, *b_flags, *b_pos, *fl, *cb;
  // scalar state (identical in every lane)
  uint32_t C, next_p, next_s, n_p, s_hw, s_count, s_freerow, iv_base, iv_hw;
  uint32_t b_hw, b_freerow, b_live, fl_n0, fl_n1, next_seg;
  uint64_t T, serial, active, requested, active_vmm, seg_bytes, s_bytes, live;
  uint32_t overflow, status;
  // peaks kept in registers
  uint64_t pk_active, pk_reserved, pk_requested, pk_active_vmm, pk_reserved_vmm;
  uint32_t mx_p, mx_s, mx_h, mx_b;

  // -------------------------------------------------------------- set-up
  GML_HDI void init(const gml_policy& pol, const Caps& c, uint8_t* arena, H* hk) {
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
    elig_n = e > 0xFFFFFFFFull ? NONE32 : (uint32_t)e;
    cap = c;
    Layout L = Layout::make(c);
    st = (gml_stats_t*)(arena + L.o_stats);
    h = (uint64_t*)(arena + L.o_h);
    bm = (uint32_t*)(arena + L.o_bm);
    p_n = (uint32_t*)(arena + L.o_pn); p_ord = (uint32_t*)(arena + L.o_pord); p_lo = (uint32_t*)(arena + L.o_plo);
    s_n = (uint32_t*)(arena + L.o_sn); s_ord = (uint32_t*)(arena + L.o_sord); s_last = (uint32_t*)(arena + L.o_slast);
    s_born = (uint32_t*)(arena + L.o_sborn); s_ivo = (uint32_t*)(arena + L.o_sivo); s_ivn = (uint32_t*)(arena + L.o_sivn);
    iv_lo = (uint32_t*)(arena + L.o_ivlo); iv_n = (uint32_t*)(arena + L.o_ivn);
    b_size = (uint32_t*)(arena + L.o_bsize); b_off = (uint32_t*)(arena + L.o_boff); b_seg = (uint32_t*)(arena + L.o_bseg);
    b_prev = (uint32_t*)(arena + L.o_bprev); b_next = (uint32_t*)(arena + L.o_bnext);
    b_flags = (uint32_t*)(arena + L.o_bflags); b_pos = (uint32_t*)(arena + L.o_bpos); fl = (uint32_t*)(arena + L.o_fl);
    cb = (uint32_t*)(arena + L.o_cb);
    C = next_p = next_s = n_p = s_hw = s_count = 0;
    s_freerow = NONE32;
    iv_base = 0; iv_hw = 0;
    b_hw = b_live = fl_n0 = fl_n1 = next_seg = 0;
    b_freerow = NONE32;
    T = serial = active = requested = active_vmm = seg_bytes = s_bytes = live = 0;
    overflow = 0; status = GML_OK;
    pk_active = pk_reserved = pk_requested = pk_active_vmm = pk_reserved_vmm = 0;
    mx_p = mx_s = mx_h = mx_b = 0;
    // zero stats, bitmap; mark every handle slot empty
    uint32_t* sw = (uint32_t*)st;
    for (uint32_t i = w.lane(); i < sizeof(gml_stats_t) / 4; i += w.width()) sw[i] = 0;
    for (uint32_t i = w.lane(); i < c.bm_words; i += w.width()) bm[i] = 0;
    for (uint32_t i = w.lane(); i < c.h; i += w.width()) h[i] = (uint64_t)HK_EMPTY << 62;
    w.sync();
  }

  GML_HD uint64_t reserved_vmm() const { return (uint64_t)C * G; }
  GML_HD uint64_t reserved() const { return reserved_vmm() + seg_bytes; }
  GML_HD void cnt(uint64_t& f, uint64_t v = 1) { if (w.leader()) f += v; }

  // ------------------------------------------------------------ bitmap
  // set / clear chunks [lo, lo+n): lanes own distinct words
  GML_HD void bm_write(uint32_t lo, uint32_t n, bool v) {
    if (n == 0) return;
    uint32_t a = lo >> 5, z = (lo + n - 1) >> 5;
    for (uint32_t wd = a + w.lane(); wd <= z; wd += w.width()) {
      uint32_t m = 0xFFFFFFFFu;
      if (wd == a) m &= 0xFFFFFFFFu << (lo & 31);
      if (wd == z) m &= 0xFFFFFFFFu >> (31 - ((lo + n - 1) & 31));
      if (v) bm[wd] |= m; else bm[wd] &= ~m;
    }
    w.sync();   // the next interval may share a word
  }
  // single-lane test: any chunk of [lo, lo+n) owned?
  GML_HD bool bm_any1(uint32_t lo, uint32_t n) const {
    uint32_t a = lo >> 5, z = (lo + n - 1) >> 5;
    for (uint32_t wd = a; wd <= z; ++wd) {
      uint32_t m = 0xFFFFFFFFu;
      if (wd == a) m &= 0xFFFFFFFFu << (lo & 31);
      if (wd == z) m &= 0xFFFFFFFFu >> (31 - ((lo + n - 1) & 31));
      if (bm[wd] & m) return true;
    }
    return false;
  }
  GML_HD bool p_active(uint32_t r) const { uint32_t lo = p_lo[r]; return (bm[lo >> 5] >> (lo & 31)) & 1u; }
  GML_HD bool s_inactive1(uint32_t r) const {   // single lane
    uint32_t o = s_ivo[r], k = s_ivn[r];
    for (uint32_t i = 0; i < k; ++i)
      if (bm_any1(iv_lo[o + i], iv_n[o + i])) return false;
    return true;
  }

  // --------------------------------------------------------- sPool rows
  GML_HD void s_evict(uint32_t r) {   // StitchFree of one sBlock
    s_bytes -= (uint64_t)s_n[r] * G;
    if (w.leader()) {
      s_n[r] = 0;
      s_born[r] = s_freerow;     // free-row link
    }
    s_freerow = r;
    s_count--;
    cnt(st->n_evict);
    cnt(st->vmm_calls[V_UNMAP]);
    cnt(st->vmm_calls[V_ADDR_FREE]);
    if (w.leader()) hooks->on_evict(r);
    w.sync();
  }

  // argmin of last_use over inactive live sBlocks (optionally excluding the
  // ones born in this malloc); NONE32 if none. last_use values are unique.
  GML_HD uint32_t s_lru(bool exclude_born) {
    uint32_t best = NONE32, row = NONE32;
    for (uint32_t r = w.lane(); r < s_hw; r += w.width()) {
      if (s_n[r] == 0) continue;
      if (exclude_born && s_born[r] == (uint32_t)serial) continue;
      uint32_t lu = s_last[r];
      if (lu < best && s_inactive1(r)) { best = lu; row = r; }
    }
    uint32_t g = w.min_u32(best);
    if (g == NONE32) return NONE32;
    uint32_t b = w.ballot(best == g && row != NONE32);
    return w.bcast(row, ctz32(b));
  }

  // D17(ii): at VMM-path malloc entry, release LRU inactive sBlocks while the
  // inactive ones hold more than the byte cap.
  GML_HD void stitch_free_bytes() {
    if (s_bytes <= spool_max_inactive) return;   // inactive bytes <= all bytes
    uint64_t part = 0;
    for (uint32_t r = w.lane(); r < s_hw; r += w.width())
      if (s_n[r] && s_inactive1(r)) part += (uint64_t)s_n[r] * G;
    uint64_t inact = w.add_u64(part);
    while (inact > spool_max_inactive) {
      uint32_t v = s_lru(false);
      inact -= (uint64_t)s_n[v] * G;
      s_evict(v);
    }
  }

  // interval arena: double-buffered; compaction copies live lists to the
  // other half (rows keep their identity).
  GML_HD bool iv_reserve(uint32_t k) {
    if (iv_hw + k <= cap.iv) return true;
    uint32_t dst = iv_base ^ cap.iv;   // other half
    uint32_t pos = 0;
    for (uint32_t r = 0; r < s_hw; ++r) {
      if (s_n[r] == 0) continue;
      uint32_t o = s_ivo[r], n = s_ivn[r];
      for (uint32_t i = w.lane(); i < n; i += w.width()) {
        iv_lo[dst + pos + i] = iv_lo[o + i];
        iv_n[dst + pos + i] = iv_n[o + i];
      }
      if (w.leader()) s_ivo[r] = dst + pos;
      pos += n;
    }
    w.sync();
    iv_base = dst;
    iv_hw = pos;
    if (iv_hw + k > cap.iv) { overflow |= OV_IV; return false; }
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
    uint32_t r;
    if (s_freerow != NONE32) {
      r = s_freerow;
      s_freerow = s_born[r];
    } else {
      if (s_hw >= cap.s) { overflow |= OV_S; return NONE32; }
      r = s_hw++;
    }
    if (!iv_reserve(k)) return NONE32;
    uint32_t o = iv_base + iv_hw;
    uint32_t tot = 0;
    for (uint32_t i = 0; i < k; ++i) tot += p_n[rows[i]];
    for (uint32_t i = w.lane(); i < k; i += w.width()) {
      iv_lo[o + i] = p_lo[rows[i]];
      iv_n[o + i] = p_n[rows[i]];
    }
    iv_hw += k;
    T++;
    if (w.leader()) {
      s_n[r] = tot; s_ord[r] = next_s; s_last[r] = (uint32_t)T; s_born[r] = (uint32_t)serial;
      s_ivo[r] = o; s_ivn[r] = k;
    }
    next_s++;
    s_count++;
    s_bytes += (uint64_t)tot * G;
    cnt(st->n_stitch);
    if (companion) cnt(st->n_companion);
    cnt(st->vmm_calls[V_RESERVE]);
    cnt(st->vmm_calls[V_MAP], tot);
    cnt(st->vmm_calls[V_ACCESS], tot);
    w.sync();
    if (w.leader()) hooks->on_stitch(r, iv_lo + o, iv_n + o, k);
    return r;
  }

  // Split: P -> F (first n chunks, keeps P's row, new
  // ordinal) + R (new row); no memory is created (D10).
  GML_HD uint32_t split(uint32_t P, uint32_t n) {
    if (n_p >= cap.p) { overflow |= OV_P; return NONE32; }
    uint32_t lo = p_lo[P], pn = p_n[P];
    uint32_t R = n_p++;
    if (w.leader()) {
      p_ord[P] = next_p; p_n[P] = n;
      p_ord[R] = next_p + 1; p_lo[R] = lo + n; p_n[R] = pn - n;
    }
    next_p += 2;
    cnt(st->n_split);
    cnt(st->vmm_calls[V_RESERVE], 2);
    cnt(st->vmm_calls[V_MAP], pn);
    cnt(st->vmm_calls[V_ACCESS], pn);
    cnt(st->vmm_calls[V_UNMAP]);
    cnt(st->vmm_calls[V_ADDR_FREE]);
    w.sync();
    if (w.leader()) hooks->on_split(P, R, lo, n);
    if (flags & GML_F_SPLIT_INVALIDATES) {   // D12 variant: drop sBlocks over P
      for (uint32_t base = 0; base < s_hw; base += w.width()) {
        uint32_t r = base + w.lane();
        bool hit = false;
        if (r < s_hw && s_n[r]) {
          uint32_t o = s_ivo[r], k = s_ivn[r];
          for (uint32_t i = 0; i < k; ++i)
            if (iv_lo[o + i] < lo + pn && lo < iv_lo[o + i] + iv_n[o + i]) hit = true;
        }
        uint32_t m = w.ballot(hit);
        while (m) {
          uint32_t j = ctz32(m);
          m &= m - 1;
          s_evict(base + j);
        }
      }
    }
    return R;
  }

  // Alloc: the only source of new chunks.
  GML_HD uint32_t alloc(uint32_t n) {
    if (n_p >= cap.p) { overflow |= OV_P; return NONE32; }
    uint32_t r = n_p++;
    if (w.leader()) { p_ord[r] = next_p; p_lo[r] = C; p_n[r] = n; }
    next_p++;
    if (w.leader()) hooks->on_alloc(r, C, n);
    C += n;
    cnt(st->n_alloc);
    cnt(st->vmm_calls[V_RESERVE]);
    cnt(st->vmm_calls[V_CREATE], n);
    cnt(st->vmm_calls[V_MAP], n);
    cnt(st->vmm_calls[V_ACCESS], n);
    w.sync();
    return r;
  }

  GML_HD void bind_p(uint32_t slot, uint32_t r, uint64_t raw) {
    bm_write(p_lo[r], p_n[r], true);
    if (w.leader()) h[slot] = ((uint64_t)HK_P << 62) | ((uint64_t)r << 40) | raw;
    uint64_t by = (uint64_t)p_n[r] * G;
    active += by; active_vmm += by; requested += raw;
    w.sync();
  }
  GML_HD void bind_s(uint32_t slot, uint32_t r, uint64_t raw) {
    uint32_t o = s_ivo[r], k = s_ivn[r];
    for (uint32_t i = 0; i < k; ++i) bm_write(iv_lo[o + i], iv_n[o + i], true);
    if (w.leader()) h[slot] = ((uint64_t)HK_S << 62) | ((uint64_t)r << 40) | raw;
    uint64_t by = (uint64_t)s_n[r] * G;
    active += by; active_vmm += by; requested += raw;
    w.sync();
  }

  // --------------------------------------------------------------- BFC
  GML_HD uint32_t& fl_n(uint32_t pool) { return pool ? fl_n1 : fl_n0; }
  GML_HD uint32_t fl_idx(uint32_t pool, uint32_t k) const { return pool ? cap.b - 1 - k : k; }
  GML_HD void fl_push(uint32_t pool, uint32_t r) {
    uint32_t k = fl_n(pool)++;
    if (w.leader()) { fl[fl_idx(pool, k)] = r; b_pos[r] = k; }
  }
  GML_HD void fl_remove(uint32_t pool, uint32_t r) {
    uint32_t k = b_pos[r];
    uint32_t last = fl_n(pool) - 1;
    uint32_t lr = fl[fl_idx(pool, last)];
    w.sync();
    if (w.leader()) { fl[fl_idx(pool, k)] = lr; b_pos[lr] = k; }
    fl_n(pool)--;
    w.sync();
  }
  GML_HD uint32_t b_newrow() {
    uint32_t r;
    if (b_freerow != NONE32) { r = b_freerow; b_freerow = b_next[r]; }
    else if (b_hw < cap.b) r = b_hw++;
    else { overflow |= OV_B; return NONE32; }
    b_live++;
    return r;
  }
  GML_HD void b_delrow(uint32_t r) {
    if (w.leader()) b_next[r] = b_freerow;
    b_freerow = r;
    b_live--;
  }

  // release every fully free segment (PyTorch release_cached_blocks on the
  // OOM path); uniform sequential walk of the free lists.
  GML_HD void bfc_release() {
    for (uint32_t pool = 0; pool < 2; ++pool) {
      uint32_t k = 0;
      while (k < fl_n(pool)) {
        uint32_t r = fl[fl_idx(pool, k)];
        if (b_prev[r] == NONE32 && b_next[r] == NONE32) {
          seg_bytes -= (uint64_t)b_size[r] * 512;
          cnt(st->n_seg_release);
          if (w.leader()) hooks->on_bfc_release(b_seg[r]);
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
    uint32_t bs = NONE32, brow = NONE32;
    uint64_t ba = ~0ull;
    uint32_t nf = fl_n(pool);
    for (uint32_t k = w.lane(); k < nf; k += w.width()) {
      uint32_t row = fl[fl_idx(pool, k)];
      uint32_t s = b_size[row];
      if (s >= ru && s <= bs) {
        uint64_t a = ((uint64_t)b_seg[row] << 32) | b_off[row];
        if (s < bs || a < ba) { bs = s; ba = a; brow = row; }
      }
    }
    uint32_t gs = w.min_u32(bs);
    uint32_t row;
    int state;
    if (gs != NONE32) {
      uint64_t ga = w.min_u64(bs == gs ? ba : ~0ull);
      uint32_t m = w.ballot(bs == gs && ba == ga);
      row = w.bcast(brow, ctz32(m));
      fl_remove(pool, row);
      state = ST_HIT;
    } else {
      uint64_t ss = bfc_segment_size(r, exact);
      if (reserved_vmm() + seg_bytes + ss > capacity) {
        bfc_release();
        if (reserved_vmm() + seg_bytes + ss > capacity) { rec = rec_oom(); cnt(st->state_count[ST_S5 - 1]); return false; }
      }
      row = b_newrow();
      if (row == NONE32) return false;
      uint32_t seg = next_seg++;
      if (w.leader()) {
        b_size[row] = (uint32_t)(ss / 512); b_off[row] = 0; b_seg[row] = seg;
        b_prev[row] = NONE32; b_next[row] = NONE32; b_flags[row] = pool ? BF_POOL1 : 0;
        hooks->on_bfc_segment(seg, ss);
      }
      seg_bytes += ss;
      cnt(st->n_seg_alloc);
      state = ST_NEWSEG;
      w.sync();
    }
    // op 2: split, front allocated, remainder stays in the pool
    uint32_t size = b_size[row];
    uint64_t rem = (uint64_t)(size - ru) * 512;
    bool do_split = (exact || pool == 0) ? rem >= 512 : rem > BFC_SMALL_SIZE;
    if (do_split) {
      uint32_t rest = b_newrow();
      if (rest == NONE32) return false;
      uint32_t nx = b_next[row];
      if (w.leader()) {
        b_size[rest] = size - ru; b_off[rest] = b_off[row] + ru; b_seg[rest] = b_seg[row];
        b_prev[rest] = row; b_next[rest] = nx; b_flags[rest] = b_flags[row] & BF_POOL1;
        if (nx != NONE32) b_prev[nx] = rest;
        b_next[row] = rest; b_size[row] = ru;
      }
      w.sync();
      fl_push(pool, rest);
      w.sync();
    }
    if (w.leader()) {
      b_flags[row] |= BF_ALLOC;
      h[slot] = ((uint64_t)HK_B << 62) | ((uint64_t)row << 40) | raw;
    }
    uint64_t by = (uint64_t)b_size[row] * 512;
    active += by; requested += raw;
    cnt(st->state_count[state - 1]);
    rec = (uint64_t)b_off[row] | ((uint64_t)HK_B << 32) | ((uint64_t)state << 34) | ((uint64_t)b_seg[row] << 40);
    w.sync();
    return true;
  }

  // BFC free + merge (PAPER.md L123-125 ops 3-4)
  GML_HD void bfc_free(uint32_t row) {
    uint32_t pool = (b_flags[row] & BF_POOL1) ? 1 : 0;
    if (w.leader()) b_flags[row] &= ~BF_ALLOC;
    w.sync();
    uint32_t p = b_prev[row];
    if (p != NONE32 && !(b_flags[p] & BF_ALLOC)) {
      fl_remove(pool, p);
      uint32_t nx = b_next[row];
      if (w.leader()) {
        b_size[p] += b_size[row];
        b_next[p] = nx;
        if (nx != NONE32) b_prev[nx] = p;
      }
      w.sync();
      b_delrow(row);
      w.sync();
      row = p;
    }
    uint32_t n = b_next[row];
    if (n != NONE32 && !(b_flags[n] & BF_ALLOC)) {
      fl_remove(pool, n);
      uint32_t nn = b_next[n];
      if (w.leader()) {
        b_size[row] += b_size[n];
        b_next[row] = nn;
        if (nn != NONE32) b_prev[nn] = row;
      }
      w.sync();
      b_delrow(n);
      w.sync();
    }
    fl_push(pool, row);
    w.sync();
  }

  // ------------------------------------------------------------ GMLake
  // next pBlock in pool order (size desc, ordinal asc) strictly after `prev`
  // among eligible inactive ones: key = (n << 32) | ~ord, take the max key
  // below prev.
  GML_HD uint64_t next_in_order(uint64_t prev_key, uint32_t& row) {
    uint64_t best = 0;
    uint32_t brow = NONE32;
    for (uint32_t r = w.lane(); r < n_p; r += w.width()) {
      uint32_t n = p_n[r];
      if (n < elig_n) continue;
      uint64_t key = ((uint64_t)n << 32) | (uint32_t)~p_ord[r];
      if (key < prev_key && key > best && !p_active(r)) { best = key; brow = r; }
    }
    // max via min of complement
    uint64_t g = ~w.min_u64(~best);
    if (g == 0) { row = NONE32; return 0; }
    uint32_t m = w.ballot(best == g && brow != NONE32);
    row = w.bcast(brow, ctz32(m));
    return g;
  }

  // GMLake malloc: Algorithm 1 + S1-S5
  GML_HD bool vmm_malloc(uint32_t slot, uint64_t raw, uint64_t& rec) {
    uint32_t b = (uint32_t)((raw + G - 1) / G);                      // D2
    stitch_free_bytes();                                             // D17(ii)
    // ---- S1: exact match, sPool then pPool (Alg. 1 L2-4; D5) ----
    bool pfirst = flags & GML_F_S1_PBLOCK_FIRST;
    for (int pass = 0; pass < 2; ++pass) {
      bool spool = (pass == 0) != pfirst;
      uint32_t bo = NONE32, brow = NONE32;
      if (spool) {
        for (uint32_t r = w.lane(); r < s_hw; r += w.width())
          if (s_n[r] == b && s_ord[r] < bo && s_inactive1(r)) { bo = s_ord[r]; brow = r; }
      } else {
        for (uint32_t r = w.lane(); r < n_p; r += w.width())
          if (p_n[r] == b && p_ord[r] < bo && !p_active(r)) { bo = p_ord[r]; brow = r; }
      }
      uint32_t g = w.min_u32(bo);
      if (g != NONE32) {
        uint32_t row = w.bcast(brow, ctz32(w.ballot(bo == g)));
        if (spool) {
          bind_s(slot, row, raw);
          T++;
          if (w.leader()) s_last[row] = (uint32_t)T;
          rec = rec_of(g, HK_S, ST_S1);
        } else {
          bind_p(slot, row, raw);
          rec = rec_of(g, HK_P, ST_S1);
        }
        cnt(st->state_count[ST_S1 - 1]);
        w.sync();
        return true;
      }
    }
    bool rr = flags & GML_F_REMAINDER_RULE;
    // ---- Alg. 1 L6-8: single block >= bSize; the replace-loop keeps the
    // smallest, ties -> highest ordinal (D6). Candidates: eligible inactive
    // pBlocks (D8), or all inactive under REMAINDER_RULE.
    {
      uint32_t bn = NONE32, bo = 0, brow = NONE32;
      for (uint32_t r = w.lane(); r < n_p; r += w.width()) {
        uint32_t n = p_n[r];
        if (n > b && (rr || n >= elig_n) && n <= bn) {
          uint32_t o = p_ord[r];
          if ((n < bn || o > bo) && !p_active(r)) { bn = n; bo = o; brow = r; }
        }
      }
      uint32_t gn = w.min_u32(bn);
      if (gn != NONE32) {
        uint32_t go = w.max_u32(bn == gn ? bo + 1 : 0) - 1;
        uint32_t P = w.bcast(brow, ctz32(w.ballot(bn == gn && bo == go)));
        // ---- S2 ----
        if (rr && (uint64_t)(gn - b) * G < limit_bytes) {
          bind_p(slot, P, raw);
          rec = rec_of(go, HK_P, ST_S2);
        } else {
          uint32_t R = split(P, b);
          if (R == NONE32) return false;
          if (!(flags & GML_F_NO_COMPANION)) {
            uint32_t pr[2] = {P, R};
            stitch(pr, 2, true);
            if (overflow) return false;
          }
          bind_p(slot, P, raw);
          rec = rec_of(p_ord[P], HK_P, ST_S2);
        }
        cnt(st->state_count[ST_S2 - 1]);
        w.sync();
        return true;
      }
    }
    // ---- Alg. 1 L9-10: greedy largest-first accumulation (no block >= b) ----
    uint32_t k = 0;
    uint64_t CBsize = 0;
    uint64_t prev = ~0ull;
    while (CBsize < b) {
      uint32_t row;
      uint64_t key = next_in_order(prev, row);
      if (row == NONE32) break;
      if (k + 1 >= cap.cb) { overflow |= OV_CB; return false; }
      if (w.leader()) cb[k] = row;
      k++;
      CBsize += p_n[row];
      prev = key;
    }
    w.sync();
    if (CBsize >= b) {
      // ---- S3: split the last candidate (D14), stitch ----
      if (CBsize > b) {
        uint32_t last = cb[k - 1];
        uint32_t n = (uint32_t)(b - (CBsize - p_n[last]));
        if (!(rr && (uint64_t)(p_n[last] - n) * G < limit_bytes)) {
          uint32_t R = split(last, n);
          if (R == NONE32) return false;
          if (!(flags & GML_F_NO_COMPANION)) {
            uint32_t pr[2] = {last, R};
            stitch(pr, 2, true);
            if (overflow) return false;
          }
        }
      }
      uint32_t s = stitch(cb, k, false);
      if (s == NONE32) return false;
      bind_s(slot, s, raw);
      rec = rec_of(s_ord[s], HK_S, ST_S3);
      cnt(st->state_count[ST_S3 - 1]);
      w.sync();
      return true;
    }
    // ---- S4: Alloc the shortfall (D15) ----
    uint32_t shortfall = (uint32_t)(b - CBsize);
    if (reserved() + (uint64_t)shortfall * G > capacity) {
      rec = rec_oom();                                               // S5 (L528, D16)
      cnt(st->state_count[ST_S5 - 1]);
      return false;
    }
    uint32_t p = alloc(shortfall);
    if (p == NONE32) return false;
    if (k == 0) {
      bind_p(slot, p, raw);
      rec = rec_of(p_ord[p], HK_P, ST_S4);
    } else {
      if (w.leader()) cb[k] = p;
      w.sync();
      uint32_t s = stitch(cb, k + 1, false);
      if (s == NONE32) return false;
      bind_s(slot, s, raw);
      rec = rec_of(s_ord[s], HK_S, ST_S4);
    }
    cnt(st->state_count[ST_S4 - 1]);
    w.sync();
    return true;
  }

  // Update: unbind, no release, no merge (D19).
  GML_HD uint64_t do_free(uint32_t slot) {
    uint64_t hv = h[slot];
    uint32_t hk = (uint32_t)(hv >> 62);
    uint32_t row = (uint32_t)((hv >> 40) & 0x3FFFFF);
    uint64_t raw = hv & MASK40;
    uint64_t by, rec;
    w.sync();
    if (hk == HK_P) {
      by = (uint64_t)p_n[row] * G;
      bm_write(p_lo[row], p_n[row], false);
      rec = rec_of(p_ord[row], HK_P, 0);
      active_vmm -= by;
    } else if (hk == HK_S) {
      by = (uint64_t)s_n[row] * G;
      uint32_t o = s_ivo[row], k = s_ivn[row];
      for (uint32_t i = 0; i < k; ++i) bm_write(iv_lo[o + i], iv_n[o + i], false);
      rec = rec_of(s_ord[row], HK_S, 0);
      active_vmm -= by;
    } else {
      by = (uint64_t)b_size[row] * 512;
      rec = (uint64_t)b_off[row] | ((uint64_t)HK_B << 32) | ((uint64_t)b_seg[row] << 40);
      bfc_free(row);
    }
    active -= by;
    requested -= raw;
    live--;
    w.sync();
    if (w.leader()) h[slot] = (uint64_t)HK_EMPTY << 62;
    w.sync();
    return rec;
  }

  // One event. Returns the assignment record; sets `status` (OOM / INVALID)
  // or `overflow` when the replay must stop.
  GML_HD uint64_t step(uint64_t ev) {
    bool is_free = ev >> 63;
    uint32_t slot = (uint32_t)((ev >> 40) & 0x7FFFFFu);
    uint64_t raw = ev & MASK40;
    if (slot >= cap.h) { overflow |= OV_H; return 0; }
    uint64_t hv = h[slot];
    bool empty = (hv >> 62) == HK_EMPTY;
    uint64_t rec = 0;
    if (is_free) {
      if (empty || raw) { status = GML_ERR_INVALID; return 0; }
      return do_free(slot);
    }
    if (!empty || raw == 0) { status = GML_ERR_INVALID; return 0; }
    serial++;
    bool ok = (kind == GML_POLICY_GMLAKE && raw >= small_thr) ? vmm_malloc(slot, raw, rec)
                                                              : bfc_malloc(slot, raw, rec);
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
    if (w.leader()) {
      st->peak_active_bytes = pk_active;
      st->peak_reserved_bytes = pk_reserved;
      st->peak_requested_bytes = pk_requested;
      st->peak_active_vmm_bytes = pk_active_vmm;
      st->peak_reserved_vmm_bytes = pk_reserved_vmm;
      st->final_active_bytes = active;
      st->final_reserved_bytes = reserved();
      st->n_events = n_events;
      st->n_events_done = n_done;
      st->oom_event = oom_event;
      st->status = status;
      st->_p = overflow;
      st->max_pblocks = mx_p;
      st->max_sblocks = mx_s;
      st->max_live_handles = mx_h;
      st->max_bfc_blocks = mx_b;
    }
    w.sync();
  }
};

}  // namespace gml
