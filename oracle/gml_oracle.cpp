// gml_oracle.cpp -- TEST INFRASTRUCTURE, NOT PRODUCT CODE.
//
// A plain, slow, single-threaded CPU simulator of the GMLake allocation engine
// (arXiv 2401.08156) and of the two BFC baselines, written directly from
// PAPER.md. It is the parity oracle for the CUDA replay kernel. Only tests/,
// __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
// may load it. It shares no code, header, table or constant generator with
// paper_2401_08156_b200/ (the product path), and the product never loads it.
//
// Data structures follow the paper's words: pPool and sPool are *sorted sets*
// "sorted by block size in descending order",
// walked front to back exactly as Algorithm 1 is written.
// Every choice the paper leaves open is fixed by a numbered reading Dn; the
// register is in DESIGN.md ("Readings of the paper") and SURVEY.md §8(c).
//
// Pins (tests/test_oracle_*.py): fig:intro worked example,
// Alg. 1 hand examples, Alg. 1 result properties checked by
// brute force on dumped pools, the no-new-peak theorem as a
// closed form on every V3 trace, invariants of PAPER.md L537-550 after every
// event, BFC tiling / coalescing / best-fit minimality by brute force, Table 1
// call counts, metric identities.
//
// Build: g++ -O2 -std=c++17 -shared -fPIC oracle/gml_oracle.cpp -o oracle/libgml_oracle.so

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <map>
#include <set>
#include <vector>

namespace {

constexpr uint32_t KIND_BFC_TORCH = 0;   // PyTorch 2.x caching allocator (baseline)
constexpr uint32_t KIND_BFC_EXACT = 1;   // BFC with segment = request
constexpr uint32_t KIND_GMLAKE = 2;      // the paper's allocator (§3-§4)

constexpr uint32_t F_S1_PBLOCK_FIRST = 1;     // D5 variant
constexpr uint32_t F_NO_COMPANION = 2;        // D11 variant
constexpr uint32_t F_SPLIT_INVALIDATES = 4;   // D12 variant
constexpr uint32_t F_REMAINDER_RULE = 8;      // D8 variant
constexpr uint32_t F_LIMIT_GATES_REQUEST = 16; // D8' (GMLake default): requests below the limit take the small path

constexpr uint64_t BFC_MIN_BLOCK = 512;                  // D21 (PyTorch kMinBlockSize)
constexpr uint64_t BFC_SMALL_SIZE = 1ull << 20;          // kSmallSize
constexpr uint64_t BFC_SMALL_BUFFER = 2ull << 20;        // kSmallBuffer
constexpr uint64_t BFC_MIN_LARGE_ALLOC = 10ull << 20;    // kMinLargeAlloc
constexpr uint64_t BFC_LARGE_BUFFER = 20ull << 20;       // kLargeBuffer
constexpr uint64_t BFC_ROUND_LARGE = 2ull << 20;         // kRoundLarge

constexpr int ST_S1 = 1, ST_S2 = 2, ST_S3 = 3, ST_S4 = 4, ST_S5 = 5, ST_HIT = 6, ST_NEWSEG = 7;
constexpr uint32_t OK = 0, ERR_OOM = 2;

}  // namespace

extern "C" {

// Field-for-field the same information as gml_policy (include/gml.h), declared
// independently here.
struct gmo_policy {
  uint32_t kind, flags;
  uint64_t capacity_bytes;
  uint64_t chunk_bytes;
  uint64_t small_threshold_bytes;
  uint64_t frag_limit_bytes;
  uint32_t spool_max_entries, _pad;
  uint64_t spool_max_inactive_bytes;
};

struct gmo_stats {
  uint64_t peak_active_bytes, peak_reserved_bytes, peak_requested_bytes;
  uint64_t peak_active_vmm_bytes, peak_reserved_vmm_bytes;
  uint64_t final_active_bytes, final_reserved_bytes;
  uint64_t n_events, n_events_done;
  int64_t oom_event;
  uint32_t status, _p;
  uint64_t state_count[7];
  uint64_t n_split, n_stitch, n_companion, n_alloc, n_evict, n_seg_alloc, n_seg_release;
  uint64_t vmm_calls[7];   // reserve, create, map, set_access, unmap, addr_free, release
  uint32_t max_pblocks, max_sblocks, max_live_handles, max_bfc_blocks;
};

}  // extern "C"

namespace {

enum { V_RESERVE, V_CREATE, V_MAP, V_ACCESS, V_UNMAP, V_ADDR_FREE, V_RELEASE };

// ------------------------------------------------------------------------
// BFC engine: PAPER.md L116-125 ops 1-4 (best fit, split, lazy free, merge).
// Used whole for V0 (torch rules) and V1 (exact rules), and as GMLake's
// small-allocation path ("we use the original PyTorch splitting method",
// PAPER.md L322; reading D3).
// ------------------------------------------------------------------------
struct BBlock {
  uint32_t seg;          // segment ordinal (segments are bump-addressed, D23)
  uint64_t off;          // byte offset inside the segment
  uint64_t size;
  bool allocated;
  int pool;              // 0 small, 1 large (torch rules); 0 only (exact)
  BBlock* prev;          // bidirectional neighbour links
  BBlock* next;
};

// PyTorch orders free blocks by (size, address); address order over bump-
// allocated segments is (segment ordinal, offset) (D21, D22, D23).
struct BCmp {
  bool operator()(const BBlock* a, const BBlock* b) const {
    if (a->size != b->size) return a->size < b->size;
    if (a->seg != b->seg) return a->seg < b->seg;
    return a->off < b->off;
  }
};

struct Segment {
  uint64_t size;
  BBlock* first;
  int pool;
};

struct Bfc {
  bool exact = false;
  std::set<BBlock*, BCmp> free_set[2];
  std::map<uint32_t, Segment> segs;   // ordinal -> segment (ascending address)
  uint64_t seg_bytes = 0;
  uint32_t next_seg = 0;
  uint64_t n_blocks = 0;

  ~Bfc() {
    for (auto& kv : segs) {
      BBlock* b = kv.second.first;
      while (b) { BBlock* n = b->next; delete b; b = n; }
    }
  }

  static uint64_t round_up(uint64_t x, uint64_t m) { return (x + m - 1) / m * m; }

  uint64_t round_size(uint64_t raw) const {
    return raw < BFC_MIN_BLOCK ? BFC_MIN_BLOCK : round_up(raw, BFC_MIN_BLOCK);
  }
  int pool_of(uint64_t r) const { return exact ? 0 : (r <= BFC_SMALL_SIZE ? 0 : 1); }
  uint64_t segment_size(uint64_t r) const {
    if (exact) return r;
    if (r <= BFC_SMALL_SIZE) return BFC_SMALL_BUFFER;
    if (r < BFC_MIN_LARGE_ALLOC) return BFC_LARGE_BUFFER;
    return round_up(r, BFC_ROUND_LARGE);
  }
  bool should_split(const BBlock* b, uint64_t r) const {
    uint64_t rem = b->size - r;
    if (exact || b->pool == 0) return rem >= BFC_MIN_BLOCK;
    return rem > BFC_SMALL_SIZE;
  }

  // Release every fully free segment (one block, not allocated), ascending
  // address order -- PyTorch's release_cached_blocks() on the OOM path.
  void release_free_segments(gmo_stats& st) {
    for (auto it = segs.begin(); it != segs.end();) {
      BBlock* b = it->second.first;
      if (!b->allocated && b->prev == nullptr && b->next == nullptr) {
        free_set[b->pool].erase(b);
        seg_bytes -= it->second.size;
        st.n_seg_release++;
        delete b;
        n_blocks--;
        it = segs.erase(it);
      } else {
        ++it;
      }
    }
  }

  // Returns the allocated block, or nullptr on OOM. other_reserved is the
  // memory held outside this engine (GMLake's pBlocks) against capacity.
  BBlock* malloc(uint64_t raw, uint64_t other_reserved, uint64_t capacity, int* state,
                 gmo_stats& st) {
    uint64_t r = round_size(raw);
    int pool = pool_of(r);
    // op 1: best fit = first free block in (size, address) order with size >= r
    BBlock* best = nullptr;
    for (BBlock* b : free_set[pool]) {
      if (b->size >= r) { best = b; break; }
    }
    if (best) {
      *state = ST_HIT;
      free_set[pool].erase(best);
    } else {
      // no fit: native allocation of a new segment
      uint64_t ss = segment_size(r);
      if (other_reserved + seg_bytes + ss > capacity) {
        release_free_segments(st);
        if (other_reserved + seg_bytes + ss > capacity) return nullptr;
      }
      uint32_t ord = next_seg++;
      best = new BBlock{ord, 0, ss, false, pool, nullptr, nullptr};
      n_blocks++;
      segs[ord] = Segment{ss, best, pool};
      seg_bytes += ss;
      st.n_seg_alloc++;
      *state = ST_NEWSEG;
    }
    // op 2: split; the front part is allocated, the remainder stays in the pool
    if (should_split(best, r)) {
      BBlock* rest = new BBlock{best->seg, best->off + r, best->size - r, false, pool, best, best->next};
      n_blocks++;
      if (best->next) best->next->prev = rest;
      best->next = rest;
      best->size = r;
      free_set[pool].insert(rest);
    }
    best->allocated = true;
    return best;
  }

  // op 3 + op 4: mark inactive, merge with inactive left / right neighbours.
  void free(BBlock* b) {
    b->allocated = false;
    BBlock* p = b->prev;
    if (p && !p->allocated) {
      free_set[p->pool].erase(p);
      p->size += b->size;
      p->next = b->next;
      if (b->next) b->next->prev = p;
      delete b;
      n_blocks--;
      b = p;
    }
    BBlock* n = b->next;
    if (n && !n->allocated) {
      free_set[n->pool].erase(n);
      b->size += n->size;
      b->next = n->next;
      if (n->next) n->next->prev = b;
      delete n;
      n_blocks--;
    }
    free_set[b->pool].insert(b);
  }
};

// ------------------------------------------------------------------------
// GMLake pools (§3.2)
// ------------------------------------------------------------------------
constexpr int64_t NONE = -1;

struct PBlock {              // primitive block: a VA over its own chunks
  uint32_t ord;              // creation ordinal (D4 tie-break)
  uint32_t lo, n;            // chunk ids [lo, lo+n) (D-a: chunk = 2 MiB granule)
  int64_t owner;             // handle slot bound to it, NONE when inactive (D18)
};

struct SBlock {              // stitched block
  uint32_t ord;
  std::vector<std::pair<uint32_t, uint32_t>> iv;   // chunk intervals it maps, in member order (D13)
  uint32_t size;             // granules = sum of the members
  uint64_t last_use;         // LRU key (D17)
  uint64_t born;             // malloc serial number that created it
};

struct PCmp {                // "sorted by block size in descending order"
  bool operator()(const PBlock* a, const PBlock* b) const {
    if (a->n != b->n) return a->n > b->n;
    return a->ord < b->ord;
  }
};
struct SCmp {
  bool operator()(const SBlock* a, const SBlock* b) const {
    if (a->size != b->size) return a->size > b->size;
    return a->ord < b->ord;
  }
};

enum HKind { H_P = 0, H_S = 1, H_B = 2 };
struct Handle {
  bool live = false;
  int kind = 0;
  PBlock* p = nullptr;
  SBlock* s = nullptr;
  BBlock* b = nullptr;
  uint64_t raw = 0;
  uint64_t bytes = 0;
};

struct Sim {
  gmo_policy pol;
  gmo_stats st;
  // GMLake state
  std::set<PBlock*, PCmp> pPool;
  std::set<SBlock*, SCmp> sPool;
  std::map<uint32_t, PBlock*> p_by_lo;     // address index of pPool, to find overlaps
  uint32_t C = 0;                          // chunks created so far (Alloc is the only growth)
  uint32_t next_p = 0, next_s = 0;
  uint64_t T = 0;                          // touch counter (LRU clock)
  uint64_t malloc_serial = 0;
  Bfc bfc;
  std::vector<Handle> h;
  uint64_t live_handles = 0;
  uint64_t active = 0, requested = 0, active_vmm = 0;
  uint64_t ev_index = 0;
  bool dead = false;

  explicit Sim(const gmo_policy& p) : pol(p) {
    std::memset(&st, 0, sizeof(st));
    st.oom_event = -1;
    bfc.exact = (pol.kind == KIND_BFC_EXACT);
  }
  ~Sim() {
    for (PBlock* p : pPool) delete p;
    for (SBlock* s : sPool) delete s;
  }

  uint64_t G() const { return pol.chunk_bytes; }
  uint64_t reserved_vmm() const { return (uint64_t)C * G(); }
  uint64_t reserved() const { return reserved_vmm() + bfc.seg_bytes; }
  bool eligible(const PBlock* p) const { return (uint64_t)p->n * G() >= pol.frag_limit_bytes; }

  // --- activity (D18): "if even one pBlock is active, all corresponding
  // sBlocks are labeled as active".
  template <class F>
  void for_overlapping(uint32_t lo, uint32_t n, F fn) {
    auto it = p_by_lo.upper_bound(lo);
    if (it != p_by_lo.begin()) --it;
    for (; it != p_by_lo.end() && it->first < lo + n; ++it) {
      PBlock* p = it->second;
      if (p->lo + p->n > lo) fn(p);
    }
  }
  bool s_inactive(SBlock* s) {
    bool act = false;
    for (auto& iv : s->iv) for_overlapping(iv.first, iv.second, [&](PBlock* p) { if (p->owner != NONE) act = true; });
    return !act;
  }
  bool s_overlaps(SBlock* s, uint32_t lo, uint32_t n) {
    for (auto& iv : s->iv)
      if (iv.first < lo + n && lo < iv.first + iv.second) return true;
    return false;
  }

  void insert_p(PBlock* p) { pPool.insert(p); p_by_lo[p->lo] = p; }
  void erase_p(PBlock* p) { pPool.erase(p); p_by_lo.erase(p->lo); }

  void evict(SBlock* s) {   // StitchFree of one sBlock
    sPool.erase(s);
    delete s;
    st.n_evict++;
    st.vmm_calls[V_UNMAP] += 1;
    st.vmm_calls[V_ADDR_FREE] += 1;
  }

  // LRU victim: the inactive sBlock with the minimum last_use, not created
  // during the current malloc (D17).
  SBlock* lru_victim() {
    SBlock* v = nullptr;
    for (SBlock* s : sPool) {
      if (s->born == malloc_serial) continue;
      if (!s_inactive(s)) continue;
      if (!v || s->last_use < v->last_use) v = s;
    }
    return v;
  }

  // D17(ii): at VMM-path malloc entry, while the inactive sBlocks hold more
  // than spool_max_inactive_bytes, release the LRU one ("StitchFree",
  // PAPER.md L563-567).
  void stitch_free_bytes() {
    uint64_t all = 0;
    for (SBlock* s : sPool) all += (uint64_t)s->size * G();
    if (all <= pol.spool_max_inactive_bytes) return;   // inactive <= all: nothing to do
    uint64_t inact = 0;
    for (SBlock* s : sPool) if (s_inactive(s)) inact += (uint64_t)s->size * G();
    while (inact > pol.spool_max_inactive_bytes) {
      SBlock* v = nullptr;
      for (SBlock* s : sPool)
        if (s_inactive(s) && (!v || s->last_use < v->last_use)) v = s;
      inact -= (uint64_t)v->size * G();
      evict(v);
    }
  }

  // Split: P -> F (first n chunks) + R (the rest); two new
  // pBlocks with new VAs over P's remapped chunks; P leaves the pPool (D10).
  std::pair<PBlock*, PBlock*> split(PBlock* P, uint32_t n) {
    PBlock* F = new PBlock{next_p++, P->lo, n, NONE};
    PBlock* R = new PBlock{next_p++, P->lo + n, P->n - n, NONE};
    uint32_t plo = P->lo, pn = P->n;
    erase_p(P);
    delete P;
    insert_p(F);
    insert_p(R);
    st.n_split++;
    st.vmm_calls[V_RESERVE] += 2;
    st.vmm_calls[V_MAP] += pn;
    st.vmm_calls[V_ACCESS] += pn;
    st.vmm_calls[V_UNMAP] += 1;
    st.vmm_calls[V_ADDR_FREE] += 1;
    if (pol.flags & F_SPLIT_INVALIDATES) {   // D12 variant
      std::vector<SBlock*> dead_s;
      for (SBlock* s : sPool) if (s_overlaps(s, plo, pn)) dead_s.push_back(s);
      for (SBlock* s : dead_s) evict(s);
    }
    return {F, R};
  }

  // Stitch: a new sBlock over the members' chunks; no new
  // physical memory. Count cap enforced at insertion (D17(i)); a companion
  // that finds no room is skipped, an allocation stitch is created anyway.
  SBlock* stitch(const std::vector<PBlock*>& L, bool companion) {
    while (sPool.size() >= pol.spool_max_entries) {
      SBlock* v = lru_victim();
      if (!v) break;
      evict(v);
    }
    if (companion && sPool.size() >= pol.spool_max_entries) return nullptr;
    SBlock* s = new SBlock{next_s++, {}, 0, ++T, malloc_serial};
    uint64_t chunks = 0;
    for (PBlock* m : L) {
      s->iv.push_back({m->lo, m->n});
      s->size += m->n;
      chunks += m->n;
    }
    sPool.insert(s);
    st.n_stitch++;
    if (companion) st.n_companion++;
    st.vmm_calls[V_RESERVE] += 1;
    st.vmm_calls[V_MAP] += chunks;
    st.vmm_calls[V_ACCESS] += chunks;
    return s;
  }

  // Alloc: the only way to create physical chunks.
  PBlock* alloc(uint32_t n) {
    PBlock* p = new PBlock{next_p++, C, n, NONE};
    C += n;
    insert_p(p);
    st.n_alloc++;
    st.vmm_calls[V_RESERVE] += 1;
    st.vmm_calls[V_CREATE] += n;
    st.vmm_calls[V_MAP] += n;
    st.vmm_calls[V_ACCESS] += n;
    return p;
  }

  void bind_p(uint32_t slot, PBlock* p, uint64_t raw) {
    p->owner = slot;
    Handle& x = h[slot];
    x = Handle{true, H_P, p, nullptr, nullptr, raw, (uint64_t)p->n * G()};
    active += x.bytes; active_vmm += x.bytes; requested += raw;
  }
  void bind_s(uint32_t slot, SBlock* s, uint64_t raw) {
    for (auto& iv : s->iv) for_overlapping(iv.first, iv.second, [&](PBlock* p) { p->owner = slot; });
    Handle& x = h[slot];
    x = Handle{true, H_S, nullptr, s, nullptr, raw, (uint64_t)s->size * G()};
    active += x.bytes; active_vmm += x.bytes; requested += raw;
  }

  static uint64_t rec(uint32_t ord, int kind, int state) {
    return (uint64_t)ord | ((uint64_t)kind << 32) | ((uint64_t)state << 34);
  }
  static uint64_t rec_b(const BBlock* b, int state) {
    return (b->off / 512) | ((uint64_t)H_B << 32) | ((uint64_t)state << 34) | ((uint64_t)b->seg << 40);
  }
  static uint64_t rec_oom() { return 0xFFFFFFFFull | ((uint64_t)ST_S5 << 34); }

  // BFC malloc for V0/V1 and for GMLake's small path.
  bool malloc_bfc(uint32_t slot, uint64_t raw, uint64_t* out) {
    int state = 0;
    BBlock* b = bfc.malloc(raw, reserved_vmm(), pol.capacity_bytes, &state, st);
    if (!b) { *out = rec_oom(); st.state_count[ST_S5 - 1]++; return false; }
    h[slot] = Handle{true, H_B, nullptr, nullptr, b, raw, b->size};
    active += b->size; requested += raw;
    st.state_count[state - 1]++;
    *out = rec_b(b, state);
    return true;
  }

  // GMLake malloc: BestFit (Algorithm 1) + the S1-S5 strategy (§4.1).
  bool malloc_gmlake(uint32_t slot, uint64_t raw, uint64_t* out) {
    if (raw < pol.small_threshold_bytes) return malloc_bfc(slot, raw, out);   // D1, D3
    // D8': "If a block is smaller than this limit, GMLake will avoid stitching
    // or splitting it" read for the REQUEST: a tensor below
    // the fragmentation limit is served by "the original PyTorch splitting
    // method", as L322 does for tensors below 2 MB.
    if ((pol.flags & F_LIMIT_GATES_REQUEST) && raw < pol.frag_limit_bytes) return malloc_bfc(slot, raw, out);
    uint32_t b = (uint32_t)((raw + G() - 1) / G());                               // D2
    stitch_free_bytes();
    // ---- Alg. 1 lines 2-4 (S1, exact match; the only use of sBlocks) ----
    bool pfirst = pol.flags & F_S1_PBLOCK_FIRST;
    for (int pass = 0; pass < 2; ++pass) {
      bool spool = (pass == 0) != pfirst;
      if (spool) {
        for (SBlock* s : sPool) {
          if (s->size == b && s_inactive(s)) {
            bind_s(slot, s, raw);
            s->last_use = ++T;
            st.state_count[ST_S1 - 1]++;
            *out = rec(s->ord, H_S, ST_S1);
            return true;
          }
        }
      } else {
        for (PBlock* p : pPool) {
          if (p->n == b && p->owner == NONE) {
            bind_p(slot, p, raw);
            st.state_count[ST_S1 - 1]++;
            *out = rec(p->ord, H_P, ST_S1);
            return true;
          }
        }
      }
    }
    // ---- Alg. 1 lines 5-11 over inactive pBlocks, fragmentation limit (D8) ----
    bool rr = pol.flags & F_REMAINDER_RULE;
    std::vector<PBlock*> CB;
    uint64_t CBsize = 0;
    for (PBlock* p : pPool) {
      if (p->owner != NONE) continue;
      if (!rr && !eligible(p)) continue;
      if (p->n >= b) {
        CB.assign(1, p);
        CBsize = p->n;
      } else if (CBsize < b) {
        if (rr && !eligible(p)) continue;   // REMAINDER_RULE: limit filters accumulation only
        CB.push_back(p);
        CBsize += p->n;
      } else {
        break;
      }
    }
    if (CB.size() == 1 && CBsize > b) {
      // ---- S2: split, companion stitch, assign the front ----
      PBlock* P = CB[0];
      if (rr && (uint64_t)(P->n - b) * G() < pol.frag_limit_bytes) {
        bind_p(slot, P, raw);
        st.state_count[ST_S2 - 1]++;
        *out = rec(P->ord, H_P, ST_S2);
        return true;
      }
      auto fr = split(P, b);
      if (!(pol.flags & F_NO_COMPANION)) stitch({fr.first, fr.second}, true);
      bind_p(slot, fr.first, raw);
      st.state_count[ST_S2 - 1]++;
      *out = rec(fr.first->ord, H_P, ST_S2);
      return true;
    }
    if (CBsize >= b) {
      // ---- S3: split the last candidate if needed, stitch ----
      if (CBsize > b) {
        PBlock* last = CB.back();
        uint32_t n = (uint32_t)(b - (CBsize - last->n));                          // D14
        if (!(rr && (uint64_t)(last->n - n) * G() < pol.frag_limit_bytes)) {
          auto fr = split(last, n);
          if (!(pol.flags & F_NO_COMPANION)) stitch({fr.first, fr.second}, true);
          CB.back() = fr.first;
        }
      }
      SBlock* s = stitch(CB, false);
      bind_s(slot, s, raw);
      st.state_count[ST_S3 - 1]++;
      *out = rec(s->ord, H_S, ST_S3);
      return true;
    }
    // ---- S4: Alloc the shortfall, stitch with the candidates ----
    uint32_t shortfall = (uint32_t)(b - CBsize);                                     // D15
    if (reserved() + (uint64_t)shortfall * G() > pol.capacity_bytes) {
      // D16: before Alloc is reported failed, the small path returns its fully
      // free cached segments (PyTorch's release of cached blocks on a failed
      // device allocation; SPEC.md "OOM last resort order" (2)-(3)); sBlocks
      // hold no physical memory, so no StitchFree here
      bfc.release_free_segments(st);
    }
    if (reserved() + (uint64_t)shortfall * G() > pol.capacity_bytes) {
      // ---- S5: "If the Alloc function call fails, GMLake
      // immediately reports an Out-of-Memory (OOM) error" (D16) ----
      st.state_count[ST_S5 - 1]++;
      *out = rec_oom();
      return false;
    }
    PBlock* p = alloc(shortfall);
    if (CB.empty()) {
      bind_p(slot, p, raw);
      st.state_count[ST_S4 - 1]++;
      *out = rec(p->ord, H_P, ST_S4);
      return true;
    }
    CB.push_back(p);
    SBlock* s = stitch(CB, false);
    bind_s(slot, s, raw);
    st.state_count[ST_S4 - 1]++;
    *out = rec(s->ord, H_S, ST_S4);
    return true;
  }

  // Free: Update on the VMM path -- unbind, no physical
  // release, no merge (D19); BFC free + merge on the small path / baselines.
  void do_free(uint32_t slot, uint64_t* out) {
    Handle& x = h[slot];
    if (x.kind == H_P) {
      x.p->owner = NONE;
      *out = rec(x.p->ord, H_P, 0);
      active_vmm -= x.bytes;
    } else if (x.kind == H_S) {
      for (auto& iv : x.s->iv) for_overlapping(iv.first, iv.second, [&](PBlock* p) { p->owner = NONE; });
      *out = rec(x.s->ord, H_S, 0);
      active_vmm -= x.bytes;
    } else {
      *out = rec_b(x.b, 0);
      bfc.free(x.b);
    }
    active -= x.bytes;
    requested -= x.raw;
    x = Handle{};
    live_handles--;
  }

  void sample() {
    st.peak_active_bytes = std::max(st.peak_active_bytes, active);
    st.peak_reserved_bytes = std::max(st.peak_reserved_bytes, reserved());
    st.peak_requested_bytes = std::max(st.peak_requested_bytes, requested);
    st.peak_active_vmm_bytes = std::max(st.peak_active_vmm_bytes, active_vmm);
    st.peak_reserved_vmm_bytes = std::max(st.peak_reserved_vmm_bytes, reserved_vmm());
    st.max_pblocks = std::max<uint32_t>(st.max_pblocks, (uint32_t)pPool.size());
    st.max_sblocks = std::max<uint32_t>(st.max_sblocks, (uint32_t)sPool.size());
    st.max_live_handles = std::max<uint32_t>(st.max_live_handles, (uint32_t)live_handles);
    st.max_bfc_blocks = std::max<uint32_t>(st.max_bfc_blocks, (uint32_t)bfc.n_blocks);
  }

  // One event; returns false once the trace has terminated (OOM).
  bool step(uint64_t ev, uint64_t* out) {
    *out = 0;
    if (dead) return false;
    bool is_free = ev >> 63;
    uint32_t slot = (uint32_t)((ev >> 40) & ((1u << 23) - 1));
    uint64_t raw = ev & ((1ull << 40) - 1);
    if (slot >= h.size()) h.resize(slot + 1);
    bool ok = true;
    if (is_free) {
      do_free(slot, out);
    } else {
      malloc_serial++;
      ok = pol.kind == KIND_GMLAKE ? malloc_gmlake(slot, raw, out) : malloc_bfc(slot, raw, out);
      if (ok) live_handles++;
    }
    if (!ok) {
      dead = true;
      st.status = ERR_OOM;
      st.oom_event = (int64_t)ev_index;
      st.n_events_done = ev_index;
      finalize();
      return false;
    }
    ev_index++;
    st.n_events_done = ev_index;
    sample();
    return true;
  }

  void finalize() {
    st.final_active_bytes = active;
    st.final_reserved_bytes = reserved();
  }
};

}  // namespace

extern "C" {

void* gmo_create(const gmo_policy* p) { return new Sim(*p); }
void gmo_destroy(void* s) { delete static_cast<Sim*>(s); }

// Process one event; *asg receives its assignment record. Returns 0, or the
// trace status once it has terminated.
uint32_t gmo_step(void* sp, uint64_t ev, uint64_t* asg) {
  Sim* s = static_cast<Sim*>(sp);
  s->step(ev, asg);
  s->finalize();
  return s->st.status;
}

void gmo_get_stats(void* sp, gmo_stats* out) {
  Sim* s = static_cast<Sim*>(sp);
  *out = s->st;
}

// Snapshot accessors for invariant tests (state dumps, not product outputs).
// pBlocks in pool order: (ord, lo, n, owner) as 4 x int64 per entry.
uint64_t gmo_dump_pblocks(void* sp, int64_t* out, uint64_t cap) {
  Sim* s = static_cast<Sim*>(sp);
  uint64_t i = 0;
  for (PBlock* p : s->pPool) {
    if (i < cap) { out[4 * i] = p->ord; out[4 * i + 1] = p->lo; out[4 * i + 2] = p->n; out[4 * i + 3] = p->owner; }
    i++;
  }
  return i;
}
// sBlocks in pool order: header (ord, size, last_use, n_iv) then n_iv pairs.
uint64_t gmo_dump_sblocks(void* sp, int64_t* out, uint64_t cap) {
  Sim* s = static_cast<Sim*>(sp);
  uint64_t k = 0;
  auto put = [&](int64_t v) { if (k < cap) out[k] = v; k++; };
  for (SBlock* b : s->sPool) {
    put(b->ord); put(b->size); put((int64_t)b->last_use); put((int64_t)b->iv.size());
    for (auto& iv : b->iv) { put(iv.first); put(iv.second); }
  }
  return k;
}
// BFC blocks by segment, address order: (seg, off, size, allocated, pool).
uint64_t gmo_dump_bfc(void* sp, int64_t* out, uint64_t cap) {
  Sim* s = static_cast<Sim*>(sp);
  uint64_t i = 0;
  for (auto& kv : s->bfc.segs) {
    for (BBlock* b = kv.second.first; b; b = b->next) {
      if (i < cap) {
        out[5 * i] = b->seg; out[5 * i + 1] = (int64_t)b->off; out[5 * i + 2] = (int64_t)b->size;
        out[5 * i + 3] = b->allocated; out[5 * i + 4] = b->pool;
      }
      i++;
    }
  }
  return i;
}
// Live handles: (slot, kind, ord-or-seg, bytes, raw) as 5 x int64.
uint64_t gmo_dump_handles(void* sp, int64_t* out, uint64_t cap) {
  Sim* s = static_cast<Sim*>(sp);
  uint64_t i = 0;
  for (size_t slot = 0; slot < s->h.size(); ++slot) {
    const Handle& x = s->h[slot];
    if (!x.live) continue;
    if (i < cap) {
      out[5 * i] = (int64_t)slot; out[5 * i + 1] = x.kind;
      out[5 * i + 2] = x.kind == H_P ? x.p->ord : x.kind == H_S ? x.s->ord : x.b->seg;
      out[5 * i + 3] = (int64_t)x.bytes; out[5 * i + 4] = (int64_t)x.raw;
    }
    i++;
  }
  return i;
}
// Scalars: active, requested, reserved, active_vmm, reserved_vmm, C, T.
void gmo_counters(void* sp, uint64_t* out) {
  Sim* s = static_cast<Sim*>(sp);
  out[0] = s->active; out[1] = s->requested; out[2] = s->reserved();
  out[3] = s->active_vmm; out[4] = s->reserved_vmm(); out[5] = s->C; out[6] = s->T;
}

// Whole-trace replay. asg (n entries) and timeline (4 x n: active, reserved,
// active_vmm, reserved_vmm after each event) are optional.
uint32_t gmo_replay(const uint64_t* ev, uint64_t n, const gmo_policy* pol, uint64_t* asg,
                    gmo_stats* out, uint64_t* timeline) {
  Sim s(*pol);
  s.st.n_events = n;
  for (uint64_t i = 0; i < n; ++i) {
    uint64_t a = 0;
    bool ok = s.step(ev[i], &a);
    if (asg) asg[i] = a;
    if (timeline) {
      timeline[4 * i] = s.active; timeline[4 * i + 1] = s.reserved();
      timeline[4 * i + 2] = s.active_vmm; timeline[4 * i + 3] = s.reserved_vmm();
    }
    if (!ok) {
      for (uint64_t j = i + 1; j < n; ++j) {
        if (asg) asg[j] = 0;
        if (timeline) for (int k = 0; k < 4; ++k) timeline[4 * j + k] = 0;
      }
      break;
    }
  }
  s.finalize();
  s.st.n_events = n;
  *out = s.st;
  return s.st.status;
}

uint64_t gmo_sizeof_stats() { return sizeof(gmo_stats); }
uint64_t gmo_sizeof_policy() { return sizeof(gmo_policy); }

}  // extern "C"
