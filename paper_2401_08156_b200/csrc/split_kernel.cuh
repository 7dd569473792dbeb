// split_kernel.cuh -- K1s: one GMLake (trace, policy) unit replayed by THREE
// warps of one CTA ("split unit", latency placement only).
//
// A GMLake unit has two allocators that share nothing but the capacity:
// requests >= vm_thr take the VMM path (Algorithm 1, S1-S5: pPool, sPool,
// chunk bitmap), smaller ones the BFC small path (D8' adds the
// fragmentation limit to the gate, L571). Each path is a serial dependence
// chain, so one warp per path halves nothing but removes the other path's
// events from the critical chain:
//
//   warp 0  Engine<Cfg<P,S,IV,4>>   -- the unit's VMM-path events, in order
//   warp 1  Engine<Cfg<4,4,4,B>>    -- the unit's small-path events, in order
//   warp 2  ledger                  -- checks the trace (every free names a
//           live slot, no malloc of a live slot), the requested-bytes and
//           live-handle peaks, then merges the two paths' active-bytes series
//           in event order (peak_active_bytes = max over events of the SUM).
//
// A malloc belongs to the VMM path iff raw >= vm_thr (the engine's own test,
// policy.cuh step); a free belongs to the path of its malloc: the engine
// finds that malloc inside the current 32-event window (match.any on the
// slot) or, for a malloc in an earlier window, in its own handle table.
//
// Exactness. The two paths interact only through the capacity checks (S4/S5
// `reserved + shortfall > capacity`, the BFC new-segment check) and through
// BFC segment releases, which happen only when such a check fails (D16,
// D21). Each warp checks its own reserved bytes only; with no failed check
// in either warp (no OOM, no release) reserved is monotone in each path, so
// if final_reserved(VMM) + final_reserved(small) <= capacity then every check
// of the interleaved replay passes too (the sum at any event is <= the final
// sum) and the decisions are identical. Any other outcome -- an OOM or
// release in either warp, the final sum over capacity, an invalid trace, a
// table overflow -- makes the host re-run the unit (serial single-warp K1 for
// the first kinds, the next size class for an overflow), so results never
// depend on the split.
#pragma once
#include "replay_kernel.cuh"

namespace gml {
namespace replay {

enum : uint32_t { OV_SERIAL = 0x100 };   // Ovf mask: re-run this unit with the single-warp K1
#ifndef GML_PATH_MINB
#define GML_PATH_MINB 3    // resident CTAs per SM of the VMM path units (168 registers, some spills: C4 -4 % vs 2)
#endif
#ifndef GML_LEDGER_NS
#define GML_LEDGER_NS 1000                 // the ledger's poll interval (ns) while a path is behind
#endif
#ifndef GML_PATH_WPC
#define GML_PATH_WPC GML_GLOBAL_WPC        // warps (units) per CTA of the path launches
#endif
#ifndef GML_PATH_PERSIST
#define GML_PATH_PERSIST 1                 // path units: persistent warps, one arena each, work counter
#endif
#ifndef GML_PATH_PIN_SMEM
#define GML_PATH_PIN_SMEM 1                // VMM path units: PIN words in shared memory
#endif
#ifndef GML_PATH_BM_SMEM
#define GML_PATH_BM_SMEM 0                 // ... and the chunk bitmap (measured: C4 167-175 vs 155 ms, the smaller L1 hurts)
#endif
#ifndef GML_PATH_FUSE
#define GML_PATH_FUSE 0                    // path units: S1 binds from the proof's lanes (Engine kFuse)
#endif
#ifndef GML_PATH_FREE_RUN
#define GML_PATH_FREE_RUN 0                // path units (global arenas): frees one by one
#endif
constexpr uint32_t kPub = 8;             // windows between a path's progress publications

// placement of the two arenas: both in shared memory, or one of them in the
// unit's global-memory workspace (L1/L2-resident)
enum SplitPlace : int { SP_BOTH = 0, SP_VMM_SMEM = 1, SP_BFC_SMEM = 2 };

template <class CF>
struct SplitCfg {
  using V = Cfg<CF::P, CF::S, CF::IV, 4>;   // VMM path: no BFC rows
  using S = Cfg<4, 4, 4, CF::B>;            // small path: VMM = false, no bitmap
  GML_HD static uint64_t a16(uint64_t x) { return (x + 15) & ~15ull; }
  GML_HD static uint64_t v_bytes(uint32_t bmw, uint32_t h) { return a16(Lay<V>::bytes(bmw, h)); }
  GML_HD static uint64_t s_bytes(uint32_t h) { return a16(Lay<S>::bytes(0, h)); }
  // slot bits + the CTA's sync words {abort, windows done by the VMM path, by the small path, -}
  GML_HD static uint64_t lv_bytes(uint32_t h) { return a16(4ull * ((h + 31) / 32) + 16); }
  // shared-memory bytes of the CTA, global bytes of the unit (arena part +
  // per-slot raw sizes + per-event active series)
  GML_HD static uint64_t smem(int place, uint32_t bmw, uint32_t h) {
    return (place == SP_BFC_SMEM ? 0 : v_bytes(bmw, h)) + (place == SP_VMM_SMEM ? 0 : s_bytes(h)) + lv_bytes(h);
  }
  GML_HD static uint64_t gpart(int place, uint32_t bmw, uint32_t h) {
    return place == SP_VMM_SMEM ? s_bytes(h) : place == SP_BFC_SMEM ? v_bytes(bmw, h) : 0;
  }
  GML_HD static uint64_t glob(int place, uint32_t bmw, uint32_t h, uint64_t n) {
    return gpart(place, bmw, h) + a16(8ull * h) + a16(4ull * n);
  }
};

// One path's warp: replays the events of its path in trace order. Records
// go to the unit's assignment row (coalesced per window, own lanes only);
// the path's active bytes after each of its events go to D (512-byte units,
// bit 31 = VMM path), for the ledger's merge.
template <bool kV, bool kSync, bool kRuns, class Eng>
__device__ __forceinline__ void split_path(Eng& E, const uint64_t* ev, uint64_t n, uint64_t* asg, uint32_t* D,
                                           volatile uint32_t* sy) {
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t lt = (1u << lane) - 1u;
  const uint64_t thr = E.vm_thr;
  const uint32_t tag = kV ? 0x80000000u : 0u;
  uint64_t cur = lane < n ? ld_event(ev + lane) : 0;
  bool stop = false;
  for (uint64_t base = 0; base < n && !stop; base += 32) {
    const uint64_t nb = base + 32 + lane;
    const uint64_t nxt = nb < n ? ld_event(ev + nb) : 0;
    const uint32_t cnt = (n - base) < 32 ? (uint32_t)(n - base) : 32u;
    const bool act = lane < cnt;
    const bool fr = cur >> 63;
    const uint32_t slot = (uint32_t)((cur >> 40) & 0x7FFFFFu);
    const bool big = !fr && (cur & MASK40) >= thr;
    const uint32_t m_slot = __match_any_sync(0xFFFFFFFFu, act ? slot : (0x80000000u | lane));
    const uint32_t pm = m_slot & lt;
    const uint32_t prev = pm ? 31u - __clz(pm) : lane;
    const bool pbig = __shfl_sync(0xFFFFFFFFu, (uint32_t)big, prev) != 0;
    bool mine;
    if (fr) mine = pm ? (pbig == kV) : ((E.H[slot] >> 62) != HK_EMPTY);
    else mine = big == kV;
    mine = mine && act;
    uint32_t m = __ballot_sync(0xFFFFFFFFu, mine);
    uint64_t myrec = 0;
    uint32_t myd = 0;
    // the VMM path unbinds runs of >= 2 consecutive own frees at once
    // (Engine::free_run); the small path's merges stay event by event
    const uint32_t mall = (kV && kRuns) ? __ballot_sync(0xFFFFFFFFu, act && !fr) : 0u;
    uint32_t skip = 0;
    while (m) {
      const uint32_t j = __ffs(m) - 1;
      if constexpr (kV && kRuns) {
        const uint32_t run = Eng::free_run_mask(m, mall) & ~skip;
        if (GML_FREE_RUN && (run & (run - 1))) {
          uint64_t r = 0;
          if (E.free_run(run, cur, r)) {
            // every event of the run records the active bytes after the
            // whole run: lower than after its own event, but the run stops
            // at the next malloc of EITHER path, so the merged sum is exact
            // at every malloc, and a free never sets the merged peak
            if ((run >> lane) & 1u) { myrec = r; myd = (uint32_t)(E.active >> 9) | tag; }
            m &= ~run;
            continue;
          }
          skip |= run;
        }
      }
      m &= m - 1;
      const uint64_t e = __shfl_sync(0xFFFFFFFFu, cur, j);
      const uint64_t r = E.step(e);
      if (lane == j) { myrec = r; myd = (uint32_t)(E.active >> 9) | tag; }
      if (E.overflow | E.status) { stop = true; break; }
    }
    if (mine) {
      if (asg) __stcs(asg + base + lane, myrec);
      D[base + lane] = myd;
    }
    cur = nxt;
    // every kPub windows (and at the end) publish the windows done to the
    // ledger, their D entries first (fence, then the progress word; every
    // window or every 8: no measurable difference on C2), and stop early if
    // another warp found a reason to re-run the unit
    const uint32_t wd = (uint32_t)(base >> 5) + 1u;
    if (kSync && ((wd & (kPub - 1)) == 0 || base + 32 >= n)) {
      __threadfence_block();
      __syncwarp();
      uint32_t ab = 0;
      if (lane == 0) {
        sy[kV ? 1 : 2] = wd;
        ab = sy[0];
      }
      if (__shfl_sync(0xFFFFFFFFu, ab, 0)) stop = true;
    }
  }
  if (kSync && stop && lane == 0) sy[0] = 1u;
}

struct Ledger {
  uint64_t pk_requested, pk_active, pk_active_vmm;
  uint32_t mx_live;
  bool valid, merged;
};

// Warp 2. Per 32-event window: (1) the trace check and the requested-bytes
// and live-handle peaks (the engine's sample(): peaks after every completed
// malloc = max over event prefixes); (2) once both paths have published the
// window, the merged active bytes: each event's value is the sum of the two
// paths' active bytes after their latest events (bit 31 of D names the
// path), the peak its maximum -- overlapped with the paths' replay.
template <bool kMerge>
__device__ __forceinline__ Ledger split_ledger(const uint64_t* ev, uint64_t n, uint32_t* LV, uint32_t h, uint64_t* RAW,
                                               const uint32_t* D, volatile uint32_t* sy) {
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t lt = (1u << lane) - 1u, le = lt | (1u << lane);
  for (uint32_t i = lane; i < (h + 31) / 32; i += 32) LV[i] = 0;
  __syncwarp();
  Ledger L{0, 0, 0, 0, true, false};
  uint64_t req = 0;
  uint32_t live = 0, cv = 0, cs = 0, pka = 0, pkv = 0;
  uint64_t cur = lane < n ? ld_event(ev + lane) : 0;
  uint64_t base = 0;
  for (; base < n; base += 32) {
    const uint64_t nb = base + 32 + lane;
    const uint64_t nxt = nb < n ? ld_event(ev + nb) : 0;
    const uint32_t cnt = (n - base) < 32 ? (uint32_t)(n - base) : 32u;
    const bool act = lane < cnt;
    const bool fr = cur >> 63;
    const uint32_t slot = (uint32_t)((cur >> 40) & 0x7FFFFFu);
    const uint64_t raw = cur & MASK40;
    const uint32_t m_slot = __match_any_sync(0xFFFFFFFFu, act ? slot : (0x80000000u | lane));
    const uint32_t pm = m_slot & lt;
    const uint32_t prev = pm ? 31u - __clz(pm) : lane;
    const bool pfree = __shfl_sync(0xFFFFFFFFu, (uint32_t)fr, prev) != 0;
    const uint64_t praw = ((uint64_t)__shfl_sync(0xFFFFFFFFu, (uint32_t)(raw >> 32), prev) << 32) |
                          __shfl_sync(0xFFFFFFFFu, (uint32_t)raw, prev);
    const bool in_h = act && slot < h;
    bool live_before = false;
    if (pm) live_before = !pfree;
    else if (in_h) live_before = (LV[slot >> 5] >> (slot & 31)) & 1u;
    const bool bad = act && (!in_h || (fr ? (!live_before || raw != 0) : (live_before || raw == 0)));
    if (__ballot_sync(0xFFFFFFFFu, bad)) { L.valid = false; break; }
    uint64_t rawm = raw;
    if (act && fr) rawm = pm ? praw : RAW[slot];
    // the last event of each slot in the window leaves the slot's state
    const bool last = act && (m_slot >> lane) == 1u;
    if (last) {
      if (fr) atomicAnd(&LV[slot >> 5], ~(1u << (slot & 31)));
      else { atomicOr(&LV[slot >> 5], 1u << (slot & 31)); RAW[slot] = raw; }
    }
    // inclusive prefix sums over the window (requested: two's complement u64)
    uint64_t dq = act ? (fr ? (uint64_t)0 - rawm : rawm) : 0;
    int32_t dl = act ? (fr ? -1 : 1) : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint64_t q = ((uint64_t)__shfl_up_sync(0xFFFFFFFFu, (uint32_t)(dq >> 32), o) << 32) |
                         __shfl_up_sync(0xFFFFFFFFu, (uint32_t)dq, o);
      const int32_t l = __shfl_up_sync(0xFFFFFFFFu, dl, o);
      if (lane >= (uint32_t)o) { dq += q; dl += l; }
    }
    const uint64_t rq = req + dq;                 // requested after each event (>= 0 on a valid trace)
    const uint32_t lv = (uint32_t)((int32_t)live + dl);
    const uint32_t mh = __reduce_max_sync(0xFFFFFFFFu, act ? (uint32_t)(rq >> 32) : 0u);
    const uint32_t ml = __reduce_max_sync(0xFFFFFFFFu, act && (uint32_t)(rq >> 32) == mh ? (uint32_t)rq : 0u);
    const uint64_t mq = ((uint64_t)mh << 32) | ml;
    if (mq > L.pk_requested) L.pk_requested = mq;
    const uint32_t ml2 = __reduce_max_sync(0xFFFFFFFFu, act ? lv : 0u);
    if (ml2 > L.mx_live) L.mx_live = ml2;
    req = ((uint64_t)__shfl_sync(0xFFFFFFFFu, (uint32_t)(rq >> 32), cnt - 1) << 32) |
          __shfl_sync(0xFFFFFFFFu, (uint32_t)rq, cnt - 1);
    live = __shfl_sync(0xFFFFFFFFu, lv, cnt - 1);
    __syncwarp();   // this window's table writes precede the next window's reads
    cur = nxt;
    if (!kMerge) continue;
    // (2) wait until both paths have published this window (or a path stopped)
    const uint32_t wi = (uint32_t)(base >> 5) + 1u;
    uint32_t ab = 0;
    if (lane == 0) {
      while ((sy[1] < wi || sy[2] < wi) && !(ab = sy[0])) __nanosleep(GML_LEDGER_NS);
      if (!ab) ab = sy[0];
    }
    if (__shfl_sync(0xFFFFFFFFu, ab, 0)) break;
    __threadfence_block();
    const uint32_t d = act ? __ldcg(D + base + lane) : 0u;
    const bool isv = act && (d >> 31);
    const uint32_t val = d & 0x7FFFFFFFu;
    const uint32_t mv = __ballot_sync(0xFFFFFFFFu, isv), ms = __ballot_sync(0xFFFFFFFFu, act && !isv);
    const uint32_t bv = mv & le, bs = ms & le;
    const uint32_t xv = __shfl_sync(0xFFFFFFFFu, val, bv ? 31u - __clz(bv) : 0u);
    const uint32_t xs = __shfl_sync(0xFFFFFFFFu, val, bs ? 31u - __clz(bs) : 0u);
    const uint32_t ma = __reduce_max_sync(0xFFFFFFFFu, act ? (bv ? xv : cv) + (bs ? xs : cs) : 0u);
    if (ma > pka) pka = ma;
    const uint32_t mvv = __reduce_max_sync(0xFFFFFFFFu, isv ? val : 0u);   // the VMM path's own peak
    if (mvv > pkv) pkv = mvv;
    if (mv) cv = __shfl_sync(0xFFFFFFFFu, val, 31u - __clz(mv));
    if (ms) cs = __shfl_sync(0xFFFFFFFFu, val, 31u - __clz(ms));
  }
  L.merged = base >= n;
  L.pk_active = (uint64_t)pka << 9;
  L.pk_active_vmm = (uint64_t)pkv << 9;
  if (kMerge && !L.valid && lane == 0) sy[0] = 1u;
  return L;
}

// the merged active-bytes peak of a finished unit from its D series (the
// merge step of split_ledger, for path units that ran in separate launches)
__device__ __forceinline__ uint64_t merge_active_peak(const uint32_t* D, uint64_t n, uint64_t* pk_vmm) {
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t le = 0xFFFFFFFFu >> (31 - lane);
  uint32_t cv = 0, cs = 0, pk = 0, pkv = 0;
  for (uint64_t base = 0; base < n; base += 32) {
    const uint32_t cnt = (n - base) < 32 ? (uint32_t)(n - base) : 32u;
    const bool act = lane < cnt;
    const uint32_t d = act ? __ldcs(D + base + lane) : 0u;
    const bool isv = act && (d >> 31);
    const uint32_t val = d & 0x7FFFFFFFu;
    const uint32_t mv = __ballot_sync(0xFFFFFFFFu, isv), ms = __ballot_sync(0xFFFFFFFFu, act && !isv);
    const uint32_t bv = mv & le, bs = ms & le;
    const uint32_t xv = __shfl_sync(0xFFFFFFFFu, val, bv ? 31u - __clz(bv) : 0u);
    const uint32_t xs = __shfl_sync(0xFFFFFFFFu, val, bs ? 31u - __clz(bs) : 0u);
    const uint32_t m = __reduce_max_sync(0xFFFFFFFFu, act ? (bv ? xv : cv) + (bs ? xs : cs) : 0u);
    if (m > pk) pk = m;
    const uint32_t mvv = __reduce_max_sync(0xFFFFFFFFu, isv ? val : 0u);
    if (mvv > pkv) pkv = mvv;
    if (mv) cv = __shfl_sync(0xFFFFFFFFu, val, 31u - __clz(mv));
    if (ms) cs = __shfl_sync(0xFFFFFFFFu, val, 31u - __clz(ms));
  }
  *pk_vmm = (uint64_t)pkv << 9;
  return (uint64_t)pk << 9;
}

// the stats record of a split unit from its two paths and its ledger;
// false if the split result is not the interleaved replay's (the unit must
// be re-run single-warp): a path stopped (OOM, invalid, overflow), a BFC
// segment release, the paths' reserved bytes over capacity, a bad trace
__device__ __forceinline__ bool split_stats_ok(const gml_stats_t& sv, const gml_stats_t& ss, bool valid,
                                               uint64_t capacity) {
  return valid && sv.status == GML_OK && ss.status == GML_OK && sv._p == 0 && ss._p == 0 &&
         ss.n_seg_release == 0 && sv.n_seg_release == 0 &&
         sv.final_reserved_bytes + ss.final_reserved_bytes <= capacity;
}
__device__ __forceinline__ void split_stats(const gml_stats_t& sv, const gml_stats_t& ss, uint64_t pk_active,
                                            uint64_t pk_active_vmm, uint64_t pk_requested, uint32_t mx_live, uint64_t n,
                                            gml_stats_t* out) {
  gml_stats_t o;
  o.peak_active_bytes = pk_active;
  o.peak_reserved_bytes = sv.final_reserved_bytes + ss.final_reserved_bytes;   // both monotone (no release)
  o.peak_requested_bytes = pk_requested;
  o.peak_active_vmm_bytes = pk_active_vmm;   // max of the VMM path's series (its own events)
  o.peak_reserved_vmm_bytes = sv.peak_reserved_vmm_bytes;
  o.final_active_bytes = sv.final_active_bytes + ss.final_active_bytes;
  o.final_reserved_bytes = sv.final_reserved_bytes + ss.final_reserved_bytes;
  o.n_events = n;
  o.n_events_done = n;
  o.oom_event = -1;
  o.status = GML_OK;
  o._p = 0;
  for (int i = 0; i < 5; ++i) o.state_count[i] = sv.state_count[i];   // S1..S5
  o.state_count[5] = ss.state_count[5];                                 // small path
  o.state_count[6] = ss.state_count[6];
  o.n_split = sv.n_split;
  o.n_stitch = sv.n_stitch;
  o.n_companion = sv.n_companion;
  o.n_alloc = sv.n_alloc;
  o.n_evict = sv.n_evict;
  o.n_seg_alloc = ss.n_seg_alloc;
  o.n_seg_release = 0;
  for (int i = 0; i < 7; ++i) o.vmm_calls[i] = sv.vmm_calls[i];
  o.max_pblocks = sv.max_pblocks;
  o.max_sblocks = sv.max_sblocks;
  o.max_live_handles = mx_live;
  o.max_bfc_blocks = ss.max_bfc_blocks;
  *out = o;
}

template <class CF, int kPlace>
__global__ void __launch_bounds__(96, 1) k_replay_split(const __grid_constant__ KParams P) {
  using SC = SplitCfg<CF>;
  using CV = typename SC::V;
  using CS = typename SC::S;
  extern __shared__ __align__(16) uint8_t smem[];
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t wid = threadIdx.x >> 5;
  const Unit u = P.units[blockIdx.x];
  const gml_policy pol = P.pols[u.policy];
  const uint32_t bmw = bm_words_of(pol);
  const uint32_t h = u.h;
  // shared-window base kept opaque (see k_replay)
  uint32_t sa = (uint32_t)__cvta_generic_to_shared(smem);
  asm volatile("" : "+r"(sa));
  uint8_t* sbase = static_cast<uint8_t*>(__cvta_shared_to_generic(sa));
  uint8_t* gbase = P.garena + u.arena_off;
  uint8_t* v_arena = kPlace == SP_BFC_SMEM ? gbase : sbase;
  uint8_t* s_arena = kPlace == SP_BFC_SMEM ? sbase : kPlace == SP_VMM_SMEM ? gbase : sbase + SC::v_bytes(bmw, h);
  uint8_t* lvp = sbase + SC::smem(kPlace, bmw, h) - SC::lv_bytes(h);
  uint32_t* LV = reinterpret_cast<uint32_t*>(lvp);
  volatile uint32_t* sy = reinterpret_cast<volatile uint32_t*>(lvp + SC::lv_bytes(h) - 16);
  uint64_t* RAW = reinterpret_cast<uint64_t*>(gbase + SC::gpart(kPlace, bmw, h));
  uint32_t* D = reinterpret_cast<uint32_t*>(gbase + SC::gpart(kPlace, bmw, h) + SC::a16(8ull * h));
  if (threadIdx.x < 4) sy[threadIdx.x] = 0u;
  __syncthreads();
  // debug probe (tools/gpu_units.sh): the VMM warp alone, so that ncu's
  // per-kernel instruction count and stall samples are the critical chain's
  if ((P.dbg & 1u) && wid != 0) return;

  const uint64_t b = P.offs[u.trace];
  const uint64_t n = P.offs[u.trace + 1] - b;
  const uint64_t* ev = P.events + b;
  uint64_t* asg = P.asg ? P.asg + (uint64_t)u.policy * P.total_events + b : nullptr;
  const long long c0 = clock64();

  Ledger L{0, 0, 0, 0, true, false};
  unsigned long long* prof = P.prof ? P.prof + 16ull * (u.trace * P.n_policies + u.policy) : nullptr;
  if (wid == 0) {
    Engine<DeviceWarp, CV, NoHooks, kPlace != SP_BFC_SMEM> E;
    E.init(pol, RtCaps{bmw, h}, v_arena, nullptr);
    if (prof) E.prof = prof;
    split_path<true, true, true>(E, ev, n, asg, D, sy);
    E.finish(n, n, -1);
  } else if (wid == 1) {
    Engine<DeviceWarp, CS, NoHooks, false> E;
    E.init(pol, RtCaps{0u, h}, s_arena, nullptr);
    split_path<false, true, false>(E, ev, n, asg, D, sy);
    E.finish(n, n, -1);
  } else {
    L = split_ledger<true>(ev, n, LV, h, RAW, D, sy);
  }
#if !defined(GML_PROF_ON)
  // debug (GML_UNIT_CYCLES): when each warp finished, cycles from the start
  if (prof && lane == 0) prof[wid] = (unsigned long long)(clock64() - c0);
#endif
  __syncthreads();
  if (wid != 2) return;   // (in the debug probe warp 0 returns here too: no result)
  const gml_stats_t& sv = *reinterpret_cast<const gml_stats_t*>(v_arena + 4ull * Lay<CV>::STATS);
  const gml_stats_t& ss = *reinterpret_cast<const gml_stats_t*>(s_arena + 4ull * Lay<CS>::STATS);
  const bool ok = sy[0] == 0u && L.merged && split_stats_ok(sv, ss, L.valid, pol.capacity_bytes);
  if (lane == 0) {
    const uint64_t unit = (uint64_t)u.trace * P.n_policies + u.policy;
    if (P.cycles) P.cycles[unit] = (unsigned long long)(clock64() - c0);
    if (!ok) {
      // a table overflow alone: the next size class, still split; anything
      // else: the single-warp replay decides (OOM, release, capacity, invalid)
      const bool only_ovf = L.valid && sv.status == GML_OK && ss.status == GML_OK && (sv._p | ss._p) != 0;
      const uint32_t k = atomicAdd(P.n_ovf, 1u);
      P.ovf[k] = Ovf{u.trace * P.n_policies + u.policy, only_ovf ? (sv._p | ss._p) : OV_SERIAL};
      return;
    }
    split_stats(sv, ss, L.pk_active, L.pk_active_vmm, L.pk_requested, L.mx_live, n, P.stats + unit);
  }
}

template <class CF, int kPlace>
gml_status launch_split_place(const KParams& kp, uint32_t smem, cudaStream_t st) {
  CK(cudaFuncSetAttribute(k_replay_split<CF, kPlace>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  k_replay_split<CF, kPlace><<<kp.n_units, 96, smem, st>>>(kp);
  CK(cudaGetLastError());
  return GML_OK;
}

template <class CF>
gml_status launch_split(int place, const KParams& kp, uint32_t smem, cudaStream_t st) {
  switch (place) {
    case SP_BOTH: return launch_split_place<CF, SP_BOTH>(kp, smem, st);
    case SP_VMM_SMEM: return launch_split_place<CF, SP_VMM_SMEM>(kp, smem, st);
    case SP_BFC_SMEM: return launch_split_place<CF, SP_BFC_SMEM>(kp, smem, st);
  }
  return GML_ERR_INVALID;
}

// K1p: one path of a path-split GMLake unit (throughput placement), one
// warp per unit in the family launches of the global-memory arenas: the
// VMM path in a GMLake-class instance, the small path in a BFC-class
// instance (Cfg::VMM = false: no VMM code, fewer registers). The unit's
// stats go to pstats[mslot][path], its active series to pd; the ledger
// (K1l) and the merge (K1m) in replay.cu finish the unit.
template <class CF>
using PathCfg = std::conditional_t<CF::VMM, Cfg<CF::P, CF::S, CF::IV, 4>, CF>;   // the VMM path: no small path

template <class CF>
__device__ __forceinline__ void path_unit(const KParams& P, const Unit& u, uint8_t* arena, uint32_t* pin_smem) {
  constexpr bool kV = CF::VMM;
  using CE = PathCfg<CF>;
  const uint32_t lane = threadIdx.x & 31u;
  const gml_policy pol = P.pols[u.policy];
  const long long c0 = clock64();
  // the VMM path keeps its PIN words in shared memory (the pPool searches'
  // loads were the largest stall site with the whole arena in global memory)
  Engine<DeviceWarp, CE, NoHooks, GML_PATH_FUSE != 0, kV && GML_PATH_PIN_SMEM, kV && GML_PATH_PIN_SMEM && GML_PATH_BM_SMEM> E;
  E.init(pol, RtCaps{kV ? bm_words_of(pol) : 0u, u.h}, arena, nullptr, pin_smem);
  const uint64_t b = P.offs[u.trace];
  const uint64_t n = P.offs[u.trace + 1] - b;
  uint64_t* asg = P.asg ? P.asg + (uint64_t)u.policy * P.total_events + b : nullptr;
  split_path<kV, false, GML_PATH_FREE_RUN != 0>(E, P.events + b, n, asg, P.pd + u.d_off, nullptr);
  E.finish(n, n, -1);
  const uint32_t* src = reinterpret_cast<const uint32_t*>(E.S());
  uint32_t* dst = reinterpret_cast<uint32_t*>(P.pstats + 2ull * u.mslot + (kV ? 0 : 1));
  for (uint32_t i = lane; i < sizeof(gml_stats_t) / 4; i += 32) dst[i] = src[i];
  if (lane == 0) {
    if (P.cycles && kV) P.cycles[u.trace * P.n_policies + u.policy] = (unsigned long long)(clock64() - c0);
    if (E.overflow) {
      const uint32_t k = atomicAdd(P.n_ovf, 1u);
      P.ovf[k] = Ovf{(u.trace * P.n_policies + u.policy) | (u.path << 30), E.overflow};
    }
  }
  __syncwarp();
}

// Persistent (GML_PATH_PERSIST): one CTA per resident slot, each warp keeps
// ONE arena and takes the next unit (longest first) from a counter until
// none is left -- a unit's tables are written over the L2-resident lines of
// the previous unit on that warp instead of new lines that are written back
// to DRAM, and the work queue balances the tail.
template <class CF>
__global__ void __launch_bounds__(32 * GML_PATH_WPC, CF::VMM ? GML_PATH_MINB : GML_BFC_MINB * 4 / GML_PATH_WPC)
    k_replay_path(const __grid_constant__ KParams P) {
  extern __shared__ __align__(16) uint32_t pin_sm[];
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t wslot = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  uint32_t* const pin_w = pin_sm + (threadIdx.x >> 5) * P.quick_words;
  if (P.next_unit) {
    if (wslot >= P.arena_slots) return;   // (the host sizes the grid in whole CTAs of arenas)
    uint8_t* arena = P.garena + (uint64_t)wslot * P.arena_stride;
    for (;;) {
      uint32_t ui = 0;
      if (lane == 0) ui = atomicAdd(P.next_unit, 1u);
      ui = __shfl_sync(0xFFFFFFFFu, ui, 0);
      if (ui >= P.n_units) break;
      path_unit<CF>(P, P.units[ui], arena, pin_w);
    }
  } else {
    if (wslot >= P.n_units) return;
    const Unit u = P.units[wslot];
    path_unit<CF>(P, u, P.garena + u.arena_off, pin_w);
  }
}

// resident CTAs per SM the launch bounds guarantee (the persistent grid)
template <class CF>
constexpr uint32_t path_ctas_per_sm() {
  return CF::VMM ? GML_PATH_MINB : GML_BFC_MINB * 4 / GML_PATH_WPC;
}

template <class CF>
gml_status launch_path(const KParams& kp, cudaStream_t st) {
  const uint32_t wpc = GML_PATH_WPC;
  uint32_t grid = (kp.n_units + wpc - 1) / wpc;
  if (kp.next_unit) grid = (uint32_t)((kp.arena_slots + wpc - 1) / wpc);
  KParams kq = kp;
  kq.quick_words = (CF::VMM && GML_PATH_PIN_SMEM)
                       ? Lay<PathCfg<CF>>::PINW + (GML_PATH_BM_SMEM ? BMS_WORDS + round4(kp.bm_words_max) : 0u)
                       : 0u;
  const uint32_t smem = 4u * wpc * kq.quick_words;
  if (smem > 48 * 1024) CK(cudaFuncSetAttribute(k_replay_path<CF>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  k_replay_path<CF><<<grid, 32 * wpc, smem, st>>>(kq);
  CK(cudaGetLastError());
  return GML_OK;
}

// classes with split instances (split_<I>.cu)
#define GML_SPLIT_CLASSES(X) X(5, C5) X(6, C6)
#define GML_SDECL(I, CF) gml_status launch_split_##I(int place, const KParams& kp, uint32_t smem, cudaStream_t st);
GML_SPLIT_CLASSES(GML_SDECL)
#undef GML_SDECL

}  // namespace replay
}  // namespace gml
