// engine_host.cpp -- TEST HARNESS (not product code): runs the product's
// allocation engine (paper_2401_08156_b200/csrc/policy.cuh) on the CPU so the
// non-GPU test suite can compare it with the oracle event by event.
//
//   width 1   Engine<HostWarp>: the executor the live allocator uses.
//   width 32  Engine<SimWarp>: 32 std::threads emulate the 32 lanes of one
//             warp; every ballot / shuffle / reduction / __syncwarp of the
//             kernel becomes a barrier exchange, lanes share the arena and
//             run the identical lane-parallel code (k-ary searches, PIN
//             bit-shifts, per-interval ownership, free-list scans). A missing
//             sync or a lane-dependent decision shows up here as a mismatch
//             or a barrier deadlock.
//
// The replay loop mirrors k_replay (replay_kernel.cuh): step, stop on
// overflow / OOM / invalid (the engine samples peaks after each malloc).
#include <atomic>
#include <barrier>
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>

#include "../paper_2401_08156_b200/csrc/policy.cuh"

using namespace gml;

namespace {

using CfgH = Cfg<65536, 32768, 65536, 65536>;
using CfgT = Cfg<64, 16, 128, 256>;   // tiny tables: the lazy-PIN stack (S entries) fills up

struct SimCtx {
  std::barrier<> bar{32};
  uint64_t v[32];
};

struct SimWarp {
  using ctr_t = uint32_t;
  static constexpr bool kReplay = false;
  SimCtx* c;
  uint32_t ln;
  uint32_t lane() const { return ln; }
  uint32_t width() const { return 32; }
  bool leader() const { return ln == 0; }
  void sync() const { c->bar.arrive_and_wait(); }
  void xchg(uint64_t x, uint64_t* out) const {
    c->v[ln] = x;
    c->bar.arrive_and_wait();
    std::memcpy(out, c->v, sizeof(c->v));
    c->bar.arrive_and_wait();
  }
  uint32_t ballot(bool p) const {
    uint64_t a[32];
    xchg(p, a);
    uint32_t m = 0;
    for (int i = 0; i < 32; ++i) m |= (a[i] ? 1u : 0u) << i;
    return m;
  }
  uint32_t shfl(uint32_t v, uint32_t s) const {
    uint64_t a[32];
    xchg(v, a);
    return (uint32_t)a[s & 31];
  }
  uint32_t wmin(uint32_t v) const {
    uint64_t a[32];
    xchg(v, a);
    uint32_t m = 0xFFFFFFFFu;
    for (int i = 0; i < 32; ++i) m = (uint32_t)a[i] < m ? (uint32_t)a[i] : m;
    return m;
  }
  uint32_t match_any(uint32_t v) const {
    uint64_t a[32];
    xchg(v, a);
    uint32_t m = 0;
    for (int i = 0; i < 32; ++i) m |= ((uint32_t)a[i] == v ? 1u : 0u) << i;
    return m;
  }
  uint64_t add_u64(uint64_t v) const {
    uint64_t a[32];
    xchg(v, a);
    uint64_t t = 0;
    for (int i = 0; i < 32; ++i) t += a[i];
    return t;
  }
  uint64_t sum_u32(uint32_t v) const { return add_u64(v); }
  uint64_t bcast64(uint64_t v) const {
    uint64_t a[32];
    xchg(v, a);
    return a[0];
  }
  uint32_t aadd(uint32_t* p, uint32_t v) const { return __atomic_fetch_add(p, v, __ATOMIC_SEQ_CST); }
  uint32_t aor(uint32_t* p, uint32_t v) const { return __atomic_fetch_or(p, v, __ATOMIC_SEQ_CST); }
  uint32_t aand(uint32_t* p, uint32_t v) const { return __atomic_fetch_and(p, v, __ATOMIC_SEQ_CST); }
};

template <class E>
void run_loop(E& e, const uint64_t* ev, uint64_t n, uint64_t* asg, bool writer) {
  uint64_t done = 0;
  int64_t oom = -1;
  for (uint64_t i = 0; i < n; ++i) {
    uint64_t r = e.step(ev[i]);
    if (writer && asg) asg[i] = r;
    if (e.overflow | e.status) {
      if (e.status == GML_ERR_OOM) oom = (int64_t)i;
      break;
    }
    ++done;
  }
  e.finish(n, done, oom);
}

// the kernel's 32-event windows (k_replay): runs of >= 2 consecutive
// VMM-path frees go through Engine::free_run, every other event through step
template <class E>
void run_loop_win(E& e, const uint64_t* ev, uint64_t n, uint64_t* asg, uint32_t lane) {
  uint64_t done = n;
  int64_t oom = -1;
  bool stop = false;
  for (uint64_t base = 0; base < n && !stop; base += 32) {
    const uint32_t cnt = (n - base) < 32 ? (uint32_t)(n - base) : 32u;
    const uint64_t cur = lane < cnt ? ev[base + lane] : 0;
    const uint32_t mall = e.w.ballot(lane < cnt && (cur >> 63) == 0);
    uint32_t m = cnt == 32 ? 0xFFFFFFFFu : (1u << cnt) - 1u, skip = 0;
    while (m) {
      const uint32_t j = ctz32(m);
      const uint32_t run = E::free_run_mask(m, mall) & ~skip;
      if (run & (run - 1)) {
        uint64_t r = 0;
        if (e.free_run(run, cur, r)) {
          if (asg && ((run >> lane) & 1u)) asg[base + lane] = r;
          m &= ~run;
          continue;
        }
        skip |= run;
      }
      m &= m - 1;
      const uint64_t r = e.step(ev[base + j]);
      if (lane == 0 && asg) asg[base + j] = r;
      if (e.overflow | e.status) {
        if (e.status == GML_ERR_OOM) oom = (int64_t)(base + j);
        stop = true;
        done = base + j;
        break;
      }
    }
  }
  e.finish(n, done, oom);
}

uint32_t max_slot(const uint64_t* ev, uint64_t n) {
  uint32_t m = 0;
  for (uint64_t i = 0; i < n; ++i) {
    uint32_t s = (uint32_t)((ev[i] >> 40) & 0x7FFFFFu) + 1;
    if (s > m) m = s;
  }
  return m ? m : 1;
}

template <class CF>
int replay_cfg(const uint64_t* ev, uint64_t n, const gml_policy* pol, int width, uint64_t* asg, gml_stats_t* st,
               uint32_t* hw) {
  if (pol->capacity_bytes / pol->chunk_bytes + 1 > kMaxChunks) return -1;
  RtCaps rc{(uint32_t)((pol->capacity_bytes / pol->chunk_bytes + 1 + 31) / 32), max_slot(ev, n)};
  std::vector<uint64_t> arena((Lay<CF>::bytes(rc.bm_words, rc.h) + 7) / 8 + 2, 0);
  uint8_t* base = reinterpret_cast<uint8_t*>(arena.data());
  NoHooks hk;
  if (width == 1) {
    Engine<HostWarp, CF> e;
    e.init(*pol, rc, base, &hk);
    run_loop(e, ev, n, asg, true);
    std::memcpy(st, e.S(), sizeof(gml_stats_t));
    st->_p = e.overflow;
    if (hw) { hw[0] = e.mx_p; hw[1] = e.mx_s; hw[2] = e.mx_iv; hw[3] = e.b_hw; hw[4] = 0; }
    return 0;
  }
  SimCtx ctx;
  std::vector<std::thread> th;
  uint32_t ovf = 0;
  for (uint32_t l = 0; l < 32; ++l) {
    th.emplace_back([&, l]() {
      Engine<SimWarp, CF> e;
      e.w = SimWarp{&ctx, l};
      e.init(*pol, rc, base, &hk);
      run_loop_win(e, ev, n, asg, l);
      if (l == 0) {
        ovf = e.overflow;
        if (hw) { hw[0] = e.mx_p; hw[1] = e.mx_s; hw[2] = e.mx_iv; hw[3] = e.b_hw; hw[4] = 0; }
      }
    });
  }
  for (auto& t : th) t.join();
  std::memcpy(st, base, sizeof(gml_stats_t));
  st->_p = ovf;
  return 0;
}

}  // namespace

extern "C" {

// Replay one trace through the product engine on the CPU. width = 1 or 32
// (large tables, CfgH), 101 or 132 (tiny tables, CfgT: width - 100).
// asg: n records (zero-initialised by the caller); *st: the stats record with
// _p = overflow bits; hw (optional): table high-water marks {pBlocks,
// sBlocks, live intervals, BFC rows, index nodes}. Returns 0, or -1 for an unsupported policy.
int eng_replay(const uint64_t* ev, uint64_t n, const gml_policy* pol, int width, uint64_t* asg, gml_stats_t* st,
               uint32_t* hw) {
  if (width > 100) return replay_cfg<CfgT>(ev, n, pol, width - 100, asg, st, hw);
  return replay_cfg<CfgH>(ev, n, pol, width, asg, st, hw);
}

}  // extern "C"
