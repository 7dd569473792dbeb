// replay.cu -- K0 (per-trace slot scan) and K1 (batched trace replay) for
// sm_100a, plus the host side of gml_replay / gml_trace_validate / metrics.
//
// K1 maps one warp to one (trace, policy) unit:
//   a1  events stream HBM -> registers, 32 per warp-wide coalesced 8-byte
//       load, the next batch prefetched while the current one is replayed;
//       event j is broadcast from lane j with one shuffle.
//   a2-a9  gml::Engine<DeviceWarp, Cfg>::step (policy.cuh) on tables in
//       shared memory (or a global-memory arena for the large size classes).
//   a10 peaks sampled after every event in registers; the record of event j
//       is kept by lane j and written back as one coalesced 256-byte store per
//       32 events; the 272-byte stats record is written at the end.
// Table capacities are compile-time size classes (all offsets immediates).
// Units whose tables overflow are re-run by the host in the next class, so a
// table size never changes a result (D30).
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <type_traits>
#include <vector>

#include "gml.h"
#include "policy.cuh"
#include "replay_kernel.cuh"
#include "split_kernel.cuh"

using namespace gml;
using namespace gml::replay;

namespace {

constexpr uint32_t kSmemMax = 227 * 1024;
thread_local uint32_t g_launches = 0;
thread_local float g_kernel_ms = 0.f;
thread_local uint32_t g_split_done = 0, g_split_reruns = 0;

// debug (GML_HOST_TIMES): host-side phase times of gml_replay on stderr
struct HostTimes {
  bool on = getenv("GML_HOST_TIMES") != nullptr;
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now(), t = t0;
  void mark(const char* what) {
    if (!on) return;
    const auto n = std::chrono::steady_clock::now();
    fprintf(stderr, "gml-host %-24s %8.3f ms\n", what, std::chrono::duration<double, std::milli>(n - t).count());
    t = n;
  }
};

// Device workspace reused across gml_replay calls (grown, never shrunk):
// per-call cudaMallocAsync / cudaFreeAsync of the arenas (hundreds of MB for
// a C4 batch) cost more than the replay launches themselves. gml_replay
// synchronises its stream before returning, so a buffer is idle between
// calls; buffers are per (thread, device).
enum { WS_SLOTS, WS_POLS, WS_OVF, WS_NOVF, WS_UNITS, WS_ARENA, WS_DBG1, WS_DBG2, WS_D, WS_PST, WS_LED, WS_LTR,
       WS_LOFF, WS_LSCR, WS_CTR, WS_N };
struct Workspace {
  void* p[WS_N] = {};
  size_t n[WS_N] = {};
  size_t free_at_start = 0;   // device memory free at the first call (cudaMemGetInfo is slow and erratic:
                              // measured 0.2-100 ms per call on the replay's critical path)
  std::vector<cudaStream_t> side;   // side streams of this device (one per class group)
};
thread_local std::map<int, Workspace> g_ws;

cudaError_t ws_get(int dev, int which, size_t bytes, void** out) {
  Workspace& w = g_ws[dev];
  if (w.n[which] < bytes) {
    if (w.p[which]) cudaFree(w.p[which]);
    w.p[which] = nullptr;
    w.n[which] = 0;
    size_t want = bytes + bytes / 4 + 256;
    cudaError_t e = cudaMalloc(&w.p[which], want);
    if (e != cudaSuccess) { w.p[which] = nullptr; return e; }
    w.n[which] = want;
  }
  *out = w.p[which];
  return cudaSuccess;
}

uint64_t class_bytes(int cls, uint32_t bm_words, uint32_t h) {
  switch (cls) {
#define GML_BYTES(I, CF) \
  case I:                \
    return Lay<CF>::bytes(bm_words, h);
    GML_CLASSES(GML_BYTES)
#undef GML_BYTES
  }
  return ~0ull;
}

// arena bytes of a path unit: the VMM path's class without BFC rows
uint64_t path_bytes(int cls, uint32_t bm_words, uint32_t h) {
  switch (cls) {
#define GML_PBYTES(I, CF) \
  case I:                 \
    return Lay<PathCfg<CF>>::bytes(bm_words, h);
    GML_CLASSES(GML_PBYTES)
#undef GML_PBYTES
  }
  return ~0ull;
}

// K0: 1 + max slot of every trace (sizes the handle table), and per trace
// the number of mallocs at or above each of up to kNThr thresholds (the
// VMM-path share of a GMLake unit: where a split unit's shared memory goes)
constexpr uint32_t kNThr = 4;
struct Thr {
  uint64_t t[kNThr];
};
__global__ void k_max_slot(const uint64_t* __restrict__ ev, const uint64_t* __restrict__ offs,
                           uint32_t n_traces, uint32_t* __restrict__ out, const __grid_constant__ Thr thr,
                           uint32_t* __restrict__ big) {
  for (uint32_t t = blockIdx.x; t < n_traces; t += gridDim.x) {
    uint64_t b = offs[t], e = offs[t + 1];
    uint32_t m = 0, c[kNThr + 1] = {0, 0, 0, 0, 0};
    for (uint64_t i = b + threadIdx.x; i < e; i += blockDim.x) {
      const uint64_t x = __ldg(ev + i);
      uint32_t s = (uint32_t)((x >> 40) & 0x7FFFFFu) + 1;
      m = max(m, s);
      if (!(x >> 63)) {
        c[kNThr]++;
#pragma unroll
        for (uint32_t k = 0; k < kNThr; ++k) c[k] += (x & MASK40) >= thr.t[k];
      }
    }
    m = __reduce_max_sync(0xFFFFFFFFu, m);
#pragma unroll
    for (uint32_t k = 0; k <= kNThr; ++k) c[k] = __reduce_add_sync(0xFFFFFFFFu, c[k]);
    __shared__ uint32_t red[32][kNThr + 2];
    if ((threadIdx.x & 31) == 0) {
      red[threadIdx.x >> 5][0] = m;
      for (uint32_t k = 0; k <= kNThr; ++k) red[threadIdx.x >> 5][k + 1] = c[k];
    }
    __syncthreads();
    if (threadIdx.x < 32) {
      const bool on = threadIdx.x < (blockDim.x >> 5);
      uint32_t v = on ? red[threadIdx.x][0] : 0;
      v = __reduce_max_sync(0xFFFFFFFFu, v);
      if (threadIdx.x == 0) out[t] = v;
      for (uint32_t k = 0; k <= kNThr; ++k) {
        uint32_t q = __reduce_add_sync(0xFFFFFFFFu, on ? red[threadIdx.x][k + 1] : 0u);
        if (threadIdx.x == 0) big[(uint64_t)t * (kNThr + 1) + k] = q;
      }
    }
    __syncthreads();
  }
}

// K1l (path units): per trace, one warp -- the trace check and the
// requested-bytes / live-handle peaks of split_ledger, without the merge
struct LedgerOut {
  uint64_t pk_requested;
  uint32_t mx_live, valid;
};
__global__ void __launch_bounds__(128) k_ledger(const uint64_t* __restrict__ ev, const uint64_t* __restrict__ offs,
                                                const uint32_t* __restrict__ traces, const uint64_t* __restrict__ scr_off,
                                                uint32_t n, const uint32_t* __restrict__ hs, uint32_t* scr, LedgerOut* out) {
  const uint32_t k = blockIdx.x * 4 + (threadIdx.x >> 5);
  if (k >= n) return;
  const uint32_t t = traces[k];
  const uint32_t h = hs[t] ? hs[t] : 1u;
  uint32_t* base = scr + scr_off[k];
  uint64_t* RAW = reinterpret_cast<uint64_t*>(base);
  uint32_t* LV = base + 2ull * h;
  const uint64_t b = offs[t];
  const Ledger L = split_ledger<false>(ev + b, offs[t + 1] - b, LV, h, RAW, nullptr, nullptr);
  if ((threadIdx.x & 31u) == 0) out[t] = LedgerOut{L.pk_requested, L.mx_live, L.valid ? 1u : 0u};
}

// K1m (path units): per unit, one warp -- the split unit's exactness test,
// the merged active-bytes peak from D, the stats record; else OV_SERIAL
__global__ void __launch_bounds__(128) k_merge(const Unit* __restrict__ mu, uint32_t n, const uint64_t* __restrict__ offs,
                                               const gml_policy* __restrict__ pols, uint32_t NP, const uint32_t* D,
                                               const gml_stats_t* pst, const LedgerOut* led, gml_stats_t* stats, Ovf* ovf,
                                               uint32_t* n_ovf) {
  const uint32_t k = blockIdx.x * 4 + (threadIdx.x >> 5);
  if (k >= n) return;
  const Unit u = mu[k];
  const gml_stats_t& sv = pst[2ull * u.mslot];
  const gml_stats_t& ss = pst[2ull * u.mslot + 1];
  const LedgerOut lo = led[u.trace];
  const uint64_t len = offs[u.trace + 1] - offs[u.trace];
  const bool ok = split_stats_ok(sv, ss, lo.valid != 0, pols[u.policy].capacity_bytes);
  uint64_t pkv = 0;
  const uint64_t pk = ok ? merge_active_peak(D + u.d_off, len, &pkv) : 0;
  if ((threadIdx.x & 31u) == 0) {
    const uint32_t unit = u.trace * NP + u.policy;
    if (ok) {
      split_stats(sv, ss, pk, pkv, lo.pk_requested, lo.mx_live, len, stats + unit);
    } else {
      const uint32_t q = atomicAdd(n_ovf, 1u);
      ovf[q] = Ovf{unit, OV_SERIAL};
    }
  }
}

uint32_t path_ctas_cls(int cls) {
  switch (cls) {
#define GML_PC(I, CF) \
  case I:             \
    return path_ctas_##I();
    GML_CLASSES(GML_PC)
#undef GML_PC
  }
  return 1;
}

gml_status launch_path_cls(int cls, const KParams& kp, cudaStream_t st) {
  switch (cls) {
#define GML_PL(I, CF) \
  case I:             \
    return launch_path_##I(kp, st);
    GML_CLASSES(GML_PL)
#undef GML_PL
  }
  return GML_ERR_INVALID;
}

// default classes of throughput placement (C8 / C2: every C4 unit fits them)
constexpr int kDefaultGlobalVmm = 8;
constexpr int kDefaultGlobalBfc = 2;

uint32_t bmw_max(const gml_trace_batch* B) {
  uint32_t m = 1;
  for (uint32_t p = 0; p < B->n_policies; ++p)
    m = std::max<uint32_t>(m, (uint32_t)((B->policies[p].capacity_bytes / B->policies[p].chunk_bytes + 1 + 31) / 32));
  return m;
}

// smallest class of the policy's family that covers the hint
int pick_class(const gml_policy& p, const gml_replay_caps* hint) {
  bool vmm = p.kind == GML_POLICY_GMLAKE;
  uint32_t np = 0, ns = 0, niv = 0, nb = 0;
  if (hint) { np = hint->pblocks; ns = hint->sblocks; niv = hint->intervals; nb = hint->bfc_blocks; }
  int lo = vmm ? kFirstVmm : 0, hi = vmm ? kNumClasses : kFirstVmm;
  if (!hint || (np | ns | niv | nb) == 0) return lo + 1;   // no hint: the middle class
  for (int c = lo; c < hi; ++c) {
    const ClassInfo& k = kClasses[c];
    if ((!vmm || (k.p >= np && k.s >= ns && k.iv >= niv)) && k.b >= nb) return c;
  }
  return hi - 1;
}

// two-path units carry a path's active bytes in 31 bits of 512-byte units
// (active <= reserved <= capacity): capacities from 2^40 bytes run single-warp
constexpr uint64_t kSplitCapMax = 1ull << 40;

// the VMM-path gate of a GMLake policy (Engine::init)
uint64_t vm_thr_of(const gml_policy& p) {
  uint64_t t = p.small_threshold_bytes;
  if ((p.flags & GML_F_LIMIT_GATES_REQUEST) && p.frag_limit_bytes > t) t = p.frag_limit_bytes;
  return t;
}

bool has_split(int cls) {
#define GML_HAS(I, CF) if (cls == I) return true;
  GML_SPLIT_CLASSES(GML_HAS)
#undef GML_HAS
  return false;
}
uint64_t split_smem(int cls, int place, uint32_t bmw, uint32_t h) {
#define GML_SB(I, CF) if (cls == I) return SplitCfg<CF>::smem(place, bmw, h);
  GML_SPLIT_CLASSES(GML_SB)
#undef GML_SB
  return ~0ull;
}
uint64_t split_glob(int cls, int place, uint32_t bmw, uint32_t h, uint64_t n) {
#define GML_SG(I, CF) if (cls == I) return SplitCfg<CF>::glob(place, bmw, h, n);
  GML_SPLIT_CLASSES(GML_SG)
#undef GML_SG
  return ~0ull;
}
gml_status launch_split_cls(int cls, int place, const KParams& kp, uint32_t smem, cudaStream_t st) {
#define GML_SL(I, CF) if (cls == I) return launch_split_##I(place, kp, smem, st);
  GML_SPLIT_CLASSES(GML_SL)
#undef GML_SL
  return GML_ERR_INVALID;
}

gml_status launch(int cls, bool smem, const KParams& kp, uint32_t stride, cudaStream_t st) {
  switch (cls) {
#define GML_LAUNCH(I, CF) \
  case I:                 \
    return launch_cls_##I(smem, kp, stride, st);
    GML_CLASSES(GML_LAUNCH)
#undef GML_LAUNCH
  }
  return GML_ERR_INVALID;
}

}  // namespace

extern "C" {

const char* gml_status_string(gml_status s) {
  switch (s) {
    case GML_OK: return "ok";
    case GML_ERR_INVALID: return "invalid argument or trace";
    case GML_ERR_OOM: return "out of memory (S5)";
    case GML_ERR_CUDA: return "CUDA error";
    case GML_ERR_TABLE_OVERFLOW: return "replay table overflow";
    case GML_ERR_UNSUPPORTED: return "unsupported";
  }
  return "unknown status";
}

gml_status gml_trace_validate(const uint64_t* ev, uint64_t n, uint32_t* max_slots) {
  if (!max_slots || (n && !ev)) return GML_ERR_INVALID;
  std::vector<uint8_t> live;
  uint32_t mx = 0;
  for (uint64_t i = 0; i < n; ++i) {
    bool f = ev[i] >> 63;
    uint32_t s = (uint32_t)((ev[i] >> 40) & 0x7FFFFFu);
    uint64_t raw = ev[i] & gml::MASK40;
    if (s >= live.size()) live.resize((size_t)s + 1, 0);
    if (f ? (raw != 0 || !live[s]) : (raw == 0 || live[s])) {
      *max_slots = (uint32_t)std::min<uint64_t>(i, 0xFFFFFFFFu);
      return GML_ERR_INVALID;
    }
    live[s] = f ? 0 : 1;
    mx = std::max(mx, s + 1);
  }
  *max_slots = mx;
  return GML_OK;
}

double gml_utilization(const gml_stats_t* s) {
  if (!s) return 0.0;
  if (s->peak_reserved_bytes == 0) return 1.0;
  return (double)s->peak_active_bytes / (double)s->peak_reserved_bytes;
}

double gml_fragmentation(const gml_stats_t* s) { return 1.0 - gml_utilization(s); }

uint32_t gml_last_launch_count(void) { return g_launches; }
float gml_last_kernel_ms(void) { return g_kernel_ms; }
uint32_t gml_last_split_count(uint32_t* serial_reruns) {
  if (serial_reruns) *serial_reruns = g_split_reruns;
  return g_split_done;
}

gml_status gml_replay(const gml_trace_batch* B) {
  g_launches = 0;
  g_kernel_ms = 0.f;
  g_split_done = g_split_reruns = 0;
  HostTimes ht;
  if (!B || !B->events || !B->trace_offsets || !B->policies || !B->stats || B->n_traces == 0 ||
      B->n_policies == 0)
    return GML_ERR_INVALID;
  for (uint32_t p = 0; p < B->n_policies; ++p) {
    const gml_policy& q = B->policies[p];
    if (q.kind > GML_POLICY_GMLAKE || q.chunk_bytes == 0 || q.chunk_bytes % 512 || q.spool_max_entries == 0)
      return GML_ERR_INVALID;
    if (q.capacity_bytes / q.chunk_bytes + 1 > kMaxChunks) return GML_ERR_UNSUPPORTED;
  }
  cudaStream_t st = (cudaStream_t)B->stream;
  const uint32_t NT = B->n_traces, NP = B->n_policies;
  const uint64_t NU = (uint64_t)NT * NP;

  // trace offsets + per-trace slot counts (K0)
  std::vector<uint64_t> offs(NT + 1);
  CK(cudaMemcpyAsync(offs.data(), B->trace_offsets, 8ull * (NT + 1), cudaMemcpyDeviceToHost, st));
  uint32_t *d_slots = nullptr, *d_novf = nullptr;
  gml_policy* d_pols = nullptr;
  int cur_dev = 0;
  CK(cudaGetDevice(&cur_dev));
  // distinct VMM-path gates of the batch's GMLake policies (K0 counts the
  // mallocs at or above each: a split unit's placement)
  Thr thr;
  std::vector<uint64_t> gates;
  for (uint32_t p = 0; p < NP; ++p)
    if (B->policies[p].kind == GML_POLICY_GMLAKE && gates.size() < kNThr &&
        std::find(gates.begin(), gates.end(), vm_thr_of(B->policies[p])) == gates.end())
      gates.push_back(vm_thr_of(B->policies[p]));
  for (uint32_t k = 0; k < kNThr; ++k) thr.t[k] = k < gates.size() ? gates[k] : ~0ull;
  CK(ws_get(cur_dev, WS_SLOTS, 4ull * NT * (kNThr + 2), (void**)&d_slots));
  k_max_slot<<<std::min<uint32_t>(NT, 148 * 8), 256, 0, st>>>(B->events, B->trace_offsets, NT, d_slots, thr,
                                                              d_slots + NT);
  g_launches++;
  CK(cudaGetLastError());
  std::vector<uint32_t> slots(NT), nbig((size_t)NT * (kNThr + 1));
  CK(cudaMemcpyAsync(slots.data(), d_slots, 4ull * NT, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(nbig.data(), d_slots + NT, 4ull * NT * (kNThr + 1), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  ht.mark("K0 + offsets");
  const uint64_t total = offs[NT];
  for (uint32_t t = 0; t < NT; ++t)
    if (offs[t + 1] < offs[t]) return GML_ERR_INVALID;

  CK(ws_get(cur_dev, WS_POLS, sizeof(gml_policy) * NP, (void**)&d_pols));
  CK(cudaMemcpyAsync(d_pols, B->policies, sizeof(gml_policy) * NP, cudaMemcpyHostToDevice, st));

  std::vector<int> cls(NU), cls_s(NU);
  std::vector<uint32_t> hcap(NU);
  for (uint32_t t = 0; t < NT; ++t)
    for (uint32_t p = 0; p < NP; ++p) {
      uint64_t i = (uint64_t)t * NP + p;
      const gml_replay_caps* hint = B->caps ? &B->caps[i] : nullptr;
      cls[i] = pick_class(B->policies[p], hint);
      gml_policy bp = B->policies[p];
      bp.kind = GML_POLICY_BFC_TORCH;
      cls_s[i] = pick_class(bp, hint);   // the small path's class if the unit is path-split
      hcap[i] = std::max<uint32_t>(slots[t], 1);
    }

  std::vector<uint32_t> bmw(NP);
  for (uint32_t p = 0; p < NP; ++p)
    bmw[p] = (uint32_t)((B->policies[p].capacity_bytes / B->policies[p].chunk_bytes + 1 + 31) / 32);

  Ovf* d_ovf = nullptr;
  CK(ws_get(cur_dev, WS_OVF, sizeof(Ovf) * 2 * NU, (void**)&d_ovf));
  CK(ws_get(cur_dev, WS_NOVF, 4, (void**)&d_novf));
  gml_status rc = GML_OK;
  const bool dbg_cycles = getenv("GML_UNIT_CYCLES") != nullptr;
  unsigned long long* d_cycles = nullptr;
  unsigned long long* d_prof = nullptr;
  if (dbg_cycles) {
    CK(ws_get(cur_dev, WS_DBG1, 8 * NU, (void**)&d_cycles));
    CK(ws_get(cur_dev, WS_DBG2, 8 * 16 * NU, (void**)&d_prof));
    CK(cudaMemsetAsync(d_prof, 0, 8 * 16 * NU, st));
  }

  // side streams (of this device) so that the per-class launches run concurrently
  std::vector<cudaStream_t>& side = g_ws[cur_dev].side;
  while (side.size() < 4 * kNumClasses + 1) {
    cudaStream_t s;
    CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    side.push_back(s);
  }

  // Small batches (fewer units than 4 per SM) keep each unit's tables in
  // the shared memory of its own CTA when they fit ("latency" placement);
  // batches that fill the GPU keep them in HBM/L2 so that more units are
  // resident per SM (measured faster on C4). GML_FORCE_GLOBAL /
  // GML_FORCE_SMEM override.
  int n_sm = 148;
  {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
  }
  const bool force_global = getenv("GML_FORCE_GLOBAL") != nullptr;
  const bool force_smem = getenv("GML_FORCE_SMEM") != nullptr;
  const bool latency = NU < (uint64_t)n_sm * 4;
  const bool no_split_env = getenv("GML_NO_SPLIT") != nullptr;
  const uint32_t dbg_flags = getenv("GML_SPLIT_VMM_ONLY") ? 1u : 0u;   // debug probe: no results
  const bool persist = GML_PATH_PERSIST && getenv("GML_NO_PERSIST") == nullptr;

  // Split units (split_kernel.cuh): in the latency placement a GMLake unit
  // of a class with split instances runs its VMM path and its small path on
  // two warps of one CTA; the part with more work (K0's malloc counts, a
  // VMM-path event costing about twice a small-path one) gets the shared
  // memory if both do not fit. A unit that reports OV_SERIAL is re-run with
  // the single-warp K1. GML_NO_SPLIT disables it.
  const bool split_on = latency && !force_global && !B->timeline && !no_split_env;
  // Path units (throughput placement): a GMLake unit's VMM path and small
  // path are two units of the two family launches -- the small path in the
  // BFC family, whose instances carry no VMM code (about half the
  // registers, twice the resident warps) -- followed by a per-trace ledger
  // (K1l) and a per-unit merge (K1m) with the split unit's exactness test.
  const bool path_on = !latency && !force_smem && !B->timeline && !no_split_env && NU < (1u << 30);
  std::vector<uint8_t> no_split(NU, 0);
  std::vector<uint32_t> mslot(NU, NONE32);
  std::vector<uint64_t> d_off(NU, 0);
  std::vector<uint32_t> led_traces;
  uint32_t n_path = 0;
  uint64_t d_words = 0;
  if (path_on) {
    std::vector<uint8_t> led(NT, 0);
    for (uint64_t i = 0; i < NU; ++i)
      if (B->policies[i % NP].kind == GML_POLICY_GMLAKE && B->policies[i % NP].capacity_bytes < kSplitCapMax) {
        const uint32_t t = (uint32_t)(i / NP);
        mslot[i] = n_path++;
        d_off[i] = d_words;
        d_words += (offs[t + 1] - offs[t] + 31) & ~31ull;
        led[t] = 1;
      }
    for (uint32_t t = 0; t < NT; ++t)
      if (led[t]) led_traces.push_back(t);
  }
  g_split_done += n_path;

  // path units' per-event series D, path stats, the ledgers (persist across rounds)
  uint32_t* d_D = nullptr;
  gml_stats_t* d_pst = nullptr;
  LedgerOut* d_led = nullptr;
  if (n_path) {
    CK(ws_get(cur_dev, WS_D, 4ull * d_words, (void**)&d_D));
    CK(ws_get(cur_dev, WS_PST, sizeof(gml_stats_t) * 2ull * n_path, (void**)&d_pst));
    CK(ws_get(cur_dev, WS_LED, sizeof(LedgerOut) * NT, (void**)&d_led));
    // K1l first: per trace scratch = per-slot raw sizes + slot bits
    std::vector<uint64_t> lo(led_traces.size());
    uint64_t sw = 0;
    for (size_t k = 0; k < led_traces.size(); ++k) {
      lo[k] = sw;
      const uint32_t h = std::max<uint32_t>(slots[led_traces[k]], 1);
      sw += 2ull * h + ((h + 31) / 32 + 3) / 4 * 4;   // u32 words: RAW (2 per slot) then LV
    }
    uint32_t* d_lt = nullptr;
    uint64_t* d_lo = nullptr;
    uint32_t* d_ls = nullptr;
    CK(ws_get(cur_dev, WS_LTR, 4ull * led_traces.size(), (void**)&d_lt));
    CK(ws_get(cur_dev, WS_LOFF, 8ull * led_traces.size(), (void**)&d_lo));
    CK(ws_get(cur_dev, WS_LSCR, 4ull * sw + 16, (void**)&d_ls));
    CK(cudaMemcpyAsync(d_lt, led_traces.data(), 4ull * led_traces.size(), cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(d_lo, lo.data(), 8ull * lo.size(), cudaMemcpyHostToDevice, st));
    const uint32_t nl = (uint32_t)led_traces.size();
    cudaEvent_t l0, l1;
    CK(cudaEventCreate(&l0));
    CK(cudaEventCreate(&l1));
    CK(cudaEventRecord(l0, st));
    k_ledger<<<(nl + 3) / 4, 128, 0, st>>>(B->events, B->trace_offsets, d_lt, d_lo, nl, d_slots, d_ls, d_led);
    CK(cudaGetLastError());
    g_launches++;
    CK(cudaEventRecord(l1, st));
    std::vector<LedgerOut> led(NT);
    CK(cudaMemcpyAsync(led.data(), d_led, sizeof(LedgerOut) * NT, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, l0, l1));
    g_kernel_ms += ms;
    cudaEventDestroy(l0);
    cudaEventDestroy(l1);
    ht.mark("ledger");
    // a trace whose requested bytes exceed a policy's capacity OOMs under it
    // (reserved >= active >= requested), and a bad trace stops: such units
    // would only fall back after the merge (a tail launch); they run
    // single-warp from the start instead
    for (uint64_t i = 0; i < NU; ++i) {
      if (mslot[i] == NONE32) continue;
      const LedgerOut& L = led[i / NP];
      if (!L.valid || L.pk_requested > B->policies[i % NP].capacity_bytes) {
        mslot[i] = NONE32;
        g_split_done--;
      }
    }
  }

  // tasks: unit index | path << 30 (0 whole unit, 1 VMM path, 2 small path)
  std::vector<uint32_t> todo;
  for (uint64_t i = 0; i < NU; ++i) {
    if (mslot[i] != NONE32) {
      todo.push_back((uint32_t)i | (1u << 30));
      todo.push_back((uint32_t)i | (2u << 30));
    } else {
      todo.push_back((uint32_t)i);
    }
  }
  auto task_cls = [&](uint32_t tk) -> int& { return (tk >> 30) == 2 ? cls_s[tk & 0x3FFFFFFFu] : cls[tk & 0x3FFFFFFFu]; };

  // Throughput placement (global-memory arenas): one size class per family
  // for (nearly) the whole batch -- the class covering 99 % of the units'
  // needs, and at least a large default -- so that each family is ONE launch
  // whose units run longest-first, instead of one launch per class whose
  // tails add up (measured on C4: 240 ms vs 280 ms with per-unit classes; a
  // larger class only spreads the same touched rows over more address
  // space). Units that need more keep their own larger class (a second,
  // short launch) rather than dragging every arena up. The arenas must fit
  // a budget of device memory, else every unit keeps its own smallest class.
  if (!latency && !force_smem) {
    std::vector<int> need_f[2];   // [bfc family, vmm family]
    for (uint32_t tk : todo) need_f[kClasses[task_cls(tk)].vmm ? 1 : 0].push_back(task_cls(tk));
    const int dflt[2] = {kDefaultGlobalBfc, kDefaultGlobalVmm};
    int want[2] = {0, 0};
    for (int f = 0; f < 2; ++f) {
      std::vector<int>& v = need_f[f];
      if (v.empty()) continue;
      std::sort(v.begin(), v.end());
      want[f] = std::max(dflt[f], v[(size_t)((v.size() - 1) * 0.99)]);
    }
    Workspace& wsp = g_ws[cur_dev];
    if (!wsp.free_at_start) {
      size_t total_b = 0;
      cudaMemGetInfo(&wsp.free_at_start, &total_b);
    }
    const uint64_t budget = (uint64_t)wsp.free_at_start / 4;
    uint32_t hmax = 1;
    for (uint64_t i = 0; i < NU; ++i) hmax = std::max(hmax, hcap[i]);
    const uint32_t bw = bmw_max(B);
    auto need = [&](const int* wv) {
      uint64_t t = 4ull * d_words;
      for (uint32_t tk : todo) {
        const int c = task_cls(tk);
        const int f = kClasses[c].vmm ? 1 : 0;
        t += class_bytes(std::max(c, wv[f]), bw, hmax) + 256;
      }
      return t;
    };
    // step the defaults down (never below the families' smallest class) until the arenas fit
    const int lo_f[2] = {0, kFirstVmm};
    for (int f = 1; f >= 0; --f)
      while (!need_f[f].empty() && need(want) > budget && want[f] > lo_f[f]) want[f]--;
    if (need(want) <= budget)
      for (uint32_t tk : todo) {
        int& c = task_cls(tk);
        c = std::max(c, want[kClasses[c].vmm ? 1 : 0]);
      }
  }

  // mode of a task: 0 single warp, global arena; 1 single warp, shared
  // memory; 2 + SplitPlace: split unit; 5 / 6: VMM / small path unit
  auto unit_mode = [&](uint32_t tk, uint64_t* smem_b, uint64_t* glob_b) -> int {
    const uint32_t ui = tk & 0x3FFFFFFFu, path = tk >> 30;
    const uint32_t t = ui / NP, p = ui % NP;
    const gml_policy& q = B->policies[p];
    if (path) {
      *smem_b = 0;
      *glob_b = path_bytes(task_cls(tk), path == 1 ? bmw[p] : 0u, hcap[ui]);
      return 4 + (int)path;
    }
    if (split_on && !no_split[ui] && q.kind == GML_POLICY_GMLAKE && q.capacity_bytes < kSplitCapMax && has_split(cls[ui])) {
      const uint64_t n = offs[t + 1] - offs[t];
      int place = SP_BOTH;
      if (split_smem(cls[ui], SP_BOTH, bmw[p], hcap[ui]) > kSmemMax) {
        uint64_t nv = 0;
        for (uint32_t k = 0; k < gates.size(); ++k)
          if (gates[k] == vm_thr_of(q)) nv = nbig[(uint64_t)t * (kNThr + 1) + k];
        const uint64_t nm = nbig[(uint64_t)t * (kNThr + 1) + kNThr];
        place = 2 * nv >= nm - nv ? SP_VMM_SMEM : SP_BFC_SMEM;
      }
      const uint64_t sb = split_smem(cls[ui], place, bmw[p], hcap[ui]);
      if (sb <= kSmemMax) {
        *smem_b = sb;
        *glob_b = split_glob(cls[ui], place, bmw[p], hcap[ui], n);
        return 2 + place;
      }
    }
    const uint64_t by = class_bytes(cls[ui], bmw[p], hcap[ui]);
    const bool sm = by <= kSmemMax && (latency ? !force_global : force_smem);
    *smem_b = sm ? by : 0;
    *glob_b = sm ? 0 : by;
    return sm ? 1 : 0;
  };

  ht.mark("placement");
  auto run_rounds = [&](std::vector<uint32_t>& todo) -> gml_status {
    for (int round = 0; !todo.empty() && round < 2 * kNumClasses + 2; ++round) {
      // group tasks by (class, mode)
      std::map<std::pair<int, int>, std::vector<Unit>> groups;
      std::map<std::pair<int, int>, uint64_t> gmax, smax;
      std::map<uint32_t, uint64_t> uglob;   // split units: their own global bytes
      for (uint32_t tk : todo) {
        const uint32_t ui = tk & 0x3FFFFFFFu, path = tk >> 30;
        Unit u{ui / NP, ui % NP, hcap[ui], path, 0, d_off[ui], mslot[ui] == NONE32 ? 0u : mslot[ui], 0};
        uint64_t sb = 0, gb = 0;
        const int mode = unit_mode(tk, &sb, &gb);
        auto key = std::make_pair(task_cls(tk), mode);
        groups[key].push_back(u);
        gmax[key] = std::max<uint64_t>(gmax[key], gb);
        smax[key] = std::max<uint64_t>(smax[key], sb);
        if (mode >= 2 && mode <= 4) { uglob[ui] = gb; g_split_done++; }
      }
      // longest units first inside a group: the CTA scheduler starts them
      // early and the tail of the launch shrinks. A unit's length is its
      // trace's event count; a path unit's, its path's share (K0's counts of
      // the mallocs at or above the policy's gate; a free follows its malloc)
      auto work = [&](const Unit& u) -> uint64_t {
        const uint64_t n = offs[u.trace + 1] - offs[u.trace];
        if (!u.path) return n;
        uint64_t nv = 0;
        for (uint32_t k = 0; k < gates.size(); ++k)
          if (gates[k] == vm_thr_of(B->policies[u.policy])) nv = 2ull * nbig[(uint64_t)u.trace * (kNThr + 1) + k];
        nv = std::min(nv, n);
        return u.path == 1 ? nv : n - nv;
      };
      for (auto& g : groups)
        std::stable_sort(g.second.begin(), g.second.end(), [&](const Unit& x, const Unit& y) { return work(x) > work(y); });
      uint64_t n_all = 0, gbytes = 0;
      // persistent path launches: one arena per resident warp (GML_PATH_PERSIST)
      std::map<std::pair<int, int>, std::pair<uint64_t, uint64_t>> pgrid;   // group -> (base, slots)
      for (auto& g : groups) {
        const int mode = g.first.second;
        if (mode >= 5 && persist) {
          const uint64_t stride = (gmax[g.first] + 255) & ~255ull;
          // every warp of the grid owns an arena: whole CTAs
          const uint64_t want = std::min<uint64_t>(g.second.size(),
                                                   (uint64_t)path_ctas_cls(g.first.first) * n_sm * GML_PATH_WPC);
          const uint64_t slots = (want + GML_PATH_WPC - 1) / GML_PATH_WPC * GML_PATH_WPC;
          pgrid[g.first] = {gbytes, slots};
          gbytes += slots * stride;
        } else if (mode == 0 || mode >= 5)
          for (Unit& u : g.second) { u.arena_off = gbytes; gbytes += (gmax[g.first] + 255) & ~255ull; }
        if (mode >= 2 && mode <= 4)
          for (Unit& u : g.second) {
            u.arena_off = gbytes;
            gbytes += (uglob[u.trace * NP + u.policy] + 255) & ~255ull;
          }
        n_all += g.second.size();
      }
      CK(cudaMemsetAsync(d_novf, 0, 4, st));
      Unit* d_units = nullptr;
      uint8_t* d_garena = nullptr;
      CK(ws_get(cur_dev, WS_UNITS, sizeof(Unit) * n_all, (void**)&d_units));
      if (gbytes) CK(ws_get(cur_dev, WS_ARENA, gbytes, (void**)&d_garena));
      {
        uint64_t o = 0;
        for (auto& g : groups) {
          CK(cudaMemcpyAsync(d_units + o, g.second.data(), sizeof(Unit) * g.second.size(),
                             cudaMemcpyHostToDevice, st));
          o += g.second.size();
        }
      }
      ht.mark("round: groups + arena");
      cudaEvent_t ev0, ev1, fork;
      CK(cudaEventCreate(&ev0));
      CK(cudaEventCreate(&ev1));
      CK(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming));
      CK(cudaEventRecord(ev0, st));
      CK(cudaEventRecord(fork, st));
      KParams kp{B->events, B->trace_offsets, d_pols, nullptr, 0, NP, total, B->assignments, B->timeline, B->stats,
                 d_garena, 0, d_ovf, d_novf, d_cycles, d_prof, d_D, d_pst, dbg_flags};
      kp.bm_words_max = bmw_max(B);
      // launch the groups of the largest size classes (the longest units:
      // GMLake tables that grew, long traces) first, so that the CTA scheduler
      // starts them before the short BFC units and the tail of the step shrinks
      std::map<std::pair<int, int>, uint64_t> goff;
      {
        uint64_t o = 0;
        for (auto& g : groups) { goff[g.first] = o; o += g.second.size(); }
      }
      std::vector<std::pair<std::pair<int, int>, std::vector<Unit>*>> order;
      for (auto& g : groups) order.push_back({g.first, &g.second});
      // VMM classes first, then by class (largest first)
      std::stable_sort(order.begin(), order.end(), [](const auto& x, const auto& y) {
        const bool vx = kClasses[x.first.first].vmm, vy = kClasses[y.first.first].vmm;
        if (vx != vy) return vx;
        return x.first > y.first;
      });
      size_t gi = 0, ci = 0;
      uint32_t* d_ctr = nullptr;
      if (!pgrid.empty()) {
        CK(ws_get(cur_dev, WS_CTR, 4 * pgrid.size(), (void**)&d_ctr));
        CK(cudaMemsetAsync(d_ctr, 0, 4 * pgrid.size(), st));
      }
      CK(cudaEventRecord(fork, st));   // (after the counters' reset)
      std::vector<cudaEvent_t> joins;
      for (auto& g : order) {
        cudaStream_t ss = groups.size() == 1 ? st : side[gi++];
        if (ss != st) CK(cudaStreamWaitEvent(ss, fork, 0));
        kp.units = d_units + goff[g.first];
        kp.n_units = (uint32_t)g.second->size();
        const int mode = g.first.second, c = g.first.first;
        kp.smem_stride = (uint32_t)(((mode == 0 || mode >= 5 ? gmax[g.first] : smax[g.first]) + 15) & ~15ull);
        kp.garena = d_garena;
        kp.next_unit = nullptr;
        if (pgrid.count(g.first)) {
          kp.garena = d_garena + pgrid[g.first].first;
          kp.next_unit = d_ctr + ci++;
          kp.arena_stride = (gmax[g.first] + 255) & ~255ull;
          kp.arena_slots = pgrid[g.first].second;
        }
        gml_status r = mode >= 5   ? launch_path_cls(c, kp, ss)
                       : mode >= 2 ? launch_split_cls(c, mode - 2, kp, kp.smem_stride, ss)
                                   : launch(c, mode == 1, kp, kp.smem_stride, ss);
        if (r != GML_OK) return r;
        g_launches++;
        if (ss != st) {
          cudaEvent_t j;
          CK(cudaEventCreateWithFlags(&j, cudaEventDisableTiming));
          CK(cudaEventRecord(j, ss));
          joins.push_back(j);
        }
      }
      for (cudaEvent_t j : joins) {
        CK(cudaStreamWaitEvent(st, j, 0));
        cudaEventDestroy(j);
      }
      CK(cudaEventRecord(ev1, st));
      ht.mark("round: launches");
      uint32_t novf = 0;
      CK(cudaMemcpyAsync(&novf, d_novf, 4, cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      ht.mark("round: kernels (sync)");
      {
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, ev0, ev1));
        g_kernel_ms += ms;
        cudaEventDestroy(ev0);
        cudaEventDestroy(ev1);
        cudaEventDestroy(fork);
      }
      std::vector<Ovf> ov(novf);
      if (novf) {
        CK(cudaMemcpyAsync(ov.data(), d_ovf, sizeof(Ovf) * novf, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
      }
      // grow: handle table in place, pools to the next class of the family
      todo.clear();
      for (const Ovf& v : ov) {
        const uint32_t tk = v.unit, ui = tk & 0x3FFFFFFFu;
        if (v.mask & OV_SERIAL) {   // a split unit the single-warp replay must decide
          no_split[ui] = 1;
          g_split_reruns++;
          g_split_done--;
          todo.push_back(ui);
          continue;
        }
        if (v.mask & OV_H) hcap[ui] *= 2;
        if (uglob.count(ui)) g_split_done--;   // an overflowed split unit is counted again when it re-runs
        if (v.mask & ~OV_H) {
          int& c = task_cls(tk);
          int top = kClasses[c].vmm ? kNumClasses - 1 : kFirstVmm - 1;
          if (c >= top) { rc = GML_ERR_TABLE_OVERFLOW; continue; }
          c++;
        }
        todo.push_back(tk);
      }
      std::sort(todo.begin(), todo.end());
    }
    if (!todo.empty()) rc = GML_ERR_TABLE_OVERFLOW;
    return GML_OK;
  };

  {
    gml_status r = run_rounds(todo);
    if (r != GML_OK) return r;
  }
  std::vector<Unit> mu;   // K1m: merge each path-split unit (after its two paths and its ledger);
  for (uint64_t i = 0; i < NU; ++i)   // units whose split result is not the interleaved replay's are re-run
    if (mslot[i] != NONE32) mu.push_back(Unit{(uint32_t)(i / NP), (uint32_t)(i % NP), hcap[i], 0, 0, d_off[i], mslot[i], 0});
  if (!mu.empty()) {
    Unit* d_mu = nullptr;
    CK(ws_get(cur_dev, WS_UNITS, sizeof(Unit) * mu.size(), (void**)&d_mu));
    CK(cudaMemcpyAsync(d_mu, mu.data(), sizeof(Unit) * mu.size(), cudaMemcpyHostToDevice, st));
    CK(cudaMemsetAsync(d_novf, 0, 4, st));
    cudaEvent_t m0, m1;
    CK(cudaEventCreate(&m0));
    CK(cudaEventCreate(&m1));
    CK(cudaEventRecord(m0, st));
    k_merge<<<(uint32_t)((mu.size() + 3) / 4), 128, 0, st>>>(d_mu, (uint32_t)mu.size(), B->trace_offsets, d_pols, NP,
                                                            d_D, d_pst, d_led, B->stats, d_ovf, d_novf);
    CK(cudaGetLastError());
    g_launches++;
    CK(cudaEventRecord(m1, st));
    uint32_t novf = 0;
    CK(cudaMemcpyAsync(&novf, d_novf, 4, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, m0, m1));
    g_kernel_ms += ms;
    cudaEventDestroy(m0);
    cudaEventDestroy(m1);
    std::vector<Ovf> ov(novf);
    if (novf) {
      CK(cudaMemcpyAsync(ov.data(), d_ovf, sizeof(Ovf) * novf, cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
    }
    ht.mark("merge");
    std::vector<uint32_t> again;
    for (const Ovf& v : ov) {
      no_split[v.unit] = 1;
      mslot[v.unit] = NONE32;
      g_split_reruns++;
      g_split_done--;
      again.push_back(v.unit);
    }
    std::sort(again.begin(), again.end());
    gml_status r = run_rounds(again);
    if (r != GML_OK) return r;
  }
  if (dbg_cycles) {
    std::vector<unsigned long long> cy(NU), pr(16 * NU);
    CK(cudaMemcpyAsync(cy.data(), d_cycles, 8 * NU, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(pr.data(), d_prof, 8 * 16 * NU, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    for (uint64_t i = 0; i < NU; ++i) {
      fprintf(stderr, "gml-unit trace %llu policy %llu class %d cycles %llu events %llu phases",
              (unsigned long long)(i / NP), (unsigned long long)(i % NP), cls[i], cy[i],
              (unsigned long long)(offs[i / NP + 1] - offs[i / NP]));
      for (int k = 0; k < 16; ++k) fprintf(stderr, " %llu", pr[16 * i + k]);
      fprintf(stderr, "\n");
    }
  }
  if (B->caps)
    for (uint64_t i = 0; i < NU; ++i) {
      const ClassInfo& k = kClasses[cls[i]];
      const uint32_t bb = (k.vmm && path_on && B->policies[i % NP].kind == GML_POLICY_GMLAKE) ? kClasses[cls_s[i]].b : k.b;
      B->caps[i] = gml_replay_caps{k.vmm ? k.p : 0, k.vmm ? k.s : 0, k.vmm ? k.iv : 0, bb};
    }
  CK(cudaStreamSynchronize(st));
  ht.mark("end");
  return rc;
}

}  // extern "C"
