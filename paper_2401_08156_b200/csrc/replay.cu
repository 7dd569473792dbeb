// replay.cu -- K0 (per-trace slot scan) and K1 (batched trace replay) for
// sm_100a, plus the host side of gml_replay / gml_trace_validate / metrics.
//
// K1 maps one warp to one (trace, policy) unit:
//   a1  events stream HBM -> registers, 32 per warp-wide coalesced 8-byte
//       load, the next batch prefetched while the current one is replayed;
//       event j is broadcast from lane j with one shuffle.
//   a2-a9  gml::Engine<DeviceWarp>::step (policy.cuh) on tables in shared
//       memory (or, when a unit's tables do not fit, a global-memory arena).
//   a10 peaks sampled after every event in registers; the record of event j
//       is kept by lane j and written back as one coalesced 256-byte store per
//       32 events; the 272-byte stats record is written at the end.
// Units whose tables overflow are re-run by the host with larger tables, so a
// table size never changes a result (D30).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <vector>

#include "gml.h"
#include "policy.cuh"

using gml::Caps;
using gml::DeviceWarp;
using gml::Engine;
using gml::Layout;

namespace {

constexpr uint32_t kSmemMax = 227 * 1024;
thread_local uint32_t g_launches = 0;

struct Unit {
  uint32_t trace, policy;
  Caps caps;
  uint64_t arena_off;   // global-arena offset (global kernel only)
};

struct Ovf {
  uint32_t unit, mask;
};

// K0: 1 + max slot of every trace (sizes the handle table).
__global__ void k_max_slot(const uint64_t* __restrict__ ev, const uint64_t* __restrict__ offs,
                           uint32_t n_traces, uint32_t* __restrict__ out) {
  for (uint32_t t = blockIdx.x; t < n_traces; t += gridDim.x) {
    uint64_t b = offs[t], e = offs[t + 1];
    uint32_t m = 0;
    for (uint64_t i = b + threadIdx.x; i < e; i += blockDim.x) {
      uint32_t s = (uint32_t)((__ldg(ev + i) >> 40) & 0x7FFFFFu) + 1;
      m = max(m, s);
    }
    m = __reduce_max_sync(0xFFFFFFFFu, m);
    __shared__ uint32_t red[32];
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x < 32) {
      uint32_t v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0;
      v = __reduce_max_sync(0xFFFFFFFFu, v);
      if (threadIdx.x == 0) out[t] = v;
    }
    __syncthreads();
  }
}

struct KParams {
  const uint64_t* events;
  const uint64_t* offs;
  const gml_policy* pols;
  const Unit* units;
  uint32_t n_units;
  uint32_t n_policies;
  uint64_t total_events;
  uint64_t* asg;
  gml_stats_t* stats;
  uint8_t* garena;
  uint32_t smem_stride;
  Ovf* ovf;
  uint32_t* n_ovf;
};

template <bool kSmem>
__global__ void __launch_bounds__(128) k_replay(KParams P) {
  extern __shared__ __align__(16) uint8_t smem[];
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t wpc = blockDim.x >> 5;
  const uint32_t ui = blockIdx.x * wpc + (threadIdx.x >> 5);
  if (ui >= P.n_units) return;
  const Unit u = P.units[ui];
  uint8_t* arena = kSmem ? smem + (threadIdx.x >> 5) * P.smem_stride : P.garena + u.arena_off;
  const gml_policy pol = P.pols[u.policy];

  Engine<DeviceWarp> E;
  E.init(pol, u.caps, arena, nullptr);

  const uint64_t b = P.offs[u.trace];
  const uint64_t n = P.offs[u.trace + 1] - b;
  const uint64_t* ev = P.events + b;
  uint64_t* asg = P.asg ? P.asg + (uint64_t)u.policy * P.total_events + b : nullptr;

  uint64_t done = 0;
  int64_t oom_event = -1;
  bool stop = false;
  uint64_t cur = lane < n ? __ldcs(ev + lane) : 0;
  uint64_t base = 0;
  for (; base < n && !stop; base += 32) {
    const uint64_t nb = base + 32 + lane;
    const uint64_t nxt = nb < n ? __ldcs(ev + nb) : 0;     // prefetch the next batch
    const uint32_t cnt = (n - base) < 32 ? (uint32_t)(n - base) : 32u;
    uint64_t myrec = 0;
    for (uint32_t j = 0; j < cnt; ++j) {
      const uint64_t e = __shfl_sync(0xFFFFFFFFu, cur, j);
      const uint64_t r = E.step(e);
      if (lane == j) myrec = r;
      if (E.overflow | E.status) {
        if (E.status == GML_ERR_OOM) oom_event = (int64_t)(base + j);
        stop = true;
        break;
      }
      E.sample();
      ++done;
    }
    if (asg && base + lane < n) __stcs(asg + base + lane, myrec);
    cur = nxt;
  }
  if (stop && asg && !E.overflow) {   // records after the terminating event are 0
    for (uint64_t i = base + lane; i < n; i += 32) __stcs(asg + i, 0ull);
  }
  E.finish(n, done, oom_event);
  // stats record -> global
  const uint32_t* src = reinterpret_cast<const uint32_t*>(E.st);
  uint32_t* dst = reinterpret_cast<uint32_t*>(P.stats + (uint64_t)u.trace * P.n_policies + u.policy);
  for (uint32_t i = lane; i < sizeof(gml_stats_t) / 4; i += 32) dst[i] = src[i];
  if (lane == 0) {
    dst[offsetof(gml_stats_t, _p) / 4] = 0;
    if (E.overflow) {
      uint32_t k = atomicAdd(P.n_ovf, 1u);
      P.ovf[k] = Ovf{u.trace * P.n_policies + u.policy, E.overflow};
    }
  }
}

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e_ = (x);                                                       \
    if (e_ != cudaSuccess) {                                                    \
      fprintf(stderr, "gml: %s failed: %s\n", #x, cudaGetErrorString(e_));      \
      return GML_ERR_CUDA;                                                      \
    }                                                                           \
  } while (0)

Caps default_caps(const gml_policy& p, uint32_t max_slots, const gml_replay_caps* hint) {
  Caps c{};
  uint64_t chunks = p.capacity_bytes / p.chunk_bytes + 1;
  c.bm_words = (uint32_t)((chunks + 31) / 32);
  c.h = std::max<uint32_t>(max_slots, 1);
  bool vmm = p.kind == GML_POLICY_GMLAKE;
  c.p = vmm ? 1024 : 1;
  c.s = vmm ? 512 : 1;
  c.iv = vmm ? 1024 : 1;
  c.b = vmm ? 512 : 2048;
  if (hint) {
    if (vmm && hint->pblocks) c.p = hint->pblocks;
    if (vmm && hint->sblocks) c.s = hint->sblocks;
    if (vmm && hint->intervals) c.iv = hint->intervals;
    if (hint->bfc_blocks) c.b = hint->bfc_blocks;
  }
  c.cb = c.p + 2;
  return c;
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

gml_status gml_replay(const gml_trace_batch* B) {
  g_launches = 0;
  if (!B || !B->events || !B->trace_offsets || !B->policies || !B->stats || B->n_traces == 0 ||
      B->n_policies == 0)
    return GML_ERR_INVALID;
  for (uint32_t p = 0; p < B->n_policies; ++p) {
    const gml_policy& q = B->policies[p];
    if (q.kind > GML_POLICY_GMLAKE || q.chunk_bytes == 0 || q.chunk_bytes % 512 ||
        q.capacity_bytes / q.chunk_bytes >= (1ull << 31) || q.spool_max_entries == 0)
      return GML_ERR_INVALID;
  }
  cudaStream_t st = (cudaStream_t)B->stream;
  const uint32_t NT = B->n_traces, NP = B->n_policies;
  const uint64_t NU = (uint64_t)NT * NP;

  // trace offsets + per-trace slot counts (K0)
  std::vector<uint64_t> offs(NT + 1);
  CK(cudaMemcpyAsync(offs.data(), B->trace_offsets, 8ull * (NT + 1), cudaMemcpyDeviceToHost, st));
  uint32_t *d_slots = nullptr, *d_novf = nullptr;
  gml_policy* d_pols = nullptr;
  CK(cudaMallocAsync(&d_slots, 4ull * NT, st));
  k_max_slot<<<std::min<uint32_t>(NT, 148 * 8), 256, 0, st>>>(B->events, B->trace_offsets, NT, d_slots);
  g_launches++;
  CK(cudaGetLastError());
  std::vector<uint32_t> slots(NT);
  CK(cudaMemcpyAsync(slots.data(), d_slots, 4ull * NT, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  const uint64_t total = offs[NT];
  for (uint32_t t = 0; t < NT; ++t)
    if (offs[t + 1] < offs[t]) return GML_ERR_INVALID;

  CK(cudaMallocAsync(&d_pols, sizeof(gml_policy) * NP, st));
  CK(cudaMemcpyAsync(d_pols, B->policies, sizeof(gml_policy) * NP, cudaMemcpyHostToDevice, st));

  std::vector<Caps> caps(NU);
  for (uint32_t t = 0; t < NT; ++t)
    for (uint32_t p = 0; p < NP; ++p)
      caps[(uint64_t)t * NP + p] =
          default_caps(B->policies[p], slots[t], B->caps ? &B->caps[(uint64_t)t * NP + p] : nullptr);

  std::vector<uint32_t> todo(NU);
  for (uint64_t i = 0; i < NU; ++i) todo[i] = (uint32_t)i;
  Ovf* d_ovf = nullptr;
  CK(cudaMallocAsync(&d_ovf, sizeof(Ovf) * NU, st));
  CK(cudaMallocAsync(&d_novf, 4, st));
  gml_status rc = GML_OK;

  for (int round = 0; !todo.empty() && round < 24; ++round) {
    // split the work into shared-memory and global-arena launches
    std::vector<Unit> us, ug;
    uint32_t smax = 0;
    uint64_t gbytes = 0;
    for (uint32_t ui : todo) {
      Unit u{ui / NP, ui % NP, caps[ui], 0};
      uint64_t by = Layout::make(u.caps).bytes;
      if (by <= kSmemMax) {
        us.push_back(u);
        smax = std::max<uint32_t>(smax, (uint32_t)by);
      } else {
        u.arena_off = gbytes;
        gbytes += (by + 255) & ~255ull;
        ug.push_back(u);
      }
    }
    CK(cudaMemsetAsync(d_novf, 0, 4, st));
    Unit* d_units = nullptr;
    uint8_t* d_garena = nullptr;
    CK(cudaMallocAsync(&d_units, sizeof(Unit) * (us.size() + ug.size()), st));
    if (!us.empty())
      CK(cudaMemcpyAsync(d_units, us.data(), sizeof(Unit) * us.size(), cudaMemcpyHostToDevice, st));
    if (!ug.empty())
      CK(cudaMemcpyAsync(d_units + us.size(), ug.data(), sizeof(Unit) * ug.size(), cudaMemcpyHostToDevice, st));
    if (gbytes) CK(cudaMallocAsync(&d_garena, gbytes, st));
    KParams kp{B->events, B->trace_offsets, d_pols, nullptr, 0, NP, total, B->assignments, B->stats,
               d_garena, 0, d_ovf, d_novf};
    if (!us.empty()) {
      kp.units = d_units;
      kp.n_units = (uint32_t)us.size();
      kp.smem_stride = (smax + 15) & ~15u;
      const uint32_t wpc = 1;
      CK(cudaFuncSetAttribute(k_replay<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)(kp.smem_stride * wpc)));
      uint32_t grid = (uint32_t)((us.size() + wpc - 1) / wpc);
      k_replay<true><<<grid, 32 * wpc, kp.smem_stride * wpc, st>>>(kp);
      g_launches++;
      CK(cudaGetLastError());
    }
    if (!ug.empty()) {
      kp.units = d_units + us.size();
      kp.n_units = (uint32_t)ug.size();
      const uint32_t wpc = 4;
      uint32_t grid = (uint32_t)((ug.size() + wpc - 1) / wpc);
      k_replay<false><<<grid, 32 * wpc, 0, st>>>(kp);
      g_launches++;
      CK(cudaGetLastError());
    }
    uint32_t novf = 0;
    CK(cudaMemcpyAsync(&novf, d_novf, 4, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    std::vector<Ovf> ov(novf);
    if (novf) {
      CK(cudaMemcpyAsync(ov.data(), d_ovf, sizeof(Ovf) * novf, cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
    }
    CK(cudaFreeAsync(d_units, st));
    if (d_garena) CK(cudaFreeAsync(d_garena, st));
    // map launch-local unit indices back and grow the overflowed tables
    todo.clear();
    for (const Ovf& o : ov) {
      uint32_t ui = o.unit;
      Caps& c = caps[ui];
      if (o.mask & gml::OV_P) { c.p *= 2; c.cb = c.p + 2; }
      if (o.mask & gml::OV_S) c.s *= 2;
      if (o.mask & gml::OV_IV) c.iv *= 2;
      if (o.mask & gml::OV_B) c.b *= 2;
      if (o.mask & gml::OV_CB) c.cb *= 2;
      if (o.mask & gml::OV_H) c.h *= 2;
      todo.push_back(ui);
    }
    std::sort(todo.begin(), todo.end());
    if (round == 23 && !todo.empty()) rc = GML_ERR_TABLE_OVERFLOW;
  }
  if (B->caps)
    for (uint64_t i = 0; i < NU; ++i)
      B->caps[i] = gml_replay_caps{caps[i].p, caps[i].s, caps[i].iv, caps[i].b};
  CK(cudaFreeAsync(d_slots, st));
  CK(cudaFreeAsync(d_pols, st));
  CK(cudaFreeAsync(d_ovf, st));
  CK(cudaFreeAsync(d_novf, st));
  CK(cudaStreamSynchronize(st));
  return rc;
}

}  // extern "C"
