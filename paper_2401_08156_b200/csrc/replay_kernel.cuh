// replay_kernel.cuh -- K1 kernel template and its launcher, included by the
// per-size-class translation units (classes_*.cu) so that the 40 kernel
// instances compile in parallel.
#pragma once
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <type_traits>

#include "gml.h"
#include "policy.cuh"

#ifndef GML_GLOBAL_WPC
#define GML_GLOBAL_WPC 4    // units (warps) per CTA for global-arena units
#endif
#ifndef GML_GLOBAL_MINB
#define GML_GLOBAL_MINB (8 / GML_GLOBAL_WPC)   // 8 resident units per SM (254 registers)
#endif
#ifndef GML_BFC_MINB
#define GML_BFC_MINB 4      // BFC-family instances carry no VMM path (Cfg::VMM): fewer registers, more CTAs
#endif
#ifndef GML_FREE_RUN
#define GML_FREE_RUN 1      // split units' VMM warp: runs of consecutive frees through Engine::free_run
#endif                      // (the single-warp K1 steps frees one by one: measured C4 +10 %, C3 +4 % with runs)
#ifndef GML_EV_LOAD
#define GML_EV_LOAD 1       // event loads: 0 = evict-first (__ldcs), 1 = default (__ldg, measured: C4 DRAM reads 1.04 -> 0.69 GB), 2 = L2 evict_last
#endif

namespace gml {
namespace replay {

// ---- size classes: BFC family (policies without pools) and GMLake family ----
using C0 = Cfg<4, 4, 4, 1024>;
using C1 = Cfg<4, 4, 4, 2048>;
using C2 = Cfg<4, 4, 4, 4096>;
using C3 = Cfg<4, 4, 4, 32768>;
using C4 = Cfg<4, 4, 4, 262144>;
using C5 = Cfg<512, 256, 1024, 512>;
using C6 = Cfg<1024, 512, 2048, 2048>;     // C2 / C3 GMLake units: 164 KiB + handles, in shared memory
using C7 = Cfg<2048, 1024, 4096, 2048>;
using C8 = Cfg<4096, 2048, 8192, 4096>;
using C9 = Cfg<65536, 32768, 65536, 32768>;
using C10 = Cfg<131072, 65536, 131072, 131072>;   // every chunk of a 256 GiB pool its own pBlock
#define GML_CLASSES(X) \
  X(0, C0) X(1, C1) X(2, C2) X(3, C3) X(4, C4) X(5, C5) X(6, C6) X(7, C7) X(8, C8) X(9, C9) X(10, C10)

struct ClassInfo {
  uint32_t p, s, iv, b;
  bool vmm;
};
constexpr int kNumClasses = 11;
constexpr int kFirstVmm = 5;
#define GML_INFO(I, CF) {CF::P, CF::S, CF::IV, CF::B, I >= kFirstVmm},
const ClassInfo kClasses[kNumClasses] = {GML_CLASSES(GML_INFO)};
#undef GML_INFO


#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e_ = (x);                                                       \
    if (e_ != cudaSuccess) {                                                    \
      fprintf(stderr, "gml: %s failed: %s\n", #x, cudaGetErrorString(e_));      \
      return GML_ERR_CUDA;                                                      \
    }                                                                           \
  } while (0)

struct Unit {
  uint32_t trace, policy, h;
  uint32_t path;        // 0 whole unit; 1 / 2: the VMM / small path of a path-split unit
  uint64_t arena_off;   // global-arena offset (global launches only)
  uint64_t d_off;       // path units: the unit's per-event series in KParams::pd (u32 words)
  uint32_t mslot, _pad; // path units: the unit's pair of records in KParams::pstats
};

struct Ovf {
  uint32_t unit, mask;
};

struct KParams {
  const uint64_t* events;
  const uint64_t* offs;
  const gml_policy* pols;
  const Unit* units;
  uint32_t n_units;
  uint32_t n_policies;
  uint64_t total_events;
  uint64_t* asg;
  uint64_t* tl;                 // optional (active, reserved) per event
  gml_stats_t* stats;
  uint8_t* garena;
  uint32_t smem_stride;
  Ovf* ovf;
  uint32_t* n_ovf;
  unsigned long long* cycles;   // optional per-unit clock64 deltas (GML_UNIT_CYCLES debug)
  unsigned long long* prof;     // optional per-unit phase counters [16] (GML_PHASE_PROF builds)
  uint32_t* pd;                 // path units: per-event active series (split_kernel.cuh)
  gml_stats_t* pstats;          // path units: [unit][VMM path, small path] stats records
  uint32_t dbg;                 // debug (GML_SPLIT_VMM_ONLY): split units run their VMM warp alone, no result
  uint32_t* next_unit;          // persistent path launches: the work counter (else NULL)
  uint64_t arena_stride;        // persistent path launches: bytes per warp arena
  uint64_t arena_slots;         // persistent path launches: warps (= arenas) of the grid
  uint32_t bm_words_max;        // chunk-bitmap words of the largest policy capacity
  uint32_t quick_words;         // path launches: shared-memory words per warp (PIN [+ bitmap])
};


// One warp per (trace, policy) unit. Shared-memory arenas: one unit (warp)
// per CTA, the whole shared memory of an SM slot for its tables; global-memory
// arenas (L1/L2-resident): GML_GLOBAL_WPC units per CTA, GML_GLOBAL_MINB CTAs per SM.
__device__ __forceinline__ uint32_t bm_words_of(const gml_policy& p) {
  return (uint32_t)((p.capacity_bytes / p.chunk_bytes + 1 + 31) / 32);
}

// event stream loads: the V policy units of a trace read the same events
__device__ __forceinline__ uint64_t ld_event(const uint64_t* p) {
#if GML_EV_LOAD == 0
  return __ldcs(p);
#elif GML_EV_LOAD == 1
  return __ldg(p);
#else
  uint64_t v, pol;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  asm volatile("ld.global.nc.L2::cache_hint.u64 %0, [%1], %2;" : "=l"(v) : "l"(p), "l"(pol));
  return v;
#endif
}

template <class CF, bool kSmem>
__global__ void __launch_bounds__(kSmem ? 32 : 32 * GML_GLOBAL_WPC, kSmem ? 1 : (CF::VMM ? GML_GLOBAL_MINB : GML_BFC_MINB * 4 / GML_GLOBAL_WPC))
    k_replay(const __grid_constant__ KParams P) {
  extern __shared__ __align__(16) uint8_t smem[];
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t wpc = blockDim.x >> 5;
  const uint32_t slot_in_cta = threadIdx.x >> 5;
  const uint32_t ui = blockIdx.x * wpc + slot_in_cta;
  if (ui >= P.n_units) return;
  const Unit u = P.units[ui];
  uint8_t* arena = P.garena + u.arena_off;
  if (kSmem) {
    // the shared-window address of the arena, made opaque so that it stays in
    // a register: otherwise ptxas rematerializes it (S2R SR_CgaCtaId + LEA)
    // at every block that touches the arena, on the unit's dependent chain
    // (measured: C2 units 4-7 % slower)
    uint32_t sa = (uint32_t)__cvta_generic_to_shared(smem);
    asm volatile("" : "+r"(sa));
    arena = static_cast<uint8_t*>(__cvta_shared_to_generic(sa));
  }
  const gml_policy pol = P.pols[u.policy];

  const long long c0 = clock64();
  Engine<DeviceWarp, CF, NoHooks, kSmem> E;
  E.init(pol, RtCaps{bm_words_of(pol), u.h}, arena, nullptr);
  if (P.prof) E.prof = P.prof + 16ull * (u.trace * P.n_policies + u.policy);

  const uint64_t b = P.offs[u.trace];
  const uint64_t n = P.offs[u.trace + 1] - b;
  const uint64_t* ev = P.events + b;
  uint64_t* asg = P.asg ? P.asg + (uint64_t)u.policy * P.total_events + b : nullptr;
  ulonglong2* tl = P.tl ? reinterpret_cast<ulonglong2*>(P.tl) + (uint64_t)u.policy * P.total_events + b : nullptr;

  int64_t oom_event = -1;
  bool stop = false;
  uint64_t stop_at = n;    // events completed before the terminating one
  uint64_t cur = lane < n ? ld_event(ev + lane) : 0;
  uint64_t base = 0;
  for (; base < n && !stop; base += 32) {
    const uint64_t nb = base + 32 + lane;
    const uint64_t nxt = nb < n ? ld_event(ev + nb) : 0;   // prefetch the next batch
    const uint32_t cnt = (n - base) < 32 ? (uint32_t)(n - base) : 32u;
    uint64_t myrec = 0;
    for (uint32_t j = 0; j < cnt; ++j) {
      const uint64_t e = __shfl_sync(0xFFFFFFFFu, cur, j);
      const uint64_t r = E.step(e);
      if (lane == j) myrec = r;
      // timeline (optional): a store cannot be speculated, so without a
      // timeline this costs one branch per event
      if (tl) {
        if (lane == 0) __stcs(tl + base + j, make_ulonglong2(E.active, E.reserved()));
      }
      if (E.overflow | E.status) {
        if (E.status == GML_ERR_OOM) oom_event = (int64_t)(base + j);
        stop = true;
        stop_at = base + j;
        break;
      }
    }
    if (asg && base + lane < n) __stcs(asg + base + lane, myrec);
    cur = nxt;
  }
  if (stop && asg && !E.overflow) {   // records after the terminating event are 0
    for (uint64_t i = base + lane; i < n; i += 32) __stcs(asg + i, 0ull);
  }
  if (stop && tl && !E.overflow) {   // (the terminating event keeps its sample)
    for (uint64_t i = stop_at + 1 + lane; i < n; i += 32) __stcs(tl + i, make_ulonglong2(0ull, 0ull));
  }
  const uint64_t done = stop_at;
  E.finish(n, done, oom_event);
  // stats record -> global
  const uint32_t* src = reinterpret_cast<const uint32_t*>(E.S());
  uint32_t* dst = reinterpret_cast<uint32_t*>(P.stats + (uint64_t)u.trace * P.n_policies + u.policy);
  for (uint32_t i = lane; i < sizeof(gml_stats_t) / 4; i += 32) dst[i] = src[i];
  if (lane == 0) {
    if (P.cycles) P.cycles[u.trace * P.n_policies + u.policy] = (unsigned long long)(clock64() - c0);
    dst[offsetof(gml_stats_t, _p) / 4] = 0;
    if (E.overflow) {
      uint32_t k = atomicAdd(P.n_ovf, 1u);
      P.ovf[k] = Ovf{u.trace * P.n_policies + u.policy, E.overflow};
    }
  }
}


template <class CF, bool kSmem>
gml_status launch_class(const KParams& kp, uint32_t smem_stride, cudaStream_t st) {
  const uint32_t wpc = kSmem ? 1 : GML_GLOBAL_WPC;
  if (kSmem) {
    CK(cudaFuncSetAttribute(k_replay<CF, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_stride));
  }
  // GML_GLOBAL_SMEM_PAD (experiments only): unused dynamic shared memory per
  // global-arena CTA, to cap resident CTAs per SM
  static const uint32_t pad = [] { const char* e = getenv("GML_GLOBAL_SMEM_PAD"); return e ? (uint32_t)atoi(e) : 0u; }();
  if (!kSmem && pad) CK(cudaFuncSetAttribute(k_replay<CF, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pad));
  uint32_t grid = (kp.n_units + wpc - 1) / wpc;
  k_replay<CF, kSmem><<<grid, 32 * wpc, kSmem ? smem_stride : pad, st>>>(kp);
  CK(cudaGetLastError());
  return GML_OK;
}


// per-class entry points (defined in classes_<I>.cu)
#define GML_DECL(I, CF) \
  gml_status launch_cls_##I(bool smem, const KParams& kp, uint32_t stride, cudaStream_t st); \
  gml_status launch_path_##I(const KParams& kp, cudaStream_t st); \
  uint32_t path_ctas_##I();
GML_CLASSES(GML_DECL)
#undef GML_DECL

}  // namespace replay
}  // namespace gml
