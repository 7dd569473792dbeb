// live.cu -- the live GMLake allocator over the CUDA VMM driver API
// (SURVEY §8(a) row a12): gml_create / gml_malloc / gml_free / gml_stats /
// gml_destroy. Decisions come from the same gml::Engine as the replay kernel
// (policy.cuh), instantiated with a width-1 HostWarp and hooks that turn them
// into driver calls:
//
//   Alloc(n chunks)  cuMemAddressReserve + n x (cuMemCreate(chunk) + cuMemMap)
//                    + ONE cuMemSetAccess over the range.
//                    Every 2 MiB chunk is its own physical handle (L319):
//                    cuMemMap maps whole handles (offset 0), so a chunk is the
//                    unit any later Split / Stitch can re-map.
//   Split            no call: F and R are sub-ranges of the parent's mapping
//                    (the paper re-reserves and remaps, L378).
//   Stitch           cuMemAddressReserve(sum) + one cuMemMap per member chunk
//                    + ONE cuMemSetAccess for the whole range (L381-387;
//                    Table 1 shows set-access dominating, L241). A stitch whose members are contiguous
//                    inside one Alloc (the [F, R] companion) reuses that VA.
//   StitchFree       cuMemUnmap per chunk + cuMemAddressFree of the sBlock VA;
//                    the chunks stay with their pBlocks (L490). The unmap is
//                    deferred behind an event on the allocator's stream
//                    (gml_set_stream): work queued before the sBlock's last
//                    free may still read through the VA. No device-wide sync.
//
// A failed driver call (cuMemCreate / cuMemMap / cudaMalloc out of memory) is
// rolled back inside the hook, the engine commits nothing and reports S5
// ("If the Alloc function call fails, GMLake immediately reports an OOM",
// L528): gml_malloc returns GML_ERR_OOM and the allocator stays usable.
//   small path       cudaMalloc / cudaFree segments (PyTorch's BFC, L322).
//
// The driver API is reached through cudaGetDriverEntryPoint, so libgml.so
// does not link libcuda and loads on machines without a GPU.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <chrono>
#include <cstring>
#include <map>
#include <new>
#include <unordered_map>
#include <vector>

#include "gml.h"
#include "policy.cuh"

using namespace gml;

namespace {

// tables for the host engine: worst case 180 GiB / 2 MiB chunks
using CfgLive = Cfg<131072, 65536, 131072, 131072>;
constexpr uint32_t kLiveSlots = 1u << 20;

struct Drv {
  bool ok = false;
  CUresult (*reserve)(CUdeviceptr*, size_t, size_t, CUdeviceptr, unsigned long long) = nullptr;
  CUresult (*create)(CUmemGenericAllocationHandle*, size_t, const CUmemAllocationProp*, unsigned long long) = nullptr;
  CUresult (*map)(CUdeviceptr, size_t, size_t, CUmemGenericAllocationHandle, unsigned long long) = nullptr;
  CUresult (*set_access)(CUdeviceptr, size_t, const CUmemAccessDesc*, size_t) = nullptr;
  CUresult (*unmap)(CUdeviceptr, size_t) = nullptr;
  CUresult (*addr_free)(CUdeviceptr, size_t) = nullptr;
  CUresult (*release)(CUmemGenericAllocationHandle) = nullptr;
  CUresult (*granularity)(size_t*, const CUmemAllocationProp*, CUmemAllocationGranularity_flags) = nullptr;
  CUresult (*device_get)(CUdevice*, int) = nullptr;
  CUresult (*device_attr)(int*, CUdevice_attribute, CUdevice) = nullptr;
};

bool load_driver(Drv& d) {
  auto get = [](const char* name, void** fn) {
    cudaDriverEntryPointQueryResult q;
    return cudaGetDriverEntryPoint(name, fn, cudaEnableDefault, &q) == cudaSuccess &&
           q == cudaDriverEntryPointSuccess && *fn;
  };
  d.ok = get("cuMemAddressReserve", (void**)&d.reserve) && get("cuMemCreate", (void**)&d.create) &&
         get("cuMemMap", (void**)&d.map) && get("cuMemSetAccess", (void**)&d.set_access) &&
         get("cuMemUnmap", (void**)&d.unmap) && get("cuMemAddressFree", (void**)&d.addr_free) &&
         get("cuMemRelease", (void**)&d.release) &&
         get("cuMemGetAllocationGranularity", (void**)&d.granularity) &&
         get("cuDeviceGet", (void**)&d.device_get) && get("cuDeviceGetAttribute", (void**)&d.device_attr);
  return d.ok;
}

enum { D_RESERVE, D_CREATE, D_MAP, D_ACCESS, D_UNMAP, D_ADDR_FREE, D_RELEASE };

struct AllocRec {             // one Alloc: its chunks [lo, lo+n) and their mapping
  uint32_t lo, n;
  CUdeviceptr va;
};

struct SRec {
  CUdeviceptr va = 0;
  size_t bytes = 0;
  bool borrowed = false;      // VA of an existing Alloc mapping (no calls)
};

}  // namespace

struct gml_allocator;

namespace {

struct LiveHooks {
  static constexpr bool kCanFail = true;
  gml_allocator* a;
  bool on_alloc(uint32_t row, uint32_t lo, uint32_t n);
  void on_split(uint32_t, uint32_t, uint32_t, uint32_t) {}
  bool on_stitch(uint32_t row, const uint32_t* lo, const uint32_t* n, uint32_t k);
  void on_evict(uint32_t row);
  bool on_bfc_segment(uint32_t seg, uint64_t bytes);
  void on_bfc_release(uint32_t seg);
};

struct Pending {              // an evicted sBlock VA, unmapped once `ev` completed
  CUdeviceptr va;
  size_t bytes;
  cudaEvent_t ev;
};

}  // namespace

struct gml_allocator {
  int device = 0;
  gml_policy pol{};
  Drv drv;
  CUmemAllocationProp prop{};
  CUmemAccessDesc access{};
  uint8_t* arena = nullptr;
  Engine<HostWarp, CfgLive, LiveHooks> E;
  LiveHooks hooks{};
  std::map<uint32_t, AllocRec> allocs;           // by first chunk
  std::vector<CUmemGenericAllocationHandle> chunk;  // physical handle of every chunk
  std::vector<SRec> sva;                          // by sBlock row
  std::unordered_map<uint32_t, void*> segs;       // BFC segment ordinal -> cudaMalloc pointer
  std::unordered_map<uintptr_t, uint32_t> slot_of; // live pointer -> slot
  std::vector<uint32_t> free_slots;
  uint32_t next_slot = 0;
  uint64_t calls[7] = {0, 0, 0, 0, 0, 0, 0};
  cudaStream_t stream = nullptr;                  // gml_set_stream (default: the legacy default stream)
  std::vector<Pending> pending;                   // deferred StitchFree unmaps
  uint64_t n_driver_failures = 0;
  uint64_t last_rec = 0;                          // assignment record of the last malloc / free

  const AllocRec& alloc_of(uint32_t chunk) const {
    auto it = allocs.upper_bound(chunk);
    --it;
    return it->second;
  }
  CUdeviceptr va_of_chunk(uint32_t chunk) const {
    const AllocRec& r = alloc_of(chunk);
    return r.va + (CUdeviceptr)(chunk - r.lo) * pol.chunk_bytes;
  }
  bool ok(CUresult r, const char* what) {
    if (r == CUDA_SUCCESS) return true;
    n_driver_failures++;
    if (getenv("GML_LIVE_VERBOSE")) fprintf(stderr, "gml live: %s failed (%d)\n", what, (int)r);
    return false;
  }
};

namespace {

void unmap_range(gml_allocator& A, CUdeviceptr va, size_t bytes, size_t mapped);

bool LiveHooks::on_alloc(uint32_t, uint32_t lo, uint32_t n) {
  gml_allocator& A = *a;
  const size_t G = A.pol.chunk_bytes;
  size_t bytes = (size_t)n * G;
  AllocRec rec{lo, n, 0};
  A.calls[D_RESERVE]++;
  if (!A.ok(A.drv.reserve(&rec.va, bytes, 0, 0, 0), "cuMemAddressReserve")) return false;
  if (A.chunk.size() < (size_t)lo + n) A.chunk.resize((size_t)lo + n, 0);
  uint32_t c = 0;
  bool good = true;
  for (; c < n; ++c) {
    A.calls[D_CREATE]++;
    if (!A.ok(A.drv.create(&A.chunk[lo + c], G, &A.prop, 0), "cuMemCreate")) { good = false; break; }
    A.calls[D_MAP]++;
    if (!A.ok(A.drv.map(rec.va + (size_t)c * G, G, 0, A.chunk[lo + c], 0), "cuMemMap")) {
      A.drv.release(A.chunk[lo + c]);
      good = false;
      break;
    }
  }
  if (good) {
    A.calls[D_ACCESS]++;
    good = A.ok(A.drv.set_access(rec.va, bytes, &A.access, 1), "cuMemSetAccess");
  }
  if (!good) {   // roll back: the c chunks created and mapped so far, then the VA
    unmap_range(A, rec.va, bytes, (size_t)c * G);
    for (uint32_t i = 0; i < c; ++i) { A.drv.release(A.chunk[lo + i]); A.chunk[lo + i] = 0; }
    return false;
  }
  A.allocs[lo] = rec;
  return true;
}

bool LiveHooks::on_stitch(uint32_t row, const uint32_t* lo, const uint32_t* n, uint32_t k) {
  gml_allocator& A = *a;
  const size_t G = A.pol.chunk_bytes;
  if (A.sva.size() <= row) A.sva.resize(row + 1);
  SRec s;
  size_t total = 0;
  bool contiguous = true;
  const AllocRec& first = A.alloc_of(lo[0]);
  for (uint32_t i = 0; i < k; ++i) {
    total += (size_t)n[i] * G;
    if (i && lo[i] != lo[i - 1] + n[i - 1]) contiguous = false;
    if (lo[i] < first.lo || lo[i] + n[i] > first.lo + first.n) contiguous = false;
  }
  s.bytes = total;
  if (contiguous) {                      // e.g. the [F, R] companion: already mapped
    s.va = A.va_of_chunk(lo[0]);
    s.borrowed = true;
  } else {
    A.calls[D_RESERVE]++;
    if (!A.ok(A.drv.reserve(&s.va, total, 0, 0, 0), "cuMemAddressReserve")) { A.sva[row] = SRec{}; return false; }
    size_t off = 0;
    bool good = true;
    for (uint32_t i = 0; i < k && good; ++i)
      for (uint32_t c = 0; c < n[i]; ++c, off += G) {
        A.calls[D_MAP]++;
        if (!A.ok(A.drv.map(s.va + off, G, 0, A.chunk[lo[i] + c], 0), "cuMemMap")) { good = false; break; }
      }
    if (good) {
      A.calls[D_ACCESS]++;
      good = A.ok(A.drv.set_access(s.va, total, &A.access, 1), "cuMemSetAccess");
    }
    if (!good) {
      unmap_range(A, s.va, total, off);
      A.sva[row] = SRec{};
      return false;
    }
  }
  A.sva[row] = s;
  return true;
}

// unmap the first `mapped` bytes of [va, va+bytes) chunk by chunk, free the VA
void unmap_range(gml_allocator& A, CUdeviceptr va, size_t bytes, size_t mapped) {
  const size_t G = A.pol.chunk_bytes;
  for (size_t off = 0; off < mapped; off += G) {
    A.ok(A.drv.unmap(va + off, G), "cuMemUnmap");
    A.calls[D_UNMAP]++;
  }
  A.ok(A.drv.addr_free(va, bytes), "cuMemAddressFree");
  A.calls[D_ADDR_FREE]++;
}

// unmap the evicted VAs whose event completed (all of them when `wait`)
void drain_pending(gml_allocator& A, bool wait) {
  size_t keep = 0;
  for (size_t i = 0; i < A.pending.size(); ++i) {
    Pending& p = A.pending[i];
    if (wait) cudaEventSynchronize(p.ev);
    const bool done = wait || cudaEventQuery(p.ev) == cudaSuccess;
    if (!done) cudaGetLastError();   // cudaErrorNotReady is not an error: clear it
    if (done) {
      unmap_range(A, p.va, p.bytes, p.bytes);
      cudaEventDestroy(p.ev);
    } else {
      A.pending[keep++] = p;
    }
  }
  A.pending.resize(keep);
}

void LiveHooks::on_evict(uint32_t row) {
  gml_allocator& A = *a;
  SRec& s = A.sva[row];
  if (!s.borrowed && s.va) {
    // the sBlock is inactive, but work queued before its last tensor was
    // freed may still read through this VA: unmap once the allocator's
    // stream has passed this point (no device-wide synchronisation)
    cudaEvent_t ev = nullptr;
    if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) == cudaSuccess &&
        cudaEventRecord(ev, A.stream) == cudaSuccess) {
      A.pending.push_back(Pending{s.va, s.bytes, ev});
    } else {   // cannot order it: wait for the stream instead
      if (ev) cudaEventDestroy(ev);
      cudaStreamSynchronize(A.stream);
      unmap_range(A, s.va, s.bytes, s.bytes);
    }
  }
  s = SRec{};
}

bool LiveHooks::on_bfc_segment(uint32_t seg, uint64_t bytes) {
  void* p = nullptr;
  if (cudaMalloc(&p, bytes) != cudaSuccess) {
    cudaGetLastError();   // clear the sticky-free OOM error
    a->ok(CUDA_ERROR_OUT_OF_MEMORY, "cudaMalloc");
    return false;
  }
  a->segs[seg] = p;
  return true;
}

void LiveHooks::on_bfc_release(uint32_t seg) {
  auto it = a->segs.find(seg);
  if (it != a->segs.end()) {
    cudaFree(it->second);
    a->segs.erase(it);
  }
}

void snapshot(const gml_allocator* a, gml_stats_t* out) {
  const auto& E = a->E;
  *out = *E.S();
  for (int i = 0; i < 7; ++i) out->state_count[i] = E.sc[i];
  out->peak_active_bytes = E.pk_active;
  out->peak_reserved_bytes = E.pk_reserved;
  out->peak_requested_bytes = E.pk_requested;
  out->peak_active_vmm_bytes = E.pk_active_vmm;
  out->peak_reserved_vmm_bytes = E.pk_reserved_vmm;
  out->final_active_bytes = E.active;
  out->final_reserved_bytes = E.reserved();
  out->n_events = E.serial;
  out->n_events_done = E.serial;
  out->oom_event = -1;
  out->status = GML_OK;
  out->_p = 0;
  out->max_pblocks = E.mx_p;
  out->max_sblocks = E.mx_s;
  out->max_live_handles = E.mx_h;
  out->max_bfc_blocks = E.mx_b;
}

}  // namespace

extern "C" {

gml_status gml_create(int device, const gml_policy* p, gml_allocator** out) {
  if (!out) return GML_ERR_INVALID;
  *out = nullptr;
  if (!p || p->kind != GML_POLICY_GMLAKE || p->chunk_bytes == 0 || p->spool_max_entries == 0)
    return GML_ERR_INVALID;
  if (p->capacity_bytes / p->chunk_bytes + 1 > kMaxChunks) return GML_ERR_UNSUPPORTED;
  if (cudaSetDevice(device) != cudaSuccess) return GML_ERR_CUDA;
  cudaFree(0);   // make sure the primary context exists
  gml_allocator* a = new (std::nothrow) gml_allocator();
  if (!a) return GML_ERR_OOM;
  int vmm = 0;
  CUdevice cu_dev = 0;
  if (!load_driver(a->drv) || a->drv.device_get(&cu_dev, device) != CUDA_SUCCESS ||
      a->drv.device_attr(&vmm, CU_DEVICE_ATTRIBUTE_VIRTUAL_MEMORY_MANAGEMENT_SUPPORTED, cu_dev) != CUDA_SUCCESS ||
      !vmm) {
    delete a;
    return GML_ERR_UNSUPPORTED;
  }
  a->device = device;
  a->pol = *p;
  a->prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  a->prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  a->prop.location.id = device;
  a->access.location = a->prop.location;
  a->access.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  size_t gran = 0;
  if (a->drv.granularity(&gran, &a->prop, CU_MEM_ALLOC_GRANULARITY_MINIMUM) != CUDA_SUCCESS || !gran ||
      p->chunk_bytes % gran) {
    delete a;
    return GML_ERR_UNSUPPORTED;   // the chunk must be a multiple of the VMM granularity
  }
  RtCaps rc{(uint32_t)((p->capacity_bytes / p->chunk_bytes + 1 + 31) / 32), kLiveSlots};
  uint64_t bytes = Lay<CfgLive>::bytes(rc.bm_words, rc.h);
  a->arena = (uint8_t*)aligned_alloc(64, (bytes + 63) & ~63ull);
  if (!a->arena) { delete a; return GML_ERR_OOM; }
  a->hooks.a = a;
  a->E.init(*p, rc, a->arena, &a->hooks);
  *out = a;
  return GML_OK;
}

gml_status gml_malloc(gml_allocator* a, size_t bytes, void** out_ptr) {
  if (out_ptr) *out_ptr = nullptr;
  if (!a || !out_ptr || bytes == 0 || bytes > gml::MASK40) return GML_ERR_INVALID;
  if (!a->pending.empty()) drain_pending(*a, false);
  uint32_t slot;
  if (!a->free_slots.empty()) { slot = a->free_slots.back(); a->free_slots.pop_back(); }
  else if (a->next_slot < kLiveSlots) slot = a->next_slot++;
  else return GML_ERR_TABLE_OVERFLOW;
  auto& E = a->E;
  a->last_rec = E.step(((uint64_t)slot << 40) | bytes);
  if (E.overflow) {                       // a host table is full: nothing was committed
    E.overflow = 0;
    a->free_slots.push_back(slot);
    return GML_ERR_TABLE_OVERFLOW;
  }
  if (E.status == GML_ERR_OOM) {          // S5 (capacity or a failed driver call): the allocator stays usable
    E.status = GML_OK;
    a->free_slots.push_back(slot);
    return GML_ERR_OOM;
  }
  uint64_t hv = E.H[slot];
  uint32_t kind = (uint32_t)(hv >> 62), row = (uint32_t)((hv >> 40) & 0x3FFFFF);
  using L = Lay<CfgLive>;
  void* p;
  if (kind == HK_P) {
    p = (void*)a->va_of_chunk(E.A[L::PLO + row]);
  } else if (kind == HK_S) {
    p = (void*)a->sva[row].va;
  } else {
    void* base = a->segs[E.A[L::BSEG + row]];
    p = (uint8_t*)base + (size_t)E.A[L::BOFF + row] * 512;
  }
  a->slot_of[(uintptr_t)p] = slot;
  *out_ptr = p;
  return GML_OK;
}

gml_status gml_free(gml_allocator* a, void* ptr) {
  if (!a) return GML_ERR_INVALID;
  auto it = a->slot_of.find((uintptr_t)ptr);
  if (it == a->slot_of.end()) return GML_ERR_INVALID;     // unknown pointer / double free
  uint32_t slot = it->second;
  a->slot_of.erase(it);
  a->last_rec = a->E.step((1ull << 63) | ((uint64_t)slot << 40));
  a->free_slots.push_back(slot);
  return GML_OK;
}

gml_status gml_live_trace(gml_allocator* a, const uint64_t* events, uint64_t n, uint64_t* records, uint64_t* ns,
                          uint64_t* n_done) {
  if (!a || (n && !events)) return GML_ERR_INVALID;
  using clk = std::chrono::steady_clock;
  std::vector<void*> ptr;
  gml_status rc = GML_OK;
  uint64_t i = 0;
  for (; i < n; ++i) {
    const uint64_t ev = events[i];
    const uint32_t slot = (uint32_t)((ev >> 40) & 0x7FFFFFu);
    if (slot >= ptr.size()) ptr.resize((size_t)slot + 1, nullptr);
    const bool is_free = ev >> 63;
    if (is_free && !ptr[slot]) { rc = GML_ERR_INVALID; break; }
    const auto t0 = clk::now();
    if (is_free) {
      rc = gml_free(a, ptr[slot]);
    } else {
      rc = gml_malloc(a, (size_t)(ev & gml::MASK40), &ptr[slot]);
    }
    const auto t1 = clk::now();
    if (rc != GML_OK) {
      if (records) records[i] = rc == GML_ERR_OOM ? gml::rec_oom() : 0;
      break;
    }
    if (is_free) ptr[slot] = nullptr;
    if (records) records[i] = a->last_rec;
    if (ns) ns[i] = (uint64_t)std::chrono::duration_cast<std::chrono::nanoseconds>(t1 - t0).count();
  }
  if (n_done) *n_done = i;
  for (void* p : ptr)
    if (p) gml_free(a, p);
  return rc;
}

gml_status gml_cudamalloc_trace(int device, const uint64_t* events, uint64_t n, uint64_t* ns, uint64_t* n_done) {
  if (n && !events) return GML_ERR_INVALID;
  if (cudaSetDevice(device) != cudaSuccess) return GML_ERR_CUDA;
  using clk = std::chrono::steady_clock;
  std::vector<void*> ptr;
  gml_status rc = GML_OK;
  uint64_t i = 0;
  for (; i < n; ++i) {
    const uint64_t ev = events[i];
    const uint32_t slot = (uint32_t)((ev >> 40) & 0x7FFFFFu);
    if (slot >= ptr.size()) ptr.resize((size_t)slot + 1, nullptr);
    const bool is_free = ev >> 63;
    const auto t0 = clk::now();
    cudaError_t e = is_free ? cudaFree(ptr[slot]) : cudaMalloc(&ptr[slot], (size_t)(ev & gml::MASK40));
    const auto t1 = clk::now();
    if (e != cudaSuccess) { cudaGetLastError(); rc = e == cudaErrorMemoryAllocation ? GML_ERR_OOM : GML_ERR_CUDA; break; }
    if (is_free) ptr[slot] = nullptr;
    if (ns) ns[i] = (uint64_t)std::chrono::duration_cast<std::chrono::nanoseconds>(t1 - t0).count();
  }
  if (n_done) *n_done = i;
  for (void* p : ptr)
    if (p) cudaFree(p);
  return rc;
}

gml_status gml_set_stream(gml_allocator* a, void* stream) {
  if (!a) return GML_ERR_INVALID;
  a->stream = (cudaStream_t)stream;
  return GML_OK;
}

gml_status gml_stats(const gml_allocator* a, gml_stats_t* out) {
  if (!a || !out) return GML_ERR_INVALID;
  snapshot(a, out);
  return GML_OK;
}

gml_status gml_driver_calls(const gml_allocator* a, uint64_t out[7]) {
  if (!a || !out) return GML_ERR_INVALID;
  memcpy(out, a->calls, sizeof(a->calls));
  return GML_OK;
}

gml_status gml_vmm_profile(int device, uint64_t bytes, uint64_t chunk, int reps, double* out_us) {
  if (!out_us || !chunk || !bytes || bytes % chunk || reps <= 0) return GML_ERR_INVALID;
  if (cudaSetDevice(device) != cudaSuccess) return GML_ERR_CUDA;
  cudaFree(0);
  Drv d;
  CUdevice cu_dev = 0;
  int vmm = 0;
  if (!load_driver(d) || d.device_get(&cu_dev, device) != CUDA_SUCCESS ||
      d.device_attr(&vmm, CU_DEVICE_ATTRIBUTE_VIRTUAL_MEMORY_MANAGEMENT_SUPPORTED, cu_dev) != CUDA_SUCCESS || !vmm)
    return GML_ERR_UNSUPPORTED;
  CUmemAllocationProp prop{};
  prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  prop.location.id = device;
  CUmemAccessDesc acc{};
  acc.location = prop.location;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  size_t gran = 0;
  if (d.granularity(&gran, &prop, CU_MEM_ALLOC_GRANULARITY_MINIMUM) != CUDA_SUCCESS || !gran || chunk % gran)
    return GML_ERR_UNSUPPORTED;
  using clk = std::chrono::steady_clock;
  auto us = [](clk::time_point a, clk::time_point b) { return std::chrono::duration<double, std::micro>(b - a).count(); };
  const size_t n = bytes / chunk;
  std::vector<std::vector<double>> t(8);
  std::vector<CUmemGenericAllocationHandle> h(n);
  for (int r = 0; r < reps; ++r) {
    void* p = nullptr;
    cudaDeviceSynchronize();
    auto a = clk::now();
    if (cudaMalloc(&p, bytes) != cudaSuccess) return GML_ERR_OOM;
    auto b = clk::now();
    cudaFree(p);
    auto c = clk::now();
    t[0].push_back(us(a, b));
    t[1].push_back(us(b, c));
    CUdeviceptr va = 0;
    a = clk::now();
    if (d.reserve(&va, bytes, 0, 0, 0) != CUDA_SUCCESS) return GML_ERR_CUDA;
    b = clk::now();
    t[2].push_back(us(a, b));
    double tc = 0, tm = 0, ta = 0;
    for (size_t i = 0; i < n; ++i) {
      auto x = clk::now();
      if (d.create(&h[i], chunk, &prop, 0) != CUDA_SUCCESS) return GML_ERR_OOM;
      auto y = clk::now();
      if (d.map(va + i * chunk, chunk, 0, h[i], 0) != CUDA_SUCCESS) return GML_ERR_CUDA;
      auto z = clk::now();
      if (d.set_access(va + i * chunk, chunk, &acc, 1) != CUDA_SUCCESS) return GML_ERR_CUDA;
      auto q = clk::now();
      tc += us(x, y); tm += us(y, z); ta += us(z, q);
    }
    t[3].push_back(tc);
    t[4].push_back(tm);
    t[5].push_back(ta);
    // the whole range once more (already accessible: measures one call over n chunks)
    a = clk::now();
    d.set_access(va, bytes, &acc, 1);
    b = clk::now();
    t[6].push_back(us(a, b));
    a = clk::now();
    for (size_t i = 0; i < n; ++i) {
      d.unmap(va + i * chunk, chunk);
      d.release(h[i]);
    }
    d.addr_free(va, bytes);
    b = clk::now();
    t[7].push_back(us(a, b));
  }
  for (int k = 0; k < 8; ++k) {
    std::sort(t[k].begin(), t[k].end());
    out_us[k] = t[k][t[k].size() / 2];
  }
  out_us[8] = out_us[2] + out_us[3] + out_us[4] + out_us[5];
  out_us[9] = out_us[2] + out_us[3] + out_us[4] + out_us[6];
  return GML_OK;
}

gml_status gml_destroy(gml_allocator* a) {
  if (!a) return GML_ERR_INVALID;
  if (!a->slot_of.empty()) return GML_ERR_INVALID;
  cudaSetDevice(a->device);
  cudaDeviceSynchronize();
  drain_pending(*a, true);
  for (SRec& s : a->sva)
    if (s.va && !s.borrowed) unmap_range(*a, s.va, s.bytes, s.bytes);
  for (auto& kv : a->allocs) {
    const size_t b = (size_t)kv.second.n * a->pol.chunk_bytes;
    unmap_range(*a, kv.second.va, b, b);
  }
  for (CUmemGenericAllocationHandle h : a->chunk) {
    if (!h) continue;
    a->drv.release(h);
    a->calls[D_RELEASE]++;
  }
  for (auto& kv : a->segs) cudaFree(kv.second);
  free(a->arena);
  delete a;
  return GML_OK;
}

}  // extern "C"
