// torch_alloc.cu -- PyTorch pluggable-allocator backend over the live
// GMLake allocator (GMLake is a
// drop-in replacement of PyTorch's caching allocator for tensor
// (de)allocation). torch.cuda.memory.CUDAPluggableAllocator(libgml.so,
// "gml_torch_malloc", "gml_torch_free") routes every tensor allocation of the
// process here; each device gets one gml_allocator (live.cu), created on its
// first request. Host code only.
#include <cuda_runtime.h>

#include <cstddef>
#include <cstring>
#include <map>
#include <mutex>

#include "gml.h"

namespace {

std::mutex g_mu;
std::map<int, gml_allocator*> g_alloc;
bool g_have_policy = false;
gml_policy g_policy{};

gml_allocator* allocator_of(int device) {
  auto it = g_alloc.find(device);
  if (it != g_alloc.end()) return it->second;
  gml_policy p = g_policy;
  if (!g_have_policy) {   // GMLake V2 defaults over the whole device
    size_t free_b = 0, total_b = 0;
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(device);
    cudaMemGetInfo(&free_b, &total_b);
    cudaSetDevice(prev);
    const uint64_t chunk = 2ull << 20;
    p = gml_policy{GML_POLICY_GMLAKE, 0, (uint64_t)total_b / chunk * chunk, chunk, 2ull << 20, 128ull << 20,
                   4096, 0, (uint64_t)total_b / chunk * chunk};
  }
  gml_allocator* a = nullptr;
  if (gml_create(device, &p, &a) != GML_OK) a = nullptr;
  g_alloc[device] = a;
  return a;
}

}  // namespace

extern "C" {

void* gml_torch_malloc(ptrdiff_t size, int device, void* /*stream*/) {
  if (size <= 0) return nullptr;
  std::lock_guard<std::mutex> lk(g_mu);
  gml_allocator* a = allocator_of(device);
  if (!a) return nullptr;
  void* p = nullptr;
  if (gml_malloc(a, (size_t)size, &p) != GML_OK) return nullptr;
  return p;
}

void gml_torch_free(void* ptr, ptrdiff_t /*size*/, int device, void* /*stream*/) {
  if (!ptr) return;
  std::lock_guard<std::mutex> lk(g_mu);
  auto it = g_alloc.find(device);
  if (it != g_alloc.end() && it->second) gml_free(it->second, ptr);
}

gml_status gml_torch_configure(const gml_policy* p) {
  if (!p || p->kind != GML_POLICY_GMLAKE) return GML_ERR_INVALID;
  std::lock_guard<std::mutex> lk(g_mu);
  if (!g_alloc.empty()) return GML_ERR_INVALID;
  g_policy = *p;
  g_have_policy = true;
  return GML_OK;
}

gml_status gml_torch_stats(int device, gml_stats_t* out) {
  if (!out) return GML_ERR_INVALID;
  std::lock_guard<std::mutex> lk(g_mu);
  auto it = g_alloc.find(device);
  if (it == g_alloc.end() || !it->second) return GML_ERR_INVALID;
  return gml_stats(it->second, out);
}

}  // extern "C"
