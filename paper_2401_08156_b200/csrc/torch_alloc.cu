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

struct Dev {
  gml_allocator* a = nullptr;
  cudaStream_t main = nullptr;   // the stream of the device's first request
  bool have_main = false;
};

std::mutex g_mu;
std::map<int, Dev> g_dev;
bool g_have_policy = false;
gml_policy g_policy{};

Dev& dev_of(int device) {
  auto it = g_dev.find(device);
  if (it != g_dev.end()) return it->second;
  gml_policy p = g_policy;
  if (!g_have_policy) {   // GMLake V2 (tracegen/policies.py) over the device's free memory
    size_t free_b = 0, total_b = 0;
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(device);
    cudaMemGetInfo(&free_b, &total_b);
    cudaSetDevice(prev);
    const uint64_t chunk = 2ull << 20;
    uint64_t head = free_b / 100 > (256ull << 20) ? free_b / 100 : (256ull << 20);
    uint64_t cap = free_b > head ? (free_b - head) / chunk * chunk : chunk;
    p = gml_policy{GML_POLICY_GMLAKE, GML_F_LIMIT_GATES_REQUEST, cap, chunk, 2ull << 20, 128ull << 20,
                   4096, 0, cap};
  }
  Dev d;
  if (gml_create(device, &p, &d.a) != GML_OK) d.a = nullptr;
  return g_dev[device] = d;
}

// make `waiter` wait for the work queued on `src` so far (no host sync)
void order_after(cudaStream_t waiter, cudaStream_t src) {
  cudaEvent_t ev;
  if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess) {
    cudaStreamSynchronize(src);
    return;
  }
  cudaEventRecord(ev, src);
  cudaStreamWaitEvent(waiter, ev, 0);
  cudaEventDestroy(ev);   // released once it completes; the wait stays valid
}

}  // namespace

extern "C" {

void* gml_torch_malloc(ptrdiff_t size, int device, void* stream) {
  if (size <= 0) return nullptr;
  std::lock_guard<std::mutex> lk(g_mu);
  Dev& d = dev_of(device);
  if (!d.a) return nullptr;
  cudaStream_t s = (cudaStream_t)stream;
  if (!d.have_main) {
    d.main = s;
    d.have_main = true;
    gml_set_stream(d.a, s);
  } else if (s != d.main) {
    // a block may have been freed on the main stream with work still queued:
    // this stream's later work waits for the main stream's work so far
    order_after(s, d.main);
  }
  void* p = nullptr;
  if (gml_malloc(d.a, (size_t)size, &p) != GML_OK) return nullptr;
  return p;
}

void gml_torch_free(void* ptr, ptrdiff_t /*size*/, int device, void* stream) {
  if (!ptr) return;
  std::lock_guard<std::mutex> lk(g_mu);
  auto it = g_dev.find(device);
  if (it == g_dev.end() || !it->second.a) return;
  Dev& d = it->second;
  cudaStream_t s = (cudaStream_t)stream;
  // the block is reusable at once: the main stream (and through it every
  // later request) waits for the work this stream queued on it
  if (d.have_main && s != d.main) order_after(d.main, s);
  gml_free(d.a, ptr);
}

gml_status gml_torch_configure(const gml_policy* p) {
  if (!p || p->kind != GML_POLICY_GMLAKE) return GML_ERR_INVALID;
  std::lock_guard<std::mutex> lk(g_mu);
  if (!g_dev.empty()) return GML_ERR_INVALID;
  g_policy = *p;
  g_have_policy = true;
  return GML_OK;
}

gml_status gml_torch_stats(int device, gml_stats_t* out) {
  if (!out) return GML_ERR_INVALID;
  std::lock_guard<std::mutex> lk(g_mu);
  auto it = g_dev.find(device);
  if (it == g_dev.end() || !it->second.a) return GML_ERR_INVALID;
  return gml_stats(it->second.a, out);
}

}  // extern "C"
