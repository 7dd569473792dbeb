// stream_bw.cu -- K2: streaming copy kernel used to show that stitched VMM
// buffers stream at the same HBM bandwidth as cudaMalloc'd ones (north star;
// SURVEY §8(d) C5). 16-byte vector loads/stores, grid-stride, grid sized to a
// multiple of the 148 SMs.
#include <cuda_runtime.h>

#include "gml.h"

namespace {
__global__ void __launch_bounds__(512) k_stream_copy(const uint4* __restrict__ src, uint4* __restrict__ dst,
                                                     size_t n16) {
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  size_t stride = (size_t)gridDim.x * blockDim.x;
#pragma unroll 4
  for (; i < n16; i += stride) __stcs(dst + i, __ldcs(src + i));
}
}  // namespace

extern "C" gml_status gml_stream_copy(const void* src, void* dst, size_t n, int iters, void* stream,
                                      float* ms) {
  if (!src || !dst || (n & 15) || ((uintptr_t)src & 15) || ((uintptr_t)dst & 15) || iters <= 0)
    return GML_ERR_INVALID;
  cudaStream_t st = (cudaStream_t)stream;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaEvent_t a, b;
  if (cudaEventCreate(&a) != cudaSuccess || cudaEventCreate(&b) != cudaSuccess) return GML_ERR_CUDA;
  size_t n16 = n / 16;
  unsigned grid = (unsigned)sms * 4;
  cudaEventRecord(a, st);
  for (int i = 0; i < iters; ++i)
    k_stream_copy<<<grid, 512, 0, st>>>((const uint4*)src, (uint4*)dst, n16);
  cudaEventRecord(b, st);
  cudaError_t e = cudaEventSynchronize(b);
  float t = 0;
  cudaEventElapsedTime(&t, a, b);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  if (e != cudaSuccess || cudaGetLastError() != cudaSuccess) return GML_ERR_CUDA;
  if (ms) *ms = t / iters;
  return GML_OK;
}
