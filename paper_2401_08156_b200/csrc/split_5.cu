// split_5.cu -- K1s (three-warp split unit) instances of size class 5 (see split_kernel.cuh).
#include "split_kernel.cuh"

namespace gml {
namespace replay {
gml_status launch_split_5(int place, const KParams& kp, uint32_t smem, cudaStream_t st) {
  return launch_split<C5>(place, kp, smem, st);
}
}  // namespace replay
}  // namespace gml
