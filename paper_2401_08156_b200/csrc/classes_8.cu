// classes_8.cu -- K1 instances of size class 8 (see replay_kernel.cuh).
#include "split_kernel.cuh"

namespace gml {
namespace replay {
gml_status launch_cls_8(bool smem, const KParams& kp, uint32_t stride, cudaStream_t st) {
  return smem ? launch_class<C8, true>(kp, stride, st) : launch_class<C8, false>(kp, stride, st);
}
gml_status launch_path_8(const KParams& kp, cudaStream_t st) { return launch_path<C8>(kp, st); }
uint32_t path_ctas_8() { return path_ctas_per_sm<C8>(); }
}  // namespace replay
}  // namespace gml
