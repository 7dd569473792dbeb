// classes_3.cu -- K1 instances of size class 3 (see replay_kernel.cuh).
#include "split_kernel.cuh"

namespace gml {
namespace replay {
gml_status launch_cls_3(bool smem, const KParams& kp, uint32_t stride, cudaStream_t st) {
  return smem ? launch_class<C3, true>(kp, stride, st) : launch_class<C3, false>(kp, stride, st);
}
gml_status launch_path_3(const KParams& kp, cudaStream_t st) { return launch_path<C3>(kp, st); }
uint32_t path_ctas_3() { return path_ctas_per_sm<C3>(); }
}  // namespace replay
}  // namespace gml
