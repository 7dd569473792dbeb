// classes_7.cu -- K1 instances of size class 7 (see replay_kernel.cuh).
#include "split_kernel.cuh"

namespace gml {
namespace replay {
gml_status launch_cls_7(bool smem, const KParams& kp, uint32_t stride, cudaStream_t st) {
  return smem ? launch_class<C7, true>(kp, stride, st) : launch_class<C7, false>(kp, stride, st);
}
gml_status launch_path_7(const KParams& kp, cudaStream_t st) { return launch_path<C7>(kp, st); }
uint32_t path_ctas_7() { return path_ctas_per_sm<C7>(); }
}  // namespace replay
}  // namespace gml
