// classes_5.cu -- K1 instances of size class 5 (see replay_kernel.cuh).
#include "split_kernel.cuh"

namespace gml {
namespace replay {
gml_status launch_cls_5(bool smem, const KParams& kp, uint32_t stride, cudaStream_t st) {
  return smem ? launch_class<C5, true>(kp, stride, st) : launch_class<C5, false>(kp, stride, st);
}
gml_status launch_path_5(const KParams& kp, cudaStream_t st) { return launch_path<C5>(kp, st); }
uint32_t path_ctas_5() { return path_ctas_per_sm<C5>(); }
}  // namespace replay
}  // namespace gml
