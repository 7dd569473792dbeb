// classes_6.cu -- K1 instances of size class 6 (see replay_kernel.cuh).
#include "split_kernel.cuh"

namespace gml {
namespace replay {
gml_status launch_cls_6(bool smem, const KParams& kp, uint32_t stride, cudaStream_t st) {
  return smem ? launch_class<C6, true>(kp, stride, st) : launch_class<C6, false>(kp, stride, st);
}
gml_status launch_path_6(const KParams& kp, cudaStream_t st) { return launch_path<C6>(kp, st); }
uint32_t path_ctas_6() { return path_ctas_per_sm<C6>(); }
}  // namespace replay
}  // namespace gml
