// classes_9.cu -- K1 instances of size class 9 (see replay_kernel.cuh).
#include "split_kernel.cuh"

namespace gml {
namespace replay {
gml_status launch_cls_9(bool smem, const KParams& kp, uint32_t stride, cudaStream_t st) {
  return smem ? launch_class<C9, true>(kp, stride, st) : launch_class<C9, false>(kp, stride, st);
}
gml_status launch_path_9(const KParams& kp, cudaStream_t st) { return launch_path<C9>(kp, st); }
uint32_t path_ctas_9() { return path_ctas_per_sm<C9>(); }
}  // namespace replay
}  // namespace gml
