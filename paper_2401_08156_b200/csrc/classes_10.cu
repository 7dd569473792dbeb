// classes_10.cu -- K1 instances of size class 10 (see replay_kernel.cuh).
#include "split_kernel.cuh"

namespace gml {
namespace replay {
gml_status launch_cls_10(bool smem, const KParams& kp, uint32_t stride, cudaStream_t st) {
  return smem ? launch_class<C10, true>(kp, stride, st) : launch_class<C10, false>(kp, stride, st);
}
gml_status launch_path_10(const KParams& kp, cudaStream_t st) { return launch_path<C10>(kp, st); }
uint32_t path_ctas_10() { return path_ctas_per_sm<C10>(); }
}  // namespace replay
}  // namespace gml
