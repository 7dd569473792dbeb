// classes_1.cu -- K1 instances of size class 1 (see replay_kernel.cuh).
#include "split_kernel.cuh"

namespace gml {
namespace replay {
gml_status launch_cls_1(bool smem, const KParams& kp, uint32_t stride, cudaStream_t st) {
  return smem ? launch_class<C1, true>(kp, stride, st) : launch_class<C1, false>(kp, stride, st);
}
gml_status launch_path_1(const KParams& kp, cudaStream_t st) { return launch_path<C1>(kp, st); }
uint32_t path_ctas_1() { return path_ctas_per_sm<C1>(); }
}  // namespace replay
}  // namespace gml
