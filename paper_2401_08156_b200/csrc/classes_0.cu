// classes_0.cu -- K1 instances of size class 0 (see replay_kernel.cuh).
#include "split_kernel.cuh"

namespace gml {
namespace replay {
gml_status launch_cls_0(bool smem, const KParams& kp, uint32_t stride, cudaStream_t st) {
  return smem ? launch_class<C0, true>(kp, stride, st) : launch_class<C0, false>(kp, stride, st);
}
gml_status launch_path_0(const KParams& kp, cudaStream_t st) { return launch_path<C0>(kp, st); }
uint32_t path_ctas_0() { return path_ctas_per_sm<C0>(); }
}  // namespace replay
}  // namespace gml
