// classes_2.cu -- K1 instances of size class 2 (see replay_kernel.cuh).
#include "split_kernel.cuh"

namespace gml {
namespace replay {
gml_status launch_cls_2(bool smem, const KParams& kp, uint32_t stride, cudaStream_t st) {
  return smem ? launch_class<C2, true>(kp, stride, st) : launch_class<C2, false>(kp, stride, st);
}
gml_status launch_path_2(const KParams& kp, cudaStream_t st) { return launch_path<C2>(kp, st); }
uint32_t path_ctas_2() { return path_ctas_per_sm<C2>(); }
}  // namespace replay
}  // namespace gml
