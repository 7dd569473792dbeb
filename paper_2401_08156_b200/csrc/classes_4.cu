// classes_4.cu -- K1 instances of size class 4 (see replay_kernel.cuh).
#include "split_kernel.cuh"

namespace gml {
namespace replay {
gml_status launch_cls_4(bool smem, const KParams& kp, uint32_t stride, cudaStream_t st) {
  return smem ? launch_class<C4, true>(kp, stride, st) : launch_class<C4, false>(kp, stride, st);
}
gml_status launch_path_4(const KParams& kp, cudaStream_t st) { return launch_path<C4>(kp, st); }
uint32_t path_ctas_4() { return path_ctas_per_sm<C4>(); }
}  // namespace replay
}  // namespace gml
