// classes_6.cu -- K1 instances of size class 6 (see replay_kernel.cuh).
#include "replay_kernel.cuh"

namespace gml {
namespace replay {
gml_status launch_cls_6(bool smem, bool latency, const KParams& kp, uint32_t stride, cudaStream_t st) {
  if (latency)
    return smem ? launch_class<C6, true, kLatencyWarps>(kp, stride, st)
                : launch_class<C6, false, kLatencyWarps>(kp, stride, st);
  return smem ? launch_class<C6, true, 0>(kp, stride, st) : launch_class<C6, false, 0>(kp, stride, st);
}
}  // namespace replay
}  // namespace gml
