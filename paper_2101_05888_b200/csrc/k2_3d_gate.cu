// k2_3d_gate.cu -- one K2 instantiation family (see k2_launch.cuh).
#include <type_traits>

#include "k2_launch.cuh"

namespace sasbp {
cudaError_t k2_launch_3d_gate(const TdbpParams& prm, const TmaDesc& tmap, const K2Launch& L) {
  return launch_family<SASBP_T3D, true, true, false>(prm, tmap, L);
}
}  // namespace sasbp
