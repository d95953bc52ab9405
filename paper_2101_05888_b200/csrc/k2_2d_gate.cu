// k2_2d_gate.cu -- one K2 instantiation family (see k2_launch.cuh).
#include <type_traits>

#include "k2_launch.cuh"

namespace sasbp {
cudaError_t k2_launch_2d_gate(const TdbpParams& prm, const TmaDesc& tmap, const K2Launch& L) {
  return launch_family<SASBP_T2D, false, true, false>(prm, tmap, L);
}
}  // namespace sasbp
