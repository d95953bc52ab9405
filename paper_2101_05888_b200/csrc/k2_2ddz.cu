// k2_2ddz.cu -- one K2 instantiation family (see k2_launch.cuh).
#include <type_traits>

#include "k2_launch.cuh"

namespace sasbp {
cudaError_t k2_launch_2ddz(const TdbpParams& prm, const TmaDesc& tmap, const K2Launch& L) {
  return launch_family<SASBP_T2D, true, false, false>(prm, tmap, L);
}
}  // namespace sasbp
