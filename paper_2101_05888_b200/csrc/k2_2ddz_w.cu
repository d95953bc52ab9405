// k2_2ddz_w.cu -- K2 with the spreading weight R_tx R_rx (NEXT-4, reading R18), one tile variant,
// gated and dense (see k2_launch.cuh).
#include <type_traits>

#include "k2_launch.cuh"

namespace sasbp {
cudaError_t k2_launch_2ddz_w(const TdbpParams& prm, const TmaDesc& tmap, const K2Launch& L) {
  return prm.gate ? launch_family<SASBP_T2D, true, true, true>(prm, tmap, L) : launch_family<SASBP_T2D, true, false, true>(prm, tmap, L);
}
}  // namespace sasbp
