// Instantiations of the large-m CTA-per-block DMMA kernel for kMatern25.
#include "vgp_big_kernel.cuh"

namespace vgp {
cudaError_t launch_big_k25(const Plan& p, const CovParams& cp, int64_t e_lo, int64_t e_hi,
                            cudaStream_t stream, bool cache) {
  return big::launch_kind<kMatern25>(p, cp, e_lo, e_hi, stream, cache, p.d_gscratch, p.gscratch_slots);
}
}  // namespace vgp
