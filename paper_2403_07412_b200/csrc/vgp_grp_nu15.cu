// Instantiation of the lock-step group DMMA kernel for kMatern15
// (split per smoothness so the unrolled kernels compile in parallel).
#include "vgp_grp_kernel.cuh"

namespace vgp {
cudaError_t launch_grp_kMatern15(const Plan& p, const CovParams& cp, int64_t e_lo, int64_t e_hi,
                                 cudaStream_t stream) {
  return grp::launch_kind<kMatern15>(p, cp, e_lo, e_hi, stream);
}
}  // namespace vgp
