// Instantiation of the scheduler-aware warp-specialised DMMA kernel for the
// general-nu Matern (covariances from the per-evaluation table, vgp_ktab.cuh).
#include "vgp_ws3_kernel.cuh"

namespace vgp {
cudaError_t launch_ws3_kMaternGen(const Plan& p, const CovParams& cp, int64_t e_lo, int64_t e_hi,
                                  cudaStream_t stream, bool cache) {
  if (!p.d_ktab) return cudaErrorNotSupported;
  return ws3::launch_kind<kMaternGen>(p, cp, e_lo, e_hi, stream, cache);
}
}  // namespace vgp
