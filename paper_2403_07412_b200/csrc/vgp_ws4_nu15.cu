// Instantiation of the split-scheduler warp-specialised DMMA kernel for kMatern15
// (split per smoothness so the unrolled kernels compile in parallel).
#include "vgp_ws4_kernel.cuh"

namespace vgp {
cudaError_t launch_ws4_kMatern15(const Plan& p, const CovParams& cp, int64_t e_lo, int64_t e_hi,
                                 cudaStream_t stream, bool cache) {
  return ws4::launch_kind<kMatern15>(p, cp, e_lo, e_hi, stream, cache);
}
}  // namespace vgp
