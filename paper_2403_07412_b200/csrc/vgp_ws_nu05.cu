// Instantiation of the warp-specialised DMMA kernel for kMatern05 (split per smoothness
// so the large unrolled kernels compile in parallel).
#include "vgp_ws_kernel.cuh"

namespace vgp {
cudaError_t launch_ws_kMatern05(const Plan& p, const CovParams& cp, int64_t e_lo, int64_t e_hi,
                              cudaStream_t stream, bool cache) {
  return ws::launch_kind<kMatern05>(p, cp, e_lo, e_hi, stream, cache);
}
}  // namespace vgp
