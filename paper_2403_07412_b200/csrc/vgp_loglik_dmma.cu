// Warp-per-block DMMA likelihood kernel (placeholder until the tensor-core
// path lands; the generic kernel covers every shape meanwhile).
#include "vgp_internal.cuh"

namespace vgp {

bool dmma_supported(int m, int kind) {
  (void)m;
  (void)kind;
  return false;
}

cudaError_t launch_loglik_dmma(const Plan& p, const CovParams& cp, int64_t e_lo, int64_t e_hi,
                               cudaStream_t stream) {
  (void)p; (void)cp; (void)e_lo; (void)e_hi; (void)stream;
  return cudaErrorNotSupported;
}

}  // namespace vgp
