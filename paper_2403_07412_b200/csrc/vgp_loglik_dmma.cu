// Dispatch for the warp-per-block DMMA kernels (vgp_ll_kernel.cuh, vgp_dmma_kernel.cuh).
#include "vgp_internal.cuh"

namespace vgp {

cudaError_t launch_dmma_kMatern05(const Plan&, const CovParams&, int64_t, int64_t, cudaStream_t);
cudaError_t launch_dmma_kMatern15(const Plan&, const CovParams&, int64_t, int64_t, cudaStream_t);
cudaError_t launch_dmma_kMatern25(const Plan&, const CovParams&, int64_t, int64_t, cudaStream_t);

cudaError_t launch_ws_kMatern05(const Plan&, const CovParams&, int64_t, int64_t, cudaStream_t, bool);
cudaError_t launch_ws_kMatern15(const Plan&, const CovParams&, int64_t, int64_t, cudaStream_t, bool);
cudaError_t launch_ws_kMatern25(const Plan&, const CovParams&, int64_t, int64_t, cudaStream_t, bool);

cudaError_t launch_loglik_ws(const Plan& p, const CovParams& cp, int64_t e_lo, int64_t e_hi,
                             cudaStream_t stream, bool cache) {
  if (!dmma_supported(p.m, cp.kind)) return cudaErrorNotSupported;
  if (e_hi <= e_lo) return cudaSuccess;
  switch (cp.kind) {
    case kMatern05: return launch_ws_kMatern05(p, cp, e_lo, e_hi, stream, cache);
    case kMatern15: return launch_ws_kMatern15(p, cp, e_lo, e_hi, stream, cache);
    default: return launch_ws_kMatern25(p, cp, e_lo, e_hi, stream, cache);
  }
}

cudaError_t launch_ws3_kMatern05(const Plan&, const CovParams&, int64_t, int64_t, cudaStream_t, bool);
cudaError_t launch_ws3_kMatern15(const Plan&, const CovParams&, int64_t, int64_t, cudaStream_t, bool);
cudaError_t launch_ws3_kMatern25(const Plan&, const CovParams&, int64_t, int64_t, cudaStream_t, bool);

cudaError_t launch_ws3_kMaternGen(const Plan&, const CovParams&, int64_t, int64_t, cudaStream_t, bool);

bool ws3_supported(int m, int kind) {
  return dmma_supported(m, kind) || (m >= 1 && m + 2 <= 64 && kind == kMaternGen);
}

cudaError_t launch_loglik_ws3(const Plan& p, const CovParams& cp, int64_t e_lo, int64_t e_hi,
                              cudaStream_t stream, bool cache) {
  if (!ws3_supported(p.m, cp.kind)) return cudaErrorNotSupported;
  if (e_hi <= e_lo) return cudaSuccess;
  switch (cp.kind) {
    case kMatern05: return launch_ws3_kMatern05(p, cp, e_lo, e_hi, stream, cache);
    case kMatern15: return launch_ws3_kMatern15(p, cp, e_lo, e_hi, stream, cache);
    case kMatern25: return launch_ws3_kMatern25(p, cp, e_lo, e_hi, stream, cache);
    default: return launch_ws3_kMaternGen(p, cp, e_lo, e_hi, stream, cache);
  }
}

bool dmma_supported(int m, int kind) {
  return m >= 1 && m + 2 <= 64 && (kind == kMatern05 || kind == kMatern15 || kind == kMatern25);
}

cudaError_t launch_loglik_dmma(const Plan& p, const CovParams& cp, int64_t e_lo, int64_t e_hi,
                               cudaStream_t stream) {
  if (!dmma_supported(p.m, cp.kind)) return cudaErrorNotSupported;
  if (e_hi <= e_lo) return cudaSuccess;
  switch (cp.kind) {
    case kMatern05: return launch_dmma_kMatern05(p, cp, e_lo, e_hi, stream);
    case kMatern15: return launch_dmma_kMatern15(p, cp, e_lo, e_hi, stream);
    default: return launch_dmma_kMatern25(p, cp, e_lo, e_hi, stream);
  }
}

}  // namespace vgp
