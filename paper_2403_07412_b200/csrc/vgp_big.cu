// Instantiations of the large-m CTA-per-block DMMA kernel (vgp_big_kernel.cuh).
#include "vgp_big_kernel.cuh"

namespace vgp {

bool big_supported(int m, int kind) {
  return m >= 1 && m <= 4096;  // every kernel family (vg/kernels.py:59-91)
}

bool big_needs_scratch(int m) { return big::use_global_tiles(m); }
int64_t big_scratch_doubles(int m) { return big::tile_doubles(m); }

cudaError_t launch_loglik_big(const Plan& p, const CovParams& cp, int64_t e_lo, int64_t e_hi,
                              cudaStream_t stream, bool cache) {
  if (!big_supported(p.m, cp.kind)) return cudaErrorNotSupported;
  if (e_hi <= e_lo) return cudaSuccess;
  switch (cp.kind) {
    case kMatern05:
      return big::launch_kind<kMatern05>(p, cp, e_lo, e_hi, stream, cache, p.d_gscratch, p.gscratch_slots);
    case kMatern15:
      return big::launch_kind<kMatern15>(p, cp, e_lo, e_hi, stream, cache, p.d_gscratch, p.gscratch_slots);
    case kMatern25:
      return big::launch_kind<kMatern25>(p, cp, e_lo, e_hi, stream, cache, p.d_gscratch, p.gscratch_slots);
    case kMaternGen:
      return big::launch_kind<kMaternGen>(p, cp, e_lo, e_hi, stream, cache, p.d_gscratch, p.gscratch_slots);
    default:
      return big::launch_kind<kPowExp>(p, cp, e_lo, e_hi, stream, cache, p.d_gscratch, p.gscratch_slots);
  }
}

}  // namespace vgp
