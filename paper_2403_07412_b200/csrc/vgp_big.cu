// Instantiations of the large-m CTA-per-block DMMA kernel (vgp_big_kernel.cuh).
#include "vgp_big_kernel.cuh"

namespace vgp {

bool big_supported(int m, int kind) {
  return m >= 1 && m <= 4096;  // every kernel family (vg/kernels.py:59-91)
}

bool big_needs_scratch(int m) { return big::use_global_tiles(m); }

namespace big {
bool point_map(const double4* pts, int64_t n, CUtensorMap* map) {
  using Encode = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static Encode encode = nullptr;
  if (!encode) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn)
      return false;
    encode = reinterpret_cast<Encode>(fn);
  }
  const cuuint64_t dims[2] = {4, (cuuint64_t)n};
  const cuuint64_t strides[1] = {sizeof(double4)};
  const cuuint32_t box[2] = {4, 1};
  const cuuint32_t estr[2] = {1, 1};
  return encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double4*>(pts), dims, strides, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
}  // namespace big
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
