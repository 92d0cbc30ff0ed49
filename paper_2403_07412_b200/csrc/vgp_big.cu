// Large-m CTA-per-block DMMA kernel (vgp_big_kernel.cuh): host helpers and the
// family dispatch (instantiations in vgp_big_k*.cu, compiled in parallel).
#include <mutex>
#include <vector>

#include "vgp_big_kernel.cuh"

namespace vgp {

bool big_supported(int m, int kind) {
  return m >= 1 && m <= 4096;  // every kernel family (vg/kernels.py:59-91)
}

bool big_needs_scratch(int m) { return big::use_global_tiles(m); }

namespace big {
int big_slot_map(int nt, SlotMap* map) {
  // lifetimes in tile-column steps: tile (I, k) is written by the look-ahead
  // at step k - 1 and last read at step I - 1 (the diagonal tile at step k)
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  static int cached_nt = -1, cached_slots = 0;
  static SlotMap cached;
  if (nt == cached_nt) {
    *map = cached;
    return cached_slots;
  }
  if (nt * (nt + 1) / 2 > kMaxSlotTiles) return -1;
  std::vector<int> slot_end;
  // tiles in order of first use (column, then row)
  for (int k = 0; k < nt; ++k) {
    for (int I = k; I < nt; ++I) {
      const int s0 = k > 0 ? k - 1 : 0, e0 = I == k ? k : I - 1;
      int chosen = -1;
      for (size_t j = 0; j < slot_end.size(); ++j)
        if (slot_end[j] < s0) {
          chosen = (int)j;
          break;
        }
      if (chosen < 0) {
        chosen = (int)slot_end.size();
        slot_end.push_back(e0);
      } else {
        slot_end[chosen] = e0;
      }
      map->s[I * kSlotStride + k] = chosen * 64 * (int)sizeof(double);
    }
  }
  cached_nt = nt;
  cached_slots = (int)slot_end.size();
  cached = *map;
  return cached_slots;
}

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

cudaError_t launch_big_k05(const Plan&, const CovParams&, int64_t, int64_t, cudaStream_t, bool);
cudaError_t launch_big_k15(const Plan&, const CovParams&, int64_t, int64_t, cudaStream_t, bool);
cudaError_t launch_big_k25(const Plan&, const CovParams&, int64_t, int64_t, cudaStream_t, bool);
cudaError_t launch_big_kgen(const Plan&, const CovParams&, int64_t, int64_t, cudaStream_t, bool);
cudaError_t launch_big_kpow(const Plan&, const CovParams&, int64_t, int64_t, cudaStream_t, bool);

cudaError_t launch_loglik_big(const Plan& p, const CovParams& cp, int64_t e_lo, int64_t e_hi,
                              cudaStream_t stream, bool cache) {
  if (!big_supported(p.m, cp.kind)) return cudaErrorNotSupported;
  if (e_hi <= e_lo) return cudaSuccess;
  switch (cp.kind) {
    case kMatern05: return launch_big_k05(p, cp, e_lo, e_hi, stream, cache);
    case kMatern15: return launch_big_k15(p, cp, e_lo, e_hi, stream, cache);
    case kMatern25: return launch_big_k25(p, cp, e_lo, e_hi, stream, cache);
    case kMaternGen: return launch_big_kgen(p, cp, e_lo, e_hi, stream, cache);
    default: return launch_big_kpow(p, cp, e_lo, e_hi, stream, cache);
  }
}

}  // namespace vgp
