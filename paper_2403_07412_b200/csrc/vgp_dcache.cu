// Plan-time distance cache for the fused kernel: for every block of the
// plan, the distances of the strictly lower part of rows 1..m of its
// conditioning block (compact order, entry (a, b) at a (a-1)/2 + b; row m is
// the target's cross-distances v).  Distances depend on the locations and the
// neighbour table only, not on theta, so an MLE loop evaluates hundreds of
// likelihoods against one cache.  Bit-identical to the on-the-fly distances
// of vgp_dmma_kernel.cuh (same formula), so cached and uncached evaluations
// agree bit for bit.
#include "vgp_fastmath.cuh"
#include "vgp_internal.cuh"

namespace vgp {
namespace {

constexpr int kWarps = 4;

__global__ void __launch_bounds__(kWarps * 32)
build_dcache_kernel(const double4* __restrict__ pts, const int32_t* __restrict__ nbr, int m,
                    int64_t e_lo, int64_t e_hi, int64_t rest_lo, double* __restrict__ cache,
                    int64_t cstride) {
  extern __shared__ double2 sxy[];  // kWarps x (m + 1)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double2* XY = sxy + warp * (m + 1);
  const int nent = m * (m + 1) / 2;
  for (int64_t e = e_lo + (int64_t)blockIdx.x * kWarps + warp; e < e_hi;
       e += (int64_t)gridDim.x * kWarps) {
    const int32_t* J = nbr + (e - 1 - rest_lo) * (int64_t)m;
    for (int a = lane; a <= m; a += 32) {
      const double4 p = pts[a < m ? (int64_t)J[a] : (int64_t)(m + e - 1)];
      XY[a] = make_double2(p.x, p.y);
    }
    __syncwarp();
    double* out = cache + (e - 1 - rest_lo) * cstride;
    int a = 1, b = lane;
    while (a <= m && b >= a) {
      b -= a;
      ++a;
    }
    for (int idx = lane; idx < nent; idx += 32) {
      const double2 pa = XY[a], pb = XY[b];
      const double dx = pa.x - pb.x;
      const double dy = pa.y - pb.y;
      out[idx] = sqrt_pos_nz(fma(dx, dx, fma(dy, dy, 0x1p-1000)));
      b += 32;
      while (a <= m && b >= a) {
        b -= a;
        ++a;
      }
    }
    __syncwarp();
  }
}

__global__ void diff_kernel(const double* __restrict__ a, const double* __restrict__ b, int64_t n,
                            int* __restrict__ flag) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    if (__double_as_longlong(a[i]) != __double_as_longlong(b[i])) *flag = 1;
}

}  // namespace

int64_t dcache_stride(int m) { return ((int64_t)m * (m + 1) / 2 + 1) & ~int64_t(1); }

cudaError_t launch_build_dcache(const Plan& p, cudaStream_t stream) {
  const int64_t e_lo = p.rest_lo + 1, e_hi = p.rest_hi + 1;
  if (e_hi <= e_lo) return cudaSuccess;
  const int64_t want = (e_hi - e_lo + kWarps - 1) / kWarps;
  const int grid = (int)(want < (int64_t)p.num_sms * 8 ? want : (int64_t)p.num_sms * 8);
  const size_t sm = sizeof(double2) * kWarps * (p.m + 1);
  build_dcache_kernel<<<grid, kWarps * 32, sm, stream>>>(p.d_pts, p.d_nbr, p.m, e_lo, e_hi,
                                                          p.rest_lo, p.d_dcache, p.dcache_stride);
  return cudaGetLastError();
}

cudaError_t launch_diff(const double* a, const double* b, int64_t n, int* flag,
                        cudaStream_t stream) {
  diff_kernel<<<296, 256, 0, stream>>>(a, b, n, flag);
  return cudaGetLastError();
}

}  // namespace vgp
