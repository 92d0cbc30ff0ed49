// Plan-time distance cache for the fused kernel: for every block of the
// plan, the distances of the lower triangle (with the diagonal) of rows 0..m
// of its conditioning block, in the warp-specialised kernel's shared-memory
// tile layout (vgp_ws_kernel.cuh: 8x8 tiles of the lower tile triangle,
// swizzled 16-byte chunks; row m is the target's cross-distances v).  Distances depend on the locations and the
// neighbour table only, not on theta, so an MLE loop evaluates hundreds of
// likelihoods against one cache.  Bit-identical to the on-the-fly distances
// of vgp_ws_kernel.cuh (same formula), so cached and uncached evaluations
// agree bit for bit.
#include "vgp_internal.cuh"
#include "vgp_math.cuh"
#include "vgp_ws_kernel.cuh"

namespace vgp {
namespace {

constexpr int kWarps = 4;

__global__ void __launch_bounds__(kWarps * 32)
build_dcache_kernel(const double4* __restrict__ pts, const int32_t* __restrict__ nbr, int m,
                    int64_t e_lo, int64_t e_hi, int64_t rest_lo, double* __restrict__ cache,
                    int64_t cstride, int metric, double radius,
                    unsigned long long* __restrict__ dmax) {
  double dm = 0.0;  // largest cached distance (the K_nu table's shared window)
  extern __shared__ double2 sxy[];  // kWarps x (m + 1)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double2* XY = sxy + warp * (m + 1);
  for (int64_t e = e_lo + (int64_t)blockIdx.x * kWarps + warp; e < e_hi;
       e += (int64_t)gridDim.x * kWarps) {
    const int32_t* J = nbr + (e - 1 - rest_lo) * (int64_t)m;
    for (int a = lane; a <= m; a += 32) {
      const double4 p = pts[a < m ? (int64_t)J[a] : (int64_t)(m + e - 1)];
      XY[a] = make_double2(p.x, p.y);
    }
    __syncwarp();
    double* out = cache + (e - 1 - rest_lo) * cstride;
    // tile (I, J), J <= I < NT, row r, column col: d(8I + r, 8J + col) on and
    // below the diagonal for rows <= m, else 0; ws::chunk_off swizzle
    const int nt = (m + 2 + 7) / 8;
    const int total = ws::ntri(nt) * 64;
    for (int idx = lane; idx < total; idx += 32) {
      const int t = idx >> 6, w = idx & 63;
      int J = 0, tt = t;
      while (tt >= nt - J) tt -= nt - J++;
      const int I = J + tt;
      const int rr = w >> 3, col = w & 7;
      const int i = 8 * I + rr, k = 8 * J + col;
      double d = 0.0;
      if (k <= i && i <= m) {
        if (metric == VGP_METRIC_GREAT_CIRCLE) {
          // haversine, vg/geo.py:70-79 (degrees; 0 for coincident points)
          d = dist_gcd(XY[k].x, XY[k].y, XY[i].x, XY[i].y, radius);
        } else {
          const double dx = XY[i].x - XY[k].x;
          const double dy = XY[i].y - XY[k].y;
          d = sqrt_pos_nz(fma(dx, dx, fma(dy, dy, 0x1p-1000)));  // as vgp_ws_kernel.cuh
        }
      }
      out[t * 64 + ws::chunk_off(rr, col >> 1) + (col & 1)] = d;
      dm = fmax(dm, d);
    }
    __syncwarp();
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) dm = fmax(dm, __shfl_xor_sync(0xffffffffu, dm, off));
  if (lane == 0 && dmax) atomicMax(dmax, (unsigned long long)__double_as_longlong(dm));
}

__global__ void diff_kernel(const double* __restrict__ a, const double* __restrict__ b, int64_t n,
                            int* __restrict__ flag) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    if (__double_as_longlong(a[i]) != __double_as_longlong(b[i])) *flag = 1;
}

}  // namespace

int64_t dcache_stride(int m) { return (int64_t)ws::ntri((m + 2 + 7) / 8) * 64; }

cudaError_t launch_build_dcache(const Plan& p, cudaStream_t stream) {
  const int64_t e_lo = p.rest_lo + 1, e_hi = p.rest_hi + 1;
  if (e_hi <= e_lo) return cudaSuccess;
  const int64_t want = (e_hi - e_lo + kWarps - 1) / kWarps;
  const int grid = (int)(want < (int64_t)p.num_sms * 8 ? want : (int64_t)p.num_sms * 8);
  const size_t sm = sizeof(double2) * kWarps * (p.m + 1);
  if (p.d_flag) cudaMemsetAsync(p.d_flag + 2, 0, sizeof(unsigned long long), stream);
  build_dcache_kernel<<<grid, kWarps * 32, sm, stream>>>(
      p.d_pts, p.d_nbr, p.m, e_lo, e_hi, p.rest_lo, p.d_dcache, p.dcache_stride, p.metric, p.radius,
      p.d_flag ? reinterpret_cast<unsigned long long*>(p.d_flag + 2) : nullptr);
  return cudaGetLastError();
}

cudaError_t launch_diff(const double* a, const double* b, int64_t n, int* flag,
                        cudaStream_t stream) {
  diff_kernel<<<296, 256, 0, stream>>>(a, b, n, flag);
  return cudaGetLastError();
}

}  // namespace vgp
