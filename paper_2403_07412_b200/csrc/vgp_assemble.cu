// Materialised conditioning batches (vecchia.assemble, vg/vecchia.py:106-166)
// for the unfused stage API (assemble -> _numeric_stage -> _reduction_stage,
// the path cli.cmd_bench times, vg/cli.py:259-263).  The fused likelihood
// kernels never build this workspace; this is the compatibility path.
//
// Entry 0: Sigma = C(d(a, b)), a, b < m; v = yJ = obs[0:m].  Entry e >= 1
// (target t = m + e - 1, J = nbr[e - 1]): Sigma[a][b] = C(d(J[a], J[b])),
// v[a] = C(d(t, J[a])), yJ[a] = obs[J[a]].  Column-major matrices (element
// (a, b) at b * m + a, vg/batchla.py:74-82).  One thread per element, HBM-
// write bound: consecutive threads write consecutive a.
#include <algorithm>

#include "vgp_internal.cuh"
#include "vgp_math.cuh"

namespace vgp {
namespace {

__global__ void assemble_sigma_kernel(const double2* __restrict__ pts, int m, const int64_t* __restrict__ nbr,
                                      int64_t e0, int64_t ne, int metric, double radius, CovParams cp,
                                      double* __restrict__ S) {
  const int64_t mm = (int64_t)m * m;
  const int64_t total = ne * mm;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = idx / mm;
    const int64_t r = idx - k * mm;
    const int b = (int)(r / m), a = (int)(r - (int64_t)b * m);
    const int64_t e = e0 + k;
    int64_t ia = a, ib = b;
    if (e > 0) {
      const int64_t* J = nbr + (e - 1) * (int64_t)m;
      ia = J[a];
      ib = J[b];
    }
    const double2 pa = pts[ia], pb = pts[ib];
    S[idx] = cov_ref(cp, point_dist(metric, radius, pa.x, pa.y, pb.x, pb.y));
  }
}

__global__ void assemble_vec_kernel(const double2* __restrict__ pts, const double* __restrict__ obs, int m,
                                    const int64_t* __restrict__ nbr, int64_t e0, int64_t ne, int metric,
                                    double radius, CovParams cp, double* __restrict__ v,
                                    double* __restrict__ yJ) {
  const int64_t total = ne * m;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = idx / m;
    const int a = (int)(idx - k * m);
    const int64_t e = e0 + k;
    if (e == 0) {
      v[idx] = obs[a];
      yJ[idx] = obs[a];
    } else {
      const int64_t t = m + e - 1;
      const int64_t j = nbr[(e - 1) * (int64_t)m + a];
      const double2 pt = pts[t], pj = pts[j];
      v[idx] = cov_ref(cp, point_dist(metric, radius, pt.x, pt.y, pj.x, pj.y));
      yJ[idx] = obs[j];
    }
  }
}

}  // namespace

cudaError_t launch_assemble(const double2* d_pts, const double* d_obs, int m, const int64_t* d_nbr, int64_t e0,
                            int64_t ne, int metric, double radius, const CovParams& cp, double* d_S,
                            double* d_v, double* d_y, int num_sms, cudaStream_t s) {
  const int bs = 256;
  const int64_t els = ne * (int64_t)m * m;
  const int64_t gs = std::min<int64_t>((els + bs - 1) / bs, (int64_t)num_sms * 16);
  assemble_sigma_kernel<<<(unsigned)std::max<int64_t>(gs, 1), bs, 0, s>>>(d_pts, m, d_nbr, e0, ne, metric, radius,
                                                                          cp, d_S);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  const int64_t gv = std::min<int64_t>((ne * m + bs - 1) / bs, (int64_t)num_sms * 16);
  assemble_vec_kernel<<<(unsigned)std::max<int64_t>(gv, 1), bs, 0, s>>>(d_pts, d_obs, m, d_nbr, e0, ne, metric,
                                                                        radius, cp, d_v, d_y);
  return cudaGetLastError();
}

}  // namespace vgp
