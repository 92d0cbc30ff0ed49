// Generic fused Vecchia block kernel: any conditioning size m.
//
// One CTA per batch entry e (grid-stride).  The entry's conditioning block is
// generated straight into an augmented column-major matrix
//     rows 0..m-1 : Sigma_e = C(||s_Ja - s_Jb||)          (vg/vecchia.py:154-160)
//     row  m      : v_e     = C(||s_t - s_Ja||)            (vg/vecchia.py:160-161)
//     row  m+1    : yJ_e    = y[J]                          (vg/vecchia.py:162)
// which lives in shared memory when it fits and in a per-CTA global
// workspace slot otherwise (the reference's full-conditioning tests use
// m up to n-1).  The right-looking sweep on the first m columns is the
// reference's _potrf_sweep (vg/batchla.py:141-156): pivot test !(piv > 0),
// sqrt, divide the column, rank-1 update the trailing part; applied to the
// two extra rows it is exactly batch_trsv's forward substitution
// (vg/batchla.py:196-207), so v' and y' come out of the same sweep.  The two
// dots accumulate in ascending index order like batch_dot
// (vg/batchla.py:223-226).  Entry 0 is the joint block with v = yJ = y[:m]
// and produces block_first (vg/vecchia.py:202-204).
//
// This path is arithmetic-for-arithmetic the reference's (true divisions,
// reference association) and serves large m and the correctness baseline; the
// m <= 62 hot path is the warp/DMMA kernel in vgp_loglik_dmma.cu.
#include "vgp_math.cuh"
#include "vgp_pairwise.cuh"

namespace vgp {

namespace {

constexpr int kGenThreads = 128;

template <bool kShared>
__global__ void __launch_bounds__(kGenThreads)
loglik_generic_kernel(const double4* __restrict__ pts, const int32_t* __restrict__ nbr, int m,
                      int64_t e_lo, int64_t e_hi, int64_t rest_lo, CovParams cp, int metric,
                      double radius, double* __restrict__ work, int ld,
                      double* __restrict__ rest, double* __restrict__ mu_out,
                      double* __restrict__ sig_out, double* __restrict__ scalars,
                      unsigned long long* __restrict__ fail) {
  extern __shared__ double smem[];
  // shared layout: [coords 3*(m+1)] [A ld*(m+2) if kShared]
  double* px = smem;
  double* py = px + (m + 1);
  double* pv = py + (m + 1);
  double* A = kShared ? (pv + (m + 1)) : (work + (size_t)blockIdx.x * ld * (m + 2));
  __shared__ int s_fail;
  __shared__ double s_piv;
  const int P = m + 2;

  for (int64_t e = e_lo + blockIdx.x; e < e_hi; e += gridDim.x) {
    const bool joint = (e == 0);
    // ---- gather the conditioning set (index m = target) ----
    for (int a = threadIdx.x; a <= m; a += blockDim.x) {
      int64_t src;
      if (joint) {
        src = (a < m) ? a : 0;
      } else {
        src = (a < m) ? (int64_t)nbr[(e - 1 - rest_lo) * (int64_t)m + a] : (m + e - 1);
      }
      double4 p = pts[src];
      px[a] = p.x;
      py[a] = p.y;
      pv[a] = p.z;
    }
    if (threadIdx.x == 0) s_fail = 0;
    __syncthreads();
    // ---- generate lower triangle of the augmented matrix ----
    // column-major: A[i + k*ld], i >= k
    for (int k = 0; k < m; ++k) {
      for (int i = k + threadIdx.x; i < P; i += blockDim.x) {
        double val;
        if (i < m) {
          val = (i == k) ? cp.s2
                         : cov_ref(cp, point_dist(metric, radius, px[i], py[i], px[k], py[k]));
        } else if (i == m) {
          // v: entry 0 holds y (vg/vecchia.py:149); else C(||s_t - s_Jk||)
          val = joint ? pv[k]
                      : cov_ref(cp, point_dist(metric, radius, px[m], py[m], px[k], py[k]));
        } else {
          val = pv[k];  // yJ
        }
        A[i + (size_t)k * ld] = val;
      }
    }
    __syncthreads();
    // ---- right-looking sweep over the first m columns ----
    int failed_col = -1;
    for (int j = 0; j < m; ++j) {
      if (threadIdx.x == 0) {
        double piv = A[j + (size_t)j * ld];
        if (!(piv > 0.0)) {
          s_fail = 1 + j;
        } else {
          s_piv = sqrt(piv);
          A[j + (size_t)j * ld] = s_piv;
        }
      }
      __syncthreads();
      if (s_fail) {
        failed_col = s_fail - 1;
        break;
      }
      const double d = s_piv;
      for (int i = j + 1 + threadIdx.x; i < P; i += blockDim.x) A[i + (size_t)j * ld] /= d;
      __syncthreads();
      // trailing update: A[i][k] -= A[i][j] * A[k][j], j < k <= min(i, m-1)
      for (int i = j + 1 + threadIdx.x; i < P; i += blockDim.x) {
        const double lij = A[i + (size_t)j * ld];
        const int kmax = i < m ? i : m - 1;
        for (int k = j + 1; k <= kmax; ++k)
          A[i + (size_t)k * ld] = __dsub_rn(A[i + (size_t)k * ld], __dmul_rn(lij, A[k + (size_t)j * ld]));
      }
      __syncthreads();
    }
    if (failed_col >= 0) {
      if (threadIdx.x == 0) atomicMin(&fail[0], npd_key(e, failed_col, m));
      __syncthreads();
      continue;
    }
    if (threadIdx.x == 0) {
      // batch_dot in ascending order, vg/batchla.py:223-226
      double accm = 0.0, accs = 0.0;
      for (int k = 0; k < m; ++k) {
        double vk = A[m + (size_t)k * ld];
        double yk = A[m + 1 + (size_t)k * ld];
        accm = __dadd_rn(accm, __dmul_rn(yk, vk));  // no contraction: numpy rounds each op
        accs = __dadd_rn(accs, __dmul_rn(vk, vk));
      }
      if (joint) {
        // block_first = -half_log_det(L0) - mu'0/2 - (m/2) log 2pi, vg/vecchia.py:202-204
        // log of the diagonal into the (now free) coordinate scratch
        for (int k = 0; k < m; ++k) px[k] = log(A[k + (size_t)k * ld]);
        double hld = pairwise_rec(px, m);
        scalars[1] = -hld - 0.5 * accm - 0.5 * m * kLog2Pi;
      } else {
        int64_t k = e - 1 - rest_lo;
        double sg = cp.s2 - accs;  // vg/vecchia.py:206
        mu_out[k] = accm;
        sig_out[k] = sg;
        if (!(sg > 0.0)) {
          atomicMin(&fail[1], (unsigned long long)e);
          rest[k] = 0.0;
        } else {
          double resid = pv[m] - accm;  // ordered_obs[m:] - mu_new, vg/vecchia.py:211
          rest[k] = -0.5 * (resid * resid / sg + kLog2Pi + log(sg));
        }
      }
    }
    __syncthreads();
  }
}

}  // namespace

cudaError_t launch_loglik_generic(const Plan& p, const CovParams& cp, int64_t e_lo, int64_t e_hi,
                                  cudaStream_t stream) {
  if (e_hi <= e_lo) return cudaSuccess;
  const int m = p.m;
  const int P = m + 2;
  const int ld = P | 1;  // odd leading dimension: conflict-free column walks
  size_t coord_bytes = sizeof(double) * 3 * (m + 1);
  size_t mat_bytes = sizeof(double) * (size_t)ld * P;
  int64_t count = e_hi - e_lo;
  if (coord_bytes + mat_bytes <= 200 * 1024) {
    size_t sm = coord_bytes + mat_bytes;
    cudaError_t err = cudaFuncSetAttribute(loglik_generic_kernel<true>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (err != cudaSuccess) return err;
    int64_t grid = count < (int64_t)p.num_sms * 64 ? count : (int64_t)p.num_sms * 64;
    loglik_generic_kernel<true><<<(unsigned)grid, kGenThreads, sm, stream>>>(
        p.d_pts, p.d_nbr, m, e_lo, e_hi, p.rest_lo, cp, p.metric, p.radius, nullptr, ld,
        p.d_rest, p.d_mu, p.d_sig, p.d_scalars, p.d_fail);
  } else {
    if (!p.d_work || p.work_slots < 1) return cudaErrorMemoryAllocation;
    cudaError_t err = cudaFuncSetAttribute(loglik_generic_kernel<false>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)coord_bytes);
    if (err != cudaSuccess) return err;
    int64_t grid = count < p.work_slots ? count : p.work_slots;
    loglik_generic_kernel<false><<<(unsigned)grid, kGenThreads, coord_bytes, stream>>>(
        p.d_pts, p.d_nbr, m, e_lo, e_hi, p.rest_lo, cp, p.metric, p.radius, p.d_work, ld,
        p.d_rest, p.d_mu, p.d_sig, p.d_scalars, p.d_fail);
  }
  return cudaGetLastError();
}

}  // namespace vgp
