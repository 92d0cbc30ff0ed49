// Thread-per-block kernel for small conditioning sets (m <= 12), variant 13.
//
// At small m a block is a few hundred flops, and the warp-per-block DMMA
// kernels spend ~1,300 issue cycles per block on 8x8-tile bookkeeping and
// padding (profiles/r01_smallm_variants.txt).  Here one thread owns one block
// (vg/vecchia.py:154-162 assemble, :180-190 _numeric_stage, :193-214
// _reduction_stage) with the augmented lower triangle in registers — rows
// 0..m-1 Sigma_e, row m the cross-covariances v_e (diagonal sigma^2), row
// m+1 the neighbour observations yJ — fully unrolled at compile-time m:
// after the m pivot columns, row m holds v' = L^-1 v and sigma_new = s2 - v'.v',
// row m+1 holds y' and -mu = -y'.v' (Schur complement).  Pivots use a true
// sqrt and division.  Euclidean distances from coordinates, closed-form
// Matern (cov_lean, exp table in shared memory); NPD reporting and outputs
// as the other block kernels (npd_key, rest / mu / sig).
#include "vgp_internal.cuh"
#include "vgp_ll_kernel.cuh"

namespace vgp {
namespace tiny {

constexpr int kThreads = 128;
constexpr int kMaxM = 12;  // m = 11, 12 spill a few bytes at 254 registers and still run 3x the warp kernel

template <int M>
struct Tri {
  static constexpr int kRows = M + 2;
  __host__ __device__ static constexpr int idx(int i, int j) { return i * (i + 1) / 2 + j; }
  static constexpr int kN = idx(M + 1, M) + 1;
};

template <int M, int KIND>
__global__ void __launch_bounds__(kThreads)
loglik_tiny_kernel(const double4* __restrict__ pts, const int32_t* __restrict__ nbr, int64_t e_lo, int64_t e_hi,
                   int64_t rest_lo, double s2, double inv_beta, double* __restrict__ rest,
                   double* __restrict__ mu_out, double* __restrict__ sig_out,
                   unsigned long long* __restrict__ fail) {
  __shared__ double tab[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) tab[i] = s2 * kExp2Table[i];
  __syncthreads();
  using T = Tri<M>;
  for (int64_t e = e_lo + (int64_t)blockIdx.x * kThreads + threadIdx.x; e < e_hi;
       e += (int64_t)gridDim.x * kThreads) {
    const int64_t kk = e - 1 - rest_lo;
    double px[M + 1], py[M + 1], a[T::kN];
    double ob[M];
    const int32_t* J = nbr + kk * M;
#pragma unroll
    for (int i = 0; i < M; ++i) {
      const double4 p = pts[J[i]];
      px[i] = p.x;
      py[i] = p.y;
      ob[i] = p.z;
    }
    const double4 tp = pts[M + e - 1];
    px[M] = tp.x;
    py[M] = tp.y;
    // generate: Sigma (rows 0..M-1), v (row M, diagonal s2), yJ (row M+1)
#pragma unroll
    for (int i = 0; i <= M; ++i) {
#pragma unroll
      for (int j = 0; j <= i; ++j) {
        if (i == j) {
          a[T::idx(i, j)] = s2;
        } else {
          const double dx = px[i] - px[j], dy = py[i] - py[j];
          a[T::idx(i, j)] = ll::cov_lean<KIND>(sqrt_pos_nz(fma(dx, dx, fma(dy, dy, 0x1p-1000))), inv_beta, tab);
        }
      }
    }
#pragma unroll
    for (int j = 0; j < M; ++j) a[T::idx(M + 1, j)] = ob[j];
    a[T::idx(M + 1, M)] = 0.0;
    // right-looking Cholesky over the M pivot columns
    int fj = -1;
#pragma unroll
    for (int k = 0; k < M; ++k) {
      const double piv = a[T::idx(k, k)];
      if (fj < 0 && !(piv > 0.0)) fj = k;
      const double d = sqrt(piv);
      const double inv = 1.0 / d;
      a[T::idx(k, k)] = d;
#pragma unroll
      for (int i = 1; i <= M + 1; ++i)
        if (i > k) a[T::idx(i, k)] *= inv;
#pragma unroll
      for (int i = 1; i <= M + 1; ++i) {
#pragma unroll
        for (int j = 1; j <= M; ++j)
          if (i > k && j > k && j <= i) a[T::idx(i, j)] = fma(-a[T::idx(i, k)], a[T::idx(j, k)], a[T::idx(i, j)]);
      }
    }
    if (fj >= 0) {
      atomicMin(&fail[0], npd_key(e, fj, M));
      continue;
    }
    const double sg = a[T::idx(M, M)];
    const double mu = -a[T::idx(M + 1, M)];
    mu_out[kk] = mu;
    sig_out[kk] = sg;
    if (!(sg > 0.0)) {
      atomicMin(&fail[1], (unsigned long long)e);
      rest[kk] = 0.0;
    } else {
      const double resid = tp.z - mu;
      rest[kk] = -0.5 * (resid * resid / sg + kLog2Pi + log(sg));
    }
  }
}

template <int M, int KIND>
cudaError_t launch_m(const Plan& p, const CovParams& cp, int64_t e_lo, int64_t e_hi, cudaStream_t s) {
  const int64_t count = e_hi - e_lo;
  const int64_t want = (count + kThreads - 1) / kThreads;
  const int64_t cap = (int64_t)p.num_sms * 16;
  const int grid = (int)(want < cap ? want : cap);
  loglik_tiny_kernel<M, KIND><<<grid, kThreads, 0, s>>>(p.d_pts, p.d_nbr, e_lo, e_hi, p.rest_lo, cp.s2,
                                                         cp.inv_beta, p.d_rest, p.d_mu, p.d_sig, p.d_fail);
  return cudaGetLastError();
}

template <int KIND>
cudaError_t launch_kind(const Plan& p, const CovParams& cp, int64_t e_lo, int64_t e_hi, cudaStream_t s) {
  switch (p.m) {
    case 1: return launch_m<1, KIND>(p, cp, e_lo, e_hi, s);
    case 2: return launch_m<2, KIND>(p, cp, e_lo, e_hi, s);
    case 3: return launch_m<3, KIND>(p, cp, e_lo, e_hi, s);
    case 4: return launch_m<4, KIND>(p, cp, e_lo, e_hi, s);
    case 5: return launch_m<5, KIND>(p, cp, e_lo, e_hi, s);
    case 6: return launch_m<6, KIND>(p, cp, e_lo, e_hi, s);
    case 7: return launch_m<7, KIND>(p, cp, e_lo, e_hi, s);
    case 8: return launch_m<8, KIND>(p, cp, e_lo, e_hi, s);
    case 9: return launch_m<9, KIND>(p, cp, e_lo, e_hi, s);
    case 10: return launch_m<10, KIND>(p, cp, e_lo, e_hi, s);
    case 11: return launch_m<11, KIND>(p, cp, e_lo, e_hi, s);
    case 12: return launch_m<12, KIND>(p, cp, e_lo, e_hi, s);
    default: return cudaErrorNotSupported;
  }
}

}  // namespace tiny

bool tiny_supported(int m, int kind) { return m >= 1 && m <= tiny::kMaxM && kind <= kMatern25; }

cudaError_t launch_loglik_tiny(const Plan& p, const CovParams& cp, int64_t e_lo, int64_t e_hi,
                               cudaStream_t stream) {
  if (!tiny_supported(p.m, cp.kind) || p.metric != VGP_METRIC_EUCLIDEAN) return cudaErrorNotSupported;
  if (e_hi <= e_lo) return cudaSuccess;
  switch (cp.kind) {
    case kMatern05: return tiny::launch_kind<kMatern05>(p, cp, e_lo, e_hi, stream);
    case kMatern15: return tiny::launch_kind<kMatern15>(p, cp, e_lo, e_hi, stream);
    default: return tiny::launch_kind<kMatern25>(p, cp, e_lo, e_hi, stream);
  }
}

}  // namespace vgp
