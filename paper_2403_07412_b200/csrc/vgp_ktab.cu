// Per-evaluation table of the general-nu Matern covariance (vgp_ktab.cuh).
#include "vgp_ktab.cuh"

namespace vgp {

namespace {

// one thread per segment: values at the 8 Chebyshev nodes (device Bessel K),
// Chebyshev coefficients, then the power basis in t (Horner form)
__global__ void ktab_build_kernel(CovParams cp, double* __restrict__ out) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= kKtabSegments) return;
  constexpr int N = kKtabDeg + 1;
  const int ex = kKtabOMin + s / kKtabSeg;
  const int k = s % kKtabSeg;
  // u = 2^ex (1 + (k + 1/2 + t/2) / 64): centre and half width
  const double scale = ldexp(1.0, ex);
  const double mid = scale * (1.0 + (k + 0.5) / kKtabSeg);
  const double hw = scale * 0.5 / kKtabSeg;
  double f[N];
#pragma unroll
  for (int j = 0; j < N; ++j) {
    const double x = cos(kPi * (j + 0.5) / N);
    const double u = mid + hw * x;
    // u >= 1: C(u) / s2 (the evaluation multiplies by s2);
    // u < 1: s2 - C(u), so the small deviation from s2 that a smooth kernel's
    // near-singular blocks hinge on is interpolated to RELATIVE accuracy
    const double v = ex >= 0 ? cp.coef * pow(u, cp.nu) * bessel_k(cp, u)
                             : cp.s2 - cp.s2 * cp.coef * pow(u, cp.nu) * bessel_k(cp, u);
    f[j] = v;
  }
  // Chebyshev coefficients c_i = (2/N) sum_j f_j T_i(x_j) (c_0 halved)
  double c[N];
#pragma unroll
  for (int i = 0; i < N; ++i) {
    double acc = 0.0;
#pragma unroll
    for (int j = 0; j < N; ++j) acc += f[j] * cos(kPi * i * (j + 0.5) / N);
    c[i] = (i == 0 ? 1.0 : 2.0) * acc / N;
  }
  // power basis: p(t) = sum_i c_i T_i(t), T_{i+1} = 2 t T_i - T_{i-1}
  double p[N] = {}, tm[N] = {}, t0[N] = {}, t1[N] = {};
  t0[0] = 1.0;  // T_0
  t1[1] = 1.0;  // T_1
#pragma unroll
  for (int d = 0; d < N; ++d) p[d] += c[0] * t0[d] + c[1] * t1[d];
#pragma unroll
  for (int i = 2; i < N; ++i) {
#pragma unroll
    for (int d = 0; d < N; ++d) tm[d] = (d > 0 ? 2.0 * t1[d - 1] : 0.0) - t0[d];
#pragma unroll
    for (int d = 0; d < N; ++d) {
      p[d] += c[i] * tm[d];
      t0[d] = t1[d];
      t1[d] = tm[d];
    }
  }
#pragma unroll
  for (int d = 0; d < N; ++d) out[(size_t)s * N + d] = p[d];
}

}  // namespace

cudaError_t launch_ktab_build(const CovParams& cp, double* d_ktab, cudaStream_t stream) {
  ktab_build_kernel<<<(kKtabSegments + 127) / 128, 128, 0, stream>>>(cp, d_ktab);
  return cudaGetLastError();
}

}  // namespace vgp
