// Lean FP64 math for the fused covariance generation.  Every routine is
// within ~2 ulp of the correctly rounded value over the domain the kernel
// uses (checked against numpy in tests/test_gpu_kernels.py), has no
// special-case branches, and spends at most a third of libdevice's FP64
// instructions:
//   sqrt_pos      MUFU.RSQ64H seed + two Newton steps on the root    6 FP64
//   sqrt_pos_nz   MUFU.RSQ64H seed + one third-order step             5 FP64
//   rsqrt_pos     MUFU.RSQ64H seed + two Newton steps                 8 FP64
//   exp_neg_tab   exp(-u) = T[j] * p(r) * 2^e, 256-entry 2^(j/256)
//                 table, Cody-Waite reduction, degree-4 polynomial     9 FP64
#pragma once

#include "vgp_exp_table.cuh"

namespace vgp {

__device__ __forceinline__ double rsqrt_seed(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  return y;
}

// sqrt(x) for x >= 0; x below the normal range (duplicate points) gives 0.
__device__ __forceinline__ double sqrt_pos(double x) {
  const double y = rsqrt_seed(x);
  const double h = 0.5 * y;
  double s = x * y;
  double r = fma(-s, s, x);
  s = fma(r, h, s);
  r = fma(-s, s, x);
  s = fma(r, h, s);
  return (__double2hiint(x) < 0x00100000) ? 0.0 : s;
}

// sqrt(x) for normal x > 0 (no zero guard: callers add 2^-1000 to squared
// distances, so exact duplicates come out as d ~ 1e-150, i.e. C(d) = C(0)).
// One third-order step on s = x y0: sqrt(x) = s (1 - e)^(-1/2) with
// e = 1 - s y0 (the rounding of s cancels), truncated after 3 e^2 / 8
// (|e| < 2^-21, so the next term is ~2^-65): 5 FP64, 4 deep.
__device__ __forceinline__ double sqrt_pos_nz(double x) {
  const double y = rsqrt_seed(x);
  const double s = x * y;
  const double e = fma(-s, y, 1.0);
  const double p = fma(e, 0.375, 0.5);
  return fma(s * e, p, s);
}

// 1/sqrt(x) for normal x > 0.
__device__ __forceinline__ double rsqrt_pos(double x) {
  double y = rsqrt_seed(x);
  double e = fma(-(x * y), y, 1.0);
  y = fma(0.5 * y, e, y);
  e = fma(-(x * y), y, 1.0);
  y = fma(0.5 * y, e, y);
  return y;
}

// 1/sqrt(x) for normal x > 0 with one third-order (Halley-type) step:
// e = 1 - x y0^2, y = y0 (1 + e/2 + 3 e^2 / 8); the dependent chain is 5
// FP64 ops instead of 8 (it sits on the Cholesky pivot critical path).
__device__ __forceinline__ double rsqrt_pos3(double x) {
  const double y0 = rsqrt_seed(x);
  const double e = fma(-(x * y0), y0, 1.0);
  const double p = fma(e, 0.375, 0.5);
  return fma(y0, e * p, y0);
}

// tab[j] = scale * 2^(j/256) (shared memory).  Returns scale * exp(-u) for
// u >= 0 (results below ~1e-290 are not guaranteed exact; see below).
__device__ __forceinline__ double exp_neg_tab(double u, const double* __restrict__ tab) {
  const double shift = 0x1.8p52;
  const double t = fma(-u, k256OverLn2, shift);  // round(-u * 256 / ln 2) in the low word
  const double kf = t - shift;
  const int ki = __double2loint(t);
  double r = fma(-kf, kLn2Over256Hi, -u);
  r = fma(-kf, kLn2Over256Lo, r);
  double p = fma(r, 1.0 / 24.0, 1.0 / 6.0);
  p = fma(p, r, 0.5);
  p = fma(p, r, 1.0);
  p = fma(p, r, 1.0);
  const double v = tab[ki & 255] * p;
  // 2^e by adding e to the exponent field (one IMAD); e is clamped at -1000
  // so deep underflow returns ~1e-301 * v instead of wrapping (such entries
  // are below any Cholesky rounding and the reference's exp underflows them).
  const int e = max(ki >> 8, -1000);
  return __hiloint2double(__double2hiint(v) + e * 0x100000, __double2loint(v));
}

}  // namespace vgp
