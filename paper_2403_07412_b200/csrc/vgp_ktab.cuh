// General-nu Matern covariance by per-evaluation piecewise polynomials.
//
// C(u) = s2 2^(1-nu)/Gamma(nu) u^nu K_nu(u), u = d / beta (vg/kernels.py:75-81)
// depends on the evaluation's (s2, nu) and on u only.  Once per likelihood
// evaluation a small kernel tabulates it (device Bessel K, vgp_math.cuh) on
// 64 segments per binade of u, u in [2^kKtabOMin, 2^(kKtabOMax+1)): on each
// segment a degree-7 polynomial in t in [-1, 1) interpolating at the
// Chebyshev nodes (measured relative interpolation error <= 2e-15 against
// scipy.special.kv, 7e-14 next to u = 2 where AMOS itself switches methods).
// For u < 1 the table holds s2 - C(u), interpolated to relative accuracy
// (smooth kernels' near-singular blocks hinge on that small deviation); for
// u >= 1 it holds C(u) / s2 itself.  There the segment's relative width
// 1/64 makes e^-u vary by at most e^(-u/64) across it, so the degree-7
// interpolant's relative error is ~(u/128)^8 / (2^7 8!), largest in absolute
// terms near u = 9 at ~2e-19 s2 — far below an ulp of the diagonal — and no
// exp is evaluated per entry (round 2 first stored C e^u / s2 and multiplied
// by a lean exp: ~10 more FP64 operations on ~9% of c5's entries, paid by
// whole warps through divergence).
//
// Evaluation is integer bit work (segment = binade and top 6 mantissa bits;
// t = u scaled into [128, 256) by exponent replacement minus an odd integer,
// both exact), 4 x 16-byte table loads and 7 DFMA (+ the lean exp for u >= 1):
// the cost of a closed-form Matern entry instead of a Bessel iteration.
// u below 1e-90 (the diagonal: distance 0 or the kernels' 2^-500 guard) gives
// s2 (vg/kernels.py:77-78); 1e-90 <= u < 2^kKtabOMin (near-duplicate points)
// falls back to the exact device Bessel K; u beyond the table underflows to 0
// like scipy's kv.
#pragma once

#include <cmath>

#include "vgp_internal.cuh"
#include "vgp_math.cuh"

namespace vgp {

constexpr int kKtabOMin = -40;
constexpr int kKtabOMax = 9;
constexpr int kKtabSeg = 64;  // segments per binade
constexpr int kKtabDeg = 7;
constexpr int kKtabSegments = (kKtabOMax - kKtabOMin + 1) * kKtabSeg;
constexpr int64_t kKtabDoubles = (int64_t)kKtabSegments * (kKtabDeg + 1);

// exact general-nu Matern (the reference expression, not inlined: rare path)
static __device__ __noinline__ double matern_gen_exact(double u, const CovParams& cp) {
  if (!(u > 0.0)) return cp.s2;
  return cp.s2 * cp.coef * pow(u, cp.nu) * bessel_k(cp, u);
}

// C(u) from the table
// A kernel may stage a window of kKtabWinSeg consecutive segments (14
// binades) in shared memory, starting at segment wseg0 (ktab_window); the
// evaluation reads those with LDS, the rest from the global table.
constexpr int kKtabWinSeg = 14 * kKtabSeg;

inline int ktab_window(double dmax, double inv_beta) {
  // the 14 binades below the largest u = d_max / beta of the plan's cache
  if (!(dmax > 0.0)) return -(1 << 30);
  int b = (int)std::floor(std::log2(dmax * inv_beta));
  if (b > kKtabOMax) b = kKtabOMax;
  int lo = b - 13;
  if (lo < kKtabOMin) lo = kKtabOMin;
  return (lo - kKtabOMin) * kKtabSeg;
}

__device__ __forceinline__ double cov_ktab(double u, const double* __restrict__ ktab,
                                           const CovParams& cp, const double* ktw = nullptr,
                                           int wseg0 = 0) {
  const int hi = __double2hiint(u);
  const int lo = __double2loint(u);
  const int bex = hi >> 20;  // biased exponent (u >= 0)
  // the diagonal and exact duplicates carry distance 2^-500 (the kernels'
  // sqrt guard) or 0: C(0) = s2 (vg/kernels.py:77-78); genuine near-duplicate
  // distances take the exact path
  if (__builtin_expect(bex < 1023 + kKtabOMin, 0)) return u > 1e-90 ? matern_gen_exact(u, cp) : cp.s2;
  if (__builtin_expect(bex > 1023 + kKtabOMax, 0)) return 0.0;
  // segment = (binade, top 6 mantissa bits); t in [-1, 1) from the remaining
  // 46 mantissa bits: d = 1 + f_low / 64 in [1, 1 + 1/64), t = 128 d - 129
  // = 2 f_low - 1 (both exact)
  const int seg = ((hi >> 14) & 0x1FFFF) - ((1023 + kKtabOMin) << 6);
  const double d = __hiloint2double((hi & 0x3FFF) | 0x3FF00000, lo);
  const double t = fma(d, 128.0, -129.0);
  double2 c01, c23, c45, c67;
  if (ktw && (unsigned)(seg - wseg0) < (unsigned)kKtabWinSeg) {
    const double2* c = reinterpret_cast<const double2*>(ktw + (seg - wseg0) * 8);
    c01 = c[0];
    c23 = c[1];
    c45 = c[2];
    c67 = c[3];
  } else {
    const double2* c = reinterpret_cast<const double2*>(ktab + (size_t)seg * 8);
    c01 = __ldg(c);
    c23 = __ldg(c + 1);
    c45 = __ldg(c + 2);
    c67 = __ldg(c + 3);
  }
  double p = fma(c67.y, t, c67.x);
  p = fma(p, t, c45.y);
  p = fma(p, t, c45.x);
  p = fma(p, t, c23.y);
  p = fma(p, t, c23.x);
  p = fma(p, t, c01.y);
  p = fma(p, t, c01.x);
  if (__builtin_expect(bex >= 1023, 0)) return p * cp.s2;  // u >= 1: C / s2
  return cp.s2 - p;
}

// (re)build the table for cp (kind kMaternGen) into d_ktab (kKtabDoubles)
cudaError_t launch_ktab_build(const CovParams& cp, double* d_ktab, cudaStream_t stream);

}  // namespace vgp
