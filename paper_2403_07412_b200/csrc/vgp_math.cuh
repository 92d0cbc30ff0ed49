// Device-side FP64 math for the Vecchia covariance: distances, Matern closed
// forms, general-nu Matern via a device Bessel K_nu, power exponential.
// Every function states the reference expression it reproduces.
#pragma once

#include "vgp_internal.cuh"

namespace vgp {

// np.hypot(a_x - b_x, a_y - b_y), vg/geo.py:98.  sqrt of an FMA-accumulated
// square sum: within 1 ulp of hypot for non-extreme inputs.
__device__ __forceinline__ double dist_euclid(double ax, double ay, double bx, double by) {
  double dx = ax - bx;
  double dy = ay - by;
  return sqrt(fma(dx, dx, dy * dy));
}

// Haversine great-circle distance, vg/geo.py:70-79 (inputs in degrees).
__device__ __forceinline__ double dist_gcd(double lon1, double lat1, double lon2, double lat2,
                                           double radius) {
  const double r = kPi / 180.0;
  double p1 = lat1 * r, p2 = lat2 * r, l1 = lon1 * r, l2 = lon2 * r;
  double s1 = sin((p2 - p1) / 2.0);
  double s2 = sin((l2 - l1) / 2.0);
  double h = s1 * s1 + cos(p1) * cos(p2) * s2 * s2;
  h = fmin(fmax(h, 0.0), 1.0);
  return 2.0 * radius * asin(sqrt(h));
}

__device__ __forceinline__ double point_dist(int metric, double radius, double ax, double ay,
                                             double bx, double by) {
  return metric == VGP_METRIC_GREAT_CIRCLE ? dist_gcd(ax, ay, bx, by, radius)
                                           : dist_euclid(ax, ay, bx, by);
}

// K_mu(x), K_{mu+1}(x) for |mu| <= 1/2 and then upward recurrence to K_nu,
// nu = mu + nl.  Temme's series for x < 2, Steed's continued fraction CF2
// otherwise (the method of scipy's reference AMOS zbesk is different; parity
// with scipy.special.kv, the routine vg/kernels.py:81 calls, is checked in
// tests at 1e-12 relative).  Returns 0 when e^-x underflows (u >~ 745), as
// scipy's kv does, so s2 * coef * u^nu * K stays finite.
// SCALED: K_nu(x) e^x instead (no under/overflow for large x; table build).
template <bool SCALED = false>
__device__ inline double bessel_k(const CovParams& c, double x) {
  const double eps = 1.0e-16;
  const double mu = c.mu;
  const double xi = 1.0 / x;
  const double xi2 = 2.0 * xi;
  double rkmu, rk1;
  if (x < 2.0) {
    double x2 = 0.5 * x;
    double d = -log(x2);
    double e = mu * d;
    double fact2 = fabs(e) < eps ? 1.0 : sinh(e) / e;
    double ff = c.fact * (c.gam1 * cosh(e) + c.gam2 * fact2 * d);
    double sum = ff;
    e = exp(e);
    double p = 0.5 * e / c.gampl;
    double q = 0.5 / (e * c.gammi);
    double cc = 1.0;
    d = x2 * x2;
    double sum1 = p;
    for (int i = 1; i <= 500; ++i) {
      double di = (double)i;
      ff = (di * ff + p + q) / (di * di - mu * mu);
      cc *= d / di;
      p /= (di - mu);
      q /= (di + mu);
      double del = cc * ff;
      sum += del;
      double del1 = cc * (p - di * ff);
      sum1 += del1;
      if (fabs(del) < fabs(sum) * eps) break;
    }
    rkmu = sum;
    rk1 = sum1 * xi2;
    if (SCALED) {
      const double ex = exp(x);
      rkmu *= ex;
      rk1 *= ex;
    }
  } else {
    double b = 2.0 * (1.0 + x);
    double d = 1.0 / b;
    double h = d, delh = d;
    double q1 = 0.0, q2 = 1.0;
    double a1 = 0.25 - mu * mu;
    double q = a1, cc = a1;
    double a = -a1;
    double s = 1.0 + q * delh;
    for (int i = 2; i <= 10000; ++i) {
      double di = (double)i;
      a -= 2.0 * (di - 1.0);
      cc = -a * cc / di;
      double qnew = (q1 - b * q2) / a;
      q1 = q2;
      q2 = qnew;
      q += cc * qnew;
      b += 2.0;
      d = 1.0 / (b + a * d);
      delh = (b * d - 1.0) * delh;
      h += delh;
      double dels = q * delh;
      s += dels;
      if (fabs(dels / s) < eps) break;
    }
    h = a1 * h;
    rkmu = SCALED ? sqrt(kPi / (2.0 * x)) / s : sqrt(kPi / (2.0 * x)) * exp(-x) / s;
    rk1 = rkmu * (mu + x + 0.5 - h) * xi;
  }
  for (int i = 1; i <= c.nl; ++i) {
    double t = (mu + i) * xi2 * rk1 + rkmu;
    rkmu = rk1;
    rk1 = t;
  }
  return rkmu;
}

// Per-evaluation reciprocal tables for bessel_k_tab: every division in the
// series / continued-fraction iterations is by a quantity that depends on
// the iteration index and mu only, so it becomes a multiplication.
constexpr int kBesselTab = 64;
// t[0..63] 1/(i^2 - mu^2), [64..127] 1/i, [128..191] 1/(i - mu),
// [192..255] 1/(i + mu), [256..319] 1/a_i of Steed's CF2 (a_1 = -(1/4 - mu^2),
// a_i = a_{i-1} - 2(i-1)); entry i at index i (entry 0 unused).
__device__ inline void bessel_fill_tab(const CovParams& c, double* t, int tid, int nthreads) {
  const double mu = c.mu;
  for (int i = tid; i < kBesselTab; i += nthreads) {
    const double di = (double)i;
    t[i] = i ? 1.0 / (di * di - mu * mu) : 0.0;
    t[64 + i] = i ? 1.0 / di : 0.0;
    t[128 + i] = i ? 1.0 / (di - mu) : 0.0;
    t[192 + i] = i ? 1.0 / (di + mu) : 0.0;
    // a_i = -(1/4 - mu^2) - (i - 1) i (closed form of the CF2 recursion)
    t[256 + i] = i >= 2 ? 1.0 / (-(0.25 - mu * mu) - (di - 1.0) * di) : 0.0;
  }
}

// bessel_k with the iteration divisions replaced by table multiplications
// (same series and continued fraction, within a few ulp of bessel_k).
__device__ inline double bessel_k_tab(const CovParams& c, double x, const double* __restrict__ t) {
  const double eps = 1.0e-16;
  const double mu = c.mu;
  const double xi = 1.0 / x;
  const double xi2 = 2.0 * xi;
  double rkmu, rk1;
  if (x < 2.0) {
    double x2 = 0.5 * x;
    double d = -log(x2);
    double e = mu * d;
    double fact2 = fabs(e) < eps ? 1.0 : sinh(e) / e;
    double ff = c.fact * (c.gam1 * cosh(e) + c.gam2 * fact2 * d);
    double sum = ff;
    e = exp(e);
    double p = 0.5 * e / c.gampl;
    double q = 0.5 / (e * c.gammi);
    double cc = 1.0;
    d = x2 * x2;
    double sum1 = p;
    for (int i = 1; i <= 500; ++i) {
      double di = (double)i;
      if (i < kBesselTab) {
        ff = (di * ff + p + q) * t[i];
        cc *= d * t[64 + i];
        p *= t[128 + i];
        q *= t[192 + i];
      } else {
        ff = (di * ff + p + q) / (di * di - mu * mu);
        cc *= d / di;
        p /= (di - mu);
        q /= (di + mu);
      }
      double del = cc * ff;
      sum += del;
      double del1 = cc * (p - di * ff);
      sum1 += del1;
      if (fabs(del) < fabs(sum) * eps) break;
    }
    rkmu = sum;
    rk1 = sum1 * xi2;
  } else {
    double b = 2.0 * (1.0 + x);
    double d = 1.0 / b;
    double h = d, delh = d;
    double q1 = 0.0, q2 = 1.0;
    double a1 = 0.25 - mu * mu;
    double q = a1, cc = a1;
    double a = -a1;
    double s = 1.0 + q * delh;
    for (int i = 2; i <= 10000; ++i) {
      double di = (double)i;
      a -= 2.0 * (di - 1.0);
      double qnew;
      if (i < kBesselTab) {
        cc = -a * cc * t[64 + i];
        qnew = (q1 - b * q2) * t[256 + i];
      } else {
        cc = -a * cc / di;
        qnew = (q1 - b * q2) / a;
      }
      q1 = q2;
      q2 = qnew;
      q += cc * qnew;
      b += 2.0;
      d = 1.0 / (b + a * d);
      delh = (b * d - 1.0) * delh;
      h += delh;
      double dels = q * delh;
      s += dels;
      if (fabs(dels / s) < eps) break;
    }
    h = a1 * h;
    rkmu = sqrt(kPi / (2.0 * x)) * exp(-x) / s;
    rk1 = rkmu * (mu + x + 0.5 - h) * xi;
  }
  for (int i = 1; i <= c.nl; ++i) {
    double tt = (mu + i) * xi2 * rk1 + rkmu;
    rkmu = rk1;
    rk1 = tt;
  }
  return rkmu;
}

// kernels.cov(d, spec), vg/kernels.py:59-98, evaluated exactly as the
// reference writes it (u = d / beta with a true division, same association).
__device__ inline double cov_ref(const CovParams& c, double d) {
  switch (c.kind) {
    case kMatern05: {
      double u = d / c.beta;
      return c.s2 * exp(-u);
    }
    case kMatern15: {
      double u = d / c.beta;
      return c.s2 * (1.0 + u) * exp(-u);
    }
    case kMatern25: {
      double u = d / c.beta;
      return c.s2 * (1.0 + u + u * u / 3.0) * exp(-u);
    }
    case kMaternGen: {
      double u = d / c.beta;
      if (!(u > 0.0)) return c.s2;
      return c.s2 * c.coef * pow(u, c.nu) * bessel_k(c, u);
    }
    default:  // kPowExp
      return c.s2 * exp(-pow(d, c.nu) / c.beta);
  }
}

}  // namespace vgp
