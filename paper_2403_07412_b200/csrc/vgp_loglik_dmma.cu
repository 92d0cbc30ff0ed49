// Warp-per-block FP64 tensor-core (DMMA) Vecchia kernel, m + 2 <= 64.
//
// One warp owns one conditioning block e >= 1 end to end; nothing but the
// block's 8-byte log-density (plus mu / sigma) ever leaves the SM:
//
//   gather   J = NBR[e-1] (int32), (x, y, obs) of the m neighbours and of the
//            target into per-warp shared memory (vg/vecchia.py:154-162);
//   generate the augmented (8*NT) x (8*NT) lower-triangular matrix
//              rows 0..m-1 Sigma_e, row m v_e, row m+1 yJ, zero padding
//            directly into registers as m8n8 DMMA accumulator fragments
//            (lane (r, q) = (lane/4, lane%4) holds entries (r, 2q), (r, 2q+1)
//            of every 8x8 tile (I, J), I >= J);
//   factor   right-looking blocked Cholesky over 8-wide tile columns:
//              panel  : column-by-column on the diagonal tile and the tiles
//                       below it (pivot test !(piv > 0) -> NPD at that column,
//                       vg/batchla.py:146-151), warp shuffles within quads;
//              update : A_IJ -= L_Ic L_Jc^T for c < J <= I with
//                       mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4), two per tile;
//            rows m and m+1 ride along, so the sweep is also the two
//            triangular solves (v' = L^-1 v, y' = L^-1 yJ) and the Schur
//            complements give sigma_new = A[m][m] and -mu = A[m+1][m];
//   reduce   l_e = -1/2 ((y_t - mu)^2 / sigma_new + log 2pi + log sigma_new)
//            (vg/vecchia.py:206-212).
//
// sm_100a has no FP64 tcgen05 kind (ptxas rejects .kind::f64), so the legacy
// DMMA path is the FP64 tensor path on B200; measured peak 37.0 TFLOP/s,
// identical to DFMA's (profiles/r01_fp64_peak.jsonl), but one DMMA issues
// 256 FMAs, which leaves the issue slots to the covariance generation.
#include "vgp_math.cuh"

namespace vgp {
namespace {

constexpr int kWarps = 4;  // warps (blocks in flight) per CTA

__device__ __forceinline__ void dmma_884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ double neg(double x) {
  return __hiloint2double(__double2hiint(x) ^ 0x80000000, __double2loint(x));
}

__device__ __forceinline__ double shfl(double v, int src) {
  return __shfl_sync(0xffffffffu, v, src);
}

// Closed-form Matern at distance d (kind is warp-uniform and hoisted by the
// caller's specialisation); u = d / beta as in vg/kernels.py:67.
template <int KIND>
__device__ __forceinline__ double cov_closed(double d, double s2, double inv_beta) {
  // u = d * (1/beta): within 1 ulp of the reference's d / beta
  double u = d * inv_beta;
  double e = exp(-u);
  if (KIND == kMatern05) return s2 * e;
  if (KIND == kMatern15) return s2 * (1.0 + u) * e;
  return s2 * (1.0 + u + u * u * (1.0 / 3.0)) * e;
}

constexpr int tidx(int I, int J) { return I * (I + 1) / 2 + J; }

template <int NT, int KIND>
__global__ void __launch_bounds__(kWarps * 32)
loglik_dmma_kernel(const double4* __restrict__ pts, const int32_t* __restrict__ nbr, int m,
                   int64_t e_lo, int64_t e_hi, int64_t rest_lo, double s2, double inv_beta,
                   double* __restrict__ rest, double* __restrict__ mu_out,
                   double* __restrict__ sig_out, unsigned long long* __restrict__ fail) {
  constexpr int P = 8 * NT;
  constexpr int NTILE = NT * (NT + 1) / 2;
  __shared__ double s_x[kWarps][P];
  __shared__ double s_y[kWarps][P];
  __shared__ double s_o[kWarps][P];
  __shared__ double s_out[kWarps][2];

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int r = lane >> 2;  // fragment row
  const int q = lane & 3;   // fragment column pair
  double* X = s_x[warp];
  double* Y = s_y[warp];
  double* O = s_o[warp];

  const int64_t stride = (int64_t)gridDim.x * kWarps;
  for (int64_t e = e_lo + (int64_t)blockIdx.x * kWarps + warp; e < e_hi; e += stride) {
    // ---------------- gather (index m = target) ----------------
    const int32_t* J = nbr + (e - 1 - rest_lo) * (int64_t)m;
    for (int a = lane; a < P; a += 32) {
      double4 p = make_double4(0.0, 0.0, 0.0, 0.0);
      if (a < m) p = pts[J[a]];
      else if (a == m) p = pts[m + e - 1];
      X[a] = p.x;
      Y[a] = p.y;
      O[a] = p.z;
    }
    __syncwarp();

    // ---------------- generate the augmented lower triangle ----------------
    double t[NTILE][2];
#pragma unroll
    for (int I = 0; I < NT; ++I) {
      const int a = 8 * I + r;
      const double xa = X[a], ya = Y[a];
#pragma unroll
      for (int Jt = 0; Jt <= I; ++Jt) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int b = 8 * Jt + 2 * q + h;
          double val = 0.0;
          if (a <= m && b < a) {
            val = cov_closed<KIND>(dist_euclid(xa, ya, X[b], Y[b]), s2, inv_beta);
          } else if (a == b && a <= m) {
            val = s2;  // C(0) = sigma^2 (vg/kernels.py:77-78 continuous limit)
          } else if (a == m + 1 && b < m) {
            val = O[b];  // yJ row
          }
          t[tidx(I, Jt)][h] = val;
        }
      }
    }

    // ---------------- blocked right-looking Cholesky ----------------
    int failed = -1;
#pragma unroll
    for (int c = 0; c < NT; ++c) {
      const int jmax = m - 8 * c;  // pivots in this tile column (<= 0: none)
      if (jmax > 0 && failed < 0) {
        // panel: diagonal tile (c, c) and tiles (I, c), I > c, column by column
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          if (j < jmax && failed < 0) {
            const int src_piv = 4 * j + (j >> 1);
            const double piv = shfl(t[tidx(c, c)][j & 1], src_piv);
            if (!(piv > 0.0)) {
              failed = 8 * c + j;
            } else {
              const double inv = rsqrt(piv);
              const double ljj = piv * inv;
              // L[col][j] of the diagonal tile for this lane's two columns
              // (read before this step's scaling: scale here instead)
              const double lc0 = shfl(t[tidx(c, c)][j & 1], 4 * (2 * q) + (j >> 1)) * inv;
              const double lc1 = shfl(t[tidx(c, c)][j & 1], 4 * (2 * q + 1) + (j >> 1)) * inv;
#pragma unroll
              for (int I = c; I < NT; ++I) {
                double& v0 = t[tidx(I, c)][0];
                double& v1 = t[tidx(I, c)][1];
                // L[r][j] of tile (I, c) from the quad lane owning column j
                const double raw = shfl(t[tidx(I, c)][j & 1], (lane & ~3) | (j >> 1));
                const double lrj = raw * inv;
                // write back column j (diagonal entry of the diagonal tile = sqrt(piv))
                if (q == (j >> 1)) {
                  const double nv = (I == c && r == j) ? ljj : ((I == c && r < j) ? 0.0 : lrj);
                  if (j & 1) v1 = nv; else v0 = nv;
                }
                // rank-1 update of the columns right of j (rows below j on the diagonal tile)
                const int c0 = 2 * q, c1 = 2 * q + 1;
                if (c0 > j && (I > c || r >= c0)) v0 = fma(neg(lrj), lc0, v0);
                if (c1 > j && (I > c || r >= c1)) v1 = fma(neg(lrj), lc1, v1);
              }
            }
          }
        }
        if (failed < 0) {
          // A-fragments of the panel: frag_k(T) = T[r][k0 + q] for k0 = 0, 4
          double fa[NT][2];
#pragma unroll
          for (int I = c + 1; I < NT; ++I) {
#pragma unroll
            for (int kk = 0; kk < 2; ++kk) {
              const int src = (lane & ~3) | (2 * kk + (q >> 1));
              const double w0 = shfl(t[tidx(I, c)][0], src);
              const double w1 = shfl(t[tidx(I, c)][1], src);
              fa[I][kk] = (q & 1) ? w1 : w0;
            }
          }
          // trailing update A_IJ -= L_Ic L_Jc^T, c < J <= I
#pragma unroll
          for (int I = c + 1; I < NT; ++I) {
#pragma unroll
            for (int Jt = c + 1; Jt <= I; ++Jt) {
#pragma unroll
              for (int kk = 0; kk < 2; ++kk)
                dmma_884(t[tidx(I, Jt)][0], t[tidx(I, Jt)][1], neg(fa[I][kk]), fa[Jt][kk]);
            }
          }
        }
      }
    }

    // ---------------- per-block log-density ----------------
    const int64_t k = e - 1 - rest_lo;
    if (failed >= 0) {
      if (lane == 0) atomicMin(&fail[0], npd_key(e, failed, m));
    } else {
      // sigma_new = A[m][m], -mu = A[m+1][m]: fetch via shared memory
      const int im = m >> 3, rm = m & 7;
      const int im1 = (m + 1) >> 3, rm1 = (m + 1) & 7;
#pragma unroll
      for (int I = 0; I < NT; ++I) {
        if (I == im && q == (rm >> 1) && r == rm)
          s_out[warp][0] = (rm & 1) ? t[tidx(I, I)][1] : t[tidx(I, I)][0];
#pragma unroll
        for (int Jt = 0; Jt <= I; ++Jt) {
          if (I == im1 && Jt == im && q == (rm >> 1) && r == rm1)
            s_out[warp][1] = (rm & 1) ? t[tidx(I, Jt)][1] : t[tidx(I, Jt)][0];
        }
      }
      __syncwarp();
      if (lane == 0) {
        const double sg = s_out[warp][0];
        const double mu = -s_out[warp][1];
        mu_out[k] = mu;
        sig_out[k] = sg;
        if (!(sg > 0.0)) {
          atomicMin(&fail[1], (unsigned long long)e);
          rest[k] = 0.0;
        } else {
          const double resid = O[m] - mu;
          rest[k] = -0.5 * (resid * resid / sg + kLog2Pi + log(sg));
        }
      }
    }
    __syncwarp();
  }
}

template <int NT, int KIND>
cudaError_t launch_nt(const Plan& p, const CovParams& cp, int64_t e_lo, int64_t e_hi,
                      cudaStream_t stream) {
  int64_t count = e_hi - e_lo;
  int64_t want = (count + kWarps - 1) / kWarps;
  int64_t cap = (int64_t)p.num_sms * 16;
  int grid = (int)(want < cap ? want : cap);
  loglik_dmma_kernel<NT, KIND><<<grid, kWarps * 32, 0, stream>>>(
      p.d_pts, p.d_nbr, p.m, e_lo, e_hi, p.rest_lo, cp.s2, cp.inv_beta, p.d_rest, p.d_mu, p.d_sig,
      p.d_fail);
  return cudaGetLastError();
}

template <int KIND>
cudaError_t launch_kind(const Plan& p, const CovParams& cp, int64_t e_lo, int64_t e_hi,
                        cudaStream_t stream) {
  switch ((p.m + 2 + 7) / 8) {
    case 1: return launch_nt<1, KIND>(p, cp, e_lo, e_hi, stream);
    case 2: return launch_nt<2, KIND>(p, cp, e_lo, e_hi, stream);
    case 3: return launch_nt<3, KIND>(p, cp, e_lo, e_hi, stream);
    case 4: return launch_nt<4, KIND>(p, cp, e_lo, e_hi, stream);
    case 5: return launch_nt<5, KIND>(p, cp, e_lo, e_hi, stream);
    case 6: return launch_nt<6, KIND>(p, cp, e_lo, e_hi, stream);
    case 7: return launch_nt<7, KIND>(p, cp, e_lo, e_hi, stream);
    case 8: return launch_nt<8, KIND>(p, cp, e_lo, e_hi, stream);
    default: return cudaErrorNotSupported;
  }
}

}  // namespace

bool dmma_supported(int m, int kind) {
  return m >= 1 && m + 2 <= 64 && (kind == kMatern05 || kind == kMatern15 || kind == kMatern25);
}

cudaError_t launch_loglik_dmma(const Plan& p, const CovParams& cp, int64_t e_lo, int64_t e_hi,
                               cudaStream_t stream) {
  if (!dmma_supported(p.m, cp.kind)) return cudaErrorNotSupported;
  if (e_hi <= e_lo) return cudaSuccess;
  switch (cp.kind) {
    case kMatern05: return launch_kind<kMatern05>(p, cp, e_lo, e_hi, stream);
    case kMatern15: return launch_kind<kMatern15>(p, cp, e_lo, e_hi, stream);
    default: return launch_kind<kMatern25>(p, cp, e_lo, e_hi, stream);
  }
}

}  // namespace vgp
