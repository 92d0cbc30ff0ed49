// Warp-per-block FP64 tensor-core (DMMA) Vecchia kernel, m + 2 <= 64.
//
// One warp owns one conditioning block e >= 1 end to end; only the block's
// log-density, mu and sigma (24 bytes) leave the SM:
//
//   gather    J = NBR[e-1] (int32) and (x, y, obs) of the m neighbours and the
//             target into per-warp shared memory (vg/vecchia.py:154-162);
//   generate  the strictly lower part of the augmented covariance
//               rows 0..m-1 Sigma_e (C(||s_Ja - s_Jb||)), row m v_e (C(||s_t - s_Ja||))
//             spread evenly over the 32 lanes (m(m+1)/2 entries, no padding
//             work), with the lean FP64 sqrt / table exp of vgp_fastmath.cuh,
//             into a per-warp shared tile store; the diagonal (sigma^2) and
//             the yJ row (obs) are plain stores;
//   load      every 8x8 tile (I, J), I >= J, of the (8 NT)^2 augmented matrix
//             into registers as an m8n8 DMMA accumulator fragment: lane
//             (r, q) = (lane/4, lane%4) holds (r, 2q), (r, 2q+1);
//   factor    right-looking blocked Cholesky over 8-wide tile columns:
//               panel  : column by column over the diagonal tile and the tiles
//                        below it, quad shuffles; pivot test !(piv > 0) ->
//                        NPD at that column (vg/batchla.py:146-151);
//               update : A_IJ -= L_Ic L_Jc^T for c < J <= I with two
//                        mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4) per tile;
//             rows m (v) and m+1 (yJ) ride along, so the same sweep performs
//             both triangular solves (v' = L^-1 v, y' = L^-1 yJ, batch_trsv)
//             and the Schur complements leave sigma_new = A[m][m] and
//             -mu = A[m+1][m] (vg/vecchia.py:186-189, :206);
//   reduce    l_e = -1/2 ((y_t - mu)^2 / sigma_new + log 2pi + log sigma_new)
//             (vg/vecchia.py:211-212).
//
// sm_100a has no FP64 tcgen05 kind (ptxas rejects .kind::f64), so DMMA is
// the FP64 tensor path on B200: measured 37.0 TFLOP/s, the same as DFMA
// (profiles/r01_fp64_peak.jsonl), but one instruction issues 256 FMAs.
#pragma once

#include "vgp_fastmath.cuh"
#include "vgp_math.cuh"

namespace vgp {
namespace dmma {

constexpr int kWarps = 4;  // warps (= blocks in flight) per CTA

__device__ __forceinline__ void mma884(double& d0, double& d1, double a, double b) {
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

constexpr int tidx(int I, int J) { return I * (I + 1) / 2 + J; }

// shared-memory tile store address of entry (i, k), i >= k: tile-packed,
// row-major inside a tile, so a lane's fragment pair is one 16-byte word.
__device__ __forceinline__ int tile_addr(int i, int k) {
  const int I = i >> 3, J = k >> 3;
  return (I * (I + 1) / 2 + J) * 64 + (i & 7) * 8 + (k & 7);
}

// Matern closed forms (vg/kernels.py:69-74) on top of tab = sigma^2 * 2^(j/256).
template <int KIND>
__device__ __forceinline__ double cov_fast(double d, double inv_beta,
                                           const double* __restrict__ tab) {
  const double u = d * inv_beta;  // within 1 ulp of the reference's d / beta
  const double e = exp_neg_tab(u, tab);
  if (KIND == kMatern05) return e;
  if (KIND == kMatern15) return (1.0 + u) * e;
  return fma(u, fma(u, 1.0 / 3.0, 1.0), 1.0) * e;
}

template <int NT>
struct Smem {
  static constexpr int kP = 8 * NT;
  static constexpr int kTiles = NT * (NT + 1) / 2;
  static constexpr int kPanelLd = 10;  // panel row stride (doubles): conflict-free LDS.128 rows
  // per warp: tile store (reused as the panel), (x, y) pairs, obs, 2 outputs
  static constexpr int kWarpDoubles = kTiles * 64 + 2 * kP + kP + 2;
  static constexpr int kMaxEntries = (kP - 2) * (kP - 1) / 2;  // m (m+1) / 2 with m <= P - 2
  // [256 exp table][entry table (u32, padded to doubles)][warps]
  static constexpr size_t entry_doubles() { return ((kMaxEntries + 3) / 4) * 2; }  // 16 B aligned
  static constexpr size_t bytes() {
    return sizeof(double) * (256 + entry_doubles() + (size_t)kWarps * kWarpDoubles);
  }
};

template <int NT, int KIND>
__global__ void __launch_bounds__(kWarps * 32)
loglik_kernel(const double4* __restrict__ pts, const int32_t* __restrict__ nbr, int m,
              int64_t e_lo, int64_t e_hi, int64_t rest_lo, double s2, double inv_beta,
              double* __restrict__ rest, double* __restrict__ mu_out,
              double* __restrict__ sig_out, unsigned long long* __restrict__ fail) {
  using S = Smem<NT>;
  constexpr int P = S::kP;
  constexpr int NTILE = S::kTiles;
  constexpr int LD = S::kPanelLd;
  extern __shared__ __align__(16) double smem[];
  double* tab = smem;  // 256: sigma^2 * 2^(j/256)
  uint32_t* ent = reinterpret_cast<uint32_t*>(smem + 256);  // packed (i, k, tile address)
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int r = lane >> 2;  // fragment row
  const int q = lane & 3;   // fragment column pair
  double* tiles = smem + 256 + S::entry_doubles() + (size_t)warp * S::kWarpDoubles;
  double2* XY = reinterpret_cast<double2*>(tiles + NTILE * 64);
  double* O = tiles + NTILE * 64 + 2 * P;
  double* out2 = O + P;

  // per-CTA tables: exp table scaled by sigma^2 and the strictly-lower entry
  // list of rows 1..m (row m = the target's cross-covariances v)
  const int nent = m * (m + 1) / 2;
  for (int i = threadIdx.x; i < 256; i += blockDim.x) tab[i] = s2 * kExp2Table[i];
  for (int idx = threadIdx.x; idx < nent; idx += blockDim.x) {
    int i = (int)((1.0f + sqrtf(1.0f + 8.0f * (float)idx)) * 0.5f);
    while (i * (i - 1) / 2 > idx) --i;
    while ((i + 1) * i / 2 <= idx) ++i;
    const int k = idx - i * (i - 1) / 2;
    ent[idx] = (uint32_t)i | ((uint32_t)k << 8) | ((uint32_t)tile_addr(i, k) << 16);
  }
  __syncthreads();

  const int64_t stride = (int64_t)gridDim.x * kWarps;
  for (int64_t e = e_lo + (int64_t)blockIdx.x * kWarps + warp; e < e_hi; e += stride) {
    // ---------------- gather (index m = target) + zero the tile store ----------------
    const int32_t* J = nbr + (e - 1 - rest_lo) * (int64_t)m;
    for (int a = lane; a < P; a += 32) {
      double4 p = make_double4(0.0, 0.0, 0.0, 0.0);
      if (a < m) p = pts[J[a]];
      else if (a == m) p = pts[m + e - 1];
      XY[a] = make_double2(p.x, p.y);
      O[a] = p.z;
    }
#pragma unroll
    for (int T = 0; T < NTILE; ++T)
      reinterpret_cast<double2*>(tiles + T * 64)[lane] = make_double2(0.0, 0.0);
    __syncwarp();

    // ---------------- generate (entries spread evenly over lanes) ----------------
#pragma unroll 2
    for (int idx = lane; idx < nent; idx += 32) {
      const uint32_t w = ent[idx];
      const double2 a = XY[w & 0xff];
      const double2 b = XY[(w >> 8) & 0xff];
      const double dx = a.x - b.x;
      const double dy = a.y - b.y;
      const double d = sqrt_pos(fma(dx, dx, dy * dy));
      tiles[w >> 16] = cov_fast<KIND>(d, inv_beta, tab);
    }
    for (int a = lane; a <= m; a += 32) tiles[tile_addr(a, a)] = s2;          // C(0) = sigma^2
    for (int b = lane; b < m; b += 32) tiles[tile_addr(m + 1, b)] = O[b];     // yJ row
    __syncwarp();

    // ---------------- load the accumulator fragments ----------------
    double t[NTILE][2];
#pragma unroll
    for (int T = 0; T < NTILE; ++T) {
      const double2 v = reinterpret_cast<const double2*>(tiles + T * 64 + 8 * r)[q];
      t[T][0] = v.x;
      t[T][1] = v.y;
    }
    __syncwarp();
    double* pan = tiles;  // tile store is free now: reuse as the panel buffer

    // ---------------- blocked right-looking Cholesky ----------------
    int failed = -1;
#pragma unroll
    for (int c = 0; c < NT; ++c) {
      const int jmax = min(8, m - 8 * c);  // pivots in this tile column
      if (jmax > 0 && failed < 0) {
        constexpr int kMaxRows = 2;
        const int R0 = 8 * c;       // first panel row
        const int NR = P - R0;      // panel rows
        const int ROWS = (NR + 31) / 32;
        // registers -> row-major panel
#pragma unroll
        for (int I = c; I < NT; ++I)
          *reinterpret_cast<double2*>(pan + (8 * (I - c) + r) * LD + 2 * q) =
              make_double2(t[tidx(I, c)][0], t[tidx(I, c)][1]);
        __syncwarp();
        double a[kMaxRows][8];
#pragma unroll
        for (int rr = 0; rr < kMaxRows; ++rr) {
          if (rr < ROWS) {
            const int row = lane + 32 * rr;
#pragma unroll
            for (int x = 0; x < 4; ++x) {
              double2 v = make_double2(0.0, 0.0);
              if (row < NR) v = *reinterpret_cast<const double2*>(pan + row * LD + 2 * x);
              a[rr][2 * x] = v.x;
              a[rr][2 * x + 1] = v.y;
            }
          }
        }
        // column-by-column factorization of the panel; lane l owns panel rows l, l + 32
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          if (j < jmax && failed < 0) {
            const double piv = shfl(a[0][j], j);
            if (!(piv > 0.0)) {
              failed = R0 + j;
            } else {
              const double inv = rsqrt_pos(piv);
              const double ljj = piv * inv;
#pragma unroll
              for (int rr = 0; rr < kMaxRows; ++rr)
                if (rr < ROWS) a[rr][j] = (rr == 0 && lane == j) ? ljj : a[rr][j] * inv;
#pragma unroll
              for (int jp = j + 1; jp < 8; ++jp) {
                const double lc = shfl(a[0][j], jp);  // L[R0 + jp][j]
#pragma unroll
                for (int rr = 0; rr < kMaxRows; ++rr)
                  if (rr < ROWS) a[rr][jp] = fma(-a[rr][j], lc, a[rr][jp]);
              }
            }
          }
        }
        if (failed < 0) {
          // sigma_new / -mu sit in this panel when m is not a multiple of 8
          if (jmax < 8 || (m & 7) != 0) {
            const int cs = m - R0;  // panel column of index m (only meaningful if < 8)
            if (cs < 8) {
#pragma unroll
              for (int rr = 0; rr < kMaxRows; ++rr) {
                if (rr < ROWS) {
                  const int row = lane + 32 * rr;
#pragma unroll
                  for (int x = 0; x < 8; ++x) {
                    if (x == cs && row == m - R0) out2[0] = a[rr][x];
                    if (x == cs && row == m + 1 - R0) out2[1] = a[rr][x];
                  }
                }
              }
            }
          }
          // panel -> shared memory, then A-fragments frag_kk(T) = L[8I + r][4 kk + q]
          __syncwarp();
#pragma unroll
          for (int rr = 0; rr < kMaxRows; ++rr) {
            if (rr < ROWS) {
              const int row = lane + 32 * rr;
              if (row < NR) {
#pragma unroll
                for (int x = 0; x < 4; ++x)
                  *reinterpret_cast<double2*>(pan + row * LD + 2 * x) =
                      make_double2(a[rr][2 * x], a[rr][2 * x + 1]);
              }
            }
          }
          __syncwarp();
          double fa[NT][2];
#pragma unroll
          for (int I = c + 1; I < NT; ++I) {
#pragma unroll
            for (int kk = 0; kk < 2; ++kk) fa[I][kk] = pan[(8 * (I - c) + r) * LD + 4 * kk + q];
          }
          __syncwarp();
          // trailing update A_IJ -= L_Ic L_Jc^T, c < J <= I
#pragma unroll
          for (int I = c + 1; I < NT; ++I) {
            const double n0 = neg(fa[I][0]);
            const double n1 = neg(fa[I][1]);
#pragma unroll
            for (int Jt = c + 1; Jt <= I; ++Jt) {
              mma884(t[tidx(I, Jt)][0], t[tidx(I, Jt)][1], n0, fa[Jt][0]);
              mma884(t[tidx(I, Jt)][0], t[tidx(I, Jt)][1], n1, fa[Jt][1]);
            }
          }
        }
      }
    }

    // ---------------- per-block log-density ----------------
    const int64_t kk = e - 1 - rest_lo;
    if (failed >= 0) {
      if (lane == 0) atomicMin(&fail[0], npd_key(e, failed, m));
    } else {
      if ((m & 7) == 0) {
        // m = 8 (NT - 1): sigma_new = tile (NT-1, NT-1)[0][0], -mu = [1][0]
        if (lane == 0) out2[0] = t[tidx(NT - 1, NT - 1)][0];
        if (lane == 4) out2[1] = t[tidx(NT - 1, NT - 1)][0];
      }
      __syncwarp();
      if (lane == 0) {
        const double sg = out2[0];
        const double mu = -out2[1];
        mu_out[kk] = mu;
        sig_out[kk] = sg;
        if (!(sg > 0.0)) {
          atomicMin(&fail[1], (unsigned long long)e);
          rest[kk] = 0.0;
        } else {
          const double resid = O[m] - mu;
          rest[kk] = -0.5 * (resid * resid / sg + kLog2Pi + log(sg));
        }
      }
    }
    __syncwarp();
  }
}

template <int NT, int KIND>
cudaError_t launch(const Plan& p, const CovParams& cp, int64_t e_lo, int64_t e_hi,
                   cudaStream_t stream) {
  const size_t sm = Smem<NT>::bytes();
  static bool configured[64] = {};  // per device ordinal
  const int dev = p.device & 63;
  if (!configured[dev]) {
    cudaError_t err = cudaFuncSetAttribute(loglik_kernel<NT, KIND>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (err != cudaSuccess) return err;
    configured[dev] = true;
  }
  const int64_t count = e_hi - e_lo;
  const int64_t want = (count + kWarps - 1) / kWarps;
  const int64_t cap = (int64_t)p.num_sms * 16;
  const int grid = (int)(want < cap ? want : cap);
  loglik_kernel<NT, KIND><<<grid, kWarps * 32, sm, stream>>>(
      p.d_pts, p.d_nbr, p.m, e_lo, e_hi, p.rest_lo, cp.s2, cp.inv_beta, p.d_rest, p.d_mu,
      p.d_sig, p.d_fail);
  return cudaGetLastError();
}

template <int KIND>
cudaError_t launch_kind(const Plan& p, const CovParams& cp, int64_t e_lo, int64_t e_hi,
                        cudaStream_t stream) {
  switch ((p.m + 2 + 7) / 8) {
    case 1: return launch<1, KIND>(p, cp, e_lo, e_hi, stream);
    case 2: return launch<2, KIND>(p, cp, e_lo, e_hi, stream);
    case 3: return launch<3, KIND>(p, cp, e_lo, e_hi, stream);
    case 4: return launch<4, KIND>(p, cp, e_lo, e_hi, stream);
    case 5: return launch<5, KIND>(p, cp, e_lo, e_hi, stream);
    case 6: return launch<6, KIND>(p, cp, e_lo, e_hi, stream);
    case 7: return launch<7, KIND>(p, cp, e_lo, e_hi, stream);
    case 8: return launch<8, KIND>(p, cp, e_lo, e_hi, stream);
    default: return cudaErrorNotSupported;
  }
}

}  // namespace dmma
}  // namespace vgp
