// Register-light warp-per-block FP64 tensor-core (DMMA) Vecchia kernel,
// m + 2 <= 64 ("grouped" kernel, the default fast path).
//
// One warp owns one conditioning block e >= 1 end to end (vg/vecchia.py:
// 154-162 assemble, :180-190 _numeric_stage, :193-214 _reduction_stage); only
// the block's log-density, mu and sigma leave the SM.  The augmented
// (8 NT)^2 matrix (rows 0..m-1 Sigma_e, row m v_e, row m+1 yJ, zero padding)
// is factored by a blocked Cholesky over 8-wide tile columns, processed in
// groups of GW tile columns:
//
//   across groups  left-looking: a group's tiles are generated, then updated
//                  with every earlier tile column's L (DMMA operands read
//                  from shared memory);
//   inside a group right-looking: panel (row-owner layout, one pivot chain)
//                  then the group's remaining tile columns are updated from
//                  the fresh L (mma.sync.m8n8k4.f64 -> SASS DMMA.8x8x4).
//
// Only one group's tiles (at most 15 for GW = 2) live in registers, against
// 36 for a fully right-looking sweep, so 12 warps fit per SM instead of 8:
// the pivot chains of 3 warps per scheduler overlap each other's DMMA and
// covariance work.  L is written back into the same per-warp shared buffer
// the distances arrive in:
//
//   buf   rows 0..m of the augmented matrix, compact lower triangle with the
//         diagonal, each row padded to an even length (row i starts at
//         rowoff(i)), so every lane's (2q, 2q+1) fragment pair and every
//         8-column panel row is a 16-byte LDS/STS;
//   O     row m+1 (yJ, then L of that row);
//   Z     a zero row shared by the CTA (padding rows read it);
//   S     staging of the last group's panels (buf is then already being
//         refilled with the next block's distances by a TMA bulk copy).
//
// L is stored with each 8-column group permuted (positions 2q, 2q+1 hold
// columns q, q+4), so the two k=4 slices of a DMMA operand are one LDS.128.
//
// Distances: with the plan-time distance cache (vgp_dcache.cu, same layout as
// buf, theta-independent) each warp streams its next block's distances into
// buf with one cp.async.bulk (SASS UBLKCP) + mbarrier; otherwise they are
// computed from the gathered coordinates with the same formula, so cached
// and uncached evaluations agree bit for bit.
#pragma once

#include "vgp_dmma_kernel.cuh"

namespace vgp {
namespace ll {

using dmma::bulk_load;
using dmma::cov_fast;
using dmma::mbar_init;
using dmma::mbar_wait;
using dmma::neg;
using dmma::shfl;

constexpr int kWarps = 4;  // warps (= blocks in flight) per CTA
constexpr int kSLd = 10;   // last-group staging row stride (conflict-free LDS.128 rows)
constexpr int kHead = 256 + 64;  // exp table + zero row

// start of row i in the padded compact layout (row i holds columns 0..i,
// padded to an even length): 2t(t+1) for i = 2t, 2(t+1)^2 for i = 2t+1.
__host__ __device__ constexpr int rowoff(int i) {
  return (i & 1) ? 2 * ((i >> 1) + 1) * ((i >> 1) + 1) : 2 * (i >> 1) * ((i >> 1) + 1);
}

__device__ __forceinline__ double2 ld2(const double* p) {
  return *reinterpret_cast<const double2*>(p);
}
__device__ __forceinline__ void st2(double* p, double a, double b) {
  *reinterpret_cast<double2*>(p) = make_double2(a, b);
}

// Matern closed forms (vg/kernels.py:69-74) on tab = sigma^2 2^(j/256):
// exp(-u) = 2^(k/256) e^r with one-step reduction r = -u - k ln2/256 (the
// rounding of ln2/256 costs u 2^-53 relative, i.e. < 0.4 ulp of sigma^2 in
// absolute terms since u e^-u <= 1/e), degree-4 polynomial; 10 FP64 ops for
// nu = 1.5 including u = d / beta (as d * (1/beta), within 1 ulp).
template <int KIND>
__device__ __forceinline__ double cov_lean(double d, double inv_beta, const double* __restrict__ tab) {
  const double u = d * inv_beta;
  const double shift = 0x1.8p52;
  const double t = fma(-u, k256OverLn2, shift);
  const double kf = t - shift;
  const int ki = __double2loint(t);
  const double r = fma(-kf, kLn2Over256, -u);
  double p = fma(r, 1.0 / 24.0, 1.0 / 6.0);
  p = fma(p, r, 0.5);
  p = fma(p, r, 1.0);
  p = fma(p, r, 1.0);
  double v = tab[ki & 255] * p;
  const int ex = max(ki >> 8, -1000);
  v = __hiloint2double(__double2hiint(v) + ex * 0x100000, __double2loint(v));
  if (KIND == kMatern05) return v;
  if (KIND == kMatern15) return fma(u, v, v);
  return fma(u, fma(u, 1.0 / 3.0, 1.0), 1.0) * v;
}

// 1/sqrt(x) with one third-order step, arranged for a 4-deep FP64 chain
// (it sits on the pivot-to-pivot critical path): y = y0 + (y0 e)(1/2 + 3e/8).
__device__ __forceinline__ double rsqrt_chain(double x) {
  const double y0 = rsqrt_seed(x);
  const double e = fma(-(x * y0), y0, 1.0);
  const double t = y0 * e;
  const double p = fma(e, 0.375, 0.5);
  return fma(t, p, y0);
}

// D = A B + D on an 8x8 tile (SASS DMMA.8x8x4); not volatile, so the
// scheduler may interleave independent tile updates
__device__ __forceinline__ void mma(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}

// first tile column of the last group / rows of its staging area
__host__ __device__ constexpr int last_c0(int nc, int gw) { return gw * ((nc - 1) / gw); }

struct WarpLayout {
  int buf_n;   // doubles of buf (= cache stride)
  int s_rows;  // staging rows
  int stride;  // doubles per warp
  static __host__ __device__ WarpLayout make(int m, int nt, int gw) {
    WarpLayout w{};
    const int p = 8 * nt;
    const int nc = (m + 8) >> 3;
    w.buf_n = rowoff(m + 1);
    w.s_rows = p - 8 * last_c0(nc, gw);
    int s = w.s_rows * kSLd;
    if (s < 2 * p) s = 2 * p;  // S doubles as the coordinate stage (uncached variant)
    w.stride = (w.buf_n + p + s + 4 + 1) & ~1;
    return w;
  }
};

template <int NT, int KIND, int MC, int GW, bool CACHE, int MINB>
__global__ void __launch_bounds__(kWarps * 32, MINB)
loglik_ll_kernel(const double4* __restrict__ pts, const int32_t* __restrict__ nbr, int m_rt,
                 int64_t e_lo, int64_t e_hi, int64_t rest_lo, double s2, double inv_beta,
                 double* __restrict__ rest, double* __restrict__ mu_out,
                 double* __restrict__ sig_out, unsigned long long* __restrict__ fail,
                 const double* __restrict__ dcache, int64_t cstride) {
  constexpr int P = 8 * NT;
  constexpr int NG = (NT + GW - 1) / GW;
  const int m = MC > 0 ? MC : m_rt;
  const int NC = (m + 8) >> 3;  // tile columns holding pivots or the Schur column
  const int G = (NC + GW - 1) / GW;
  const int C0L = last_c0(NC, GW);
  const WarpLayout wl = WarpLayout::make(m, NT, GW);
  extern __shared__ __align__(16) double smem[];
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int r = lane >> 2;  // fragment row
  const int q = lane & 3;   // fragment column pair
  // offsets (in doubles) into smem
  constexpr int kZ = 256;
  const int kB = kHead + warp * wl.stride;  // buf
  const int kO = kB + wl.buf_n;             // row m+1
  const int kS = kO + P;                    // staging / coordinates
  const int kMisc = kS + ((wl.s_rows * kSLd < 2 * P) ? 2 * P : wl.s_rows * kSLd);
  double* out2 = smem + kMisc;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + kMisc + 2);
  double2* XY = reinterpret_cast<double2*>(smem + kS);

  for (int i = threadIdx.x; i < 256; i += blockDim.x) smem[i] = s2 * kExp2Table[i];
  for (int i = threadIdx.x; i < 64; i += blockDim.x) smem[kZ + i] = 0.0;
  if (CACHE && lane == 0) mbar_init(bar);
  __syncthreads();
  const double* tab = smem;
  const uint32_t cbytes = (uint32_t)(cstride * sizeof(double));
  uint32_t cphase = 0;

  // smem offset of row i of the augmented matrix
  auto rowo = [&](int i) -> int { return i <= m ? kB + rowoff(i) : (i == m + 1 ? kO : kZ); };

  const int64_t stride = (int64_t)gridDim.x * kWarps;
  // Software-pipelined gather: next block's neighbour indices early, its
  // points late; lane owns slots lane and lane + 32 (slot m = target).
  auto slot_index = [&](int64_t eb, int a) -> int {
    if (a < m) return nbr[(eb - 1 - rest_lo) * (int64_t)m + a];
    return a == m ? (int)(m + eb - 1) : -1;
  };
  auto slot_point = [&](int idx) -> double4 {
    return idx >= 0 ? pts[idx] : make_double4(0.0, 0.0, 0.0, 0.0);
  };
  int64_t e = e_lo + (int64_t)blockIdx.x * kWarps + warp;
  int ni0 = -1, ni1 = -1;
  double4 pf0 = make_double4(0.0, 0.0, 0.0, 0.0), pf1 = pf0;
  if (e < e_hi) {
    if (CACHE && lane == 0) bulk_load(smem + kB, dcache + (e - 1 - rest_lo) * cstride, cbytes, bar);
    pf0 = slot_point(slot_index(e, lane));
    if (P > 32) pf1 = slot_point(slot_index(e, lane + 32));
  }
  for (; e < e_hi; e += stride) {
    const int64_t en = e + stride;
    // ---------------- stage the block's yJ row (and coordinates) ----------------
    double yt = 0.0;  // target observation (lane m % 32 holds it)
    {
      if (lane < P) smem[kO + lane] = lane < m ? pf0.z : 0.0;
      if (P > 32 && lane + 32 < P) smem[kO + lane + 32] = lane + 32 < m ? pf1.z : 0.0;
      if (!CACHE) {
        if (lane < P) XY[lane] = make_double2(pf0.x, pf0.y);
        if (P > 32 && lane + 32 < P) XY[lane + 32] = make_double2(pf1.x, pf1.y);
      }
      yt = (m < 32) ? pf0.z : pf1.z;
      yt = shfl(yt, m & 31);
    }
    if (en < e_hi) {
      ni0 = slot_index(en, lane);
      if (P > 32) ni1 = slot_index(en, lane + 32);
      if (CACHE) {  // only the observations are needed: load them a whole block ahead
        pf0.z = ni0 >= 0 ? pts[ni0].z : 0.0;
        if (P > 32) pf1.z = ni1 >= 0 ? pts[ni1].z : 0.0;
      }
    }
    if (CACHE) {
      mbar_wait(bar, cphase);
      cphase ^= 1;
    }
    __syncwarp();

    // covariance entries (8I + r, 8J + 2q + h) of tile (I, J) (vg/vecchia.py:154-162)
    auto gen_tile = [&](const int I, const int J, double& v0, double& v1) {
      const int i = 8 * I + r;
      if (CACHE) {
        const double2 dv = ld2(smem + rowo(i) + 8 * J + 2 * q);
        v0 = cov_lean<KIND>(dv.x, inv_beta, tab);
        v1 = cov_lean<KIND>(dv.y, inv_beta, tab);
        if (I == NT - 1 && i > m) {  // row m+1: yJ values; padding: 0
          v0 = dv.x;
          v1 = dv.y;
        }
      } else {
        const double2 pa = XY[i];
        const double4 pb = *reinterpret_cast<const double4*>(XY + 8 * J + 2 * q);
        double dx = pa.x - pb.x, dy = pa.y - pb.y;
        v0 = cov_lean<KIND>(sqrt_pos_nz(fma(dx, dx, fma(dy, dy, 0x1p-1000))), inv_beta, tab);
        dx = pa.x - pb.z;
        dy = pa.y - pb.w;
        v1 = cov_lean<KIND>(sqrt_pos_nz(fma(dx, dx, fma(dy, dy, 0x1p-1000))), inv_beta, tab);
        if (I == NT - 1 && i > m) {
          const double2 ov = ld2(smem + rowo(i) + 8 * J + 2 * q);
          v0 = ov.x;
          v1 = ov.y;
        }
      }
    };
    double pre[GW][NT][2];  // next group's tiles, generated during this group's panels
    int fj = -1;            // first non-positive pivot column
#pragma unroll
    for (int g = 0; g < NG; ++g) {
      if (g < G) {
        const int c0 = g * GW;
        const bool last = (g == G - 1);
        // ---------------- the group's tiles (I, J), J in [c0, c0+GW) ----------------
        // group 0 is generated here; later groups were generated during the
        // previous group's pivot chains (below)
        double acc[GW][NT][2];
#pragma unroll
        for (int jj = 0; jj < GW; ++jj) {
          const int J = c0 + jj;
#pragma unroll
          for (int I = 0; I < NT; ++I) {
            if (J < NT && I >= J && J < NC) {
              if (g == 0) {
                gen_tile(I, J, acc[jj][I][0], acc[jj][I][1]);
              } else {
                acc[jj][I][0] = pre[jj][I][0];
                acc[jj][I][1] = pre[jj][I][1];
              }
            }
          }
        }
        // ---------------- left-looking update from earlier groups ----------------
#pragma unroll
        for (int k = 0; k < NT; ++k) {
          if (k < c0) {
            double2 f[NT];
#pragma unroll
            for (int I = 0; I < NT; ++I)
              if (I >= c0) f[I] = ld2(smem + rowo(8 * I + r) + 8 * k + 2 * q);
            // kk outer: consecutive DMMAs hit different accumulators
#pragma unroll
            for (int kk = 0; kk < 2; ++kk) {
#pragma unroll
              for (int jj = 0; jj < GW; ++jj) {
                const int J = c0 + jj;
#pragma unroll
                for (int I = 0; I < NT; ++I) {
                  if (J < NT && I >= J && J < NC)
                    mma(acc[jj][I][0], acc[jj][I][1], neg(kk ? f[I].y : f[I].x), kk ? f[J].y : f[J].x);
                }
              }
            }
          }
        }
        if (last) {
          // buf and the yJ row are no longer read: stream in the next block
          __syncwarp();
          if (CACHE && lane == 0 && en < e_hi)
            bulk_load(smem + kB, dcache + (en - 1 - rest_lo) * cstride, cbytes, bar);
        }
        // ---------------- the group's panels, right-looking inside ----------------
#pragma unroll
        for (int jj = 0; jj < GW; ++jj) {
          const int c = c0 + jj;
          if (c < NT && c < NC) {
            const int R0 = 8 * c;
            const int NR = P - R0;
            const int jmax = min(8, m - R0);  // pivots in this tile column
            if (!CACHE && last && (jj == GW - 1 || c + 1 >= NC) && en < e_hi) {
              pf0 = slot_point(ni0);
              if (P > 32) pf1 = slot_point(ni1);
            }
            // panel row base (column 8c + x of row i at base(i) + x)
            auto pbase = [&](int i) -> int {
              return last ? kS + (i - 8 * c0) * kSLd : rowo(i) + R0;
            };
            // stage tile column c into row layout
#pragma unroll
            for (int I = 0; I < NT; ++I) {
              if (I >= c) {
                const int i = 8 * I + r;
                if (last) {
                  st2(smem + pbase(i) + 2 * q, acc[jj][I][0], acc[jj][I][1]);
                } else if (I == c) {
                  const int k = R0 + 2 * q;
                  if (i <= m + 1) {
                    if (k <= i) smem[pbase(i) + 2 * q] = acc[jj][I][0];
                    if (k + 1 <= i) smem[pbase(i) + 2 * q + 1] = acc[jj][I][1];
                  }
                } else if (I < NT - 1 || i <= m + 1) {
                  st2(smem + pbase(i) + 2 * q, acc[jj][I][0], acc[jj][I][1]);
                }
              }
            }
            __syncwarp();
            constexpr int kMaxRows = 2;
            double a[kMaxRows][8];
#pragma unroll
            for (int rr = 0; rr < kMaxRows; ++rr) {
              const int row = R0 + lane + 32 * rr;
#pragma unroll
              for (int x = 0; x < 4; ++x) {
                double2 v = make_double2(0.0, 0.0);
                if (rr * 32 < NR && row < P) v = ld2(smem + pbase(row) + 2 * x);
                a[rr][2 * x] = v.x;
                a[rr][2 * x + 1] = v.y;
              }
            }
            // the next group's tile column c + GW: independent work that fills
            // the latency of this panel's pivot chain
            if (c + GW < NC) {
#pragma unroll
              for (int I = 0; I < NT; ++I)
                if (I >= c + GW) gen_tile(I, c + GW, pre[jj][I][0], pre[jj][I][1]);
            }
            if (jmax > 0) {
              double piv = shfl(a[0][0], 0);
#pragma unroll
              for (int j = 0; j < 8; ++j) {
                if (j < jmax) {
                  const double inv = rsqrt_chain(piv);
#pragma unroll
                  for (int rr = 0; rr < kMaxRows; ++rr)
                    if (rr * 32 < NR) a[rr][j] *= inv;
                  if (j + 1 < 8) {
                    const double nxt = fma(-a[0][j], a[0][j], a[0][j + 1]);
                    piv = shfl(nxt, j + 1);
                  }
#pragma unroll
                  for (int jp = j + 1; jp < 8; ++jp) {
                    const double lc = shfl(a[0][j], jp);  // L[R0 + jp][R0 + j]
#pragma unroll
                    for (int rr = 0; rr < kMaxRows; ++rr)
                      if (rr * 32 < NR) a[rr][jp] = fma(-a[rr][j], lc, a[rr][jp]);
                  }
                }
              }
            }
            // pivot test !(piv > 0) (vg/batchla.py:146-151): a non-positive or NaN
            // pivot makes L_jj = piv * rsqrt(piv) NaN (and every later pivot);
            // lane j holds L_jj, so one test per panel finds the first one
            if (jmax > 0) {
              double ljj = a[0][0];
#pragma unroll
              for (int x = 1; x < 8; ++x)
                if (lane == x) ljj = a[0][x];
              const unsigned bad = __ballot_sync(0xffffffffu, lane < jmax && !(ljj > 0.0));
              if (bad && fj < 0) fj = R0 + __ffs(bad) - 1;
            }
            // sigma_new / -mu sit in the first unfactored column of the last panel
            if (c == NC - 1) {
              const int cs = m - R0;
#pragma unroll
              for (int rr = 0; rr < kMaxRows; ++rr) {
                if (rr * 32 < NR) {
                  const int row = R0 + lane + 32 * rr;
#pragma unroll
                  for (int x = 0; x < 8; ++x) {
                    if (x == cs && row == m) out2[0] = a[rr][x];
                    if (x == cs && row == m + 1) out2[1] = a[rr][x];
                  }
                }
              }
            }
            if (c + 1 < NC) {
              __syncwarp();
              // L rows below the diagonal tile back to shared memory, permuted
#pragma unroll
              for (int rr = 0; rr < kMaxRows; ++rr) {
                const int row = R0 + lane + 32 * rr;
                if (rr * 32 < NR && row >= R0 + 8 && row < P && (last || row <= m + 1)) {
                  const int b = pbase(row);
                  st2(smem + b + 0, a[rr][0], a[rr][4]);
                  st2(smem + b + 2, a[rr][1], a[rr][5]);
                  st2(smem + b + 4, a[rr][2], a[rr][6]);
                  st2(smem + b + 6, a[rr][3], a[rr][7]);
                }
              }
              __syncwarp();
              // right-looking update of the group's later tile columns
              if (jj + 1 < GW) {
                double2 f[NT];
#pragma unroll
                for (int I = 0; I < NT; ++I)
                  if (I > c) f[I] = ld2(smem + pbase(8 * I + r) + 2 * q);
#pragma unroll
                for (int kk = 0; kk < 2; ++kk) {
#pragma unroll
                  for (int j2 = jj + 1; j2 < GW; ++j2) {
                    const int J = c0 + j2;
#pragma unroll
                    for (int I = 0; I < NT; ++I) {
                      if (J < NT && I >= J && J < NC)
                        mma(acc[j2][I][0], acc[j2][I][1], neg(kk ? f[I].y : f[I].x),
                            kk ? f[J].y : f[J].x);
                    }
                  }
                }
              }
            }
          }
        }
      }
    }

    // ---------------- per-block log-density ----------------
    const int64_t kk = e - 1 - rest_lo;
    __syncwarp();
    if (fj >= 0) {
      if (lane == 0) atomicMin(&fail[0], npd_key(e, fj, m));
    } else if (lane == 0) {
      const double sg = out2[0];
      const double mu = -out2[1];
      mu_out[kk] = mu;
      sig_out[kk] = sg;
      if (!(sg > 0.0)) {
        atomicMin(&fail[1], (unsigned long long)e);
        rest[kk] = 0.0;
      } else {
        const double resid = yt - mu;
        rest[kk] = -0.5 * (resid * resid / sg + kLog2Pi + log(sg));
      }
    }
    __syncwarp();
  }
}

template <int NT, int GW>
struct Occupancy {
  // register budget: 3 CTAs (12 warps) per SM for the large shapes
  static constexpr int kMinCtas = NT >= 7 ? 3 : (NT >= 5 ? 4 : 6);
};

template <int NT, int KIND, int MC, int GW, bool CACHE>
cudaError_t launch(const Plan& p, const CovParams& cp, int64_t e_lo, int64_t e_hi,
                   cudaStream_t stream) {
  constexpr int MINB = Occupancy<NT, GW>::kMinCtas;
  const WarpLayout wl = WarpLayout::make(p.m, NT, GW);
  const size_t sm = sizeof(double) * ((size_t)kHead + (size_t)kWarps * wl.stride);
  static size_t configured[64] = {};
  const int dev = p.device & 63;
  auto kern = loglik_ll_kernel<NT, KIND, MC, GW, CACHE, MINB>;
  if (configured[dev] < sm) {
    cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (err != cudaSuccess) return err;
    configured[dev] = sm;
  }
  int per_sm = 0;
  cudaError_t err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kWarps * 32, sm);
  if (err != cudaSuccess) return err;
  if (per_sm < 1) per_sm = 1;
  const int64_t count = e_hi - e_lo;
  const int64_t want = (count + kWarps - 1) / kWarps;
  const int64_t cap = (int64_t)p.num_sms * per_sm;
  const int grid = (int)(want < cap ? want : cap);
  kern<<<grid, kWarps * 32, sm, stream>>>(p.d_pts, p.d_nbr, p.m, e_lo, e_hi, p.rest_lo, cp.s2,
                                         cp.inv_beta, p.d_rest, p.d_mu, p.d_sig, p.d_fail,
                                         p.d_dcache, p.dcache_stride);
  return cudaGetLastError();
}

template <int NT, int KIND, int MC>
cudaError_t launch_c(const Plan& p, const CovParams& cp, int64_t e_lo, int64_t e_hi,
                     cudaStream_t stream, bool cache) {
  if (cache) return launch<NT, KIND, MC, 2, true>(p, cp, e_lo, e_hi, stream);
  return launch<NT, KIND, MC, 2, false>(p, cp, e_lo, e_hi, stream);
}

template <int KIND>
cudaError_t launch_kind(const Plan& p, const CovParams& cp, int64_t e_lo, int64_t e_hi,
                        cudaStream_t stream, bool cache) {
  if (p.m == 60) return launch_c<8, KIND, 60>(p, cp, e_lo, e_hi, stream, cache);
  if (p.m == 30) return launch_c<4, KIND, 30>(p, cp, e_lo, e_hi, stream, cache);
  switch ((p.m + 2 + 7) / 8) {
    case 1: return launch_c<1, KIND, 0>(p, cp, e_lo, e_hi, stream, cache);
    case 2: return launch_c<2, KIND, 0>(p, cp, e_lo, e_hi, stream, cache);
    case 3: return launch_c<3, KIND, 0>(p, cp, e_lo, e_hi, stream, cache);
    case 4: return launch_c<4, KIND, 0>(p, cp, e_lo, e_hi, stream, cache);
    case 5: return launch_c<5, KIND, 0>(p, cp, e_lo, e_hi, stream, cache);
    case 6: return launch_c<6, KIND, 0>(p, cp, e_lo, e_hi, stream, cache);
    case 7: return launch_c<7, KIND, 0>(p, cp, e_lo, e_hi, stream, cache);
    case 8: return launch_c<8, KIND, 0>(p, cp, e_lo, e_hi, stream, cache);
    default: return cudaErrorNotSupported;
  }
}

}  // namespace ll
}  // namespace vgp
