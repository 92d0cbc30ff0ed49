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
  static constexpr int kPanelLd = 10;  // panel row stride (doubles): conflict-free LDS.128 rows
  // per warp: panel (kP rows), (x, y) pairs, obs, 2 outputs, mbarrier
  static constexpr int kWarpDoubles = kP * kPanelLd + 2 * kP + kP + 2 + 2;
  // distance-cache buffer per warp (doubles), 16-byte aligned
  static constexpr int cache_doubles(int m) { return ((m * (m + 1) / 2) + 1) & ~1; }
  static size_t bytes(bool cache, int m) {
    return sizeof(double) *
           (256 + (size_t)kWarps * (kWarpDoubles + (cache ? cache_doubles(m) : 0)));
  }
};

// ---- TMA bulk copy (cp.async.bulk, SASS UBLKCP) + mbarrier helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes,
                                          uint64_t* bar) {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  }
}

// minimum resident CTAs per SM (register cap 65536 / (128 * kMinCtas)): the
// 36 accumulator tiles of NT = 8 alone take 144 registers, and a 168 cap
// (3 CTAs) spilled and measured slower than 2 CTAs without spills.
template <int NT>
struct Occupancy {
  static constexpr int kMinCtas = NT >= 7 ? 2 : (NT >= 5 ? 3 : (NT >= 3 ? 4 : 6));
};

// MC > 0 compiles the kernel for m == MC exactly: every panel extent, the
// location of sigma_new / -mu and all padding tests fold away, leaving
// branch-free straight-line code for the hot configurations (m = 30, 60).
// CACHE: the plan holds every block's distances (compact strictly-lower order,
// rows 1..m, built once per dataset by build_dcache_kernel); each warp streams
// the next block's row of the cache into shared memory with a 1D TMA bulk copy
// (cp.async.bulk + mbarrier) while it factors the current one, and the
// generation skips the coordinate gather, the distance and the square root.
template <int NT, int KIND, int MC, int MINB = Occupancy<NT>::kMinCtas, bool CACHE = false>
__global__ void __launch_bounds__(kWarps * 32, MINB)
loglik_kernel(const double4* __restrict__ pts, const int32_t* __restrict__ nbr, int m_rt,
              int64_t e_lo, int64_t e_hi, int64_t rest_lo, double s2, double inv_beta,
              double* __restrict__ rest, double* __restrict__ mu_out,
              double* __restrict__ sig_out, unsigned long long* __restrict__ fail,
              const double* __restrict__ dcache, int64_t cstride) {
  using S = Smem<NT>;
  constexpr int P = S::kP;
  constexpr int NTILE = NT * (NT + 1) / 2;
  constexpr int LD = S::kPanelLd;
  const int m = MC > 0 ? MC : m_rt;
  extern __shared__ __align__(16) double smem[];
  double* tab = smem;  // 256: sigma^2 * 2^(j/256)
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int r = lane >> 2;  // fragment row
  const int q = lane & 3;   // fragment column pair
  double* pan = smem + 256 + (size_t)warp * S::kWarpDoubles;
  double2* XY = reinterpret_cast<double2*>(pan + P * LD);
  double* O = pan + P * LD + 2 * P;
  double* out2 = O + P;
  uint64_t* bar = reinterpret_cast<uint64_t*>(out2 + 2);
  double* dbuf = smem + 256 + (size_t)kWarps * S::kWarpDoubles + (size_t)warp * cstride;

  for (int i = threadIdx.x; i < 256; i += blockDim.x) tab[i] = s2 * kExp2Table[i];
  if (CACHE && lane == 0) mbar_init(bar);
  __syncthreads();
  const uint32_t cbytes = (uint32_t)(cstride * sizeof(double));
  uint32_t cphase = 0;

  const int64_t stride = (int64_t)gridDim.x * kWarps;
  // Software-pipelined gather: block e+stride's neighbour indices are read
  // during block e's first panel and its points during the second-to-last
  // panel, so the dependent L2 round trips overlap the factorization.
  // Lane owns conditioning-set slots lane and lane + 32 (index m = target).
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
    if (CACHE && lane == 0) bulk_load(dbuf, dcache + (e - 1 - rest_lo) * cstride, cbytes, bar);
    pf0 = slot_point(slot_index(e, lane));
    if (P > 32) pf1 = slot_point(slot_index(e, lane + 32));
  }
  for (; e < e_hi; e += stride) {
    const int64_t en = e + stride;
    // ---------------- gather (from the prefetch registers) ----------------
    if (lane < P) {
      XY[lane] = make_double2(pf0.x, pf0.y);
      O[lane] = pf0.z;
    }
    if (P > 32 && lane + 32 < P) {
      XY[lane + 32] = make_double2(pf1.x, pf1.y);
      O[lane + 32] = pf1.z;
    }
    __syncwarp();

    // ---------------- generate straight into accumulator fragments ----------------
    // lane (r, q) owns entries (8I + r, 8J + 2q + h) of tile (I, J), I >= J.
    // Rows below 8 (NT - 1) are always covariance rows (m >= 8 NT - 9), so
    // only the diagonal tiles and the last tile row need entry tests.
    double t[NTILE][2];
    if (CACHE) {
      mbar_wait(bar, cphase);
      cphase ^= 1;
#pragma unroll
      for (int I = 0; I < NT; ++I) {
        const int a = 8 * I + r;
        const int rowbase = a * (a - 1) / 2;  // compact index of (a, 0)
#pragma unroll
        for (int Jt = 0; Jt <= I; ++Jt) {
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int b = 8 * Jt + 2 * q + h;
            const bool lower = (I < NT - 1 && Jt < I) || (b < a && a <= m);
            double val = 0.0;
            if (lower) val = cov_fast<KIND>(dbuf[rowbase + b], inv_beta, tab);
            if (I == NT - 1 || Jt == I) {
              if (a == b && a <= m) val = s2;       // C(0) = sigma^2
              if (a == m + 1 && b < m) val = O[b];  // yJ row
            }
            t[tidx(I, Jt)][h] = val;
          }
        }
      }
      __syncwarp();
      if (lane == 0 && en < e_hi)
        bulk_load(dbuf, dcache + (en - 1 - rest_lo) * cstride, cbytes, bar);
    } else {
#pragma unroll
    for (int I = 0; I < NT; ++I) {
      const int a = 8 * I + r;
      const double2 pa = XY[a];
#pragma unroll
      for (int Jt = 0; Jt <= I; ++Jt) {
        const double4 pb = *reinterpret_cast<const double4*>(XY + 8 * Jt + 2 * q);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int b = 8 * Jt + 2 * q + h;
          const double dx = pa.x - (h ? pb.z : pb.x);
          const double dy = pa.y - (h ? pb.w : pb.y);
          // + 2^-1000: exact duplicates give d ~ 1e-150, C = sigma^2 to the last bit
          const double d2 = fma(dx, dx, fma(dy, dy, 0x1p-1000));
          double val = cov_fast<KIND>(sqrt_pos_nz(d2), inv_beta, tab);
          if (I == NT - 1 || Jt == I) {
            if (!(a <= m && b < a)) val = 0.0;
            if (a == b && a <= m) val = s2;       // C(0) = sigma^2
            if (a == m + 1 && b < m) val = O[b];  // yJ row
          }
          t[tidx(I, Jt)][h] = val;
        }
      }
    }
    }

    // ---------------- blocked right-looking Cholesky with look-ahead ----------------
    // Panel c lives in registers in row-owner layout (lane l: panel rows l, l+32)
    // and is factored column by column; the next pivot is formed by its owner
    // from its own row, so one shuffle sits on the pivot-to-pivot chain.  After
    // panel c, tile column c+1 is updated first and handed to the next panel;
    // the rest of the trailing update is issued after, where it overlaps the
    // next panel's dependent chain.  Failures are tracked without branching
    // (fj: first non-positive pivot column) and acted on once per block.
    constexpr int kMaxRows = 2;
    int fj = -1;
    double a[kMaxRows][8];
    auto load_panel = [&](const int c) {
      const int NR = P - 8 * c;
#pragma unroll
      for (int I = c; I < NT; ++I)
        *reinterpret_cast<double2*>(pan + (8 * (I - c) + r) * LD + 2 * q) =
            make_double2(t[tidx(I, c)][0], t[tidx(I, c)][1]);
      __syncwarp();
#pragma unroll
      for (int rr = 0; rr < kMaxRows; ++rr) {
        const int row = lane + 32 * rr;
#pragma unroll
        for (int x = 0; x < 4; ++x) {
          double2 v = make_double2(0.0, 0.0);
          if (rr * 32 < NR && row < NR) v = *reinterpret_cast<const double2*>(pan + row * LD + 2 * x);
          a[rr][2 * x] = v.x;
          a[rr][2 * x + 1] = v.y;
        }
      }
      __syncwarp();
    };
    load_panel(0);
#pragma unroll
    for (int c = 0; c < NT; ++c) {
      const int R0 = 8 * c;
      const int NR = P - R0;
      const int jmax = min(8, m - R0);  // pivots in this tile column
      if (c == 0 && en < e_hi) {
        ni0 = slot_index(en, lane);
        if (P > 32) ni1 = slot_index(en, lane + 32);
      }
      if (c == (NT >= 2 ? NT - 2 : 0) && en < e_hi) {
        pf0 = slot_point(ni0);
        if (P > 32) pf1 = slot_point(ni1);
      }
      if (jmax > 0) {
        double piv = shfl(a[0][0], 0);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          if (j < jmax) {
            if (!(piv > 0.0) && fj < 0) fj = R0 + j;
            const double inv = rsqrt_pos3(piv);
#pragma unroll
            for (int rr = 0; rr < kMaxRows; ++rr)
              if (rr * 32 < NR) a[rr][j] *= inv;  // the pivot row's own entry becomes piv * inv = L_jj
            if (j + 1 < 8) {
              const double nxt = fma(-a[0][j], a[0][j], a[0][j + 1]);  // lane j+1's pivot
              piv = shfl(nxt, j + 1);
            }
#pragma unroll
            for (int jp = j + 1; jp < 8; ++jp) {
              const double lc = shfl(a[0][j], jp);  // L[R0 + jp][j]
#pragma unroll
              for (int rr = 0; rr < kMaxRows; ++rr)
                if (rr * 32 < NR) a[rr][jp] = fma(-a[rr][j], lc, a[rr][jp]);
            }
          }
        }
        // sigma_new / -mu sit in this panel's first unfactored column
        if (m - R0 < 8) {
          const int cs = m - R0;
#pragma unroll
          for (int rr = 0; rr < kMaxRows; ++rr) {
            if (rr * 32 < NR) {
              const int row = lane + 32 * rr;
#pragma unroll
              for (int x = 0; x < 8; ++x) {
                if (x == cs && row == m - R0) out2[0] = a[rr][x];
                if (x == cs && row == m + 1 - R0) out2[1] = a[rr][x];
              }
            }
          }
        }
        if (c + 1 < NT) {
          // L panel -> shared memory -> A-fragments frag_kk(T) = L[8I + r][4 kk + q]
#pragma unroll
          for (int rr = 0; rr < kMaxRows; ++rr) {
            const int row = lane + 32 * rr;
            if (rr * 32 < NR && row < NR) {
#pragma unroll
              for (int x = 0; x < 4; ++x)
                *reinterpret_cast<double2*>(pan + row * LD + 2 * x) =
                    make_double2(a[rr][2 * x], a[rr][2 * x + 1]);
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
          // look-ahead: tile column c+1 first, then hand it to the next panel
#pragma unroll
          for (int I = c + 1; I < NT; ++I) {
            mma884(t[tidx(I, c + 1)][0], t[tidx(I, c + 1)][1], neg(fa[I][0]), fa[c + 1][0]);
            mma884(t[tidx(I, c + 1)][0], t[tidx(I, c + 1)][1], neg(fa[I][1]), fa[c + 1][1]);
          }
          if (m - 8 * (c + 1) > 0) load_panel(c + 1);
          // remaining trailing update A_IJ -= L_Ic L_Jc^T, c + 1 < J <= I
#pragma unroll
          for (int I = c + 2; I < NT; ++I) {
            const double n0 = neg(fa[I][0]);
            const double n1 = neg(fa[I][1]);
#pragma unroll
            for (int Jt = c + 2; Jt <= I; ++Jt) {
              mma884(t[tidx(I, Jt)][0], t[tidx(I, Jt)][1], n0, fa[Jt][0]);
              mma884(t[tidx(I, Jt)][0], t[tidx(I, Jt)][1], n1, fa[Jt][1]);
            }
          }
        }
      }
    }

    // ---------------- per-block log-density ----------------
    const int64_t kk = e - 1 - rest_lo;
    if (fj >= 0) {
      if (lane == 0) atomicMin(&fail[0], npd_key(e, fj, m));
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

template <int NT, int KIND, int MC, int MINB = Occupancy<NT>::kMinCtas, bool CACHE = false>
cudaError_t launch(const Plan& p, const CovParams& cp, int64_t e_lo, int64_t e_hi,
                   cudaStream_t stream) {
  const size_t sm = Smem<NT>::bytes(CACHE, p.m);
  static size_t configured[64] = {};  // per device ordinal: smem size set
  const int dev = p.device & 63;
  if (configured[dev] < sm) {
    cudaError_t err = cudaFuncSetAttribute(loglik_kernel<NT, KIND, MC, MINB, CACHE>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (err != cudaSuccess) return err;
    configured[dev] = sm;
  }
  const int64_t count = e_hi - e_lo;
  const int64_t want = (count + kWarps - 1) / kWarps;
  const int64_t cap = (int64_t)p.num_sms * 16;
  const int grid = (int)(want < cap ? want : cap);
  loglik_kernel<NT, KIND, MC, MINB, CACHE><<<grid, kWarps * 32, sm, stream>>>(
      p.d_pts, p.d_nbr, p.m, e_lo, e_hi, p.rest_lo, cp.s2, cp.inv_beta, p.d_rest, p.d_mu,
      p.d_sig, p.d_fail, p.d_dcache, p.dcache_stride);
  return cudaGetLastError();
}

template <int NT, int KIND, int MC>
cudaError_t launch_c(const Plan& p, const CovParams& cp, int64_t e_lo, int64_t e_hi,
                     cudaStream_t stream) {
  // the distance cache is laid out for the grouped kernel (vgp_ll_kernel.cuh);
  // this all-register kernel always computes distances from coordinates
  return launch<NT, KIND, MC, Occupancy<NT>::kMinCtas, false>(p, cp, e_lo, e_hi, stream);
}

template <int KIND>
cudaError_t launch_kind(const Plan& p, const CovParams& cp, int64_t e_lo, int64_t e_hi,
                        cudaStream_t stream) {
  if (p.m == 60) return launch_c<8, KIND, 60>(p, cp, e_lo, e_hi, stream);
  if (p.m == 30) return launch_c<4, KIND, 30>(p, cp, e_lo, e_hi, stream);
  switch ((p.m + 2 + 7) / 8) {
    case 1: return launch_c<1, KIND, 0>(p, cp, e_lo, e_hi, stream);
    case 2: return launch_c<2, KIND, 0>(p, cp, e_lo, e_hi, stream);
    case 3: return launch_c<3, KIND, 0>(p, cp, e_lo, e_hi, stream);
    case 4: return launch_c<4, KIND, 0>(p, cp, e_lo, e_hi, stream);
    case 5: return launch_c<5, KIND, 0>(p, cp, e_lo, e_hi, stream);
    case 6: return launch_c<6, KIND, 0>(p, cp, e_lo, e_hi, stream);
    case 7: return launch_c<7, KIND, 0>(p, cp, e_lo, e_hi, stream);
    case 8: return launch_c<8, KIND, 0>(p, cp, e_lo, e_hi, stream);
    default: return cudaErrorNotSupported;
  }
}

}  // namespace dmma
}  // namespace vgp
