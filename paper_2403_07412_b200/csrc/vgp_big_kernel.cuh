// CTA-per-block FP64 tensor-core (DMMA) Vecchia kernel for large conditioning
// sets (m + 2 > 64; BASELINE configs 3-4: m = 90..400).
//
// One CTA of 4 warps owns one conditioning block e >= 1 at a time
// (vg/vecchia.py:154-162 assemble, :180-190 _numeric_stage, :193-214
// _reduction_stage); the augmented (8 NT)^2 matrix (rows 0..m-1 Sigma_e, row
// m v_e, row m+1 yJ, zero padding) is factored left-looking over 8-wide tile
// columns:
//
//   column   (look-ahead: during column c's diagonal phase) the tiles (I, c+1)
//            are dealt to warps 1..3 round-robin, kGroup at a time; each tile is generated (lean FP64 Matern) and updated
//            with every earlier tile column's L, mma.sync.m8n8k4.f64 (SASS
//            DMMA.8x8x4), kGroup independent accumulators per warp;
//   diagonal warp 0 factors the 8x8 diagonal tile (one rsqrt / shuffle pivot
//            chain) and publishes L_cc transposed + the reciprocal pivots; at
//            the last column its panel also holds rows m, m+1, whose Schur
//            complement gives sigma_new, -mu and the block's log-density;
//   solve    every warp solves 32-row chunks of the rows below the diagonal
//            tile against L_cc (row per lane, L_cc broadcast from shared
//            memory) and writes L back in DMMA-operand order.
//
// The block's points (x, y, obs, 0: 32-byte rows) are gathered by TMA
// (cp.async.bulk.tensor.2d tile::gather4, SASS UTMALDG.2D.GATHER4: each lane
// of warp 1 brings 4 rows by index) into shared memory while the previous
// block finishes, so no block starts on a dependent global-load chain.
//
// Tiles live in the ws:: swizzled layout (conflict-free fragment and row
// accesses): in shared memory while the tile triangle fits (m <= ~200,
// several CTAs per SM overlap one block's serial diagonal phase with the
// others' DMMA phases), otherwise in a per-CTA global scratch that stays in
// L2.  Distances come from the plan's cache (same tile layout, read straight
// from HBM with coalesced 512-byte tile loads) or from the gathered
// coordinates.
#pragma once

#include <cuda.h>

#include <cstdio>
#include <cstdlib>
#include <type_traits>
#include <vector>

#include "vgp_ktab.cuh"
#include "vgp_math.cuh"
#include "vgp_ws_kernel.cuh"

namespace vgp {
namespace big {

using dmma::neg;
using dmma::shfl;
using ll::cov_lean;
using ll::ld2;
using ll::mma;
using ll::rsqrt_chain;
using ll::st2;
using ws::chunk_off;
using ws::ntri;
using ws::tidx;

constexpr int kWarps = 4;
constexpr int kThreads = 32 * kWarps;
constexpr int kGroup = 4;  // tiles per warp in flight
constexpr int kTraceCtas = 16, kTraceEv = 6;
constexpr int kHead = 256 + 64 + 8 + 5 * kBesselTab;  // exp table | Lt | Iv | Bessel tables

__host__ __device__ constexpr int ntiles_of(int m) { return (m + 2 + 7) / 8; }
// doubles of the shared-memory area besides the tiles
// the Bessel tables only exist for general nu: the closed forms keep 2.5 KB
// more shared memory per CTA (m = 120: 74.6 KB, 3 CTAs per SM instead of 2)
__host__ __device__ constexpr int head_fixed(int kind) {
  return 256 + 64 + 8 + (kind == kMaternGen ? 5 * kBesselTab : 0);
}
// head | G: the block's points, 32-byte rows (P of them), 128-byte aligned
// for the TMA gather | mbarrier (+ pad)
__host__ __device__ constexpr int g_offset(int kind) { return (head_fixed(kind) + 15) & ~15; }
__host__ __device__ inline int head_doubles(int m, int kind = kMaternGen) {
  return g_offset(kind) + 4 * 8 * ntiles_of(m) + 2;
}

// Shared-memory tile slots: tile (I, J) is live from its generation (look-ahead
// at column J - 1) to its last use as L (column I - 1); tiles with disjoint
// lifetimes share a slot (greedy interval colouring on the host,
// big_slot_map).  m = 120: 73 slots instead of 136 tiles, 4 CTAs per SM
// instead of 3.  The global-scratch path keeps the plain triangle.
constexpr int kMaxSlotTiles = 528;  // NT <= 32
constexpr int kSlotStride = 32;
struct SlotMap {
  // byte offset of tile (I, J) at [I * kSlotStride + J]: row-major, so the
  // left-looking k loop walks consecutive entries (no triangular index
  // arithmetic); 32-bit, no byte permutes on the lookups
  int32_t s[kSlotStride * kSlotStride];
};
int big_slot_map(int nt, SlotMap* map);  // returns the slot count

// one 4-row TMA gather of 32-byte point rows into shared memory (tile::gather4)
__device__ __forceinline__ void gather4(void* dst, const CUtensorMap* map, int r0, int r1, int r2,
                                        int r3, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(dmma::smem_u32(dst)),
      "l"(map), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(dmma::smem_u32(bar))
      : "memory");
}
__host__ __device__ inline int64_t tile_doubles(int m) {
  const int nt = ntiles_of(m);
  return (int64_t)ntri(nt) * 64;
}

// General-nu Matern: s2 2^(1-nu)/Gamma(nu) u^nu K_nu(u), u = d / beta
// (vg/kernels.py:75-81).  Not inlined: the kernel evaluates covariances at
// 2 * kGroup unrolled sites, and eight inlined copies of the Bessel K
// iteration overflow the instruction cache (profiles/r01_ncu_c5_*.txt).
static __device__ __noinline__ double matern_gen(double d, const CovParams& cp, const double* btab) {
  const double u = d / cp.beta;
  return cp.s2 * cp.coef * pow(u, cp.nu) * bessel_k_tab(cp, u, btab);
}

// covariance at distance d: lean closed forms, or the reference expression
// (general-nu Matern via the device Bessel K_nu, power exponential;
// vg/kernels.py:59-91) with C(0) = sigma^2 exactly (d below 1e-100: the
// diagonal and exact duplicates, whose distance is 2^-500 by construction)
template <int KIND>
__device__ __forceinline__ double cov_any(double d, const CovParams& cp, const double* tab,
                                          const double* btab, const double* __restrict__ ktab) {
  if (KIND <= kMatern25) return cov_lean<KIND>(d, cp.inv_beta, tab);
  if (d < 1e-100) return cp.s2;
  if (KIND == kMaternGen) {
    // per-evaluation polynomial table (vgp_ktab.cuh) when the plan built one
    if (ktab)
      return cov_ktab(d * cp.inv_beta, ktab, cp);
    return matern_gen(d, cp, btab);
  }
  return cov_ref(cp, d);
}

// MINB > 0: minimum resident CTAs for the register budget (5 where the tile
// triangle lets 5 CTAs share the SM, e.g. m = 63..80)
template <int KIND, bool CACHE, bool GT, int MC = 0, bool SLOTS = false, bool TRACE = false, int MINB = 0>
__global__ void __launch_bounds__(kThreads, MINB > 0 ? MINB : (GT ? 3 : (SLOTS && MC == 120 ? 5 : 4)))
loglik_big_kernel(const __grid_constant__ CUtensorMap pmap, const int32_t* __restrict__ nbr,
                  int m_rt, int64_t e_lo, int64_t e_hi, int64_t rest_lo, CovParams cp,
                  double* __restrict__ rest, double* __restrict__ mu_out,
                  double* __restrict__ sig_out, unsigned long long* __restrict__ fail,
                  const double* __restrict__ dcache, int64_t cstride, double* __restrict__ gscratch,
                  const double* __restrict__ ktab, const __grid_constant__ SlotMap smap,
                  long long* __restrict__ trace = nullptr) {
  // MC > 0: conditioning size fixed at compile time (tile counts and
  // addresses fold to constants)
  const int m = MC > 0 ? MC : m_rt;
  const int NT = MC > 0 ? ntiles_of(MC) : ntiles_of(m);
  const int P = 8 * NT;
  const double s2 = cp.s2;
  const int NC = (m + 8) >> 3;  // tile columns holding pivots or the Schur column
  extern __shared__ __align__(128) double smem[];
  double* tabw = smem;
  double* Lt = smem + 256;  // L_cc transposed: Lt[8k + j] = L[j][k]
  double* Iv = Lt + 64;     // reciprocal pivots
  double* Bt = Iv + 8;      // general-nu Bessel reciprocal tables
  double4* G = reinterpret_cast<double4*>(smem + g_offset(KIND));  // the block's points
  uint64_t* gbar = reinterpret_cast<uint64_t*>(smem + g_offset(KIND) + 4 * P);
  double* T = GT ? gscratch + (size_t)blockIdx.x * tile_doubles(m) : smem + head_doubles(m, KIND);
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  // clock64 phase trace (VGP_TRACE_BIG, tools/big_trace.py): CTAs <
  // kTraceCtas, their third block, per column and warp kTraceEv events
  int iter = 0;
  auto stamp = [&](int c, int ev) {
    if (TRACE && iter == 2 && blockIdx.x < kTraceCtas && lane == 0)
      trace[((blockIdx.x * kWarps + warp) * 32 + c) * kTraceEv + ev] = clock64();
  };
  const int r = lane >> 2;  // fragment row
  const int q = lane & 3;   // fragment column pair

  for (int i = threadIdx.x; i < 256; i += blockDim.x) tabw[i] = s2 * kExp2Table[i];
  if (KIND == kMaternGen) bessel_fill_tab(cp, Bt, threadIdx.x, blockDim.x);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(dmma::smem_u32(gbar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const double* tab = smem;
  auto tile = [&](int I, int J) -> double* {
    if (SLOTS) return reinterpret_cast<double*>(reinterpret_cast<char*>(T) + smap.s[I * kSlotStride + J]);
    return T + (size_t)tidx(I, J, NT) * 64;
  };
  // block eb's point rows: lane l of warp 1 gathers rows 4l..4l+3 (P / 4 <= 32
  // lanes per pass): neighbours a < m, the target at a = m, row 0 as padding
  const uint32_t gbytes = (uint32_t)(P * sizeof(double4));
  auto row_of = [&](int64_t eb, int a) -> int {
    if (a < m) return nbr[(eb - 1 - rest_lo) * (int64_t)m + a];
    return a == m ? (int)(m + eb - 1) : 0;
  };
  auto issue_gather = [&](int64_t eb) {
    if (lane == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(dmma::smem_u32(gbar)),
                   "r"(gbytes)
                   : "memory");
    __syncwarp();
    for (int a0 = 4 * lane; a0 < P; a0 += 128)
      gather4(G + a0, &pmap, row_of(eb, a0), row_of(eb, a0 + 1), row_of(eb, a0 + 2),
              row_of(eb, a0 + 3), gbar);
  };
  uint32_t gpar = 0;
  if (warp == 1 && e_lo + blockIdx.x < e_hi) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    issue_gather(e_lo + blockIdx.x);
  }

  int fj = -1;  // warp 0: first non-positive pivot column of the current block
  for (int64_t e = e_lo + blockIdx.x; e < e_hi; e += gridDim.x) {
    const double* D = CACHE ? dcache + (e - 1 - rest_lo) * cstride : nullptr;
    // ---- this block's points (gathered while the previous block finished)
    dmma::mbar_wait(gbar, gpar);
    gpar ^= 1;
    const double y_t = G[m].z;  // target observation (G is refilled before the last panel)
    fj = -1;

    // tiles (I0 + g * st, J), g < NG: generate, apply L of tile columns
    // k <= kmax with DMMA, stage (natural column order)
    auto la_tiles = [&](const int J, const int kmax, const int I0, const int st, auto ngc) {
      constexpr int NG = decltype(ngc)::value;
      double acc[NG][2];
#pragma unroll
      for (int g = 0; g < NG; ++g) {
        const int I = I0 + g * st;
        const int i = 8 * I + r;
        double v0, v1;
        const int j0 = 8 * J + 2 * q;  // columns j0, j0 + 1
        if (CACHE) {
          const double2 dv = __ldg(reinterpret_cast<const double2*>(D + (size_t)tidx(I, J, NT) * 64 + chunk_off(r, q)));
          v0 = cov_any<KIND>(dv.x, cp, tab, Bt, ktab);
          v1 = cov_any<KIND>(dv.y, cp, tab, Bt, ktab);
        } else {
          const double2 pa = *reinterpret_cast<const double2*>(G + (i < P ? i : 0));
          const double2 pb0 = *reinterpret_cast<const double2*>(G + j0);
          const double2 pb1 = *reinterpret_cast<const double2*>(G + j0 + 1);
          double dx = pa.x - pb0.x, dy = pa.y - pb0.y;
          v0 = cov_any<KIND>(sqrt_pos_nz(fma(dx, dx, fma(dy, dy, 0x1p-1000))), cp, tab, Bt, ktab);
          dx = pa.x - pb1.x;
          dy = pa.y - pb1.y;
          v1 = cov_any<KIND>(sqrt_pos_nz(fma(dx, dx, fma(dy, dy, 0x1p-1000))), cp, tab, Bt, ktab);
        }
        if (i > m) {  // row m+1: yJ (0 from column m on); padding: 0
          v0 = (i == m + 1 && j0 < m) ? G[j0].z : 0.0;
          v1 = (i == m + 1 && j0 + 1 < m) ? G[j0 + 1].z : 0.0;
        }
        // accumulate -A + sum L L^T and negate once at the store:
        // bit-identical to A - sum L L^T (round-to-nearest is odd under
        // negation) without negating an operand per DMMA
        acc[g][0] = -v0;
        acc[g][1] = -v1;
      }
      for (int k = 0; k <= kmax; ++k) {
        const double2 b = ld2(tile(J, k) + chunk_off(r, q));
        double2 a[NG];
#pragma unroll
        for (int g = 0; g < NG; ++g) a[g] = ld2(tile(I0 + g * st, k) + chunk_off(r, q));
#pragma unroll
        for (int kk = 0; kk < 2; ++kk) {
#pragma unroll
          for (int g = 0; g < NG; ++g) mma(acc[g][0], acc[g][1], kk ? a[g].y : a[g].x, kk ? b.y : b.x);
        }
      }
#pragma unroll
      for (int g = 0; g < NG; ++g) st2(tile(I0 + g * st, J) + chunk_off(r, q), -acc[g][0], -acc[g][1]);
    };
    // a group of ng tiles runs a body unrolled for exactly that many: a
    // predicated-off DMMA still occupies the FP64 datapath (ncu: 2464 DMMA
    // issued per m = 120 block against 1360 needed when the tail groups were
    // predicated)
    auto dispatch = [&](const int ng, auto&& body) {
      static_assert(kGroup == 4, "group dispatch below");
      switch (ng) {
        case 4: body(std::integral_constant<int, 4>{}); break;
        case 3: body(std::integral_constant<int, 3>{}); break;
        case 2: body(std::integral_constant<int, 2>{}); break;
        default: body(std::integral_constant<int, 1>{}); break;
      }
    };
    // tiles (I, J), J <= I < Iend, dealt round-robin over warps
    // [w0, w0 + nw) in groups of kGroup
    auto column_work = [&](const int J, const int kmax, const int w0, const int nw, const int Iend) {
      for (int I0 = J + (warp - w0); I0 < Iend; I0 += nw * kGroup)
        dispatch(min(kGroup, (Iend - 1 - I0) / nw + 1), [&](auto ngc) { la_tiles(J, kmax, I0, nw, ngc); });
    };
    // the last left-looking step of tile column J: reload, apply L of column
    // k, stage (tiles dealt round-robin over all warps)
    auto column_finish = [&](const int J, const int k) {
      const double2 b = ld2(tile(J, k) + chunk_off(r, q));
      for (int I = J + warp; I < NT; I += kWarps) {
        double* tp = tile(I, J) + chunk_off(r, q);
        const double2 v = ld2(tp);
        const double2 a = ld2(tile(I, k) + chunk_off(r, q));
        double a0 = v.x, a1 = v.y;
        mma(a0, a1, neg(a.x), b.x);
        mma(a0, a1, neg(a.y), b.y);
        st2(tp, a0, a1);
      }
    };

    // left-looking over tile columns with look-ahead: while warp 0 factors
    // the diagonal tile of column c, warps 1..3 generate column c + 1 and
    // apply every earlier column but c; after the row solve of column c one
    // DMMA step finishes column c + 1
    // (global-memory tiles, m >~ 230: no look-ahead, the extra reload pass
    // costs more in L2 than the overlap gains)
    constexpr bool kLookAhead = !GT;
    auto la_rest = [&](const int c) { return min(max(NT - c - 1 - 3 * kGroup, 0), 3); };
    column_work(0, -1, 0, kWarps, NT);
    __syncthreads();
    for (int c = 0; c < NC; ++c) {
      const bool lastc = (c == NC - 1);
      stamp(c, 0);
      if (kLookAhead) {
        // (more than 12 tiles: warps 1..3 take 4 each and the diagonal warp,
        // whose pivot chain is shorter than a 4-tile group's look-ahead
        // (tools/big_trace.py), the last 1-3 after its panel)
        if (warp != 0 && !lastc) column_work(c + 1, c - 1, 1, kWarps - 1, NT - la_rest(c));
      } else if (c > 0) {
        column_work(c, c - 1, 0, kWarps, NT);
        __syncthreads();
      }
      // the last tile column is generated: G is free, gather the next block
      // (its points land while this block's last panels finish)
      if (warp == 1 && c == NC - 1 && e + gridDim.x < e_hi) {
        __syncwarp();
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        issue_gather(e + gridDim.x);
      }
      // ================= diagonal tile (warp 0) =================
      if (warp == 0) {
        const int R0 = 8 * c;
        const int jmax = min(8, m - R0);
        const int nrows = lastc ? P - R0 : 8;  // last column: rows m, m+1 ride along (<= 16)
        double a[8];
        {
          const int I = c + (lane >> 3);
          const double* base = tile(I < NT ? I : c, c);
#pragma unroll
          for (int x = 0; x < 4; ++x) {
            double2 v = make_double2(0.0, 0.0);
            if (lane < nrows) v = ld2(base + chunk_off(lane & 7, x));
            a[2 * x] = v.x;
            a[2 * x + 1] = v.y;
          }
        }
        double lastpiv = 1.0;
        double iv[8];
        if (jmax > 0) {
          double piv = shfl(a[0], 0);
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            if (j < jmax) {
              if (j == jmax - 1) lastpiv = piv;
              const double inv = rsqrt_chain(piv);
              iv[j] = inv;
              a[j] *= inv;
              if (j + 1 < 8) {
                const double nxt = fma(-a[j], a[j], a[j + 1]);
                piv = shfl(nxt, j + 1);
              }
              // column j of L_cc straight into its published slot (Lt[8 j + row])
              // and back to every lane with broadcast LDS.128: 4 loads instead
              // of 14 32-bit shuffles per pivot on the block's critical path
              if (lane < 8) Lt[8 * j + lane] = a[j];
              __syncwarp();
#pragma unroll
              for (int x = (j + 1) & ~1; x < 8; x += 2) {
                const double2 lv = ld2(Lt + 8 * j + x);  // L[R0 + x][R0 + j], L[R0 + x + 1][R0 + j]
                if (x >= j + 1) a[x] = fma(-a[j], lv.x, a[x]);
                if (x + 1 >= j + 1) a[x + 1] = fma(-a[j], lv.y, a[x + 1]);
              }
            }
          }
        }
        // pivot test !(piv > 0) (vg/batchla.py:146-151): a non-positive or NaN
        // pivot turns every later pivot NaN; locate the first bad column
        if (!(lastpiv > 0.0) && fj < 0) {
          double ljj = a[0];
#pragma unroll
          for (int x = 1; x < 8; ++x)
            if (lane == x) ljj = a[x];
          const unsigned bad = __ballot_sync(0xffffffffu, lane < jmax && !(ljj > 0.0));
          fj = R0 + (bad ? __ffs(bad) - 1 : jmax - 1);
        }
        if (!lastc) {
          // (L_cc itself was published column by column in the pivot loop)
          if (lane == 0) {
            st2(Iv, iv[0], iv[1]);
            st2(Iv + 2, iv[2], iv[3]);
            st2(Iv + 4, iv[4], iv[5]);
            st2(Iv + 6, iv[6], iv[7]);
          }
        } else {
          // sigma_new = A[m][m], -mu = A[m+1][m] after m pivots (vg/vecchia.py:186-189, :206)
          const int cs = m - R0;
          double v = a[0];
#pragma unroll
          for (int x = 1; x < 8; ++x)
            if (x == cs) v = a[x];
          const double sg = shfl(v, cs);
          const double mu = -shfl(v, cs + 1);
          if (lane == 0) {
            const int64_t kk = e - 1 - rest_lo;
            if (fj >= 0) {
              atomicMin(&fail[0], npd_key(e, fj, m));
            } else {
              mu_out[kk] = mu;
              sig_out[kk] = sg;
              if (!(sg > 0.0)) {
                atomicMin(&fail[1], (unsigned long long)e);
                rest[kk] = 0.0;
              } else {
                const double resid = y_t - mu;
                rest[kk] = -0.5 * (resid * resid / sg + kLog2Pi + log(sg));
              }
            }
          }
        }
      }
      if (kLookAhead && warp == 0 && !lastc) {
        const int nr = la_rest(c);
        if (nr > 0)
          dispatch(nr, [&](auto ngc) { la_tiles(c + 1, c - 1, NT - nr, 1, ngc); });
      }
      stamp(c, 1);
      __syncthreads();
      stamp(c, 2);
      if (lastc) break;

      // ================= solve the rows below the diagonal tile =================
      {
        const double2 i01 = ld2(Iv), i23 = ld2(Iv + 2), i45 = ld2(Iv + 4), i67 = ld2(Iv + 6);
        const double iv[8] = {i01.x, i01.y, i23.x, i23.y, i45.x, i45.y, i67.x, i67.y};
        for (int rb = 8 * (c + 1) + 32 * warp; rb < P; rb += 32 * kWarps) {
          const int row = rb + lane;
          const bool ok = row < P;
          double* base = tile(ok ? row >> 3 : c + 1, c);
          double a[8];
#pragma unroll
          for (int x = 0; x < 4; ++x) {
            double2 v = make_double2(0.0, 0.0);
            if (ok) v = ld2(base + chunk_off(lane & 7, x));
            a[2 * x] = v.x;
            a[2 * x + 1] = v.y;
          }
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            a[k] *= iv[k];
            if (k + 1 < 8) {
              double lt[8];
#pragma unroll
              for (int x = (k + 1) & ~1; x < 8; x += 2) {
                const double2 v = ld2(Lt + 8 * k + x);
                lt[x] = v.x;
                lt[x + 1] = v.y;
              }
#pragma unroll
              for (int j = k + 1; j < 8; ++j) a[j] = fma(-a[k], lt[j], a[j]);
            }
          }
          if (ok) {
#pragma unroll
            for (int x = 0; x < 4; ++x) st2(base + chunk_off(lane & 7, x), a[x], a[x + 4]);
          }
        }
      }
      stamp(c, 3);
      __syncthreads();
      stamp(c, 4);
      if (kLookAhead) {
        column_finish(c + 1, c);
        stamp(c, 5);
        __syncthreads();
      }
    }
    ++iter;
  }
}

// shared memory per CTA: the plain tile triangle, or (slots) the compacted
// slot set
inline size_t smem_bytes(int m, bool gt, int kind = kMaternGen, bool slots = false) {
  if (gt) return sizeof(double) * (size_t)head_doubles(m, kind);
  int tiles = (int)(tile_doubles(m) / 64);
  if (slots) {
    SlotMap map;
    tiles = big_slot_map(ntiles_of(m), &map);
    if (tiles < 0) return (size_t)1 << 40;  // beyond the slot map
  }
  return sizeof(double) * ((size_t)head_doubles(m, kind) + (size_t)tiles * 64);
}
inline int ctas_per_sm(size_t bytes, int cap = 4) {  // by shared memory (228 KB, 1 KB reserved per CTA)
  const size_t per = bytes + 1024;
  const int n = (int)((size_t)233472 / per);
  return n < cap ? n : cap;
}
// the slot layout only where it buys resident CTAs (its lookups cost ~6%)
inline bool use_slots(int m, int kind) {
  // (up to 5 resident CTAs for the closed forms, whose 96-register budget allows 5)
  const int cap = kind <= kMatern25 ? 5 : 4;
  return ctas_per_sm(smem_bytes(m, false, kind, true), cap) > ctas_per_sm(smem_bytes(m, false, kind, false), cap);
}
// tiles in shared memory up to ~200 KB per CTA (compacted when that fits),
// else the global scratch
inline bool use_global_tiles(int m) {
  return smem_bytes(m, false) > 200 * 1024 && smem_bytes(m, false, kMaternGen, true) > 200 * 1024;
}

// TMA descriptor of the plan's points: a 2-D tensor of n rows x 4 doubles
// (x, y, obs, 0), one row per box, for tile::gather4
bool point_map(const double4* pts, int64_t n, CUtensorMap* map);

template <int KIND, bool CACHE, bool GT, int MC = 0, bool SLOTS = false, bool TRACE = false, int MINB = 0>
cudaError_t launch(const Plan& p, const CovParams& cp, int64_t e_lo, int64_t e_hi,
                   cudaStream_t stream, double* gscratch, int max_grid, long long* trace = nullptr) {
  CUtensorMap map;
  if (!point_map(p.d_pts, p.n, &map)) return cudaErrorNotSupported;
  const size_t sm = smem_bytes(p.m, GT, KIND, SLOTS);
  auto kern = loglik_big_kernel<KIND, CACHE, GT, MC, SLOTS, TRACE, MINB>;
  cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (err != cudaSuccess) return err;
  int per_sm = 0;
  err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThreads, sm);
  if (err != cudaSuccess) return err;
  if (per_sm < 1) per_sm = 1;
  const int64_t count = e_hi - e_lo;
  int64_t cap = (int64_t)p.num_sms * per_sm;
  if (GT && cap > max_grid) cap = max_grid;
  const int grid = (int)(count < cap ? count : cap);
  SlotMap smap;
  if (SLOTS) big_slot_map(ntiles_of(p.m), &smap);
  kern<<<grid, kThreads, sm, stream>>>(map, p.d_nbr, p.m, e_lo, e_hi, p.rest_lo, cp,
                                       p.d_rest, p.d_mu, p.d_sig, p.d_fail,
                                       p.d_dcache, p.dcache_stride, gscratch,
                                       (KIND == kMaternGen && !p.no_ktab) ? p.d_ktab : nullptr, smap,
                                       trace);
  return cudaGetLastError();
}

// VGP_TRACE_BIG=<file>: run the launch with the clock64 phase trace and
// append it (diagnostics; tools/big_trace.py)
template <int KIND, bool CACHE, bool GT, int MC, bool SLOTS>
cudaError_t launch_traced(const Plan& p, const CovParams& cp, int64_t e_lo, int64_t e_hi,
                          cudaStream_t stream, double* gscratch, int max_grid, const char* path) {
  const size_t n = (size_t)kTraceCtas * kWarps * 32 * kTraceEv;
  long long* d = nullptr;
  cudaError_t err = cudaMalloc(&d, n * sizeof(long long));
  if (err != cudaSuccess) return err;
  err = cudaMemsetAsync(d, 0, n * sizeof(long long), stream);
  if (err == cudaSuccess) err = launch<KIND, CACHE, GT, MC, SLOTS, true>(p, cp, e_lo, e_hi, stream, gscratch, max_grid, d);
  std::vector<long long> h(n);
  if (err == cudaSuccess) err = cudaMemcpyAsync(h.data(), d, n * sizeof(long long), cudaMemcpyDeviceToHost, stream);
  if (err == cudaSuccess) err = cudaStreamSynchronize(stream);
  cudaFree(d);
  if (err != cudaSuccess) return err;
  if (FILE* f = std::fopen(path, "a")) {
    for (size_t i = 0; i < n; ++i) std::fprintf(f, "%lld%c", h[i], (i + 1) % kTraceEv ? ' ' : '\n');
    std::fclose(f);
  }
  return cudaSuccess;
}

template <int KIND>
cudaError_t launch_kind(const Plan& p, const CovParams& cp, int64_t e_lo, int64_t e_hi,
                        cudaStream_t stream, bool cache, double* gscratch, int max_grid) {
  const bool gt = use_global_tiles(p.m);
  if (gt && !gscratch) return cudaErrorInvalidValue;
  const bool slots = !gt && (use_slots(p.m, KIND) || smem_bytes(p.m, false, KIND) > 200 * 1024);
  if (cache) {
    // config 5 (m = 60, general nu, streamed distances): compile-time m
    if (p.m == 60 && KIND == kMaternGen) return launch<KIND, true, false, 60>(p, cp, e_lo, e_hi, stream, gscratch, max_grid);
    if (gt) return launch<KIND, true, true>(p, cp, e_lo, e_hi, stream, gscratch, max_grid);
    return slots ? launch<KIND, true, false, 0, true>(p, cp, e_lo, e_hi, stream, gscratch, max_grid)
                 : launch<KIND, true, false>(p, cp, e_lo, e_hi, stream, gscratch, max_grid);
  }
  // config 4 (m = 120, closed forms, distances from coordinates): compile-time
  // m, slot layout (4 CTAs per SM instead of 3)
  if (p.m == 120 && KIND <= kMatern25) {
    if (const char* path = std::getenv("VGP_TRACE_BIG"))
      return launch_traced<KIND, false, false, 120, true>(p, cp, e_lo, e_hi, stream, gscratch, max_grid, path);
    return launch<KIND, false, false, 120, true>(p, cp, e_lo, e_hi, stream, gscratch, max_grid);
  }
  if (gt) return launch<KIND, false, true>(p, cp, e_lo, e_hi, stream, gscratch, max_grid);
  if (slots) {
    if constexpr (KIND <= kMatern25) {
      if (ctas_per_sm(smem_bytes(p.m, false, KIND, true), 8) >= 5 && p.tune != 11)
        return launch<KIND, false, false, 0, true, false, 5>(p, cp, e_lo, e_hi, stream, gscratch, max_grid);
    }
    return launch<KIND, false, false, 0, true>(p, cp, e_lo, e_hi, stream, gscratch, max_grid);
  }
  // closed forms whose triangle lets 5 CTAs share the SM: a 5-CTA register
  // budget (96 registers; n = 250k: m = 64 156 -> 170, m = 75 132 -> 144
  // evals/s; at m = 90, 4 CTAs by shared memory, it only spills)
  if constexpr (KIND <= kMatern25) {
    if (ctas_per_sm(smem_bytes(p.m, false, KIND), 8) >= 5 && p.tune != 11)
      return launch<KIND, false, false, 0, false, false, 5>(p, cp, e_lo, e_hi, stream, gscratch, max_grid);
  }
  return launch<KIND, false, false>(p, cp, e_lo, e_hi, stream, gscratch, max_grid);
}

}  // namespace big
}  // namespace vgp
