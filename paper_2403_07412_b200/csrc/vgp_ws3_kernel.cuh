// Warp-specialised FP64 tensor-core (DMMA) Vecchia kernel laid out for the
// SM's four schedulers (sub-partitions), m + 2 <= 64: the default fast path.
//
// Each conditioning block e >= 1 (vg/vecchia.py:154-162 assemble, :180-190
// _numeric_stage, :193-214 _reduction_stage) is factored left-looking over
// 8-wide tile columns by two warps sharing its augmented (8 NT)^2 matrix in
// shared memory (as in vgp_ws_kernel.cuh):
//
//   worker warp  covariance generation (lean FP64 Matern) and every trailing
//                update, mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4), then hands the
//                tile column over (bar.arrive);
//   chain warp   factors the column's panel (row-owner layout: the pivot
//                chain of rsqrt / shuffle steps), writes L back; at the last
//                column it reads sigma_new, -mu off the Schur complement and
//                writes the block's log-density.
//
// Why this layout (measured, profiles/r01_contention.jsonl): a warp issuing a
// stream of DMMAs holds its scheduler's FP64 pipe; one such warp doubles the
// latency of a dependent DFMA chain on the same scheduler, two or more starve
// it (8 -> 260..30000 cycles), while DMMAs on OTHER schedulers cost nothing.
// The pivot chain is the block's critical path, so each scheduler runs
// exactly ONE worker warp, and that worker serves the two blocks whose chain
// warps sit on the same scheduler (warp w -> scheduler w % 4):
//
//   CTA = 12 warps, 1 per SM: warps 0..3 workers (slots w, w + 4),
//   warps 4..11 chains (slot w - 4, scheduler w % 4 = its worker's).
//
// The worker alternates between its two blocks column by column, so while
// one block's chain factors panel c the worker prepares the other block's
// column.  8 blocks in flight per SM (8 x 20.8 KB of shared memory).
//
// C0 (default for the cached closed forms at NT = 8): the chain generates its
// block's tile column 0 itself, straight into its row-owner registers, right
// after the previous block's epilogue; the worker starts every block at
// column 1.  A clock64 trace showed the chains idle ~2.8k cycles per block
// waiting for column 0 while the worker (never idle) finished the other
// slot's last column and generated 8 tiles: 115.5 -> 123.1 evals/s (c2),
// bit-identical.
//
// Shared memory per block: the tile triangle (tile (I, J) at
// (J NT - J (J-1)/2 + I - J) * 64 doubles, column-major, ws::chunk_off swizzle: conflict-free fragment
// and row accesses), staging S for the last panel (the tile triangle is then
// refilled with the next block's distances by one cp.async.bulk + mbarrier),
// the yJ row, coordinates (uncached variant) and the target observation.
#pragma once

#include "vgp_ktab.cuh"
#include "vgp_ws_kernel.cuh"

namespace vgp {
namespace ws3 {

using dmma::bulk_load;
using dmma::mbar_init;
using dmma::mbar_wait;
using dmma::neg;
using dmma::shfl;
using ll::cov_lean;
using ll::ld2;
using ll::mma;
using ll::rsqrt_chain;
using ll::st2;
using ws::bar_arrive;
using ws::bar_sync;
using ws::chunk_off;
using ws::ntri;
using ws::tidx;

constexpr int kSlots = 8;    // blocks in flight per CTA (= per SM)
constexpr int kWorkers = 4;  // one per scheduler
constexpr int kThreads = 32 * (kWorkers + kSlots);
constexpr int kHead = 256;   // sigma^2-scaled exp table
constexpr int kTraceBlocks = ws::kTraceBlocks;
constexpr int kTraceEvents = ws::kTraceEvents;

// covariance at distance d: lean closed forms, or the general-nu Matern from
// the per-evaluation polynomial table (vgp_ktab.cuh)
template <int KIND>
__device__ __forceinline__ double cov_gen(double d, double inv_beta, const double* tab,
                                          const double* __restrict__ ktab, const CovParams& cp,
                                          const double* ktw = nullptr, int wseg0 = 0) {
  if constexpr (KIND != kMaternGen) return cov_lean<KIND>(d, inv_beta, tab);
  return cov_ktab(d * inv_beta, ktab, cp, ktw, wseg0);
}
// the K_nu table window in shared memory (general nu, NT = 8: the smem left
// beside the eight slots holds 14 binades)
template <int KIND, int NT>
constexpr bool kTabWindow = KIND == kMaternGen && NT == 8;

struct SlotLayout {
  int tiles;   // doubles of the tile triangle (= cache stride)
  int stride;  // tiles | S (2 tiles) | O (P) | XY (2P) | yt (2) | mbarrier (2) | Lc (2 x 8) | gen mbarriers (2)
};
__host__ __device__ constexpr SlotLayout slot_layout(int nt) {
  return SlotLayout{ntri(nt) * 64, ntri(nt) * 64 + 128 + 8 * nt + 16 * nt + 2 + 2 + 16 + 2};
}

// CG: the chain warps generate half of the covariance tiles (in place over
// the cached distances, one column ahead, in the time they otherwise wait for
// their worker); the workers generate the other half and load these.
// CGK = 2: every other tile of a column; CGK = k > 2: all but every k-th tile
template <int CGK = 2>
__host__ __device__ constexpr bool chain_tile(int I, int c) {
  return CGK == 2 ? ((I - c) & 1) == 0 : (I - c) % CGK != CGK - 1;
}
template <int NT, int KIND, int MC, bool CACHE, bool TRACE = false, bool CG = false, bool C0 = false,
          int CGK = 2>
__global__ void __launch_bounds__(kThreads, 1)
loglik_ws3_kernel(const double4* __restrict__ pts, const int32_t* __restrict__ nbr, int m_rt,
                  int64_t e_lo, int64_t e_hi, int64_t rest_lo, double s2, double inv_beta,
                  double* __restrict__ rest, double* __restrict__ mu_out,
                  double* __restrict__ sig_out, unsigned long long* __restrict__ fail,
                  const double* __restrict__ dcache, int64_t cstride,
                  const double* __restrict__ ktab, const CovParams cpx, int wseg0,
                  long long* __restrict__ trace = nullptr) {
  constexpr int P = 8 * NT;
  const int m = MC > 0 ? MC : m_rt;
  const int NC = (m + 8) >> 3;  // tile columns holding pivots or the Schur column
  constexpr SlotLayout L = slot_layout(NT);
  extern __shared__ __align__(16) double smem[];
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const bool chain = warp >= kWorkers;
  auto Tb = [&](int s) { return smem + kHead + s * L.stride; };
  auto Sb = [&](int s) { return Tb(s) + L.tiles; };
  auto Ob = [&](int s) { return Sb(s) + 128; };
  auto XYb = [&](int s) { return reinterpret_cast<double2*>(Ob(s) + P); };
  auto Yb = [&](int s) { return Ob(s) + 3 * P; };  // [parity] target observation
  auto MBb = [&](int s) { return reinterpret_cast<uint64_t*>(Ob(s) + 3 * P + 2); };
  auto Lcb = [&](int s) { return Ob(s) + 3 * P + 4; };  // [pivot parity][8] column of L_cc
  auto GBb = [&](int s) { return reinterpret_cast<uint64_t*>(Ob(s) + 3 * P + 20); };  // CG: [2] column generated
  // named barriers (ids 0..15; id 0 is free again after the setup __syncthreads):
  // 2s = tile column staged (worker -> chain), 2s + 1 = L written (chain -> worker)

  for (int i = threadIdx.x; i < 256; i += blockDim.x) smem[i] = s2 * kExp2Table[i];
  double* ktw = nullptr;
  if constexpr (kTabWindow<KIND, NT>) {
    if (wseg0 >= 0) {
      ktw = smem + kHead + kSlots * L.stride;
      const double2* src = reinterpret_cast<const double2*>(ktab + (size_t)wseg0 * 8);
      const int nwin = min(kKtabWinSeg, kKtabSegments - wseg0) * 4;  // double2 per segment: 4
      for (int i = threadIdx.x; i < nwin; i += blockDim.x) reinterpret_cast<double2*>(ktw)[i] = __ldg(src + i);
    }
  }
  if (CACHE && warp < kSlots && lane == 0) mbar_init(MBb(warp));
  if (CG && warp < kSlots && lane < 2) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 32;" ::"r"(dmma::smem_u32(GBb(warp) + lane)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const double* tab = smem;

  const int64_t stride = (int64_t)gridDim.x * kSlots;
  const int64_t e0 = e_lo + (int64_t)blockIdx.x * kSlots;
  const int r = lane >> 2;  // fragment row
  const int q = lane & 3;   // fragment column pair
  int tblk = 0;
  auto mark = [&](int slot, int role, int ev) {
    if (TRACE && blockIdx.x == 0 && lane == 0 && tblk < kTraceBlocks && ev < kTraceEvents)
      trace[((slot * 2 + role) * kTraceBlocks + tblk) * kTraceEvents + ev] = clock64();
  };

  if (!chain) {
    // ============================ worker warp ============================
    const int sl[2] = {warp, warp + kWorkers};
    const uint32_t cbytes = (uint32_t)(cstride * sizeof(double));
    uint32_t phase[2] = {0, 0};
    auto slot_index = [&](int64_t eb, int a) -> int {
      if (a < m) return nbr[(eb - 1 - rest_lo) * (int64_t)m + a];
      return a == m ? (int)(m + eb - 1) : -1;
    };
    auto slot_point = [&](int idx) -> double4 {
      return idx >= 0 ? pts[idx] : make_double4(0.0, 0.0, 0.0, 0.0);
    };
    double4 pf0[2], pf1[2];
    int ni0[2] = {-1, -1}, ni1[2] = {-1, -1};
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      pf0[h] = make_double4(0.0, 0.0, 0.0, 0.0);
      pf1[h] = pf0[h];
      const int64_t e = e0 + sl[h];
      if (e < e_hi) {
        if (!CG && !C0 && CACHE && lane == 0)
          bulk_load(Tb(sl[h]), dcache + (e - 1 - rest_lo) * cstride, cbytes, MBb(sl[h]));
        pf0[h] = slot_point(slot_index(e, lane));
        if (P > 32) pf1[h] = slot_point(slot_index(e, lane + 32));
        if (CG || C0) {
          // the chain generates from O: stage it, then the distances (the
          // mbarrier's release by lane 0 after __syncwarp covers both)
          double* O = Ob(sl[h]);
          if (lane < P) O[lane] = lane < m ? pf0[h].z : 0.0;
          if (P > 32 && lane + 32 < P) O[lane + 32] = lane + 32 < m ? pf1[h].z : 0.0;
          __syncwarp();
          if (lane == 0) bulk_load(Tb(sl[h]), dcache + (e - 1 - rest_lo) * cstride, cbytes, MBb(sl[h]));
        }
      }
    }
    int par = 0;
    bool first = true;
    uint32_t gcnt[2] = {0, 0};  // CG: generated columns consumed per slot
    for (int64_t base = e0; base + sl[0] < e_hi; base += stride, par ^= 1, first = false, ++tblk) {
      bool act[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int s = sl[h];
        const int64_t e = base + s, en = e + stride;
        act[h] = e < e_hi;
        if (!act[h]) continue;
        mark(s, 1, 0);
        double* O = Ob(s);
        double2* XY = XYb(s);
        if (!CG && !C0) {
          if (lane < P) O[lane] = lane < m ? pf0[h].z : 0.0;
          if (P > 32 && lane + 32 < P) O[lane + 32] = lane + 32 < m ? pf1[h].z : 0.0;
        }
        if (!CACHE) {
          if (lane < P) XY[lane] = make_double2(pf0[h].x, pf0[h].y);
          if (P > 32 && lane + 32 < P) XY[lane + 32] = make_double2(pf1[h].x, pf1[h].y);
        }
        const double yt = shfl((m < 32) ? pf0[h].z : pf1[h].z, m & 31);
        if (lane == 0) Yb(s)[par] = yt;
        ni0[h] = ni1[h] = -1;
        if (en < e_hi) {  // next block's neighbour indices now, its points one column later
          ni0[h] = slot_index(en, lane);
          if (P > 32) ni1[h] = slot_index(en, lane + 32);
        }
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        if (!CG && CACHE && act[h]) {
          mbar_wait(MBb(sl[h]), phase[h]);
          phase[h] ^= 1;
        }
      }
      __syncwarp();

#pragma unroll
      for (int c = C0 ? 1 : 0; c < NT; ++c) {
        if (c < NC) {
          const bool lastc = (c == NC - 1);
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            if (!act[h]) continue;
            const int s = sl[h];
            const int64_t en = base + s + stride;
            double* T = Tb(s);
            if (c == (NC > 1 ? 1 : 0) && en < e_hi) {
              if (CACHE) {
                pf0[h].z = ni0[h] >= 0 ? pts[ni0[h]].z : 0.0;
                if (P > 32) pf1[h].z = ni1[h] >= 0 ? pts[ni1[h]].z : 0.0;
              } else {
                pf0[h] = slot_point(ni0[h]);
                if (P > 32) pf1[h] = slot_point(ni1[h]);
              }
            }
            // ---- generate tile column c: entries (8I + r, 8c + 2q + h)
            double acc[NT][2];
            if (CG) {
              // generated by the chain (column c of this slot's block)
              mbar_wait(GBb(s) + (gcnt[h] & 1), (gcnt[h] >> 1) & 1);
              ++gcnt[h];
#pragma unroll
              for (int I = 0; I < NT; ++I) {
                if (I >= c && chain_tile<CGK>(I, c)) {
                  const double2 v = ld2(T + tidx(I, c, NT) * 64 + chunk_off(r, q));
                  acc[I][0] = v.x;
                  acc[I][1] = v.y;
                }
              }
            }
#pragma unroll
            for (int I = 0; I < NT; ++I) {
              if (I >= c && !(CG && chain_tile<CGK>(I, c))) {
                const int i = 8 * I + r;
                double v0, v1;
                if (CACHE) {
                  const double2 dv = ld2(T + tidx(I, c, NT) * 64 + chunk_off(r, q));
                  v0 = cov_gen<KIND>(dv.x, inv_beta, tab, ktab, cpx, ktw, wseg0);
                  v1 = cov_gen<KIND>(dv.y, inv_beta, tab, ktab, cpx, ktw, wseg0);
                } else {
                  const double2* XY = XYb(s);
                  const double2 pa = XY[i];
                  const double4 pb = *reinterpret_cast<const double4*>(XY + 8 * c + 2 * q);
                  double dx = pa.x - pb.x, dy = pa.y - pb.y;
                  v0 = cov_gen<KIND>(sqrt_pos_nz(fma(dx, dx, fma(dy, dy, 0x1p-1000))), inv_beta, tab, ktab, cpx);
                  dx = pa.x - pb.z;
                  dy = pa.y - pb.w;
                  v1 = cov_gen<KIND>(sqrt_pos_nz(fma(dx, dx, fma(dy, dy, 0x1p-1000))), inv_beta, tab, ktab, cpx);
                }
                if (I == NT - 1 && i > m) {  // row m+1: yJ (0 from column m on); padding: 0
                  const double2 ov = ld2(Ob(s) + 8 * c + 2 * q);
                  v0 = i == m + 1 ? ov.x : 0.0;
                  v1 = i == m + 1 ? ov.y : 0.0;
                }
                acc[I][0] = v0;
                acc[I][1] = v1;
              }
            }
            // ---- left-looking update with L of tile columns k < c
            auto update = [&](const int k) {
              const double2 b = ld2(T + tidx(c, k, NT) * 64 + chunk_off(r, q));
              double2 a[NT];
#pragma unroll
              for (int I = 0; I < NT; ++I)
                if (I > c) a[I] = ld2(T + tidx(I, k, NT) * 64 + chunk_off(r, q));
              a[c] = b;
              if (k == c - 1) mark(s, 1, 3 + 2 * c);
#pragma unroll
              for (int kk = 0; kk < 2; ++kk) {
#pragma unroll
                for (int I = 0; I < NT; ++I)
                  if (I >= c)
                    mma(acc[I][0], acc[I][1], neg(kk ? a[I].y : a[I].x), kk ? b.y : b.x);
              }
            };
#pragma unroll
            for (int k = 0; k + 1 < c; ++k) update(k);
            if (c >= 1) {
              mark(s, 1, 2 + 2 * c);
              bar_sync(2 * s + 1, 64);  // L of column c - 1 is in T
              update(c - 1);
            }
            if (lastc) {
              // T is no longer read for this block (the last panel runs from
              // S): stream in the next block's distances (CG: and its
              // observations, which the chain generates from)
              if ((CG || C0) && en < e_hi) {
                double* O = Ob(s);
                if (lane < P) O[lane] = lane < m ? pf0[h].z : 0.0;
                if (P > 32 && lane + 32 < P) O[lane + 32] = lane + 32 < m ? pf1[h].z : 0.0;
              }
              __syncwarp();
              if (CACHE && lane == 0 && en < e_hi)
                bulk_load(T, dcache + (en - 1 - rest_lo) * cstride, cbytes, MBb(s));
            }
            // ---- hand column c over (natural column order); before a block's
            // first column, wait until the chain has taken the previous
            // block's last column (one arrival in flight per barrier; S reuse)
            if (!C0 && c == 0 && !first) bar_sync(2 * s + 1, 64);
#pragma unroll
            for (int I = 0; I < NT; ++I) {
              if (I >= c) {
                double* dst = lastc ? Sb(s) + (I - c) * 64 : T + tidx(I, c, NT) * 64;
                st2(dst + chunk_off(r, q), acc[I][0], acc[I][1]);
              }
            }
            bar_arrive(2 * s, 64);
          }
        }
      }
    }
  } else {
    // ============================ chain warp ============================
    const int s = warp - kWorkers;
    double* T = Tb(s);
    double* S = Sb(s);
    int par = 0;
    uint32_t dph = 0, gcnt = 0;
    // CG: generate tile column c in place over the cached distances and
    // hand it to the worker
    auto gen_col = [&](const int c) {
#pragma unroll
      for (int I = 0; I < NT; ++I) {
        if (I >= c && chain_tile<CGK>(I, c)) {
          const int i = 8 * I + r;
          double* tp = T + tidx(I, c, NT) * 64 + chunk_off(r, q);
          const double2 dv = ld2(tp);
          double v0 = cov_gen<KIND>(dv.x, inv_beta, tab, ktab, cpx, ktw, wseg0);
          double v1 = cov_gen<KIND>(dv.y, inv_beta, tab, ktab, cpx, ktw, wseg0);
          if (I == NT - 1 && i > m) {  // row m+1: yJ (0 from column m on); padding: 0
            const double2 ov = ld2(Ob(s) + 8 * c + 2 * q);
            v0 = i == m + 1 ? ov.x : 0.0;
            v1 = i == m + 1 ? ov.y : 0.0;
          }
          st2(tp, v0, v1);
        }
      }
      asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(dmma::smem_u32(GBb(s) + (gcnt & 1)))
                   : "memory");
      ++gcnt;
    };
    for (int64_t e = e0 + s; e < e_hi; e += stride, par ^= 1, ++tblk) {
      int fj = -1;  // first non-positive pivot column
      if (CG || C0) {
        mbar_wait(MBb(s), dph);  // this block's distances and observations
        dph ^= 1;
      }
      if (CG) {
        gen_col(0);
        if (NC > 1) gen_col(1);
      }
#pragma unroll
      for (int c = 0; c < NT; ++c) {
        if (c < NC) {
          const bool lastc = (c == NC - 1);
          const int R0 = 8 * c;
          const int NR = P - R0;
          const int jmax = min(8, m - R0);  // pivots in this tile column
          mark(s, 0, 2 * c);
          if (!(C0 && c == 0)) bar_sync(2 * s, 64);
          // lane owns panel rows R0 + lane + 32 rr: tile c + (lane + 32 rr) / 8, row lane & 7
          constexpr int kMaxRows = 2;
          double a[kMaxRows][8];
          auto row_ptr = [&](int rr) -> double* {
            const int I = c + ((lane + 32 * rr) >> 3);
            return lastc ? S + (I - c) * 64 : T + tidx(I < NT ? I : NT - 1, c, NT) * 64;
          };
          if (C0 && c == 0) {
            // C0: the chain generates tile column 0 itself, straight into its
            // row-owner registers from the cached distances (the worker starts
            // each block at column 1; column 0's distances are never read again
            // and the tiles take L(., 0) as usual)
#pragma unroll
            for (int rr = 0; rr < kMaxRows; ++rr) {
              const int row = lane + 32 * rr;
              const int I = row >> 3;
              const double* tp = T + tidx(I, 0, NT) * 64;
#pragma unroll
              for (int x = 0; x < 4; ++x) {
                const double2 dv = ld2(tp + chunk_off(lane & 7, x));
                double v0 = cov_gen<KIND>(dv.x, inv_beta, tab, ktab, cpx, ktw, wseg0);
                double v1 = cov_gen<KIND>(dv.y, inv_beta, tab, ktab, cpx, ktw, wseg0);
                if (I == NT - 1 && row > m) {  // row m+1: yJ; padding: 0
                  const double2 ov = ld2(Ob(s) + 2 * x);
                  v0 = row == m + 1 ? ov.x : 0.0;
                  v1 = row == m + 1 ? ov.y : 0.0;
                }
                a[rr][2 * x] = v0;
                a[rr][2 * x + 1] = v1;
              }
            }
          } else {
#pragma unroll
          for (int rr = 0; rr < kMaxRows; ++rr) {
            if (rr * 32 < NR) {
              const bool ok = lane + 32 * rr < NR;
              const double* rb = row_ptr(rr);
#pragma unroll
              for (int x = 0; x < 4; ++x) {
                double2 v = make_double2(0.0, 0.0);
                if (ok) v = ld2(rb + chunk_off(lane & 7, x));
                a[rr][2 * x] = v.x;
                a[rr][2 * x + 1] = v.y;
              }
            }
          }
          }
          mark(s, 0, 2 * c + 1);
          // last column: rows are in registers, S may be refilled
          if (!C0 && lastc && e + stride < e_hi) bar_arrive(2 * s + 1, 64);
          double lastpiv = 1.0;
          if (jmax > 0) {
            double piv = shfl(a[0][0], 0);
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              if (j < jmax) {
                if (j == jmax - 1) lastpiv = piv;
                const double inv = rsqrt_chain(piv);
#pragma unroll
                for (int rr = 0; rr < kMaxRows; ++rr)
                  if (rr * 32 < NR) a[rr][j] *= inv;
                if (j + 1 < 8) {
                  const double nxt = fma(-a[0][j], a[0][j], a[0][j + 1]);
                  piv = shfl(nxt, j + 1);
                }
                // column j of L_cc to every lane: the diagonal-tile lanes store
                // it, every lane reads it back with broadcast LDS.128 (4
                // instructions instead of 14 32-bit shuffles; double-buffered
                // by pivot parity, so one __syncwarp per pivot orders both
                // the reads after the store and the next-but-one overwrite)
                double* Lc = Lcb(s) + 8 * (j & 1);
                if (lane < 8) Lc[lane] = a[0][j];
                __syncwarp();
                double lcv[8];
#pragma unroll
                for (int x = (j + 1) & ~1; x < 8; x += 2) {
                  const double2 v = ld2(Lc + x);
                  lcv[x] = v.x;
                  lcv[x + 1] = v.y;
                }
#pragma unroll
                for (int jp = j + 1; jp < 8; ++jp) {
#pragma unroll
                  for (int rr = 0; rr < kMaxRows; ++rr)
                    if (rr * 32 < NR) a[rr][jp] = fma(-a[rr][j], lcv[jp], a[rr][jp]);
                }
              }
            }
          }
          // pivot test !(piv > 0) (vg/batchla.py:146-151): a non-positive or
          // NaN pivot turns every later pivot NaN, so testing the panel's
          // last pivot detects it; the rare failing panel then locates the
          // first bad column from the diagonal of L
          if (!(lastpiv > 0.0) && fj < 0) {
            double ljj = a[0][0];
#pragma unroll
            for (int x = 1; x < 8; ++x)
              if (lane == x) ljj = a[0][x];
            const unsigned bad = __ballot_sync(0xffffffffu, lane < jmax && !(ljj > 0.0));
            fj = R0 + (bad ? __ffs(bad) - 1 : jmax - 1);
          }
          if (!lastc) {
            // L rows below the diagonal tile, columns (x, x + 4) per chunk
#pragma unroll
            for (int rr = 0; rr < kMaxRows; ++rr) {
              if (rr * 32 < NR && lane + 32 * rr >= 8 && lane + 32 * rr < NR) {
                double* rb = row_ptr(rr);
#pragma unroll
                for (int x = 0; x < 4; ++x)
                  st2(rb + chunk_off(lane & 7, x), a[rr][x], a[rr][x + 4]);
              }
            }
            bar_arrive(2 * s + 1, 64);
            if (CG && c + 2 < NC) gen_col(c + 2);
          } else {
            // sigma_new = A[m][m], -mu = A[m+1][m] after m pivots (vg/vecchia.py:186-189, :206)
            const int cs = m - R0;
            double v = a[0][0];
#pragma unroll
            for (int x = 1; x < 8; ++x)
              if (x == cs) v = a[0][x];
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
                  const double resid = Yb(s)[par] - mu;
                  rest[kk] = -0.5 * (resid * resid / sg + kLog2Pi + log(sg));
                }
              }
            }
            mark(s, 0, 20);
          }
        }
      }
    }
  }
}

template <int NT, int KIND, int MC, bool CACHE, bool TRACE = false, bool CG = false, bool C0 = false,
          int CGK = 2>
cudaError_t launch(const Plan& p, const CovParams& cp, int64_t e_lo, int64_t e_hi,
                   cudaStream_t stream, long long* trace = nullptr) {
  constexpr SlotLayout L = slot_layout(NT);
  const int wseg0 = kTabWindow<KIND, NT> ? ktab_window(p.dcache_dmax, cp.inv_beta) : -(1 << 30);
  const size_t sm = sizeof(double) * ((size_t)kHead + (size_t)kSlots * L.stride +
                                      (kTabWindow<KIND, NT> ? (size_t)kKtabWinSeg * 8 : 0));
  static size_t configured[64] = {};
  const int dev = p.device & 63;
  auto kern = loglik_ws3_kernel<NT, KIND, MC, CACHE, TRACE, CG, C0, CGK>;
  if (configured[dev] < sm) {
    cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (err != cudaSuccess) return err;
    configured[dev] = sm;
  }
  const int64_t count = e_hi - e_lo;
  const int64_t want = (count + kSlots - 1) / kSlots;
  const int64_t cap = (int64_t)p.num_sms;  // one CTA per SM: the role layout assumes it
  const int grid = (int)(want < cap ? want : cap);
  kern<<<grid, kThreads, sm, stream>>>(p.d_pts, p.d_nbr, p.m, e_lo, e_hi, p.rest_lo, cp.s2,
                                       cp.inv_beta, p.d_rest, p.d_mu, p.d_sig, p.d_fail,
                                       p.d_dcache, p.dcache_stride, p.d_ktab, cp,
                                       wseg0 >= 0 ? wseg0 : -1, trace);
  return cudaGetLastError();
}

template <int KIND>
cudaError_t launch_traced(const Plan& p, const CovParams& cp, int64_t e_lo, int64_t e_hi,
                                 cudaStream_t stream, const char* path) {
  const size_t n = (size_t)kSlots * 2 * kTraceBlocks * kTraceEvents;
  long long* d = nullptr;
  cudaError_t err = cudaMalloc(&d, n * sizeof(long long));
  if (err != cudaSuccess) return err;
  cudaMemsetAsync(d, 0, n * sizeof(long long), stream);
  if constexpr (KIND == kMaternGen)
    err = launch<8, KIND, 60, true, true, true, false, 3>(p, cp, e_lo, e_hi, stream, d);
  else
    err = p.tune == 1 ? launch<8, KIND, 60, true, true>(p, cp, e_lo, e_hi, stream, d)
                      : launch<8, KIND, 60, true, true, false, true>(p, cp, e_lo, e_hi, stream, d);
  std::vector<long long> h(n);
  if (err == cudaSuccess) err = cudaMemcpyAsync(h.data(), d, n * sizeof(long long), cudaMemcpyDeviceToHost, stream);
  if (err == cudaSuccess) err = cudaStreamSynchronize(stream);
  cudaFree(d);
  if (err != cudaSuccess) return err;
  if (FILE* f = std::fopen(path, "a")) {
    for (size_t i = 0; i < n; ++i) std::fprintf(f, "%lld%c", h[i], (i + 1) % kTraceEvents ? ' ' : '\n');
    std::fclose(f);
  }
  return cudaSuccess;
}

template <int NT, int KIND, int MC>
cudaError_t launch_c(const Plan& p, const CovParams& cp, int64_t e_lo, int64_t e_hi,
                     cudaStream_t stream, bool cache) {
  if constexpr (NT == 8 && (KIND == kMatern15 || KIND == kMaternGen) && MC == 60) {
    if (cache) {
      if (const char* path = std::getenv("VGP_TRACE3")) return launch_traced<KIND>(p, cp, e_lo, e_hi, stream, path);
    }
  }
  // general nu: covariance generation (the K_nu table) is the expensive part,
  // so the chains generate in their idle time (c5: 12.2 -> 15.4 evals/s); for
  // the closed forms it only lengthens the chains (c2: 115.8 -> 106.2)
  // (the chains take 2 of every 3 tiles: they wait ~2.4k cycles per column
  // while the worker never does -- c5 18.64 -> 18.9 evals/s against every
  // other tile; 3 of 4: 18.65)
  if constexpr (KIND == kMaternGen) {
    if (cache && p.tune != 7) return launch<NT, KIND, MC, true, false, true, false, 3>(p, cp, e_lo, e_hi, stream);
  }
  if (cache && (KIND == kMaternGen || p.tune == 2))
    return launch<NT, KIND, MC, true, false, true>(p, cp, e_lo, e_hi, stream);
  // closed forms, NT = 8 (m = 55..62, so at least two tile columns): the chain
  // generates tile column 0 itself (C0; VGP_TUNE=1 selects the previous layout)
  if constexpr (NT == 8 && KIND != kMaternGen) {
    if (cache && p.tune != 1) return launch<NT, KIND, MC, true, false, false, true>(p, cp, e_lo, e_hi, stream);
  }
  if (cache) return launch<NT, KIND, MC, true>(p, cp, e_lo, e_hi, stream);
  return launch<NT, KIND, MC, false>(p, cp, e_lo, e_hi, stream);
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

}  // namespace ws3
}  // namespace vgp
