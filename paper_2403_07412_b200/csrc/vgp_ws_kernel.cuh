// Warp-specialised FP64 tensor-core (DMMA) Vecchia kernel, m + 2 <= 64 (the
// default fast path).
//
// Each conditioning block e >= 1 (vg/vecchia.py:154-162 assemble, :180-190
// _numeric_stage, :193-214 _reduction_stage) is owned by a PAIR of warps that
// share its augmented (8 NT)^2 matrix (rows 0..m-1 Sigma_e, row m v_e, row
// m+1 yJ, zero padding) in shared memory and factor it tile column by tile
// column (8 wide), left-looking:
//
//   worker warp  generates tile column c from the distances (lean FP64
//                Matern), applies every earlier tile column's L with
//                mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4), and hands the column
//                over (bar.arrive);
//   chain warp   factors the column's panel (row-owner layout: one pivot
//                chain of rsqrt / shuffle steps), writes L back and hands it
//                over (bar.arrive); at the last column it reads sigma_new and
//                -mu off the Schur complement and writes the block's
//                log-density.
//
// The chain of pivot steps (SHFL 24 + MUFU 17 + 6 dependent FP64 ops x 8
// cycles per pivot, measured, profiles/r01_latency.jsonl) is the block's
// critical path; the worker's covariance generation and DMMA updates of the
// next column run underneath it instead of after it.
//
// Shared memory per pair: the lower tile triangle, tile (I, J) at
// (J NT - J (J-1)/2 + I - J) * 64 doubles, column-major; row r of a tile is 4 16-byte chunks, chunk x
// stored at position x ^ ((r >> 1) & 3), so both the DMMA fragment accesses
// (lane (r, q) -> chunk q of row r) and the panel's row accesses (lane -> one
// row, all chunks) are bank-conflict free.  A tile holds, in turn, the
// distances (natural column order), the updated covariance handed to the
// chain (natural order) and L (columns q, q + 4 in chunk q: the two k = 4
// slices of a DMMA operand in one LDS.128).  With the plan-time distance
// cache (vgp_dcache.cu writes exactly this layout) the worker streams the
// next block's tiles in with one cp.async.bulk (SASS UBLKCP) + mbarrier as
// soon as the current block's last column has been handed over; the last
// panel runs from a side staging area.
#pragma once

#include <cstdio>
#include <cstdlib>
#include <vector>

#include "vgp_ll_kernel.cuh"

namespace vgp {
namespace ws {

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

constexpr int kPairs = 4;              // blocks in flight per CTA
constexpr int kThreads = 64 * kPairs;  // warps 0..kPairs-1 chain, kPairs..2kPairs-1 worker
constexpr int kHead = 256;             // sigma^2-scaled exp table

// tiles of the lower tile triangle, column-major: tile column J is a
// contiguous run of nt - J tiles (column 0 first, so a block's first
// column can be streamed ahead of the rest)
__host__ __device__ constexpr int ntri(int nt) { return nt * (nt + 1) / 2; }
__host__ __device__ constexpr int tidx(int I, int J, int nt) { return J * nt - J * (J - 1) / 2 + (I - J); }
// doubles offset of 16-byte chunk x (columns 2x, 2x+1 or x, x+4) of row r in a tile
__host__ __device__ constexpr int chunk_off(int r, int x) { return 8 * r + 2 * (x ^ ((r >> 1) & 3)); }

struct PairLayout {
  int tiles;   // doubles of the tile triangle (= cache stride)
  int stride;  // doubles per pair: tiles | S (2 tiles) | O (P) | XY (2P) | yt (4) | mbarrier (2)
};
__host__ __device__ constexpr PairLayout pair_layout(int nt) {
  return PairLayout{ntri(nt) * 64, ntri(nt) * 64 + 128 + 8 * nt + 16 * nt + 4 + 2 + 16};
}

__device__ __forceinline__ void bar_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void bar_arrive(int id, int n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// TRACE (profiling builds only): per-pair clock64 timeline of the first
// kTraceBlocks blocks of CTA 0 -> trace[pair][role][block][event]
constexpr int kTraceBlocks = 8;
constexpr int kTraceEvents = 24;

// SPLIT (experiment): CTA of 16 warps; chain of pair p = warp 4p (scheduler 0,
// away from DMMA traffic), worker = warp 1, 2, 3, 5; the other warps exit.
template <int NT, int KIND, int MC, bool CACHE, bool TRACE = false, bool SPLIT = false>
__global__ void __launch_bounds__(SPLIT ? 512 : kThreads, SPLIT ? 1 : 2)
loglik_ws_kernel(const double4* __restrict__ pts, const int32_t* __restrict__ nbr, int m_rt,
                 int64_t e_lo, int64_t e_hi, int64_t rest_lo, double s2, double inv_beta,
                 double* __restrict__ rest, double* __restrict__ mu_out,
                 double* __restrict__ sig_out, unsigned long long* __restrict__ fail,
                 const double* __restrict__ dcache, int64_t cstride,
                 long long* __restrict__ trace = nullptr, int active = kPairs) {
  constexpr int P = 8 * NT;
  const int m = MC > 0 ? MC : m_rt;
  const int NC = (m + 8) >> 3;  // tile columns holding pivots or the Schur column
  constexpr PairLayout L = pair_layout(NT);
  extern __shared__ __align__(16) double smem[];
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  bool chain = warp < kPairs;
  int pr = chain ? warp : warp - kPairs;
  if (SPLIT) {
    chain = (warp & 3) == 0;
    pr = chain ? warp >> 2 : (warp <= 3 ? warp - 1 : (warp == 5 ? 3 : -1));
  }
  double* T = smem + kHead + pr * L.stride;  // tile triangle
  double* S = T + L.tiles;                   // last-panel staging (2 tiles)
  double* O = S + 128;                       // yJ row (row m+1)
  double2* XY = reinterpret_cast<double2*>(O + P);
  double* misc = O + 3 * P;  // [0] sigma_new, [1] -mu, [2 + parity] target obs
  uint64_t* mbar = reinterpret_cast<uint64_t*>(misc + 4);
  double* Lcb = misc + 6;  // [pivot parity][8] column of L_cc (chain broadcast)
  const int cbar = 1 + 2 * pr;  // column c staged (worker -> chain)
  const int lbar = 2 + 2 * pr;  // L of column c written (chain -> worker)

  for (int i = threadIdx.x; i < 256; i += blockDim.x) smem[i] = s2 * kExp2Table[i];
  if (CACHE && !chain && pr >= 0 && lane == 0) mbar_init(mbar);
  __syncthreads();
  if (pr < 0 || pr >= active) return;
  const double* tab = smem;

  const int64_t stride = (int64_t)gridDim.x * active;
  int64_t e = e_lo + (int64_t)blockIdx.x * active + pr;
  const int r = lane >> 2;  // fragment row
  const int q = lane & 3;   // fragment column pair
  int tblk = 0;
  auto mark = [&](int ev) {
    if (TRACE && blockIdx.x == 0 && lane == 0 && tblk < kTraceBlocks && ev < kTraceEvents)
      trace[((pr * 2 + (chain ? 0 : 1)) * kTraceBlocks + tblk) * kTraceEvents + ev] = clock64();
  };

  if (!chain) {
    // ============================ worker warp ============================
    const uint32_t cbytes = (uint32_t)(cstride * sizeof(double));
    uint32_t phase = 0;
    auto slot_index = [&](int64_t eb, int a) -> int {
      if (a < m) return nbr[(eb - 1 - rest_lo) * (int64_t)m + a];
      return a == m ? (int)(m + eb - 1) : -1;
    };
    auto slot_point = [&](int idx) -> double4 {
      return idx >= 0 ? pts[idx] : make_double4(0.0, 0.0, 0.0, 0.0);
    };
    double4 pf0 = make_double4(0.0, 0.0, 0.0, 0.0), pf1 = pf0;
    if (e < e_hi) {
      if (CACHE && lane == 0) bulk_load(T, dcache + (e - 1 - rest_lo) * cstride, cbytes, mbar);
      pf0 = slot_point(slot_index(e, lane));
      if (P > 32) pf1 = slot_point(slot_index(e, lane + 32));
    }
    int par = 0;
    bool first = true;
    for (; e < e_hi; e += stride, par ^= 1, first = false, ++tblk) {
      const int64_t en = e + stride;
      mark(0);
      // ---- this block's yJ row, target observation (and coordinates)
      if (lane < P) O[lane] = lane < m ? pf0.z : 0.0;
      if (P > 32 && lane + 32 < P) O[lane + 32] = lane + 32 < m ? pf1.z : 0.0;
      if (!CACHE) {
        if (lane < P) XY[lane] = make_double2(pf0.x, pf0.y);
        if (P > 32 && lane + 32 < P) XY[lane + 32] = make_double2(pf1.x, pf1.y);
      }
      {
        const double yt = shfl((m < 32) ? pf0.z : pf1.z, m & 31);
        if (lane == 0) misc[2 + par] = yt;
      }
      // ---- next block's gather, a whole block ahead: neighbour indices now,
      // the dependent point loads one column later (in-order issue would
      // otherwise stall on the index load)
      int ni0 = -1, ni1 = -1;
      if (en < e_hi) {
        ni0 = slot_index(en, lane);
        if (P > 32) ni1 = slot_index(en, lane + 32);
      }
      auto gather_next = [&]() {
        if (en < e_hi) {
          if (CACHE) {
            pf0.z = ni0 >= 0 ? pts[ni0].z : 0.0;
            if (P > 32) pf1.z = ni1 >= 0 ? pts[ni1].z : 0.0;
          } else {
            pf0 = slot_point(ni0);
            if (P > 32) pf1 = slot_point(ni1);
          }
        }
      };
      if (CACHE) {
        mbar_wait(mbar, phase);
        phase ^= 1;
      }
      __syncwarp();
      mark(1);

#pragma unroll
      for (int c = 0; c < NT; ++c) {
        if (c < NC) {
          const bool lastc = (c == NC - 1);
          if (c == (NC > 1 ? 1 : 0)) gather_next();
          // ---- generate tile column c: entries (8I + r, 8c + 2q + h)
          double acc[NT][2];
#pragma unroll
          for (int I = 0; I < NT; ++I) {
            if (I >= c) {
              const int i = 8 * I + r;
              double v0, v1;
              if (CACHE) {
                const double2 dv = ld2(T + tidx(I, c, NT) * 64 + chunk_off(r, q));
                v0 = cov_lean<KIND>(dv.x, inv_beta, tab);
                v1 = cov_lean<KIND>(dv.y, inv_beta, tab);
              } else {
                const double2 pa = XY[i];
                const double4 pb = *reinterpret_cast<const double4*>(XY + 8 * c + 2 * q);
                double dx = pa.x - pb.x, dy = pa.y - pb.y;
                v0 = cov_lean<KIND>(sqrt_pos_nz(fma(dx, dx, fma(dy, dy, 0x1p-1000))), inv_beta, tab);
                dx = pa.x - pb.z;
                dy = pa.y - pb.w;
                v1 = cov_lean<KIND>(sqrt_pos_nz(fma(dx, dx, fma(dy, dy, 0x1p-1000))), inv_beta, tab);
              }
              if (I == NT - 1 && i > m) {  // row m+1: yJ (0 from column m on); padding: 0
                const double2 ov = ld2(O + 8 * c + 2 * q);
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
            if (k == c - 1) mark(3 + 2 * c);
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
            mark(2 + 2 * c);
            bar_sync(lbar, 64);  // L of column c - 1 is in T
            update(c - 1);
          }
          if (lastc) {
            // T is no longer read by either warp for this block (the last
            // panel runs from S): stream in the next block's distances
            __syncwarp();
            if (CACHE && lane == 0 && en < e_hi)
              bulk_load(T, dcache + (en - 1 - rest_lo) * cstride, cbytes, mbar);
          }
          // ---- hand column c over (natural column order); before the first
          // column of a block, wait until the chain has taken the previous
          // block's last column (keeps one bar.arrive in flight per barrier
          // and protects S)
          if (c == 0 && !first) bar_sync(lbar, 64);
#pragma unroll
          for (int I = 0; I < NT; ++I) {
            if (I >= c) {
              double* dst = lastc ? S + (I - c) * 64 : T + tidx(I, c, NT) * 64;
              st2(dst + chunk_off(r, q), acc[I][0], acc[I][1]);
            }
          }
          bar_arrive(cbar, 64);
          mark(18 + (c == 0 ? 0 : (lastc ? 1 : 2)));
        }
      }
    }
  } else {
    // ============================ chain warp ============================
    int par = 0;
    for (; e < e_hi; e += stride, par ^= 1, ++tblk) {
      int fj = -1;  // first non-positive pivot column
#pragma unroll
      for (int c = 0; c < NT; ++c) {
        if (c < NC) {
          const bool lastc = (c == NC - 1);
          const int R0 = 8 * c;
          const int NR = P - R0;
          const int jmax = min(8, m - R0);  // pivots in this tile column
          mark(2 * c);
          bar_sync(cbar, 64);
          // lane owns panel rows R0 + lane + 32 rr: tile c + (lane + 32 rr) / 8, row lane & 7
          constexpr int kMaxRows = 2;
          double a[kMaxRows][8];
          auto row_ptr = [&](int rr) -> double* {
            const int I = c + ((lane + 32 * rr) >> 3);
            return lastc ? S + (I - c) * 64 : T + tidx(I, c, NT) * 64;
          };
#pragma unroll
          for (int rr = 0; rr < kMaxRows; ++rr) {
            if (rr * 32 < NR) {
              const bool ok = lane + 32 * rr < NR;
              const double* base = row_ptr(rr);
#pragma unroll
              for (int x = 0; x < 4; ++x) {
                double2 v = make_double2(0.0, 0.0);
                if (ok) v = ld2(base + chunk_off(lane & 7, x));
                a[rr][2 * x] = v.x;
                a[rr][2 * x + 1] = v.y;
              }
            }
          }
          mark(2 * c + 1);  // after the first LDS behind the (deferred-blocking) barrier
          // last column: rows are in registers, S may be refilled
          if (lastc && e + stride < e_hi) bar_arrive(lbar, 64);
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
                // column j of L_cc through shared memory (one store, four
                // broadcast LDS.128 instead of 14 32-bit shuffles; double-
                // buffered by pivot parity, one __syncwarp per pivot)
                double* Lc = Lcb + 8 * (j & 1);
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
                double* base = row_ptr(rr);
#pragma unroll
                for (int x = 0; x < 4; ++x)
                  st2(base + chunk_off(lane & 7, x), a[rr][x], a[rr][x + 4]);
              }
            }
            bar_arrive(lbar, 64);
            mark(16 + (c & 1));
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
                  const double resid = misc[2 + par] - mu;
                  rest[kk] = -0.5 * (resid * resid / sg + kLog2Pi + log(sg));
                }
              }
            }
            mark(20);
          }
        }
      }
    }
  }
}

template <int NT, int KIND, int MC, bool CACHE, bool TRACE = false, bool SPLIT = false>
cudaError_t launch(const Plan& p, const CovParams& cp, int64_t e_lo, int64_t e_hi,
                   cudaStream_t stream, long long* trace = nullptr) {
  constexpr int kThr = SPLIT ? 512 : kThreads;
  constexpr PairLayout L = pair_layout(NT);
  const size_t sm = sizeof(double) * ((size_t)kHead + (size_t)kPairs * L.stride);
  static size_t configured[64] = {};
  const int dev = p.device & 63;
  auto kern = loglik_ws_kernel<NT, KIND, MC, CACHE, TRACE, SPLIT>;
  if (configured[dev] < sm) {
    cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (err != cudaSuccess) return err;
    configured[dev] = sm;
  }
  int per_sm = 0;
  cudaError_t err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThr, sm);
  if (err != cudaSuccess) return err;
  if (per_sm < 1) per_sm = 1;
  int active = kPairs;
  if (TRACE) {
    if (const char* a = std::getenv("VGP_ACTIVE")) active = std::atoi(a), per_sm = 1;
  }
  const int64_t count = e_hi - e_lo;
  const int64_t want = (count + active - 1) / active;
  const int64_t cap = (int64_t)p.num_sms * per_sm;
  const int grid = (int)(want < cap ? want : cap);
  kern<<<grid, kThr, sm, stream>>>(p.d_pts, p.d_nbr, p.m, e_lo, e_hi, p.rest_lo, cp.s2,
                                       cp.inv_beta, p.d_rest, p.d_mu, p.d_sig, p.d_fail,
                                       p.d_dcache, p.dcache_stride, trace, active);
  return cudaGetLastError();
}

// VGP_TRACE=<file>: one traced launch (m = 60, nu = 1.5, cache) appends the
// per-pair timeline of CTA 0 to <file> (tools/ws_trace.py reads it)
inline cudaError_t launch_traced(const Plan& p, const CovParams& cp, int64_t e_lo, int64_t e_hi,
                                 cudaStream_t stream, const char* path) {
  const size_t n = (size_t)kPairs * 2 * kTraceBlocks * kTraceEvents;
  long long* d = nullptr;
  cudaError_t err = cudaMalloc(&d, n * sizeof(long long));
  if (err != cudaSuccess) return err;
  cudaMemsetAsync(d, 0, n * sizeof(long long), stream);
  const char* split = std::getenv("VGP_SPLIT");
  if (split && split[0] == '1')
    err = launch<8, kMatern15, 60, true, true, true>(p, cp, e_lo, e_hi, stream, d);
  else
    err = launch<8, kMatern15, 60, true, true>(p, cp, e_lo, e_hi, stream, d);
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
  if (NT == 8 && KIND == kMatern15 && MC == 60 && cache) {
    if (const char* path = std::getenv("VGP_TRACE")) return launch_traced(p, cp, e_lo, e_hi, stream, path);
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

}  // namespace ws
}  // namespace vgp
