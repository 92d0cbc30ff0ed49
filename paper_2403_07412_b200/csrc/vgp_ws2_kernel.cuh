// Warp-specialised FP64 tensor-core (DMMA) Vecchia kernel with a short
// critical path, m + 2 <= 64 (the default fast path).
//
// Each conditioning block e >= 1 (vg/vecchia.py:154-162 assemble, :180-190
// _numeric_stage, :193-214 _reduction_stage) is owned by a PAIR of warps that
// share its augmented (8 NT)^2 matrix (rows 0..m-1 Sigma_e, row m v_e, row
// m+1 yJ, zero padding) in shared memory.  The blocked Cholesky over 8-wide
// tile columns is split so that only the irreducible part stays serial:
//
//   chain warp   factors the 8x8 diagonal tile of column c (lanes 0..7 own
//                its rows; 8 rsqrt / shuffle pivot steps) and publishes L_cc
//                (transposed) and the 8 reciprocal pivots; the last column's
//                panel also carries rows m, m+1, whose Schur complement gives
//                sigma_new and -mu (vg/vecchia.py:186-189, :206), and the
//                block's log-density;
//   worker warp  everything else: covariance generation (lean FP64 Matern),
//                the triangular solve of the rows below the diagonal tile
//                against L_cc (row per lane, L_cc broadcast from shared
//                memory), and the trailing updates with mma.sync.m8n8k4.f64
//                (SASS DMMA.8x8x4).  After receiving L_cc it solves, updates
//                the NEXT diagonal tile first and hands it over (look-ahead),
//                then finishes column c + 1 and generates column c + 2
//                (left-looking over the columns before).
//
// Critical path per column: the chain's 8 pivots + one 8-step row solve and
// two DMMAs in the worker (measured latencies in profiles/r01_latency.jsonl).
//
// Shared-memory tiles and the distance cache use ws::chunk_off's swizzled
// 16-byte chunks (conflict-free for fragment and row accesses); staged
// covariance is in natural column order, L in (q, q + 4) order.
#pragma once

#include "vgp_ws_kernel.cuh"

namespace vgp {
namespace ws2 {

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
using ws::tidx;

constexpr int kPairs = 4;              // blocks in flight per CTA
constexpr int kThreads = 64 * kPairs;  // warps 0..kPairs-1 chain, kPairs..2kPairs-1 worker
constexpr int kHead = 256;             // sigma^2-scaled exp table
constexpr int kTraceBlocks = ws::kTraceBlocks;
constexpr int kTraceEvents = ws::kTraceEvents;

struct PairLayout {
  int tiles;   // doubles of the tile triangle (= cache stride)
  int stride;  // tiles | S (2 tiles) | Lt (2 x 64) | inv (2 x 8) | O (P) | XY (2P) | yt (4) | mbarrier (2)
};
__host__ __device__ constexpr PairLayout pair_layout(int nt) {
  return PairLayout{tidx(nt, 0) * 64, tidx(nt, 0) * 64 + 128 + 128 + 16 + 8 * nt + 16 * nt + 4 + 2};
}

template <int NT, int KIND, int MC, bool CACHE, bool TRACE = false>
__global__ void __launch_bounds__(kThreads, 2)
loglik_ws2_kernel(const double4* __restrict__ pts, const int32_t* __restrict__ nbr, int m_rt,
                  int64_t e_lo, int64_t e_hi, int64_t rest_lo, double s2, double inv_beta,
                  double* __restrict__ rest, double* __restrict__ mu_out,
                  double* __restrict__ sig_out, unsigned long long* __restrict__ fail,
                  const double* __restrict__ dcache, int64_t cstride,
                  long long* __restrict__ trace = nullptr) {
  constexpr int P = 8 * NT;
  const int m = MC > 0 ? MC : m_rt;
  const int NC = (m + 8) >> 3;  // tile columns holding pivots or the Schur column
  constexpr PairLayout L = pair_layout(NT);
  extern __shared__ __align__(16) double smem[];
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const bool chain = warp < kPairs;
  const int pr = chain ? warp : warp - kPairs;
  double* T = smem + kHead + pr * L.stride;  // tile triangle
  double* S = T + L.tiles;                   // last column staging (2 tiles)
  double* Lt = S + 128;  // L_cc transposed, 2 buffers by column parity: Lt[8k + j] = L[j][k]
  double* Iv = Lt + 128;  // reciprocal pivots of column c, 2 buffers
  double* O = Iv + 16;    // yJ row (row m+1)
  double2* XY = reinterpret_cast<double2*>(O + P);
  double* misc = O + 3 * P;  // [2 + parity] target obs
  uint64_t* mbar = reinterpret_cast<uint64_t*>(misc + 4);
  const int cbar = 1 + 2 * pr;  // diagonal tile / last column staged (worker -> chain)
  const int lbar = 2 + 2 * pr;  // L_cc published (chain -> worker)

  for (int i = threadIdx.x; i < 256; i += blockDim.x) smem[i] = s2 * kExp2Table[i];
  if (CACHE && !chain && lane == 0) mbar_init(mbar);
  __syncthreads();
  const double* tab = smem;

  const int64_t stride = (int64_t)gridDim.x * kPairs;
  int64_t e = e_lo + (int64_t)blockIdx.x * kPairs + pr;
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
    // staged tile (I, J) base
    auto tile = [&](int I, int J) -> double* { return T + tidx(I, J) * 64; };
    // covariance entries (8I + r, 8J + 2q + h) of tile (I, J)
    auto gen_tile = [&](const int I, const int J, double& v0, double& v1) {
      const int i = 8 * I + r;
      if (CACHE) {
        const double2 dv = ld2(tile(I, J) + chunk_off(r, q));
        v0 = cov_lean<KIND>(dv.x, inv_beta, tab);
        v1 = cov_lean<KIND>(dv.y, inv_beta, tab);
      } else {
        const double2 pa = XY[i];
        const double4 pb = *reinterpret_cast<const double4*>(XY + 8 * J + 2 * q);
        double dx = pa.x - pb.x, dy = pa.y - pb.y;
        v0 = cov_lean<KIND>(sqrt_pos_nz(fma(dx, dx, fma(dy, dy, 0x1p-1000))), inv_beta, tab);
        dx = pa.x - pb.z;
        dy = pa.y - pb.w;
        v1 = cov_lean<KIND>(sqrt_pos_nz(fma(dx, dx, fma(dy, dy, 0x1p-1000))), inv_beta, tab);
      }
      if (I == NT - 1 && i > m) {  // row m+1: yJ (0 from column m on); padding: 0
        const double2 ov = ld2(O + 8 * J + 2 * q);
        v0 = i == m + 1 ? ov.x : 0.0;
        v1 = i == m + 1 ? ov.y : 0.0;
      }
    };
    // acc(I, J) -= L_Ik L_Jk^T for I in [i0, i1), operands from T (L order)
    auto update = [&](double (&acc)[NT][2], const int i0, const int i1, const int J, const int k) {
      const double2 b = ld2(tile(J, k) + chunk_off(r, q));
      double2 a[NT];
#pragma unroll
      for (int I = 0; I < NT; ++I)
        if (I >= i0 && I < i1) a[I] = I == J ? b : ld2(tile(I, k) + chunk_off(r, q));
#pragma unroll
      for (int kk = 0; kk < 2; ++kk) {
#pragma unroll
        for (int I = 0; I < NT; ++I)
          if (I >= i0 && I < i1)
            mma(acc[I][0], acc[I][1], neg(kk ? a[I].y : a[I].x), kk ? b.y : b.x);
      }
    };
    // generate column J, apply L of columns k <= kmax, stage (natural order)
    auto column = [&](const int J, const int kmax) {
      double acc[NT][2];
#pragma unroll
      for (int I = 0; I < NT; ++I)
        if (I >= J) gen_tile(I, J, acc[I][0], acc[I][1]);
#pragma unroll
      for (int k = 0; k < NT; ++k)
        if (k <= kmax) update(acc, J, NT, J, k);
#pragma unroll
      for (int I = 0; I < NT; ++I)
        if (I >= J) st2(tile(I, J) + chunk_off(r, q), acc[I][0], acc[I][1]);
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
      // ---- next block's gather: indices now, the dependent loads later
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

      // the last column is staged to S (T then takes the next block's tiles)
      auto finish_last = [&]() {
        __syncwarp();
        if (CACHE && lane == 0 && en < e_hi)
          bulk_load(T, dcache + (en - 1 - rest_lo) * cstride, cbytes, mbar);
      };

      // ---- column 0 (and 1), hand over the first diagonal tile
      if (NC == 1) {
        double acc[NT][2];
#pragma unroll
        for (int I = 0; I < NT; ++I) gen_tile(I, 0, acc[I][0], acc[I][1]);
        finish_last();
#pragma unroll
        for (int I = 0; I < NT; ++I) st2(S + I * 64 + chunk_off(r, q), acc[I][0], acc[I][1]);
      } else {
        column(0, -1);
      }
      if (!first) bar_sync(lbar, 64);  // the chain holds the previous block's last column
      bar_arrive(cbar, 64);
      if (NC > 1) column(1, -1);
      gather_next();

#pragma unroll
      for (int c = 0; c + 1 < NT; ++c) {
        if (c + 1 < NC) {
          const bool lastn = (c + 2 == NC);  // column c + 1 is the last one
          mark(2 + 2 * c);
          bar_sync(lbar, 64);  // L_cc and the reciprocal pivots are published
          // ---- triangular solve of the rows below the diagonal tile:
          // x = a L_cc^-T, lane owns row 8(c+1) + lane + 32 s
          const double* Ivc = Iv + 8 * (c & 1);
          const double* Ltc = Lt + 64 * (c & 1);
          const double2 i01 = ld2(Ivc), i23 = ld2(Ivc + 2), i45 = ld2(Ivc + 4), i67 = ld2(Ivc + 6);
          const double iv[8] = {i01.x, i01.y, i23.x, i23.y, i45.x, i45.y, i67.x, i67.y};
          auto solve = [&](const int s) {
            const int row = 8 * (c + 1) + lane + 32 * s;
            const int I = row >> 3;
            double* base = tile(I < NT ? I : NT - 1, c);
            double a[8];
#pragma unroll
            for (int x = 0; x < 4; ++x) {
              double2 v = make_double2(0.0, 0.0);
              if (row < P) v = ld2(base + chunk_off(lane & 7, x));
              a[2 * x] = v.x;
              a[2 * x + 1] = v.y;
            }
            if (s == 0) mark(3 + 2 * c);
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              a[k] *= iv[k];
              if (k + 1 < 8) {
                double lt[8];
#pragma unroll
                for (int x = (k + 1) & ~1; x < 8; x += 2) {
                  const double2 v = ld2(Ltc + 8 * k + x);
                  lt[x] = v.x;
                  lt[x + 1] = v.y;
                }
#pragma unroll
                for (int j = k + 1; j < 8; ++j) a[j] = fma(-a[k], lt[j], a[j]);
              }
            }
            if (row < P) {
#pragma unroll
              for (int x = 0; x < 4; ++x) st2(base + chunk_off(lane & 7, x), a[x], a[x + 4]);
            }
          };
          solve(0);
          __syncwarp();
          // ---- look-ahead: the next diagonal tile first
          if (!lastn) {
            double dg[NT][2];
            const double2 v = ld2(tile(c + 1, c + 1) + chunk_off(r, q));
            dg[c + 1][0] = v.x;
            dg[c + 1][1] = v.y;
            update(dg, c + 1, c + 2, c + 1, c);
            st2(tile(c + 1, c + 1) + chunk_off(r, q), dg[c + 1][0], dg[c + 1][1]);
            bar_arrive(cbar, 64);
          }
          if (8 * (c + 1) + 32 < P) {
            solve(1);
            __syncwarp();
          }
          // ---- rest of column c + 1 (all of it if it is the last column)
          {
            double acc[NT][2];
            const int i0 = lastn ? c + 1 : c + 2;
#pragma unroll
            for (int I = 0; I < NT; ++I) {
              if (I >= i0) {
                const double2 v = ld2(tile(I, c + 1) + chunk_off(r, q));
                acc[I][0] = v.x;
                acc[I][1] = v.y;
              }
            }
            update(acc, i0, NT, c + 1, c);
            if (lastn) {
              finish_last();
#pragma unroll
              for (int I = 0; I < NT; ++I)
                if (I >= c + 1)
                  st2(S + (I - c - 1) * 64 + chunk_off(r, q), acc[I][0], acc[I][1]);
              bar_arrive(cbar, 64);
            } else {
#pragma unroll
              for (int I = 0; I < NT; ++I)
                if (I >= c + 2) st2(tile(I, c + 1) + chunk_off(r, q), acc[I][0], acc[I][1]);
            }
          }
          // ---- column c + 2 (left-looking over columns <= c)
          if (c + 2 < NC) column(c + 2, c);
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
          const int jmax = min(8, m - R0);  // pivots in this tile column
          mark(2 * c);
          bar_sync(cbar, 64);
          // lastc: rows R0.. of S (lanes 0..15); else the diagonal tile (lanes 0..7)
          const int nrows = lastc ? P - R0 : 8;
          double a[8];
          {
            const double* base = lastc ? S + (lane >> 3) * 64 : T + tidx(c, c) * 64;
#pragma unroll
            for (int x = 0; x < 4; ++x) {
              double2 v = make_double2(0.0, 0.0);
              if (lane < nrows) v = ld2(base + chunk_off(lane & 7, x));
              a[2 * x] = v.x;
              a[2 * x + 1] = v.y;
            }
          }
          mark(2 * c + 1);
          if (lastc && e + stride < e_hi) bar_arrive(lbar, 64);  // S may be refilled
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
#pragma unroll
                for (int jp = j + 1; jp < 8; ++jp) {
                  const double lc = shfl(a[j], jp);  // L[R0 + jp][R0 + j]
                  a[jp] = fma(-a[j], lc, a[jp]);
                }
              }
            }
          }
          // pivot test !(piv > 0) (vg/batchla.py:146-151): a non-positive or
          // NaN pivot turns every later pivot NaN; the rare failing panel
          // locates the first bad column from the diagonal of L
          if (!(lastpiv > 0.0) && fj < 0) {
            double ljj = a[0];
#pragma unroll
            for (int x = 1; x < 8; ++x)
              if (lane == x) ljj = a[x];
            const unsigned bad = __ballot_sync(0xffffffffu, lane < jmax && !(ljj > 0.0));
            fj = R0 + (bad ? __ffs(bad) - 1 : jmax - 1);
          }
          if (!lastc) {
            // publish L_cc transposed (lane j: Lt[8k + j] = L[j][k], k < j) and 1/L_kk
            double* Ltc = Lt + 64 * (c & 1);
            double* Ivc = Iv + 8 * (c & 1);
#pragma unroll
            for (int k = 0; k < 7; ++k)
              if (lane > k && lane < 8) Ltc[8 * k + lane] = a[k];
            if (lane == 0) {
              st2(Ivc, iv[0], iv[1]);
              st2(Ivc + 2, iv[2], iv[3]);
              st2(Ivc + 4, iv[4], iv[5]);
              st2(Ivc + 6, iv[6], iv[7]);
            }
            bar_arrive(lbar, 64);
          } else {
            // sigma_new = A[m][m], -mu = A[m+1][m] after m pivots
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

template <int NT, int KIND, int MC, bool CACHE, bool TRACE = false>
cudaError_t launch(const Plan& p, const CovParams& cp, int64_t e_lo, int64_t e_hi,
                   cudaStream_t stream, long long* trace = nullptr) {
  constexpr PairLayout L = pair_layout(NT);
  const size_t sm = sizeof(double) * ((size_t)kHead + (size_t)kPairs * L.stride);
  static size_t configured[64] = {};
  const int dev = p.device & 63;
  auto kern = loglik_ws2_kernel<NT, KIND, MC, CACHE, TRACE>;
  if (configured[dev] < sm) {
    cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (err != cudaSuccess) return err;
    configured[dev] = sm;
  }
  int per_sm = 0;
  cudaError_t err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThreads, sm);
  if (err != cudaSuccess) return err;
  if (per_sm < 1) per_sm = 1;
  const int64_t count = e_hi - e_lo;
  const int64_t want = (count + kPairs - 1) / kPairs;
  const int64_t cap = (int64_t)p.num_sms * per_sm;
  const int grid = (int)(want < cap ? want : cap);
  kern<<<grid, kThreads, sm, stream>>>(p.d_pts, p.d_nbr, p.m, e_lo, e_hi, p.rest_lo, cp.s2,
                                       cp.inv_beta, p.d_rest, p.d_mu, p.d_sig, p.d_fail,
                                       p.d_dcache, p.dcache_stride, trace);
  return cudaGetLastError();
}

inline cudaError_t launch_traced(const Plan& p, const CovParams& cp, int64_t e_lo, int64_t e_hi,
                                 cudaStream_t stream, const char* path) {
  const size_t n = (size_t)kPairs * 2 * kTraceBlocks * kTraceEvents;
  long long* d = nullptr;
  cudaError_t err = cudaMalloc(&d, n * sizeof(long long));
  if (err != cudaSuccess) return err;
  cudaMemsetAsync(d, 0, n * sizeof(long long), stream);
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
    if (const char* path = std::getenv("VGP_TRACE2")) return launch_traced(p, cp, e_lo, e_hi, stream, path);
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

}  // namespace ws2
}  // namespace vgp
