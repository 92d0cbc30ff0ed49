// Split-scheduler warp-specialised FP64 DMMA Vecchia kernel, 8 <= m, m + 2 <= 64:
// the default fast path for mid-size conditioning sets (config 2: m = 60).
//
// Same per-block algorithm as vgp_ws3_kernel.cuh (vg/vecchia.py:154-162
// assemble, :180-190 _numeric_stage, :193-214 _reduction_stage): the
// augmented (8 NT)^2 matrix [Sigma_e; v_e; yJ_e] of batch entry e is factored
// left-looking over 8-wide tile columns in shared memory, the Schur
// complement leaving sigma_new and -mu.  What changes is WHERE each kind of
// FP64 work runs.  Measured on B200 (profiles/r01_contention.jsonl): one
// warp streaming DMMAs on a scheduler doubles the latency of a dependent
// DFMA chain on the same scheduler and two starve it, while DMMAs on another
// scheduler cost it nothing; ncu puts DMMA on the tensor sub-pipe and DFMA on
// the fp64 sub-pipe of the one shared FP64 pipe (profiles/r02_fp64_pipe.txt).
// So the SM is split by scheduler (warp w runs on scheduler w % 4):
//
//   schedulers 0, 1: 8 CHAIN warps, one per block slot: only the panel
//       factorisations (row-owner pivot chain: rsqrt / shuffle steps), the
//       block's critical path, with no DMMA stream beside them.
//   schedulers 2, 3: 8 WORKER warps, one per block slot: covariance
//       generation (lean FP64 Matern over the cached distances) straight into
//       the DMMA accumulators, the left-looking trailing updates with
//       mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4) — all but the last one while the
//       chain factors the previous column — the gather of the next block's
//       observations and the cp.async.bulk (SASS UBLKCP) of its distances.
//
// Hand-offs per slot go through shared-memory mbarriers (all 32 lanes
// arrive, release/acquire at CTA scope): col (column generated + updated,
// worker -> chain), lrdy (L of the column written, chain -> worker), dist
// (next block's distances and observations landed).  Each producer is at
// most one phase ahead of its consumer by construction.
#pragma once

#include "vgp_ws_kernel.cuh"

namespace vgp {
namespace ws4 {

using dmma::bulk_load;
using dmma::mbar_wait;
using dmma::neg;
using dmma::shfl;
using dmma::smem_u32;
using ll::cov_lean;
using ll::ld2;
using ll::mma;
using ll::rsqrt_chain;
using ll::st2;
using ws::chunk_off;
using ws::ntri;
using ws::tidx;

constexpr int kSlots = 8;    // blocks in flight per CTA (= per SM)
constexpr int kWarps = 16;   // 8 chain (schedulers 0, 1) + 8 worker (schedulers 2, 3)
constexpr int kThreads = 32 * kWarps;
constexpr int kHead = 256;   // sigma^2-scaled exp table

struct SlotLayout {
  int tiles;   // doubles of the tile triangle (= cache stride)
  int stride;  // tiles | S (2 tiles) | O (2 x P) | XY (2 x 2P) | Y (2) | 3 mbarriers (+3 pad)
};
__host__ __device__ constexpr SlotLayout slot_layout(int nt) {
  return SlotLayout{ntri(nt) * 64, ntri(nt) * 64 + 128 + 16 * nt + 32 * nt + 2 + 6};
}

__device__ __forceinline__ void mbar_init32(uint64_t* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 32;" ::"r"(smem_u32(bar)));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

// warp w -> slot ((w >> 2) << 1) | (w & 1); chain iff (w & 2) == 0
__device__ __forceinline__ int slot_of(int w) { return ((w >> 2) << 1) | (w & 1); }

constexpr int kTraceBlocks = 8;
constexpr int kTraceEvents = 24;

template <int NT, int KIND, int MC, bool CACHE, bool TRACE = false>
__global__ void __launch_bounds__(kThreads, 1)
loglik_ws4_kernel(const double4* __restrict__ pts, const int32_t* __restrict__ nbr, int m_rt,
                  int64_t e_lo, int64_t e_hi, int64_t rest_lo, double s2, double inv_beta,
                  double* __restrict__ rest, double* __restrict__ mu_out,
                  double* __restrict__ sig_out, unsigned long long* __restrict__ fail,
                  const double* __restrict__ dcache, int64_t cstride,
                  long long* __restrict__ trace = nullptr) {
  constexpr int P = 8 * NT;
  const int m = MC > 0 ? MC : m_rt;
  const int NC = (m + 8) >> 3;  // tile columns holding pivots or the Schur column (>= 2)
  constexpr SlotLayout L = slot_layout(NT);
  extern __shared__ __align__(16) double smem[];
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const bool chain = (warp & 2) == 0;
  const int s = slot_of(warp);
  double* T = smem + kHead + s * L.stride;
  double* S = T + L.tiles;
  double* Ob = S + 128;                                   // [par][P] observations of J
  double2* XYb = reinterpret_cast<double2*>(Ob + 2 * P);  // [par][P] coordinates (uncached)
  double* Yb = Ob + 6 * P;                                // [par] target observation
  uint64_t* MB = reinterpret_cast<uint64_t*>(Yb + 2);
  uint64_t* mb_dist = MB;
  uint64_t* mb_col = MB + 1;
  uint64_t* mb_lrdy = MB + 2;

  for (int i = threadIdx.x; i < 256; i += blockDim.x) smem[i] = s2 * kExp2Table[i];
  if (chain && lane < 3) mbar_init32(MB + lane);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  const double* tab = smem;

  const int64_t stride = (int64_t)gridDim.x * kSlots;
  const int64_t e_first = e_lo + (int64_t)blockIdx.x * kSlots + s;
  const int r = lane >> 2;  // fragment row
  const int q = lane & 3;   // fragment column pair
  const uint32_t cbytes = (uint32_t)(cstride * sizeof(double));
  int tblk = 0;
  // TRACE (profiling builds only): clock64 timeline of the first blocks of CTA 0
  auto mark = [&](int ev) {
    if (TRACE && blockIdx.x == 0 && lane == 0 && tblk < kTraceBlocks && ev < kTraceEvents)
      trace[((s * 2 + (chain ? 0 : 1)) * kTraceBlocks + tblk) * kTraceEvents + ev] = clock64();
  };

  if (!chain) {
    // ============================ worker warp ============================
    auto slot_index = [&](int64_t eb, int a) -> int {
      if (a < m) return nbr[(eb - 1 - rest_lo) * (int64_t)m + a];
      return a == m ? (int)(m + eb - 1) : -1;
    };
    auto slot_point = [&](int idx) -> double4 {
      return idx >= 0 ? pts[idx] : make_double4(0.0, 0.0, 0.0, 0.0);
    };
    // stage block eb's observations (+ coordinates) into buffer `par`, then
    // arrive on dist (lane 0 with the distance tiles' transaction bytes)
    auto publish = [&](int64_t eb, int par, double4 p0, double4 p1) {
      double* O = Ob + par * P;
      double2* XY = XYb + par * P;
      if (lane < P) O[lane] = lane < m ? p0.z : 0.0;
      if (P > 32 && lane + 32 < P) O[lane + 32] = lane + 32 < m ? p1.z : 0.0;
      if (!CACHE) {
        if (lane < P) XY[lane] = make_double2(p0.x, p0.y);
        if (P > 32 && lane + 32 < P) XY[lane + 32] = make_double2(p1.x, p1.y);
      }
      if (lane == (m & 31)) Yb[par] = (m < 32) ? p0.z : p1.z;
      if (CACHE && lane == 0)
        bulk_load(T, dcache + (eb - 1 - rest_lo) * cstride, cbytes, mb_dist);
      else
        mbar_arrive(mb_dist);
    };
    if (e_first < e_hi) {
      double4 p0 = slot_point(slot_index(e_first, lane));
      double4 p1 = P > 32 ? slot_point(slot_index(e_first, lane + 32)) : p0;
      publish(e_first, 0, p0, p1);
    }
    uint32_t lpar = 0, dpar = 0;
    int par = 0;
    for (int64_t e = e_first; e < e_hi; e += stride, par ^= 1, ++tblk) {
      const int64_t en = e + stride;
      const double* O = Ob + par * P;
      const double2* XY = XYb + par * P;
      int ni0 = -1, ni1 = -1;
      double4 pf0 = make_double4(0.0, 0.0, 0.0, 0.0), pf1 = pf0;
      if (en < e_hi) {  // next block's indices now, its points one column later
        ni0 = slot_index(en, lane);
        if (P > 32) ni1 = slot_index(en, lane + 32);
      }
      mbar_wait(mb_dist, dpar);  // this block's distances (T) and O / XY / Y
      dpar ^= 1;
      mark(1);
#pragma unroll
      for (int c = 0; c < NT; ++c) {
        if (c < NC) {
          const bool lastc = (c == NC - 1);
          if (c == 1 && en < e_hi) {
            pf0 = slot_point(ni0);
            if (P > 32) pf1 = slot_point(ni1);
          }
          // ---- generate tile column c into the accumulators: entries (8I + r, 8c + 2q + h)
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
#pragma unroll
            for (int kk = 0; kk < 2; ++kk) {
#pragma unroll
              for (int I = 0; I < NT; ++I)
                if (I >= c) mma(acc[I][0], acc[I][1], neg(kk ? a[I].y : a[I].x), kk ? b.y : b.x);
            }
          };
#pragma unroll
          for (int k = 0; k + 1 < c; ++k) update(k);
          if (c >= 1) {
            mark(2 * c);
            mbar_wait(mb_lrdy, lpar);  // L of column c - 1 is in T
            lpar ^= 1;
            mark(2 * c + 1);
            update(c - 1);
          }
#pragma unroll
          for (int I = 0; I < NT; ++I) {
            if (I >= c) {
              double* dst = lastc ? S + (I - c) * 64 : T + tidx(I, c, NT) * 64;
              st2(dst + chunk_off(r, q), acc[I][0], acc[I][1]);
            }
          }
          mbar_arrive(mb_col);
          mark(16 + c);
          if (lastc && en < e_hi) {
            // T is no longer read for this block (the last panel runs from
            // S): stage the next block into the other buffers
            __syncwarp();
            publish(en, par ^ 1, pf0, pf1);
          }
        }
      }
    }
  } else {
    // ============================ chain warp ============================
    uint32_t cpar = 0;
    int par = 0;
    for (int64_t e = e_first; e < e_hi; e += stride, par ^= 1, ++tblk) {
      int fj = -1;  // first non-positive pivot column
#pragma unroll
      for (int c = 0; c < NT; ++c) {
        if (c < NC) {
          const bool lastc = (c == NC - 1);
          const int R0 = 8 * c;
          const int NR = P - R0;
          const int jmax = min(8, m - R0);  // pivots in this tile column
          mbar_wait(mb_col, cpar);  // column c generated and updated by the worker
          cpar ^= 1;
          mark(2 + 2 * c);
          // ---- diagonal tile: every lane loads it (broadcast reads) and
          // factors it in registers, redundantly — the pivot chain then needs
          // no cross-lane traffic at all (the row-owner chain spent half its
          // time in the 16 shuffles per pivot); d[j][j] keeps 1 / L_jj
          const double* dt = lastc ? S : T + tidx(c, c, NT) * 64;
          double d[8][8];
#pragma unroll
          for (int i = 0; i < 8; ++i) {
#pragma unroll
            for (int x = 0; x < 4; ++x) {
              if (2 * x <= i) {
                const double2 v = ld2(dt + chunk_off(i, x));
                d[i][2 * x] = v.x;
                if (2 * x + 1 <= i) d[i][2 * x + 1] = v.y;
              }
            }
          }
          if (c == 2) mark(18);
          int fl = -1;  // first non-positive pivot of this panel
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            if (j < jmax) {
              // pivot test !(piv > 0) (vg/batchla.py:146-151)
              const double piv = d[j][j];
              if (!(piv > 0.0) && fl < 0) fl = j;
              const double inv = rsqrt_chain(piv);
              d[j][j] = inv;
#pragma unroll
              for (int i = j + 1; i < 8; ++i) d[i][j] *= inv;
#pragma unroll
              for (int i = j + 1; i < 8; ++i) {
#pragma unroll
                for (int k = j + 1; k <= i; ++k) d[i][k] = fma(-d[i][j], d[k][j], d[i][k]);
              }
            }
          }
          if (fl >= 0 && fj < 0) fj = R0 + fl;
          if (c == 2) mark(19);
          // ---- rows below the diagonal tile: lane owns rows R0 + 8 + lane + 32 rr,
          // forward substitution against L_cc in the order of the reference's
          // right-looking sweep (scale by 1/L_jj, then subtract from later columns)
          const int NB = NR - 8;
          double mu_row = 0.0;  // last panel: column cs of row R0 + 8 (lane 0)
#pragma unroll
          for (int rr = 0; rr < 2; ++rr) {
            if (rr * 32 < NB) {
              const int lr = 8 + lane + 32 * rr;  // row within the panel
              const bool ok = lr < NR;
              const int I = c + (lr >> 3);
              double* rb = lastc ? S + (I - c) * 64 : T + tidx(I < NT ? I : NT - 1, c, NT) * 64;
              double a[8];
#pragma unroll
              for (int x = 0; x < 4; ++x) {
                double2 v = make_double2(0.0, 0.0);
                if (ok) v = ld2(rb + chunk_off(lane & 7, x));
                a[2 * x] = v.x;
                a[2 * x + 1] = v.y;
              }
#pragma unroll
              for (int j = 0; j < 8; ++j) {
                if (j < jmax) {
                  a[j] *= d[j][j];
#pragma unroll
                  for (int jp = j + 1; jp < 8; ++jp) a[jp] = fma(-a[j], d[jp][j], a[jp]);
                }
              }
              if (!lastc) {
                // L rows, columns (x, x + 4) per chunk
                if (ok) {
#pragma unroll
                  for (int x = 0; x < 4; ++x) st2(rb + chunk_off(lane & 7, x), a[x], a[x + 4]);
                }
              } else if (rr == 0) {
                const int cs = m - R0;
#pragma unroll
                for (int x = 0; x < 8; ++x)
                  if (x == cs) mu_row = a[x];
              }
            }
          }
          if (!lastc) {
            if (c == 2) mark(20);
            mbar_arrive(mb_lrdy);
            mark(3 + 2 * c);
          } else {
            // sigma_new = A[m][m], -mu = A[m+1][m] after m pivots (vg/vecchia.py:186-189, :206)
            const int cs = m - R0;
            double sg = 0.0, nmu = 0.0;
#pragma unroll
            for (int x = 0; x < 8; ++x) {
              if (x == cs) sg = d[x][x];
              if (x + 1 < 8 && x == cs) nmu = d[x + 1][x];
            }
            if (cs == 7) nmu = shfl(mu_row, 0);
            const double mu = -nmu;
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
                  const double resid = Yb[par] - mu;
                  rest[kk] = -0.5 * (resid * resid / sg + kLog2Pi + log(sg));
                }
              }
            }
            mark(3 + 2 * c);
          }
        }
      }
    }
  }
}

template <int NT, int KIND, int MC, bool CACHE, bool TRACE = false>
cudaError_t launch(const Plan& p, const CovParams& cp, int64_t e_lo, int64_t e_hi,
                   cudaStream_t stream, long long* trace = nullptr) {
  constexpr SlotLayout L = slot_layout(NT);
  const size_t sm = sizeof(double) * ((size_t)kHead + (size_t)kSlots * L.stride);
  static size_t configured[64] = {};
  const int dev = p.device & 63;
  auto kern = loglik_ws4_kernel<NT, KIND, MC, CACHE, TRACE>;
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
                                       p.d_dcache, p.dcache_stride, trace);
  return cudaGetLastError();
}

// VGP_TRACE4=<file>: one traced launch (m = 60, nu = 1.5, cache) appends the
// clock64 timeline [slot][role][block][event] of CTA 0 (tools/ws4_trace.py)
inline cudaError_t launch_traced(const Plan& p, const CovParams& cp, int64_t e_lo, int64_t e_hi,
                                 cudaStream_t stream, const char* path) {
  const size_t n = (size_t)kSlots * 2 * kTraceBlocks * kTraceEvents;
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
    if (const char* path = std::getenv("VGP_TRACE4")) return launch_traced(p, cp, e_lo, e_hi, stream, path);
  }
  if (cache) return launch<NT, KIND, MC, true>(p, cp, e_lo, e_hi, stream);
  return launch<NT, KIND, MC, false>(p, cp, e_lo, e_hi, stream);
}

template <int KIND>
cudaError_t launch_kind(const Plan& p, const CovParams& cp, int64_t e_lo, int64_t e_hi,
                        cudaStream_t stream, bool cache) {
  if (p.m < 8) return cudaErrorNotSupported;  // needs >= 2 tile columns
  if (p.m == 60) return launch_c<8, KIND, 60>(p, cp, e_lo, e_hi, stream, cache);
  switch ((p.m + 2 + 7) / 8) {
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

}  // namespace ws4
}  // namespace vgp
