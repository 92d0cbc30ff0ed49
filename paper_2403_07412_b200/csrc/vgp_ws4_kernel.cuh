// Warp-specialised FP64 tensor-core (DMMA) Vecchia kernel with the pivot
// chains isolated on their own SM sub-partition, m + 2 <= 64.
//
// Same block algorithm as vgp_ws3_kernel.cuh (worker warp: covariance
// generation + DMMA updates; chain warp: panel pivot chain), different warp
// placement.  Measured (profiles/r01_contention.jsonl): one DMMA-streaming
// warp on a scheduler doubles every dependent DFMA / MUFU latency of the
// other warps there, two or more starve them.  So here the scheduler-0 warps
// (warp % 4 == 0) run nothing but pivot chains - each interleaves the panels
// of two blocks (ILP 2 on the chain) - and the DMMA workers run on schedulers
// 1..3 (3 + 3 + 2 blocks):
//
//   CTA = 16 warps, 1 per SM; warp 4k: chain of slots 2k, 2k + 1;
//   the other 12 warps: workers of slots 0..7 in order, 4 spare warps exit.
#pragma once

#include "vgp_ws3_kernel.cuh"

namespace vgp {
namespace ws4 {

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

constexpr int kSlots = 8;     // blocks in flight per CTA (= per SM)
constexpr int kThreads = 512;  // 16 warps
constexpr int kHead = 256;   // sigma^2-scaled exp table
constexpr int kTraceBlocks = ws::kTraceBlocks;
constexpr int kTraceEvents = ws::kTraceEvents;

using ws3::SlotLayout;
using ws3::slot_layout;

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
  const int NC = (m + 8) >> 3;  // tile columns holding pivots or the Schur column
  constexpr SlotLayout L = slot_layout(NT);
  extern __shared__ __align__(16) double smem[];
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const bool chain = (warp & 3) == 0;
  // worker index: the non-chain warps in order
  const int wslot = chain ? -1 : 3 * (warp >> 2) + (warp & 3) - 1;
  auto Tb = [&](int s) { return smem + kHead + s * L.stride; };
  auto Sb = [&](int s) { return Tb(s) + L.tiles; };
  auto Ob = [&](int s) { return Sb(s) + 128; };
  auto XYb = [&](int s) { return reinterpret_cast<double2*>(Ob(s) + P); };
  auto Yb = [&](int s) { return Ob(s) + 3 * P; };  // [parity] target observation
  auto MBb = [&](int s) { return reinterpret_cast<uint64_t*>(Ob(s) + 3 * P + 2); };
  // named barriers (ids 0..15; id 0 is free again after the setup __syncthreads):
  // 2s = tile column staged (worker -> chain), 2s + 1 = L written (chain -> worker)

  for (int i = threadIdx.x; i < 256; i += blockDim.x) smem[i] = s2 * kExp2Table[i];
  if (CACHE && warp < kSlots && lane == 0) mbar_init(MBb(warp));
  __syncthreads();
  if (!chain && wslot >= kSlots) return;
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
    const int s = wslot;
    double* T = Tb(s);
    double* S = Sb(s);
    double* O = Ob(s);
    double2* XY = XYb(s);
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
    int64_t e = e0 + s;
    if (e < e_hi) {
      if (CACHE && lane == 0) bulk_load(T, dcache + (e - 1 - rest_lo) * cstride, cbytes, MBb(s));
      pf0 = slot_point(slot_index(e, lane));
      if (P > 32) pf1 = slot_point(slot_index(e, lane + 32));
    }
    int par = 0;
    bool first = true;
    for (; e < e_hi; e += stride, par ^= 1, first = false, ++tblk) {
      const int64_t en = e + stride;
      mark(s, 1, 0);
      if (lane < P) O[lane] = lane < m ? pf0.z : 0.0;
      if (P > 32 && lane + 32 < P) O[lane + 32] = lane + 32 < m ? pf1.z : 0.0;
      if (!CACHE) {
        if (lane < P) XY[lane] = make_double2(pf0.x, pf0.y);
        if (P > 32 && lane + 32 < P) XY[lane + 32] = make_double2(pf1.x, pf1.y);
      }
      {
        const double yt = shfl((m < 32) ? pf0.z : pf1.z, m & 31);
        if (lane == 0) Yb(s)[par] = yt;
      }
      int ni0 = -1, ni1 = -1;
      if (en < e_hi) {  // next block's neighbour indices now, its points one column later
        ni0 = slot_index(en, lane);
        if (P > 32) ni1 = slot_index(en, lane + 32);
      }
      if (CACHE) {
        mbar_wait(MBb(s), phase);
        phase ^= 1;
      }
      __syncwarp();
      mark(s, 1, 1);

#pragma unroll
      for (int c = 0; c < NT; ++c) {
        if (c < NC) {
          const bool lastc = (c == NC - 1);
          if (c == (NC > 1 ? 1 : 0) && en < e_hi) {
            if (CACHE) {
              pf0.z = ni0 >= 0 ? pts[ni0].z : 0.0;
              if (P > 32) pf1.z = ni1 >= 0 ? pts[ni1].z : 0.0;
            } else {
              pf0 = slot_point(ni0);
              if (P > 32) pf1 = slot_point(ni1);
            }
          }
          // ---- generate tile column c: entries (8I + r, 8c + 2q + h)
          double acc[NT][2];
#pragma unroll
          for (int I = 0; I < NT; ++I) {
            if (I >= c) {
              const int i = 8 * I + r;
              double v0, v1;
              if (CACHE) {
                const double2 dv = ld2(T + tidx(I, c) * 64 + chunk_off(r, q));
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
            const double2 b = ld2(T + tidx(c, k) * 64 + chunk_off(r, q));
            double2 a[NT];
#pragma unroll
            for (int I = 0; I < NT; ++I)
              if (I > c) a[I] = ld2(T + tidx(I, k) * 64 + chunk_off(r, q));
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
            // S): stream in the next block's distances
            __syncwarp();
            if (CACHE && lane == 0 && en < e_hi)
              bulk_load(T, dcache + (en - 1 - rest_lo) * cstride, cbytes, MBb(s));
          }
          // ---- hand column c over (natural column order); before a block's
          // first column, wait until the chain has taken the previous
          // block's last column (one arrival in flight per barrier; S reuse)
          if (c == 0 && !first) bar_sync(2 * s + 1, 64);
#pragma unroll
          for (int I = 0; I < NT; ++I) {
            if (I >= c) {
              double* dst = lastc ? S + (I - c) * 64 : T + tidx(I, c) * 64;
              st2(dst + chunk_off(r, q), acc[I][0], acc[I][1]);
            }
          }
          bar_arrive(2 * s, 64);
        }
      }
    }
  } else {
    // ============================ chain warp ============================
    // slots s0 = 2k, s0 + 1 in lockstep: both panels of column c are factored
    // in one instruction stream (two independent pivot chains)
    const int s0 = 2 * (warp >> 2);
    int par = 0;
    for (int64_t e = e0 + s0; e < e_hi; e += stride, par ^= 1, ++tblk) {
      const bool act1 = e + 1 < e_hi;
      int fj[2] = {-1, -1};
#pragma unroll
      for (int c = 0; c < NT; ++c) {
        if (c < NC) {
          const bool lastc = (c == NC - 1);
          const int R0 = 8 * c;
          const int NR = P - R0;
          const int jmax = min(8, m - R0);  // pivots in this tile column
          mark(s0, 0, 2 * c);
          bar_sync(2 * s0, 64);
          if (act1) bar_sync(2 * s0 + 2, 64);
          constexpr int kMaxRows = 2;
          double a[2][kMaxRows][8];
          auto row_ptr = [&](int h, int rr) -> double* {
            const int I = c + ((lane + 32 * rr) >> 3);
            return lastc ? Sb(s0 + h) + (I - c) * 64 : Tb(s0 + h) + tidx(I < NT ? I : NT - 1, c) * 64;
          };
#pragma unroll
          for (int h = 0; h < 2; ++h) {
#pragma unroll
            for (int rr = 0; rr < kMaxRows; ++rr) {
              if (rr * 32 < NR) {
                const bool ok = lane + 32 * rr < NR && (h == 0 || act1);
                const double* rb = row_ptr(h, rr);
#pragma unroll
                for (int x = 0; x < 4; ++x) {
                  double2 v = make_double2(1.0, 0.0);  // inactive slot: harmless identity
                  if (ok) v = ld2(rb + chunk_off(lane & 7, x));
                  else if (h == 0 || act1) v = make_double2(0.0, 0.0);
                  a[h][rr][2 * x] = v.x;
                  a[h][rr][2 * x + 1] = v.y;
                }
              }
            }
          }
          mark(s0, 0, 2 * c + 1);
          // last column: rows are in registers, S may be refilled
          if (lastc && e + stride < e_hi) bar_arrive(2 * s0 + 1, 64);
          if (lastc && act1 && e + 1 + stride < e_hi) bar_arrive(2 * s0 + 3, 64);
          double lastpiv[2] = {1.0, 1.0};
          if (jmax > 0) {
            double piv[2];
#pragma unroll
            for (int h = 0; h < 2; ++h) piv[h] = shfl(a[h][0][0], 0);
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              if (j < jmax) {
                double inv[2];
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                  if (j == jmax - 1) lastpiv[h] = piv[h];
                  inv[h] = rsqrt_chain(piv[h]);
                }
#pragma unroll
                for (int h = 0; h < 2; ++h)
#pragma unroll
                  for (int rr = 0; rr < kMaxRows; ++rr)
                    if (rr * 32 < NR) a[h][rr][j] *= inv[h];
                if (j + 1 < 8) {
#pragma unroll
                  for (int h = 0; h < 2; ++h) {
                    const double nxt = fma(-a[h][0][j], a[h][0][j], a[h][0][j + 1]);
                    piv[h] = shfl(nxt, j + 1);
                  }
                }
#pragma unroll
                for (int jp = j + 1; jp < 8; ++jp) {
#pragma unroll
                  for (int h = 0; h < 2; ++h) {
                    const double lc = shfl(a[h][0][j], jp);  // L[R0 + jp][R0 + j]
#pragma unroll
                    for (int rr = 0; rr < kMaxRows; ++rr)
                      if (rr * 32 < NR) a[h][rr][jp] = fma(-a[h][rr][j], lc, a[h][rr][jp]);
                  }
                }
              }
            }
          }
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            // pivot test !(piv > 0) (vg/batchla.py:146-151): a non-positive or
            // NaN pivot turns every later pivot NaN; the rare failing panel
            // locates the first bad column from the diagonal of L
            if (!(lastpiv[h] > 0.0) && fj[h] < 0) {
              double ljj = a[h][0][0];
#pragma unroll
              for (int x = 1; x < 8; ++x)
                if (lane == x) ljj = a[h][0][x];
              const unsigned bad = __ballot_sync(0xffffffffu, lane < jmax && !(ljj > 0.0));
              fj[h] = R0 + (bad ? __ffs(bad) - 1 : jmax - 1);
            }
          }
          if (!lastc) {
            // L rows below the diagonal tile, columns (x, x + 4) per chunk
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              if (h == 0 || act1) {
#pragma unroll
                for (int rr = 0; rr < kMaxRows; ++rr) {
                  if (rr * 32 < NR && lane + 32 * rr >= 8 && lane + 32 * rr < NR) {
                    double* rb = row_ptr(h, rr);
#pragma unroll
                    for (int x = 0; x < 4; ++x)
                      st2(rb + chunk_off(lane & 7, x), a[h][rr][x], a[h][rr][x + 4]);
                  }
                }
              }
            }
            bar_arrive(2 * s0 + 1, 64);
            if (act1) bar_arrive(2 * s0 + 3, 64);
          } else {
            // sigma_new = A[m][m], -mu = A[m+1][m] after m pivots (vg/vecchia.py:186-189, :206)
            const int cs = m - R0;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              double v = a[h][0][0];
#pragma unroll
              for (int x = 1; x < 8; ++x)
                if (x == cs) v = a[h][0][x];
              const double sg = shfl(v, cs);
              const double mu = -shfl(v, cs + 1);
              const int64_t eh = e + h;
              if (lane == 0 && (h == 0 || act1)) {
                const int64_t kk = eh - 1 - rest_lo;
                if (fj[h] >= 0) {
                  atomicMin(&fail[0], npd_key(eh, fj[h], m));
                } else {
                  mu_out[kk] = mu;
                  sig_out[kk] = sg;
                  if (!(sg > 0.0)) {
                    atomicMin(&fail[1], (unsigned long long)eh);
                    rest[kk] = 0.0;
                  } else {
                    const double resid = Yb(s0 + h)[par] - mu;
                    rest[kk] = -0.5 * (resid * resid / sg + kLog2Pi + log(sg));
                  }
                }
              }
            }
            mark(s0, 0, 20);
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

}  // namespace ws4
}  // namespace vgp
