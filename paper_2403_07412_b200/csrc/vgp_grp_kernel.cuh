// Lock-step group FP64 DMMA Vecchia kernel, 8 <= m, m + 2 <= 64, distance
// cache: blocks are factored in groups of four that advance one tile column
// at a time together, so every stage of the left-looking blocked Cholesky is
// a batch over the group's blocks instead of a per-block dependency chain.
//
// Per block the algorithm is the one of vgp_ws3_kernel.cuh (vg/vecchia.py:154-162
// assemble, :180-190 _numeric_stage, :193-214 _reduction_stage): the augmented
// (8 NT)^2 matrix [Sigma_e; v_e; yJ_e] in shared memory, factored over 8-wide
// tile columns, the Schur complement leaving sigma_new and -mu.  Per column c
// and group (8 warps, 256 threads, one named barrier):
//
//   1. tile jobs (all 8 warps): generate tiles (I, c), I >= c, of the four
//      blocks straight into DMMA accumulators (lean FP64 Matern over the
//      cached distances) and apply L of the columns k < c with
//      mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4); store.
//   2. diagonal tiles (one warp, ONE LANE PER BLOCK): each lane factors its
//      block's 8x8 diagonal tile in registers — no shuffles, no redundancy;
//      the pivot test !(piv > 0) (vg/batchla.py:146-151) per pivot.
//   3. panel rows (all 256 threads, one row each): forward substitution of
//      the rows below the diagonal tile against L_cc, in the reference
//      sweep's order; store L.
//
// Two groups per CTA (8 blocks in flight per SM, one CTA per SM) run
// independently, so one group's latency-bound stage 2 overlaps the other's
// throughput-bound stage 1.  A group's next four blocks are staged at the end
// of its current ones: neighbour observations gathered a whole round ahead
// into registers, the distance tiles prefetched into L2 a round ahead
// (cp.async.bulk.prefetch.L2) and then copied with one cp.async.bulk per
// block (SASS UBLKCP) + mbarrier.
#pragma once

#include "vgp_ws_kernel.cuh"

namespace vgp {
namespace grp {

using dmma::bulk_load;
using dmma::mbar_wait;
using dmma::neg;
using dmma::smem_u32;
using ll::cov_lean;
using ll::ld2;
using ll::mma;
using ll::rsqrt_chain;
using ll::st2;
using ws::chunk_off;
using ws::ntri;
using ws::tidx;

constexpr int kGroupBlocks = 4;
constexpr int kGroups = 2;
constexpr int kSlots = kGroups * kGroupBlocks;  // blocks in flight per CTA (= per SM)
constexpr int kGroupWarps = 8;
constexpr int kThreads = 32 * kGroupWarps * kGroups;
constexpr int kHead = 256;  // sigma^2-scaled exp table
constexpr int kTraceRounds = 6;
constexpr int kTraceEvents = 32;

struct SlotLayout {
  int tiles;   // doubles of the tile triangle (= cache stride)
  int stride;  // tiles | LD (64) | O (P) | scalars (8)
};
__host__ __device__ constexpr SlotLayout slot_layout(int nt) {
  return SlotLayout{ntri(nt) * 64, ntri(nt) * 64 + 64 + 8 * nt + 8};
}

__device__ __forceinline__ void bar_group(int id) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(32 * kGroupWarps) : "memory");
}
__device__ __forceinline__ void mbar_init_n(uint64_t* bar, int n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(n));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}

template <int NT, int KIND, int MC, bool TRACE = false>
__global__ void __launch_bounds__(kThreads, 1)
loglik_grp_kernel(const double4* __restrict__ pts, const int32_t* __restrict__ nbr, int m_rt,
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
  const int g = warp / kGroupWarps;   // group
  const int gw = warp % kGroupWarps;  // warp within the group
  const int gt = threadIdx.x % (32 * kGroupWarps);
  uint64_t* MB = reinterpret_cast<uint64_t*>(smem + kHead + kSlots * L.stride);
  auto T_of = [&](int b) { return smem + kHead + (g * kGroupBlocks + b) * L.stride; };
  auto LD_of = [&](int b) { return T_of(b) + L.tiles; };
  auto O_of = [&](int b) { return T_of(b) + L.tiles + 64; };
  auto SC_of = [&](int b) { return T_of(b) + L.tiles + 64 + P; };  // [0] sigma, [1] -mu, [2] y_t, [3] fail col

  for (int i = threadIdx.x; i < 256; i += blockDim.x) smem[i] = s2 * kExp2Table[i];
  if (threadIdx.x < kGroups) mbar_init_n(MB + threadIdx.x, kGroupBlocks);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  const double* tab = smem;
  const int r = lane >> 2;  // fragment row
  const int q = lane & 3;   // fragment column pair
  const uint32_t cbytes = (uint32_t)(cstride * sizeof(double));
  const int bar_id = 1 + g;

  // rounds: this group's blocks are e = first + i * rstride + b, b < 4
  const int64_t rstride = (int64_t)gridDim.x * kSlots;
  const int64_t first = e_lo + (int64_t)blockIdx.x * kSlots + g * kGroupBlocks;
  // staging thread (b, a) = (gt >> 6, gt & 63): observation a of block b
  const int sb = gt >> 6, sa = gt & 63;
  auto obs_index = [&](int64_t eb) -> int {
    if (eb >= e_hi || sa > m || sa >= P) return -1;
    return sa < m ? nbr[(eb - 1 - rest_lo) * (int64_t)m + sa] : (int)(m + eb - 1);
  };
  double pf = 0.0;
  {
    const int idx = obs_index(first + sb);
    if (idx >= 0) pf = pts[idx].z;
  }
  int tround = 0;
  auto mark = [&](int ev) {
    if (TRACE && blockIdx.x == 0 && gt == 0 && tround < kTraceRounds && ev < kTraceEvents)
      trace[(g * kTraceRounds + tround) * kTraceEvents + ev] = clock64();
  };
  uint32_t mpar = 0;
  for (int64_t base = first; base < e_hi; base += rstride, mpar ^= 1, ++tround) {
    mark(0);
    // ---- stage this round's blocks: distances (TMA), observations (registers -> smem)
    if (gw == 0 && lane < kGroupBlocks) {
      const int64_t eb = base + lane;
      if (eb < e_hi)
        bulk_load(T_of(lane), dcache + (eb - 1 - rest_lo) * cstride, cbytes, MB + g);
      else
        mbar_arrive(MB + g);
      const int64_t en = eb + rstride;  // next round: into L2 now
      if (en < e_hi) prefetch_l2(dcache + (en - 1 - rest_lo) * cstride, cbytes);
    }
    if (sa < P) {
      O_of(sb)[sa] = sa < m ? pf : 0.0;
      if (sa == m) SC_of(sb)[2] = pf;
    }
    if (sa == 0) SC_of(sb)[3] = -1.0;
    {
      const int idx = obs_index(base + rstride + sb);  // next round's observation, a round ahead
      pf = idx >= 0 ? pts[idx].z : 0.0;
    }
    mbar_wait(MB + g, mpar);
    bar_group(bar_id);
    mark(1);

#pragma unroll
    for (int c = 0; c < NT; ++c) {
      if (c < NC) {
        const bool lastc = (c == NC - 1);
        const int R0 = 8 * c;
        const int jmax = min(8, m - R0);
        // ================= 1. tile jobs: (block, up to 4 tiles of column c)
        {
          constexpr int kJT = 4;  // tiles per job
          const int ntile = NT - c;
          const int nch = (ntile + kJT - 1) / kJT;
          // tile jobs run on schedulers 1-3 only (warp w -> scheduler w % 4):
          // scheduler 0 keeps the diagonal pivot chains free of DMMA streams,
          // which starve a dependent DFMA chain on the same scheduler
          // (profiles/r01_contention.jsonl)
          const int tw = gw - 1 - gw / 4;  // 0..5 for gw in {1, 2, 3, 5, 6, 7}
          for (int job = (gw % 4) ? tw : kGroupBlocks * nch; job < kGroupBlocks * nch; job += kGroupWarps - 2) {
            const int b = job / nch;
            const int I0 = c + (job % nch) * kJT;
            double* T = T_of(b);
            const double* O = O_of(b);
            double acc[kJT][2];
#pragma unroll
            for (int t = 0; t < kJT; ++t) {
              const int I = I0 + t;
              if (I < NT) {
                const int i = 8 * I + r;
                const double2 dv = ld2(T + tidx(I, c, NT) * 64 + chunk_off(r, q));
                double v0 = cov_lean<KIND>(dv.x, inv_beta, tab);
                double v1 = cov_lean<KIND>(dv.y, inv_beta, tab);
                if (I == NT - 1 && i > m) {  // row m+1: yJ (0 from column m on); padding: 0
                  const double2 ov = ld2(O + 8 * c + 2 * q);
                  v0 = i == m + 1 ? ov.x : 0.0;
                  v1 = i == m + 1 ? ov.y : 0.0;
                }
                acc[t][0] = v0;
                acc[t][1] = v1;
              }
            }
#pragma unroll
            for (int k = 0; k < NT; ++k) {
              if (k < c) {
                const double2 bb = ld2(T + tidx(c, k, NT) * 64 + chunk_off(r, q));
                double2 a[kJT];
#pragma unroll
                for (int t = 0; t < kJT; ++t)
                  if (I0 + t < NT) a[t] = ld2(T + tidx(I0 + t, k, NT) * 64 + chunk_off(r, q));
#pragma unroll
                for (int kk = 0; kk < 2; ++kk) {
#pragma unroll
                  for (int t = 0; t < kJT; ++t)
                    if (I0 + t < NT)
                      mma(acc[t][0], acc[t][1], neg(kk ? a[t].y : a[t].x), kk ? bb.y : bb.x);
                }
              }
            }
#pragma unroll
            for (int t = 0; t < kJT; ++t)
              if (I0 + t < NT) st2(T + tidx(I0 + t, c, NT) * 64 + chunk_off(r, q), acc[t][0], acc[t][1]);
          }
        }
        bar_group(bar_id);
        mark(2 + 3 * c);
        // ================= 2. diagonal tiles: one lane per block
        if (gw == 0 && lane < kGroupBlocks) {
          const int b = lane;
          const double* dt = T_of(b) + tidx(c, c, NT) * 64;
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
          int fl = -1;
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            if (j < jmax) {
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
          double* LD = LD_of(b);
#pragma unroll
          for (int i = 0; i < 8; ++i) {
#pragma unroll
            for (int j = 0; j <= i; ++j) LD[i * 8 + j] = d[i][j];
          }
          double* SC = SC_of(b);
          if (fl >= 0 && SC[3] < 0.0) SC[3] = (double)(R0 + fl);
          if (lastc) {
            const int cs = m - R0;
#pragma unroll
            for (int x = 0; x < 8; ++x) {
              if (x == cs) SC[0] = d[x][x];
              if (x + 1 < 8 && x == cs) SC[1] = d[x + 1][x];
            }
          }
        }
        bar_group(bar_id);
        mark(3 + 3 * c);
        // ================= 3. rows below the diagonal tiles: one thread per row
        {
          const int b = gt >> 6, lr = gt & 63;
          const int NB = P - R0 - 8;
          if (lr < NB) {
            const int I = c + 1 + (lr >> 3), rw = lr & 7;
            double* rb = T_of(b) + tidx(I, c, NT) * 64;
            const double* LD = LD_of(b);
            double a[8];
#pragma unroll
            for (int x = 0; x < 4; ++x) {
              const double2 v = ld2(rb + chunk_off(rw, x));
              a[2 * x] = v.x;
              a[2 * x + 1] = v.y;
            }
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              if (j < jmax) {
                a[j] *= LD[j * 8 + j];
#pragma unroll
                for (int jp = j + 1; jp < 8; ++jp) a[jp] = fma(-a[j], LD[jp * 8 + j], a[jp]);
              }
            }
            if (!lastc) {
#pragma unroll
              for (int x = 0; x < 4; ++x) st2(rb + chunk_off(rw, x), a[x], a[x + 4]);
            } else if (8 * I + rw == m + 1) {
              const int cs = m - R0;
#pragma unroll
              for (int x = 0; x < 8; ++x)
                if (x == cs) SC_of(b)[1] = a[x];
            }
          }
        }
        bar_group(bar_id);
        mark(4 + 3 * c);
      }
    }
    // ---- epilogue: the blocks' log-densities (vg/vecchia.py:186-189, :206-213)
    if (gw == 0 && lane < kGroupBlocks) {
      const int64_t e = base + lane;
      if (e < e_hi) {
        const double* SC = SC_of(lane);
        const int64_t kk = e - 1 - rest_lo;
        if (SC[3] >= 0.0) {
          atomicMin(&fail[0], npd_key(e, (int)SC[3], m));
        } else {
          const double sg = SC[0], mu = -SC[1];
          mu_out[kk] = mu;
          sig_out[kk] = sg;
          if (!(sg > 0.0)) {
            atomicMin(&fail[1], (unsigned long long)e);
            rest[kk] = 0.0;
          } else {
            const double resid = SC[2] - mu;
            rest[kk] = -0.5 * (resid * resid / sg + kLog2Pi + log(sg));
          }
        }
      }
    }
    // the next round's staging overwrites T, O, SC: everyone is past them
    bar_group(bar_id);
  }
}

template <int NT, int KIND, int MC, bool TRACE = false>
cudaError_t launch(const Plan& p, const CovParams& cp, int64_t e_lo, int64_t e_hi,
                   cudaStream_t stream, long long* trace = nullptr) {
  constexpr SlotLayout L = slot_layout(NT);
  const size_t sm = sizeof(double) * ((size_t)kHead + (size_t)kSlots * L.stride) + 8 * kGroups;
  static size_t configured[64] = {};
  const int dev = p.device & 63;
  auto kern = loglik_grp_kernel<NT, KIND, MC, TRACE>;
  if (configured[dev] < sm) {
    cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (err != cudaSuccess) return err;
    configured[dev] = sm;
  }
  const int64_t count = e_hi - e_lo;
  const int64_t want = (count + kSlots - 1) / kSlots;
  const int64_t cap = (int64_t)p.num_sms;  // one CTA per SM
  const int grid = (int)(want < cap ? want : cap);
  kern<<<grid, kThreads, sm, stream>>>(p.d_pts, p.d_nbr, p.m, e_lo, e_hi, p.rest_lo, cp.s2,
                                       cp.inv_beta, p.d_rest, p.d_mu, p.d_sig, p.d_fail,
                                       p.d_dcache, p.dcache_stride, trace);
  return cudaGetLastError();
}

// VGP_TRACEG=<file>: one traced launch (m = 60, nu = 1.5) appends the clock64
// timeline [group][round][event] of CTA 0 (tools/grp_trace.py)
inline cudaError_t launch_traced(const Plan& p, const CovParams& cp, int64_t e_lo, int64_t e_hi,
                                 cudaStream_t stream, const char* path) {
  const size_t n = (size_t)kGroups * kTraceRounds * kTraceEvents;
  long long* d = nullptr;
  cudaError_t err = cudaMalloc(&d, n * sizeof(long long));
  if (err != cudaSuccess) return err;
  cudaMemsetAsync(d, 0, n * sizeof(long long), stream);
  err = launch<8, kMatern15, 60, true>(p, cp, e_lo, e_hi, stream, d);
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

template <int KIND>
cudaError_t launch_kind(const Plan& p, const CovParams& cp, int64_t e_lo, int64_t e_hi,
                        cudaStream_t stream) {
  if (p.m < 8 || p.m + 2 > 64 || !p.d_dcache) return cudaErrorNotSupported;
  if (p.m == 60) {
    if (KIND == kMatern15)
      if (const char* path = std::getenv("VGP_TRACEG")) return launch_traced(p, cp, e_lo, e_hi, stream, path);
    return launch<8, KIND, 60>(p, cp, e_lo, e_hi, stream);
  }
  switch ((p.m + 2 + 7) / 8) {
    case 2: return launch<2, KIND, 0>(p, cp, e_lo, e_hi, stream);
    case 3: return launch<3, KIND, 0>(p, cp, e_lo, e_hi, stream);
    case 4: return launch<4, KIND, 0>(p, cp, e_lo, e_hi, stream);
    case 5: return launch<5, KIND, 0>(p, cp, e_lo, e_hi, stream);
    case 6: return launch<6, KIND, 0>(p, cp, e_lo, e_hi, stream);
    case 7: return launch<7, KIND, 0>(p, cp, e_lo, e_hi, stream);
    case 8: return launch<8, KIND, 0>(p, cp, e_lo, e_hi, stream);
    default: return cudaErrorNotSupported;
  }
}

}  // namespace grp
}  // namespace vgp
