// Exact maxmin ordering on the GPU (BASELINE config 5; the reference has only
// random / Morton / identity orderings, vg/vecchia.py:37, so this is new and
// pinned by a brute-force restatement in the tests, not by the reference).
//
// Definition (Guinness 2018): the first point is given (the caller passes
// the one nearest the centroid); then repeatedly the unselected point whose
// squared distance to the selected set is largest, ties to the smallest
// index.  Squared distances are dx*dx + dy*dy with every operation rounded
// (no FMA), so the numpy restatement reproduces the order bit for bit.
//
// The selection is inherently sequential (n steps), so the design minimises
// the per-step critical path rather than the work:
//  * points are sorted by Morton code (CUB radix sort) and cut into chunks of
//    kChunk consecutive points; each chunk keeps in shared memory its
//    bounding box and its best candidate (largest distance, smallest index);
//  * one cluster of kCtas CTAs owns all chunks (lane-owned, registers-free
//    metadata in shared memory); in step t a chunk is touched only when a
//    lower bound of the new point's distance to its box is below the chunk's
//    best distance (rounding is monotone, so the bound is conservative and
//    the skipped chunks provably do not change), i.e. a handful of chunks per
//    step once the ordering is past its first few hundred points;
//  * the CTA candidates are exchanged through distributed shared memory with
//    one cluster barrier per step (double-buffered by step parity).
#include <cooperative_groups.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#include <cub/device/device_radix_sort.cuh>

#include "vgp_internal.cuh"

namespace cg = cooperative_groups;

namespace vgp {
namespace {

constexpr int kCtas = 8;        // cluster size (portable maximum)
constexpr int kThreads = 512;   // per CTA (128 registers: a chunk's loads all in flight)
constexpr int kWarps = kThreads / 32;
constexpr int kChunk = 256;     // points per chunk (8 per lane)
constexpr int kPer = kChunk / 32;
constexpr int kMaxChunksPerCta = 3200;  // 64 B of metadata each (+1/16 padding) -> 213 KB

struct Cand {
  double d, x, y;
  int32_t orig, pos;
};

__device__ __forceinline__ bool better(double d, int32_t o, double bd, int32_t bo) {
  return d > bd || (d == bd && o < bo);
}

__device__ __forceinline__ double key2(double x, double y, double cx, double cy) {
  const double dx = __dsub_rn(x, cx);
  const double dy = __dsub_rn(y, cy);
  return __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy));
}

__device__ __forceinline__ void shfl_cand(Cand& c, int src) {
  c.d = __shfl_sync(0xffffffffu, c.d, src);
  c.x = __shfl_sync(0xffffffffu, c.x, src);
  c.y = __shfl_sync(0xffffffffu, c.y, src);
  c.orig = __shfl_sync(0xffffffffu, c.orig, src);
  c.pos = __shfl_sync(0xffffffffu, c.pos, src);
}

// Warp argmax of (d desc, orig asc); every lane ends with the winner.
__device__ __forceinline__ Cand warp_best(Cand c) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const double od = __shfl_xor_sync(0xffffffffu, c.d, off);
    const int32_t oo = __shfl_xor_sync(0xffffffffu, c.orig, off);
    if (better(od, oo, c.d, c.orig)) {
      c.d = od;
      c.orig = oo;
    }
  }
  return c;
}

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ uint32_t map_rank(uint32_t a, int rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}

// 16 bytes into a peer CTA's shared memory, completing 16 tx bytes on its
// mbarrier (both addresses shared::cluster).
__device__ __forceinline__ void st_async16(uint32_t raddr, uint64_t a, uint64_t b, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.b64 [%0], {%1, %2}, [%3];"
               :: "r"(raddr), "l"(a), "l"(b), "r"(rbar) : "memory");
}

__device__ __forceinline__ void mbar_wait_parity(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "W: mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra W;\n}\n" :: "r"(bar), "r"(parity) : "memory");
}

// Warp argmax with the winner's full record on every lane (kNone-like
// record with pos -1 when no lane holds a candidate).
__device__ __forceinline__ Cand warp_winner(const Cand& c) {
  const Cand w = warp_best(c);
  const unsigned own = __ballot_sync(0xffffffffu, c.orig == w.orig && c.d == w.d && c.pos >= 0);
  Cand full = c;
  shfl_cand(full, own ? __ffs(own) - 1 : 0);
  if (!own) full = Cand{-1.0, 0.0, 0.0, INT32_MAX, -1};
  return full;
}

// Morton code of (x, y) on a 2^21 x 2^21 grid over the bounding box.
__device__ __forceinline__ uint64_t spread21(uint64_t v) {
  v &= 0x1fffffull;  // 21 bits -> even bit positions 0..40
  v = (v | v << 16) & 0x0000ffff0000ffffull;
  v = (v | v << 8) & 0x00ff00ff00ff00ffull;
  v = (v | v << 4) & 0x0f0f0f0f0f0f0f0full;
  v = (v | v << 2) & 0x3333333333333333ull;
  v = (v | v << 1) & 0x5555555555555555ull;
  return v;
}

__global__ void morton_kernel(const double2* __restrict__ pts, int64_t n, double x0, double sx, double y0,
                              double sy, uint64_t* __restrict__ code, int32_t* __restrict__ idx) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double2 p = pts[i];
  const double fx = (p.x - x0) * sx, fy = (p.y - y0) * sy;
  const uint64_t qx = (uint64_t)fmin(fmax(fx, 0.0), 2097151.0);
  const uint64_t qy = (uint64_t)fmin(fmax(fy, 0.0), 2097151.0);
  code[i] = spread21(qx) | spread21(qy) << 1;
  idx[i] = (int32_t)i;
}

__global__ void gather_kernel(const double2* __restrict__ pts, const int32_t* __restrict__ idx, int64_t n,
                              int64_t first, double2* __restrict__ spts, int32_t* __restrict__ first_pos) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int32_t o = idx[i];
  spts[i] = pts[o];
  if (o == first) *first_pos = (int32_t)i;
}

// Chunk metadata, structure of arrays in dynamic shared memory.  Local chunk
// j is owned by warp j % kWarps, lane (j / kWarps) % 32, so a warp's lanes
// read chunks kWarps apart; chunk j lives at slot j + j / kWarps (one pad
// entry per kWarps keeps those reads on distinct banks).
__device__ __forceinline__ int mslot(int j) { return j + j / kWarps; }
__host__ __device__ constexpr int meta_slots(int cpc) { return cpc + cpc / kWarps + 1; }

struct Meta {
  double *bx0, *bx1, *by0, *by1, *cd, *cx, *cy;
  int32_t *co, *cp;
  __device__ Meta(unsigned char* base, int cap) {
    double* d = reinterpret_cast<double*>(base);
    bx0 = d;
    bx1 = d + cap;
    by0 = d + 2 * cap;
    by1 = d + 3 * cap;
    cd = d + 4 * cap;
    cx = d + 5 * cap;
    cy = d + 6 * cap;
    co = reinterpret_cast<int32_t*>(d + 7 * cap);
    cp = co + cap;
  }
};

// Phase trace (env VGP_MM_TRACE=<file>, diagnostics only): per CTA and
// step in [n/2, n/2 + kTraceSteps), clock64 at step start, last warp done
// with its chunks, after the CTA barrier, slot written, after the cluster
// wait, next point known; plus the CTA's number of chunk updates.
constexpr int kTraceSteps = 256, kTraceEv = 8;

template <bool TRACE>
__global__ void __cluster_dims__(kCtas, 1, 1) __launch_bounds__(kThreads, 1)
maxmin_cluster_kernel(const double2* __restrict__ spts, const int32_t* __restrict__ orig,
                      double* __restrict__ dist, int64_t n, const int32_t* __restrict__ first_pos,
                      int64_t* __restrict__ order, int cpc, long long* __restrict__ trace) {
  __shared__ unsigned long long tr_done, tr_ld;
  __shared__ int tr_hits;
  cg::cluster_group cluster = cg::this_cluster();
  extern __shared__ __align__(16) unsigned char smem[];
  // inbox[b][r]: CTA r's candidate of the last step with parity b, pushed
  // by CTA r itself (st.async); mbar[b] completes when all kCtas arrived
  __shared__ __align__(16) double inbox[2][kCtas][4];
  __shared__ __align__(8) unsigned long long mbar[2];
  __shared__ Cand red[kWarps];
  const int rank = (int)cluster.block_rank();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t nchunks = (n + kChunk - 1) / kChunk;
  const int64_t c_base = (int64_t)rank * cpc;
  const int64_t left = nchunks - c_base;
  const int my_chunks = left <= 0 ? 0 : (int)(left < cpc ? left : cpc);
  Meta mt(smem, meta_slots(cpc));
  const double kInf = __longlong_as_double(0x7ff0000000000000ll);
  if (threadIdx.x == 0) {
    for (int b = 0; b < 2; ++b)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_addr(&mbar[b])) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }

  // setup: bounding boxes, dist = +inf; local chunk j is owned by warp
  // j % kWarps, lane (j / kWarps) % 32 (neighbouring chunks, which a new
  // point tends to hit together, land in different warps and are updated in
  // parallel)
  for (int j0 = warp; j0 < my_chunks; j0 += kThreads) {
    for (int jj = 0; jj < 32 && j0 + jj * kWarps < my_chunks; ++jj) {
      const int64_t c = c_base + j0 + jj * kWarps;
      double ax0 = kInf, ax1 = -kInf, ay0 = kInf, ay1 = -kInf;
#pragma unroll
      for (int k = 0; k < kPer; ++k) {
        const int64_t pos = c * kChunk + lane + 32 * k;
        if (pos < n) {
          const double2 p = spts[pos];
          ax0 = fmin(ax0, p.x);
          ax1 = fmax(ax1, p.x);
          ay0 = fmin(ay0, p.y);
          ay1 = fmax(ay1, p.y);
          dist[pos] = kInf;
        }
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        ax0 = fmin(ax0, __shfl_xor_sync(0xffffffffu, ax0, off));
        ax1 = fmax(ax1, __shfl_xor_sync(0xffffffffu, ax1, off));
        ay0 = fmin(ay0, __shfl_xor_sync(0xffffffffu, ay0, off));
        ay1 = fmax(ay1, __shfl_xor_sync(0xffffffffu, ay1, off));
      }
      if (lane == jj) {
        const int j = mslot(j0 + jj * kWarps);
        mt.bx0[j] = ax0;
        mt.bx1[j] = ax1;
        mt.by0[j] = ay0;
        mt.by1[j] = ay1;
        mt.cd[j] = kInf;
        mt.cx[j] = mt.cy[j] = 0.0;
        mt.co[j] = INT32_MAX;
        mt.cp[j] = -1;
      }
    }
  }
  cluster.sync();  // barriers initialised cluster-wide, metadata ready

  Cand cur;
  cur.pos = *first_pos;
  {
    const double2 p = spts[cur.pos];
    cur.x = p.x;
    cur.y = p.y;
    cur.orig = orig[cur.pos];
    cur.d = kInf;
  }
  const int passes = (my_chunks + kThreads - 1) / kThreads;
  const Cand kNone{-1.0, 0.0, 0.0, INT32_MAX, -1};
  if (lane == 0) red[warp] = kNone;
  Cand cta_best = kNone;  // warp 0: this CTA's cached candidate
  __syncthreads();
  for (int64_t t = 0; t < n; ++t) {
    const int64_t ts = t - n / 2;
    const bool tr = TRACE && ts >= 0 && ts < kTraceSteps;
    long long* trow = tr ? trace + ((int64_t)rank * kTraceSteps + ts) * kTraceEv : nullptr;
    if (tr && threadIdx.x == 0) {
      trow[0] = clock64();
      tr_done = 0;
      tr_ld = 0;
      tr_hits = 0;
    }
    if (TRACE) __syncthreads();
    if (rank == 0 && threadIdx.x == 32) order[t] = cur.orig;
    if (threadIdx.x == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
                   :: "r"(smem_addr(&mbar[t & 1])), "r"(kCtas * 32) : "memory");
    const int64_t cur_chunk = cur.pos / kChunk;
    bool warp_changed = false;
    for (int ps = 0; ps < passes; ++ps) {
      const int j = ps * kThreads + lane * kWarps + warp;  // chunk
      const int js = mslot(j);                          // its metadata slot
      bool hit = false;
      if (j < my_chunks) {
        const double cd = mt.cd[js];
        if (c_base + j == cur_chunk) {
          hit = true;
        } else if (cd >= 0.0) {
          const double gx = fmax(fmax(__dsub_rn(mt.bx0[js], cur.x), __dsub_rn(cur.x, mt.bx1[js])), 0.0);
          const double gy = fmax(fmax(__dsub_rn(mt.by0[js], cur.y), __dsub_rn(cur.y, mt.by1[js])), 0.0);
          hit = __dadd_rn(__dmul_rn(gx, gx), __dmul_rn(gy, gy)) < cd;
        }
      }
      unsigned mask = __ballot_sync(0xffffffffu, hit);
      if (tr && lane == 0) atomicAdd(&tr_hits, __popc(mask));
      warp_changed |= mask != 0;
      while (mask) {
        const int src = __ffs(mask) - 1;
        mask &= mask - 1;
        const int64_t c = c_base + ps * kThreads + src * kWarps + warp;
        // all loads first (one L2 round trip), then the updates
        double d0[kPer];
        double2 pt[kPer];
        int32_t o[kPer];
#pragma unroll
        for (int k = 0; k < kPer; ++k) {
          const int64_t pos = c * kChunk + lane + 32 * k;
          d0[k] = -1.0;
          if (pos < n) {
            d0[k] = __ldcg(dist + pos);
            pt[k] = __ldcg(spts + pos);
            o[k] = __ldcg(orig + pos);
          }
        }
        Cand lb = kNone;
#pragma unroll
        for (int k = 0; k < kPer; ++k) {
          const int64_t pos = c * kChunk + lane + 32 * k;
          if (d0[k] >= 0.0) {
            if (pos == cur.pos) {
              dist[pos] = -1.0;
            } else {
              const double d = key2(pt[k].x, pt[k].y, cur.x, cur.y);
              double dn = d0[k];
              if (d < dn) {
                dn = d;
                dist[pos] = dn;
              }
              if (better(dn, o[k], lb.d, lb.orig)) lb = Cand{dn, pt[k].x, pt[k].y, o[k], (int32_t)pos};
            }
          }
        }
        if (tr && lane == 0) atomicMax(&tr_ld, (unsigned long long)clock64());
        const Cand full = warp_winner(lb);
        if (lane == src) {
          const int jj = mslot(ps * kThreads + src * kWarps + warp);
          mt.cd[jj] = full.d;
          mt.cx[jj] = full.x;
          mt.cy[jj] = full.y;
          mt.co[jj] = full.orig;
          mt.cp[jj] = full.pos;
        }
      }
    }
    // this warp's candidate changes only when one of its chunks did
    if (warp_changed) {
      Cand best = kNone;
      for (int ps = 0; ps < passes; ++ps) {
        const int j = ps * kThreads + lane * kWarps + warp;
        if (j < my_chunks) {
          const int js = mslot(j);
          const double cd = mt.cd[js];
          const int32_t co = mt.co[js];
          if (cd >= 0.0 && better(cd, co, best.d, best.orig)) best = Cand{cd, mt.cx[js], mt.cy[js], co, mt.cp[js]};
        }
      }
      const Cand full = warp_winner(best);
      if (lane == 0) red[warp] = full;
    }
    if (tr && lane == 0) atomicMax(&tr_done, (unsigned long long)clock64());
    const int cta_changed = __syncthreads_or(warp_changed);
    if (tr && threadIdx.x == 0) trow[2] = clock64();
    if (warp == 0) {
      if (cta_changed) cta_best = warp_winner(lane < kWarps ? red[lane] : kNone);
      // push this CTA's candidate into every CTA's inbox (lane r -> rank r)
      if (lane < kCtas) {
        const uint32_t dst = map_rank(smem_addr(&inbox[t & 1][rank][0]), lane);
        const uint32_t bar = map_rank(smem_addr(&mbar[t & 1]), lane);
        const uint64_t op = ((uint64_t)(uint32_t)cta_best.pos << 32) | (uint32_t)cta_best.orig;
        st_async16(dst, __double_as_longlong(cta_best.d), __double_as_longlong(cta_best.x), bar);
        st_async16(dst + 16, __double_as_longlong(cta_best.y), op, bar);
      }
      if (tr && lane == 0) trow[3] = clock64();
    }
    // every warp sleeps on the local mbarrier until all kCtas candidates of
    // this step have landed, then reduces them from local shared memory
    mbar_wait_parity(smem_addr(&mbar[t & 1]), (uint32_t)((t >> 1) & 1));
    if (tr && threadIdx.x == 0) trow[4] = clock64();
    {
      Cand c = kNone;
      if (lane < kCtas) {
        const double* e = inbox[t & 1][lane];
        const uint64_t op = (uint64_t)__double_as_longlong(e[3]);
        c = Cand{e[0], e[1], e[2], (int32_t)(uint32_t)op, (int32_t)(op >> 32)};
      }
      cur = warp_winner(c);
      if (tr && threadIdx.x == 0) {
        trow[5] = clock64();
        trow[1] = (long long)tr_done;
        trow[6] = tr_hits;
        trow[7] = (long long)tr_ld;
      }
      if (cur.pos < 0) break;  // nothing left (t == n - 1)
    }
  }
  cluster.sync();  // no CTA exits while a peer may still push into it
}

}  // namespace

int64_t maxmin_capacity() { return (int64_t)kCtas * kMaxChunksPerCta * kChunk; }

cudaError_t launch_maxmin(const double2* d_pts, int64_t n, int64_t first, const double bbox[4],
                          int64_t* d_order, cudaStream_t stream) {
  if (n > maxmin_capacity() || n >= INT32_MAX) return cudaErrorInvalidValue;
  // Morton grid over the bounding box (only the chunking, not the result,
  // depends on it)
  const int bs = 256;
  const int64_t nb = (n + bs - 1) / bs;
  const double x0 = bbox[0], x1 = bbox[1], y0 = bbox[2], y1 = bbox[3];
  cudaError_t e = cudaSuccess;
  const double sx = x1 > x0 ? 2097152.0 / (x1 - x0) : 0.0;
  const double sy = y1 > y0 ? 2097152.0 / (y1 - y0) : 0.0;

  uint64_t *code = nullptr, *code2 = nullptr;
  int32_t *idx = nullptr, *idx2 = nullptr, *fpos = nullptr;
  double2* spts = nullptr;
  double* dist = nullptr;
  void* tmp = nullptr;
  size_t tmp_bytes = 0;
  if (e == cudaSuccess) e = cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, code, code2, idx, idx2, (int)n, 0, 42, stream);
  auto A = [&](void** p, size_t b) {
    if (e == cudaSuccess) e = cudaMallocAsync(p, b ? b : 1, stream);
  };
  A((void**)&code, sizeof(uint64_t) * n);
  A((void**)&code2, sizeof(uint64_t) * n);
  A((void**)&idx, sizeof(int32_t) * n);
  A((void**)&idx2, sizeof(int32_t) * n);
  A((void**)&fpos, sizeof(int32_t));
  A((void**)&spts, sizeof(double2) * n);
  A((void**)&dist, sizeof(double) * n);
  A(&tmp, tmp_bytes);
  if (e == cudaSuccess) {
    morton_kernel<<<(unsigned)nb, bs, 0, stream>>>(d_pts, n, x0, sx, y0, sy, code, idx);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess)
    e = cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, code, code2, idx, idx2, (int)n, 0, 42, stream);
  if (e == cudaSuccess) {
    gather_kernel<<<(unsigned)nb, bs, 0, stream>>>(d_pts, idx2, n, first, spts, fpos);
    e = cudaGetLastError();
  }
  const int64_t nchunks = (n + kChunk - 1) / kChunk;
  const int cpc = (int)std::max<int64_t>(32, (nchunks + kCtas - 1) / kCtas);
  const size_t dyn = (size_t)meta_slots(cpc) * 64;
  const char* trace_path = std::getenv("VGP_MM_TRACE");
  long long* d_trace = nullptr;
  const size_t tn = (size_t)kCtas * kTraceSteps * kTraceEv;
  if (trace_path && e == cudaSuccess) {
    e = cudaMallocAsync((void**)&d_trace, tn * sizeof(long long), stream);
    if (e == cudaSuccess) e = cudaMemsetAsync(d_trace, 0, tn * sizeof(long long), stream);
  }
  auto kern = trace_path ? maxmin_cluster_kernel<true> : maxmin_cluster_kernel<false>;
  if (e == cudaSuccess) e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
  if (e == cudaSuccess) {
    kern<<<kCtas, kThreads, dyn, stream>>>(spts, idx2, dist, n, fpos, d_order, cpc, d_trace);
    e = cudaGetLastError();
  }
  if (d_trace) {
    std::vector<long long> h(tn);
    if (e == cudaSuccess) e = cudaMemcpyAsync(h.data(), d_trace, tn * sizeof(long long), cudaMemcpyDeviceToHost, stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
    if (e == cudaSuccess)
      if (FILE* f = std::fopen(trace_path, "a")) {
        for (size_t i = 0; i < tn; ++i) std::fprintf(f, "%lld%c", h[i], (i + 1) % kTraceEv ? ' ' : '\n');
        std::fclose(f);
      }
    cudaFreeAsync(d_trace, stream);
  }
  cudaFreeAsync(code, stream);
  cudaFreeAsync(code2, stream);
  cudaFreeAsync(idx, stream);
  cudaFreeAsync(idx2, stream);
  cudaFreeAsync(fpos, stream);
  cudaFreeAsync(spts, stream);
  cudaFreeAsync(dist, stream);
  cudaFreeAsync(tmp, stream);
  return e;
}

}  // namespace vgp
