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

#include <cub/device/device_radix_sort.cuh>

#include "vgp_internal.cuh"

namespace cg = cooperative_groups;

namespace vgp {
namespace {

constexpr int kCtas = 8;        // cluster size (portable maximum)
constexpr int kThreads = 1024;  // per CTA
constexpr int kWarps = kThreads / 32;
constexpr int kChunk = 256;     // points per chunk (8 per lane)
constexpr int kPer = kChunk / 32;
constexpr int kMaxChunksPerCta = 3200;  // 64 B of metadata each -> 200 KB

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

// Chunk metadata, structure of arrays in dynamic shared memory.
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

__global__ void __cluster_dims__(kCtas, 1, 1) __launch_bounds__(kThreads, 1)
maxmin_cluster_kernel(const double2* __restrict__ spts, const int32_t* __restrict__ orig,
                      double* __restrict__ dist, int64_t n, const int32_t* __restrict__ first_pos,
                      int64_t* __restrict__ order, int cpc) {
  cg::cluster_group cluster = cg::this_cluster();
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ Cand slot[2];
  __shared__ Cand red[kWarps];
  const int rank = (int)cluster.block_rank();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t nchunks = (n + kChunk - 1) / kChunk;
  const int64_t c_base = (int64_t)rank * cpc;
  const int64_t left = nchunks - c_base;
  const int my_chunks = left <= 0 ? 0 : (int)(left < cpc ? left : cpc);
  Meta mt(smem, cpc);
  const double kInf = __longlong_as_double(0x7ff0000000000000ll);

  // setup: bounding boxes, dist = +inf; chunk j (local) is owned by lane
  // (j % 32) of warp ((j / 32) % kWarps)
  for (int j0 = warp * 32; j0 < my_chunks; j0 += kThreads) {
    for (int jj = 0; jj < 32 && j0 + jj < my_chunks; ++jj) {
      const int64_t c = c_base + j0 + jj;
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
        const int j = j0 + jj;
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
  __syncthreads();

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
  for (int64_t t = 0; t < n; ++t) {
    if (rank == 0 && threadIdx.x == 0) order[t] = cur.orig;
    const int64_t cur_chunk = cur.pos / kChunk;
    Cand best{-1.0, 0.0, 0.0, INT32_MAX, -1};
    for (int ps = 0; ps < passes; ++ps) {
      const int j = ps * kThreads + warp * 32 + lane;
      bool hit = false;
      if (j < my_chunks) {
        const double cd = mt.cd[j];
        if (c_base + j == cur_chunk) {
          hit = true;
        } else if (cd >= 0.0) {
          const double gx = fmax(fmax(__dsub_rn(mt.bx0[j], cur.x), __dsub_rn(cur.x, mt.bx1[j])), 0.0);
          const double gy = fmax(fmax(__dsub_rn(mt.by0[j], cur.y), __dsub_rn(cur.y, mt.by1[j])), 0.0);
          hit = __dadd_rn(__dmul_rn(gx, gx), __dmul_rn(gy, gy)) < cd;
        }
      }
      unsigned mask = __ballot_sync(0xffffffffu, hit);
      while (mask) {
        const int src = __ffs(mask) - 1;
        mask &= mask - 1;
        const int64_t c = c_base + ps * kThreads + warp * 32 + src;
        Cand lb{-1.0, 0.0, 0.0, INT32_MAX, -1};
#pragma unroll
        for (int k = 0; k < kPer; ++k) {
          const int64_t pos = c * kChunk + lane + 32 * k;
          if (pos < n) {
            double d0 = dist[pos];
            if (d0 >= 0.0) {
              const double2 p = spts[pos];
              if (pos == cur.pos) {
                d0 = -1.0;
                dist[pos] = d0;
              } else {
                const double d = key2(p.x, p.y, cur.x, cur.y);
                if (d < d0) {
                  d0 = d;
                  dist[pos] = d0;
                }
                const int32_t o = orig[pos];
                if (better(d0, o, lb.d, lb.orig)) lb = Cand{d0, p.x, p.y, o, (int32_t)pos};
              }
            }
          }
        }
        // chunk winner: reduce (d, orig), then fetch its coordinates from the
        // lane holding it (that lane's local best is the winner)
        Cand w = warp_best(lb);
        const unsigned own = __ballot_sync(0xffffffffu, lb.orig == w.orig && lb.d == w.d && lb.pos >= 0);
        Cand full = lb;
        shfl_cand(full, own ? __ffs(own) - 1 : 0);
        if (!own) full = Cand{-1.0, 0.0, 0.0, INT32_MAX, -1};
        if (lane == src) {
          const int jj = ps * kThreads + warp * 32 + src;
          mt.cd[jj] = full.d;
          mt.cx[jj] = full.x;
          mt.cy[jj] = full.y;
          mt.co[jj] = full.orig;
          mt.cp[jj] = full.pos;
        }
      }
      if (j < my_chunks) {
        const double cd = mt.cd[j];
        const int32_t co = mt.co[j];
        if (cd >= 0.0 && better(cd, co, best.d, best.orig)) best = Cand{cd, mt.cx[j], mt.cy[j], co, mt.cp[j]};
      }
    }
    // CTA candidate
    {
      Cand w = warp_best(best);
      const unsigned own = __ballot_sync(0xffffffffu, best.orig == w.orig && best.d == w.d && best.pos >= 0);
      Cand full = best;
      shfl_cand(full, own ? __ffs(own) - 1 : 0);
      if (!own) full = Cand{-1.0, 0.0, 0.0, INT32_MAX, -1};
      if (lane == 0) red[warp] = full;
    }
    __syncthreads();
    if (warp == 0) {
      Cand c = red[lane];
      Cand w = warp_best(c);
      const unsigned own = __ballot_sync(0xffffffffu, c.orig == w.orig && c.d == w.d && c.pos >= 0);
      Cand full = c;
      shfl_cand(full, own ? __ffs(own) - 1 : 0);
      if (!own) full = Cand{-1.0, 0.0, 0.0, INT32_MAX, -1};
      if (lane == 0) slot[t & 1] = full;
    }
    cluster.sync();
    // every warp reduces the kCtas CTA candidates itself (no CTA barrier)
    {
      Cand c{-1.0, 0.0, 0.0, INT32_MAX, -1};
      if (lane < kCtas) {
        const Cand* rs = cluster.map_shared_rank(&slot[t & 1], lane);
        c = *rs;
      }
      Cand w = warp_best(c);
      const unsigned own = __ballot_sync(0xffffffffu, c.orig == w.orig && c.d == w.d && c.pos >= 0);
      Cand full = c;
      shfl_cand(full, own ? __ffs(own) - 1 : 0);
      cur = full;
      if (!own) break;  // nothing left (cannot happen before t == n - 1)
    }
  }
  cluster.sync();  // keep shared memory alive until every remote read is done
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
  const size_t dyn = (size_t)cpc * 64;
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(maxmin_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
  if (e == cudaSuccess) {
    maxmin_cluster_kernel<<<kCtas, kThreads, dyn, stream>>>(spts, idx2, dist, n, fpos, d_order, cpc);
    e = cudaGetLastError();
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
