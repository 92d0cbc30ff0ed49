// Exact m-nearest-neighbour search, bit-exact with the reference's numba scan
// geo._topm_plane (vg/geo.py:234-263):
//   key  = dx*dx + dy*dy  with dx = x_j - x_t, each op rounded (no FMA),
//   keep the m smallest by (key, j); a candidate tying the current worst is
//   rejected; insertion keeps equal keys in ascending-index order.
// Candidates are streamed in ascending j through shared memory; every thread
// owns one query and keeps only its admission threshold (the current m-th
// key) in a register.  The sorted top-m list lives in a global scratch laid
// out [slot][query] so the rare insertions stay coalesced across a warp.
#include <algorithm>
#include <cmath>

#include <cub/device/device_radix_sort.cuh>

#include "vgp_internal.cuh"

namespace vgp {

namespace {

constexpr int kKnnThreads = 128;
constexpr int kKnnTile = 1024;  // candidates per shared-memory tile (16 KiB)

__device__ __forceinline__ double knn_key(double2 c, double2 t) {
  double dx = __dsub_rn(c.x, t.x);
  double dy = __dsub_rn(c.y, t.y);
  return __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy));
}

// geo._topm_sphere (vg/geo.py:266-292): points are (lambda, phi, cos phi) in
// radians, computed on the host with numpy exactly as the reference's
// _topm_scan does (vg/geo.py:305-310); key = haversine of the central angle
//   sp * sp + ((cos_t * cos_j) * sl) * sl,  sp = sin((phi_j - phi_t) / 2),
//   sl = sin((lambda_j - lambda_t) / 2), every op rounded separately.
// CUDA's sin is within 1 ulp of glibc's (the reference's numba calls libm),
// so sphere neighbour sets are exact except for keys tied to the last ulp.
__device__ __forceinline__ double knn_key(double4 c, double4 t) {
  const double sp = sin(__dmul_rn(__dsub_rn(c.y, t.y), 0.5));
  const double sl = sin(__dmul_rn(__dsub_rn(c.x, t.x), 0.5));
  return __dadd_rn(__dmul_rn(sp, sp), __dmul_rn(__dmul_rn(__dmul_rn(t.z, c.z), sl), sl));
}

// pred != 0: query q (global index q_offset + q) is ordered target i = m + q
// (q_offset + q) and admits candidates j < i (nearest_neighbors, vg/geo.py:342).
// pred == 0: every candidate admissible (nearest_points, vg/geo.py:357).
// j_lo > 0 continues a search whose top-m state (cnt_in[q] entries, sorted by
// (key, index), all indices < j_lo) is already in the scratch: candidates
// j >= j_lo are larger than every stored index, so the ascending-j insertion
// rule below stays exactly the lexicographic (key, index) order.
template <typename PT>
__global__ void __launch_bounds__(kKnnThreads)
knn_kernel(const PT* __restrict__ data, int64_t nd, const PT* __restrict__ query,
           int64_t nq, int64_t q_offset, int pred, int m, int64_t* __restrict__ out,
           double* __restrict__ keys, int32_t* __restrict__ idx, int64_t j_lo,
           const int* __restrict__ cnt_in) {
  constexpr int kTile = kKnnTile * 16 / (int)sizeof(PT);
  __shared__ PT tile[kTile];
  const int64_t q = (int64_t)blockIdx.x * kKnnThreads + threadIdx.x;
  const bool active = q < nq;
  const int64_t stride = (int64_t)gridDim.x * kKnnThreads;  // slot stride in scratch
  PT pt{};
  int64_t limit = 0;
  if (active) {
    pt = query[q];
    limit = pred ? (q_offset + q + m) : nd;
  }
  // block-wide scan bound: the largest limit among this block's queries
  int64_t q_last = (int64_t)blockIdx.x * kKnnThreads + kKnnThreads - 1;
  if (q_last >= nq) q_last = nq - 1;
  const int64_t block_limit = pred ? (q_offset + q_last + m) : nd;

  double* kp = keys + q;   // keys[slot * stride + q]
  int32_t* ip = idx + q;
  int cnt = 0;
  double worst = __longlong_as_double(0x7ff0000000000000ll);  // +inf until full
  if (cnt_in && active) {
    cnt = cnt_in[q];
    if (cnt == m) worst = kp[(int64_t)(m - 1) * stride];
  }

  for (int64_t base = j_lo; base < block_limit; base += kTile) {
    int64_t tn = block_limit - base;
    if (tn > kTile) tn = kTile;
    __syncthreads();
    for (int t = threadIdx.x; t < tn; t += kKnnThreads) tile[t] = data[base + t];
    __syncthreads();
    if (!active) continue;
    int64_t jend = limit - base;
    if (jend > tn) jend = tn;
    for (int t = 0; t < jend; ++t) {
      double k = knn_key(tile[t], pt);
      if (cnt == m && !(k < worst)) continue;  // k >= keys[m-1] -> reject (vg/geo.py:252)
      int p;
      if (cnt == m) {
        p = m - 1;
      } else {
        p = cnt;
        cnt += 1;
      }
      while (p > 0) {
        double kq = kp[(int64_t)(p - 1) * stride];
        if (!(kq > k)) break;
        kp[(int64_t)p * stride] = kq;
        ip[(int64_t)p * stride] = ip[(int64_t)(p - 1) * stride];
        p -= 1;
      }
      kp[(int64_t)p * stride] = k;
      ip[(int64_t)p * stride] = (int32_t)(base + t);
      if (cnt == m) worst = kp[(int64_t)(m - 1) * stride];
    }
  }
  if (active) {
    int64_t* o = out + q * (int64_t)m;
    for (int s = 0; s < m; ++s) o[s] = (int64_t)ip[(int64_t)s * stride];
  }
}

// ---------------------------------------------------------------- grid search
// Exact predecessor kNN in index batches (targets [s, e)): each target t
// searches a uniform grid over the points [0, e) ring by ring, keeping the m
// smallest (key, index) pairs among the candidates j < t.  The search stops
// only when the current m-th key is strictly below a
// lower bound of every key outside the searched square: the bound is the
// target's distance to the square's boundary minus a slack that dominates
// the cell-assignment rounding, squared with the key's own rounding (which
// is monotone), so no candidate that could enter the top m is skipped and
// the result equals the brute-force scan bit for bit.

struct GridDesc {
  double x0, y0, hx, hy, ihx, ihy, slack;
  int g;  // g x g cells
};

__device__ __forceinline__ int cell_of(double v, double v0, double ih, int g) {
  const double f = floor((v - v0) * ih);
  return (int)fmin(fmax(f, 0.0), (double)(g - 1));
}

__global__ void grid_cell_kernel(const double2* __restrict__ pts, int64_t s, GridDesc gd,
                                 uint32_t* __restrict__ cell, int32_t* __restrict__ ids) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= s) return;
  const double2 p = pts[j];
  cell[j] = (uint32_t)(cell_of(p.y, gd.y0, gd.ihy, gd.g) * gd.g + cell_of(p.x, gd.x0, gd.ihx, gd.g));
  ids[j] = (int32_t)j;
}

__global__ void grid_bounds_kernel(const uint32_t* __restrict__ cell_sorted, int64_t s,
                                   int32_t* __restrict__ cstart, int32_t* __restrict__ cend) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= s) return;
  const uint32_t c = cell_sorted[p];
  if (p == 0 || cell_sorted[p - 1] != c) cstart[c] = (int32_t)p;
  if (p == s - 1 || cell_sorted[p + 1] != c) cend[c] = (int32_t)(p + 1);
}

__device__ __forceinline__ bool lex_less(double k, int32_t j, double kq, int32_t jq) {
  return k < kq || (k == kq && j < jq);
}

// the grid's points in cell order (coordinates next to their index), so a
// cell's candidates are one contiguous run
__global__ void grid_gather_kernel(const double2* __restrict__ pts, const int32_t* __restrict__ ids_sorted,
                                   int64_t s, double2* __restrict__ spts) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= s) return;
  spts[p] = pts[ids_sorted[p]];
}

// query q <-> ordered target t = t0 + q, candidates j < t only (the grid may
// hold later points of the batch); scratch [slot * stride + q]; the final
// table row goes to out[q * m ..]
__global__ void __launch_bounds__(kKnnThreads)
grid_query_kernel(const double2* __restrict__ pts, int64_t t0, int64_t nq, int m, GridDesc gd,
                  const int32_t* __restrict__ cstart, const int32_t* __restrict__ cend,
                  const int32_t* __restrict__ cpts, const double2* __restrict__ spts,
                  double* __restrict__ keys, int32_t* __restrict__ idx, int64_t stride,
                  int64_t* __restrict__ out) {
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nq) return;
  const int32_t t = (int32_t)(t0 + q);
  const double2 pt = pts[t];
  const int g = gd.g;
  const int cx = cell_of(pt.x, gd.x0, gd.ihx, g), cy = cell_of(pt.y, gd.y0, gd.ihy, g);
  double* kp = keys + q;
  int32_t* ip = idx + q;
  int cnt = 0;
  double wk = __longlong_as_double(0x7ff0000000000000ll);
  int32_t wj = INT32_MAX;
  const double inf = wk;
  for (int r = 0; r <= g; ++r) {
    if (r > 0) {
      // searched square: cells [cx - r + 1, cx + r - 1] x [cy - r + 1, cy + r - 1]
      const int lo_x = cx - r + 1, hi_x = cx + r - 1, lo_y = cy - r + 1, hi_y = cy + r - 1;
      if (lo_x <= 0 && hi_x >= g - 1 && lo_y <= 0 && hi_y >= g - 1) break;  // everything searched
      if (cnt == m) {
        double d = inf;
        if (lo_x > 0) d = fmin(d, __dsub_rn(pt.x, gd.x0 + lo_x * gd.hx));
        if (hi_x < g - 1) d = fmin(d, __dsub_rn(gd.x0 + (hi_x + 1) * gd.hx, pt.x));
        if (lo_y > 0) d = fmin(d, __dsub_rn(pt.y, gd.y0 + lo_y * gd.hy));
        if (hi_y < g - 1) d = fmin(d, __dsub_rn(gd.y0 + (hi_y + 1) * gd.hy, pt.y));
        d = fmax(d - gd.slack, 0.0);
        if (wk < __dmul_rn(d, d)) break;
      }
    }
    // ring r: rows cy - r and cy + r over [cx - r, cx + r], columns cx +- r over the rows between
    for (int side = 0; side < 4; ++side) {
      int ax, ay, dx, dy, len;
      if (r == 0) {
        if (side) break;
        ax = cx; ay = cy; dx = 1; dy = 0; len = 1;
      } else if (side == 0) { ax = cx - r; ay = cy - r; dx = 1; dy = 0; len = 2 * r + 1; }
      else if (side == 1) { ax = cx - r; ay = cy + r; dx = 1; dy = 0; len = 2 * r + 1; }
      else if (side == 2) { ax = cx - r; ay = cy - r + 1; dx = 0; dy = 1; len = 2 * r - 1; }
      else { ax = cx + r; ay = cy - r + 1; dx = 0; dy = 1; len = 2 * r - 1; }
      if ((dy == 0 && (ay < 0 || ay >= g)) || (dx == 0 && (ax < 0 || ax >= g))) continue;
      for (int u = 0; u < len; ++u) {
        const int ix = ax + u * dx, iy = ay + u * dy;
        if (ix < 0 || ix >= g || iy < 0 || iy >= g) continue;
        const int c = iy * g + ix;
        const int b = cstart[c], e = cend[c];
        for (int pp = b; pp < e; ++pp) {
          const int32_t j = cpts[pp];
          if (j >= t) continue;  // predecessors only (vg/geo.py:342)
          const double k = knn_key(spts[pp], pt);
          if (cnt == m && !lex_less(k, j, wk, wj)) continue;
          int p;
          if (cnt == m) {
            p = m - 1;
          } else {
            p = cnt;
            cnt += 1;
          }
          while (p > 0) {
            const double kq = kp[(int64_t)(p - 1) * stride];
            const int32_t jq = ip[(int64_t)(p - 1) * stride];
            if (!lex_less(k, j, kq, jq)) break;
            kp[(int64_t)p * stride] = kq;
            ip[(int64_t)p * stride] = jq;
            p -= 1;
          }
          kp[(int64_t)p * stride] = k;
          ip[(int64_t)p * stride] = j;
          if (cnt == m) {
            wk = kp[(int64_t)(m - 1) * stride];
            wj = ip[(int64_t)(m - 1) * stride];
          }
        }
      }
    }
  }
  int64_t* o = out + q * (int64_t)m;
  for (int x = 0; x < m; ++x) o[x] = (int64_t)ip[(int64_t)x * stride];
}

}  // namespace

cudaError_t launch_knn(const double2* d_data, int64_t nd, const double2* d_query, int64_t nq,
                       int64_t q_offset, int pred, int32_t m, int64_t* d_out, double* d_keys,
                       int32_t* d_idx, cudaStream_t stream) {
  if (nq <= 0) return cudaSuccess;
  int64_t blocks = (nq + kKnnThreads - 1) / kKnnThreads;
  knn_kernel<double2><<<(unsigned)blocks, kKnnThreads, 0, stream>>>(d_data, nd, d_query, nq, q_offset,
                                                                    pred, m, d_out, d_keys, d_idx, 0, nullptr);
  return cudaGetLastError();
}

cudaError_t launch_knn_sphere(const double4* d_data, int64_t nd, const double4* d_query, int64_t nq,
                              int64_t q_offset, int pred, int32_t m, int64_t* d_out, double* d_keys,
                              int32_t* d_idx, cudaStream_t stream) {
  if (nq <= 0) return cudaSuccess;
  int64_t blocks = (nq + kKnnThreads - 1) / kKnnThreads;
  knn_kernel<double4><<<(unsigned)blocks, kKnnThreads, 0, stream>>>(d_data, nd, d_query, nq, q_offset,
                                                                    pred, m, d_out, d_keys, d_idx, 0, nullptr);
  return cudaGetLastError();
}

}  // namespace vgp

namespace vgp {

// Predecessor kNN (Euclidean) by index batches [s, e) with a grid over the
// points [0, e): each target t searches it for candidates j < t only, so no
// brute-force pass over the batch's own earlier points is needed (round 1 ran
// one, 24x the grid search's time, profiles/r02_ncu_knn_grid.json).  Batches
// grow geometrically (e <= 2 s): at least half of every grid is admissible to
// each of its targets, and the last batches hold ~n/2 targets in one launch.
// Bit-identical to launch_knn's brute force (see grid_query_kernel).
// locations are the ORDERED points (host); out rows [row_lo, row_hi) on the host.
cudaError_t knn_pred_grid(const double2* d_pts, const double* h_locs, int64_t n, int32_t m, int64_t batch,
                          int64_t* h_out, cudaStream_t st, int64_t row_lo, int64_t row_hi) {
  // rows [row_lo, row_hi) of the table (targets m + row); only points
  // [0, m + row_hi) are ever candidates
  if (row_hi < 0) row_hi = n - m;
  n = m + row_hi;
  double x0 = h_locs[0], x1 = h_locs[0], y0 = h_locs[1], y1 = h_locs[1];
  for (int64_t i = 0; i < n; ++i) {
    x0 = std::min(x0, h_locs[2 * i]);
    x1 = std::max(x1, h_locs[2 * i]);
    y0 = std::min(y0, h_locs[2 * i + 1]);
    y1 = std::max(y1, h_locs[2 * i + 1]);
  }
  // batch boundaries: e = min(n, s + batch cap, max(s + kMinBatch, 2 s))
  constexpr int64_t kMinBatch = 4096;
  auto batch_end = [&](int64_t s0) {
    return std::min({n, s0 + batch, std::max(s0 + kMinBatch, 2 * s0)});
  };
  int64_t nqmax = 1;
  for (int64_t s0 = m + row_lo; s0 < n; s0 = batch_end(s0)) nqmax = std::max(nqmax, batch_end(s0) - s0);
  const int64_t slots = ((nqmax + kKnnThreads - 1) / kKnnThreads) * kKnnThreads;
  const int gmax = 4096;
  uint32_t *cell = nullptr, *cell_s = nullptr;
  int32_t *ids = nullptr, *ids_s = nullptr, *cs = nullptr, *ce = nullptr, *kidx = nullptr;
  double* kkey = nullptr;
  double2* spts = nullptr;
  int64_t* out = nullptr;
  void* tmp = nullptr;
  size_t tmp_bytes = 0;
  cudaError_t e = cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, cell, cell_s, ids, ids_s, (int)n, 0, 32, st);
  auto A = [&](void** p, size_t b) {
    if (e == cudaSuccess) e = cudaMallocAsync(p, b ? b : 1, st);
  };
  A((void**)&cell, sizeof(uint32_t) * n);
  A((void**)&cell_s, sizeof(uint32_t) * n);
  A((void**)&ids, sizeof(int32_t) * n);
  A((void**)&ids_s, sizeof(int32_t) * n);
  A((void**)&spts, sizeof(double2) * n);
  A((void**)&cs, sizeof(int32_t) * gmax * gmax);
  A((void**)&ce, sizeof(int32_t) * gmax * gmax);
  A((void**)&kkey, sizeof(double) * slots * m);
  A((void**)&kidx, sizeof(int32_t) * slots * m);
  A((void**)&out, sizeof(int64_t) * nqmax * m);
  A(&tmp, tmp_bytes);
  for (int64_t s0 = m + row_lo; e == cudaSuccess && s0 < n; s0 = batch_end(s0)) {
    const int64_t e0 = batch_end(s0), nq = e0 - s0;
    // grid over [0, e0): about 3 points per cell
    const int g = (int)std::max<int64_t>(1, std::min<int64_t>(gmax, (int64_t)std::sqrt((double)e0 / 3.0)));
    GridDesc gd;
    gd.g = g;
    gd.x0 = x0;
    gd.y0 = y0;
    gd.hx = x1 > x0 ? (x1 - x0) / g : 1.0;
    gd.hy = y1 > y0 ? (y1 - y0) / g : 1.0;
    gd.ihx = 1.0 / gd.hx;
    gd.ihy = 1.0 / gd.hy;
    // dominates the cell-assignment rounding (~1e-16 of the coordinate range)
    gd.slack = 1e-9 * std::max(gd.hx, gd.hy) + 1e-12 * std::max({std::fabs(x0), std::fabs(x1), std::fabs(y0),
                                                                  std::fabs(y1)});
    const int bs = 256;
    const unsigned nb = (unsigned)((e0 + bs - 1) / bs);
    grid_cell_kernel<<<nb, bs, 0, st>>>(d_pts, e0, gd, cell, ids);
    e = cudaGetLastError();
    if (e == cudaSuccess)
      e = cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, cell, cell_s, ids, ids_s, (int)e0, 0, 32, st);
    if (e == cudaSuccess) e = cudaMemsetAsync(cs, 0, sizeof(int32_t) * g * g, st);
    if (e == cudaSuccess) e = cudaMemsetAsync(ce, 0, sizeof(int32_t) * g * g, st);
    if (e == cudaSuccess) {
      grid_bounds_kernel<<<nb, bs, 0, st>>>(cell_s, e0, cs, ce);
      grid_gather_kernel<<<nb, bs, 0, st>>>(d_pts, ids_s, e0, spts);
      e = cudaGetLastError();
    }
    const int64_t stride = ((nq + kKnnThreads - 1) / kKnnThreads) * kKnnThreads;
    const unsigned qb = (unsigned)(stride / kKnnThreads);
    if (e == cudaSuccess) {
      grid_query_kernel<<<qb, kKnnThreads, 0, st>>>(d_pts, s0, nq, m, gd, cs, ce, ids_s, spts, kkey, kidx,
                                                    stride, out);
      e = cudaGetLastError();
    }
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(h_out + (s0 - m - row_lo) * m, out, sizeof(int64_t) * nq * m, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  }
  cudaFreeAsync(cell, st);
  cudaFreeAsync(cell_s, st);
  cudaFreeAsync(ids, st);
  cudaFreeAsync(ids_s, st);
  cudaFreeAsync(spts, st);
  cudaFreeAsync(cs, st);
  cudaFreeAsync(ce, st);
  cudaFreeAsync(kkey, st);
  cudaFreeAsync(kidx, st);
  cudaFreeAsync(out, st);
  cudaFreeAsync(tmp, st);
  return e;
}

}  // namespace vgp

// ---------------------------------------------------------------- sphere grid
// Great-circle predecessor kNN by index batches.  Points (lambda, phi,
// cos phi) map to unit vectors; the haversine key equals chord^2 / 4 in exact
// arithmetic, so a cube grid over [-1, 1]^3 gives a lower bound for every
// point outside the searched cube: (distance to the cube's faces, minus an
// absolute slack)^2 / 4, shrunk by a relative slack far above the key's few-
// ulp error (sin) and the unit vectors' rounding.  Shells are searched until
// the m-th key is strictly below that bound; the in-batch candidates then go
// through the sphere brute-force kernel as in the plane case.

namespace vgp {
namespace {

__global__ void sph_unit_kernel(const double4* __restrict__ pts, int64_t n, double4* __restrict__ u) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const double4 p = pts[j];  // (lambda, phi, cos phi)
  double sl, cl;
  sincos(p.x, &sl, &cl);
  u[j] = make_double4(p.z * cl, p.z * sl, sin(p.y), 0.0);
}

__device__ __forceinline__ int cell3(double v, double ih, int g) {
  const double f = floor((v + 1.0) * ih);
  return (int)fmin(fmax(f, 0.0), (double)(g - 1));
}

__global__ void grid3_cell_kernel(const double4* __restrict__ u, int64_t s, int g, double ih,
                                  uint32_t* __restrict__ cell, int32_t* __restrict__ ids) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= s) return;
  const double4 p = u[j];
  cell[j] = (uint32_t)(((int64_t)cell3(p.z, ih, g) * g + cell3(p.y, ih, g)) * g + cell3(p.x, ih, g));
  ids[j] = (int32_t)j;
}

__global__ void __launch_bounds__(kKnnThreads)
grid3_query_kernel(const double4* __restrict__ pts, const double4* __restrict__ u, int64_t t0, int64_t nq, int m,
                   int g, double h, double ih, const int32_t* __restrict__ cstart, const int32_t* __restrict__ cend,
                   const int32_t* __restrict__ cpts, double* __restrict__ keys, int32_t* __restrict__ idx,
                   int64_t stride, int* __restrict__ cnt_out) {
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nq) return;
  const double4 pt = pts[t0 + q];
  const double4 ut = u[t0 + q];
  const int c[3] = {cell3(ut.x, ih, g), cell3(ut.y, ih, g), cell3(ut.z, ih, g)};
  const double tc[3] = {ut.x, ut.y, ut.z};
  double* kp = keys + q;
  int32_t* ip = idx + q;
  int cnt = 0;
  double wk = __longlong_as_double(0x7ff0000000000000ll);
  int32_t wj = INT32_MAX;
  for (int r = 0; r <= g; ++r) {
    if (r > 0) {
      bool all = true;
      double d = __longlong_as_double(0x7ff0000000000000ll);
      for (int a = 0; a < 3; ++a) {
        const int lo = c[a] - r + 1, hi = c[a] + r - 1;
        if (lo > 0) {
          all = false;
          d = fmin(d, tc[a] - (-1.0 + lo * h));
        }
        if (hi < g - 1) {
          all = false;
          d = fmin(d, (-1.0 + (hi + 1) * h) - tc[a]);
        }
      }
      if (all) break;  // the whole cube searched
      if (cnt == m) {
        d = fmax(d - 1e-9 * h, 0.0);
        if (wk < d * d * 0.25 * (1.0 - 1e-9)) break;
      }
    }
    for (int dz = -r; dz <= r; ++dz) {
      const int iz = c[2] + dz;
      if (iz < 0 || iz >= g) continue;
      for (int dy = -r; dy <= r; ++dy) {
        const int iy = c[1] + dy;
        if (iy < 0 || iy >= g) continue;
        const bool face = (dz == -r || dz == r || dy == -r || dy == r);
        for (int dx = -r; dx <= r; dx += (face || r == 0) ? 1 : 2 * r) {
          const int ix = c[0] + dx;
          if (ix < 0 || ix >= g) continue;
          const int64_t cc = ((int64_t)iz * g + iy) * g + ix;
          const int b = cstart[cc], e = cend[cc];
          for (int pp = b; pp < e; ++pp) {
            const int32_t j = cpts[pp];
            const double k = knn_key(pts[j], pt);
            if (cnt == m && !lex_less(k, j, wk, wj)) continue;
            int p;
            if (cnt == m) {
              p = m - 1;
            } else {
              p = cnt;
              cnt += 1;
            }
            while (p > 0) {
              const double kq = kp[(int64_t)(p - 1) * stride];
              const int32_t jq = ip[(int64_t)(p - 1) * stride];
              if (!lex_less(k, j, kq, jq)) break;
              kp[(int64_t)p * stride] = kq;
              ip[(int64_t)p * stride] = jq;
              p -= 1;
            }
            kp[(int64_t)p * stride] = k;
            ip[(int64_t)p * stride] = j;
            if (cnt == m) {
              wk = kp[(int64_t)(m - 1) * stride];
              wj = ip[(int64_t)(m - 1) * stride];
            }
          }
        }
      }
    }
  }
  cnt_out[q] = cnt;
}

}  // namespace

cudaError_t knn_pred_grid_sphere(const double4* d_pts, int64_t n, int32_t m, int64_t batch, int64_t* h_out,
                                 cudaStream_t st) {
  const int64_t nqmax = std::min<int64_t>(batch, n - m);
  const int64_t slots = ((nqmax + kKnnThreads - 1) / kKnnThreads) * kKnnThreads;
  const int gmax = 320;
  const int64_t ncell_max = (int64_t)gmax * gmax * gmax;
  uint32_t *cell = nullptr, *cell_s = nullptr;
  int32_t *ids = nullptr, *ids_s = nullptr, *cs = nullptr, *ce = nullptr, *kidx = nullptr, *cnt = nullptr;
  double* kkey = nullptr;
  double4* u = nullptr;
  int64_t* out = nullptr;
  void* tmp = nullptr;
  size_t tmp_bytes = 0;
  cudaError_t e = cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, cell, cell_s, ids, ids_s, (int)n, 0, 32, st);
  auto A = [&](void** p, size_t b) {
    if (e == cudaSuccess) e = cudaMallocAsync(p, b ? b : 1, st);
  };
  A((void**)&u, sizeof(double4) * n);
  A((void**)&cell, sizeof(uint32_t) * n);
  A((void**)&cell_s, sizeof(uint32_t) * n);
  A((void**)&ids, sizeof(int32_t) * n);
  A((void**)&ids_s, sizeof(int32_t) * n);
  A((void**)&cs, sizeof(int32_t) * ncell_max);
  A((void**)&ce, sizeof(int32_t) * ncell_max);
  A((void**)&kkey, sizeof(double) * slots * m);
  A((void**)&kidx, sizeof(int32_t) * slots * m);
  A((void**)&cnt, sizeof(int) * slots);
  A((void**)&out, sizeof(int64_t) * nqmax * m);
  A(&tmp, tmp_bytes);
  const int bs = 256;
  if (e == cudaSuccess) {
    sph_unit_kernel<<<(unsigned)((n + bs - 1) / bs), bs, 0, st>>>(d_pts, n, u);
    e = cudaGetLastError();
  }
  for (int64_t s0 = m; e == cudaSuccess && s0 < n; s0 += batch) {
    const int64_t e0 = std::min(n, s0 + batch), nq = e0 - s0;
    // ~3 points per occupied cell: about 4.7 g^2 cells meet the sphere
    const int g = (int)std::max<int64_t>(1, std::min<int64_t>(gmax, (int64_t)std::sqrt((double)s0 / 14.0)));
    const double h = 2.0 / g, ih = g / 2.0;
    const int64_t ncell = (int64_t)g * g * g;
    const unsigned nb = (unsigned)((s0 + bs - 1) / bs);
    grid3_cell_kernel<<<nb, bs, 0, st>>>(u, s0, g, ih, cell, ids);
    e = cudaGetLastError();
    if (e == cudaSuccess)
      e = cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, cell, cell_s, ids, ids_s, (int)s0, 0, 32, st);
    if (e == cudaSuccess) e = cudaMemsetAsync(cs, 0, sizeof(int32_t) * ncell, st);
    if (e == cudaSuccess) e = cudaMemsetAsync(ce, 0, sizeof(int32_t) * ncell, st);
    if (e == cudaSuccess) {
      grid_bounds_kernel<<<nb, bs, 0, st>>>(cell_s, s0, cs, ce);
      e = cudaGetLastError();
    }
    const int64_t stride = ((nq + kKnnThreads - 1) / kKnnThreads) * kKnnThreads;
    const unsigned qb = (unsigned)(stride / kKnnThreads);
    if (e == cudaSuccess) {
      grid3_query_kernel<<<qb, kKnnThreads, 0, st>>>(d_pts, u, s0, nq, m, g, h, ih, cs, ce, ids_s, kkey, kidx,
                                                     stride, cnt);
      e = cudaGetLastError();
    }
    if (e == cudaSuccess) {
      knn_kernel<double4><<<qb, kKnnThreads, 0, st>>>(d_pts, n, d_pts + s0, nq, s0 - m, 1, m, out, kkey, kidx,
                                                      s0, cnt);
      e = cudaGetLastError();
    }
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(h_out + (s0 - m) * m, out, sizeof(int64_t) * nq * m, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  }
  for (void* p : {(void*)u, (void*)cell, (void*)cell_s, (void*)ids, (void*)ids_s, (void*)cs, (void*)ce,
                  (void*)kkey, (void*)kidx, (void*)cnt, (void*)out, tmp})
    cudaFreeAsync(p, st);
  return e;
}

}  // namespace vgp
