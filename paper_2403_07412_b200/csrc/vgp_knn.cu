// Exact m-nearest-neighbour search, bit-exact with the reference's numba scan
// geo._topm_plane (vg/geo.py:234-263):
//   key  = dx*dx + dy*dy  with dx = x_j - x_t, each op rounded (no FMA),
//   keep the m smallest by (key, j); a candidate tying the current worst is
//   rejected; insertion keeps equal keys in ascending-index order.
// Candidates are streamed in ascending j through shared memory; every thread
// owns one query and keeps only its admission threshold (the current m-th
// key) in a register.  The sorted top-m list lives in a global scratch laid
// out [slot][query] so the rare insertions stay coalesced across a warp.
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
template <typename PT>
__global__ void __launch_bounds__(kKnnThreads)
knn_kernel(const PT* __restrict__ data, int64_t nd, const PT* __restrict__ query,
           int64_t nq, int64_t q_offset, int pred, int m, int64_t* __restrict__ out,
           double* __restrict__ keys, int32_t* __restrict__ idx) {
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

  for (int64_t base = 0; base < block_limit; base += kTile) {
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

}  // namespace

cudaError_t launch_knn(const double2* d_data, int64_t nd, const double2* d_query, int64_t nq,
                       int64_t q_offset, int pred, int32_t m, int64_t* d_out, double* d_keys,
                       int32_t* d_idx, cudaStream_t stream) {
  if (nq <= 0) return cudaSuccess;
  int64_t blocks = (nq + kKnnThreads - 1) / kKnnThreads;
  knn_kernel<double2><<<(unsigned)blocks, kKnnThreads, 0, stream>>>(d_data, nd, d_query, nq, q_offset,
                                                                    pred, m, d_out, d_keys, d_idx);
  return cudaGetLastError();
}

cudaError_t launch_knn_sphere(const double4* d_data, int64_t nd, const double4* d_query, int64_t nq,
                              int64_t q_offset, int pred, int32_t m, int64_t* d_out, double* d_keys,
                              int32_t* d_idx, cudaStream_t stream) {
  if (nq <= 0) return cudaSuccess;
  int64_t blocks = (nq + kKnnThreads - 1) / kKnnThreads;
  knn_kernel<double4><<<(unsigned)blocks, kKnnThreads, 0, stream>>>(d_data, nd, d_query, nq, q_offset,
                                                                    pred, m, d_out, d_keys, d_idx);
  return cudaGetLastError();
}

}  // namespace vgp
