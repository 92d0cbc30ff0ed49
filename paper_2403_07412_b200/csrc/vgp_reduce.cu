// Small glue kernels: device-side dataset permutation (Dataset.permute,
// vg/geo.py:145-149, done once per upload instead of once per evaluation),
// the deterministic ordered reduction of block_rest (vecchia._ordered_sum,
// vg/vecchia.py:169-177) and covariance evaluation at given distances
// (kernels.cov, vg/kernels.py:94-98).
#include "vgp_math.cuh"
#include "vgp_pairwise.cuh"

namespace vgp {

namespace {

__global__ void permute_kernel(const double* __restrict__ raw, const int64_t* __restrict__ order,
                               int64_t n, double4* __restrict__ pts) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  // raw = [(x, y) * n | obs * n] in original order
  int64_t s = order[i];
  double2 xy = reinterpret_cast<const double2*>(raw)[s];
  pts[i] = make_double4(xy.x, xy.y, raw[2 * n + s], 0.0);
}

// observations only (the locations are unchanged): pts[i].z
__global__ void permute_obs_kernel(const double* __restrict__ obs, const int64_t* __restrict__ order,
                                   int64_t n, double4* __restrict__ pts) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  reinterpret_cast<double*>(pts)[4 * i + 2] = obs[order[i]];
}

// One warp per 4096-chunk.  A full chunk is a perfect binary tree of 32
// numpy 128-blocks: lane l sums block l with numpy's 8-accumulator rule and
// the xor-shuffle tree reproduces numpy's split-in-half recursion exactly.
// A short tail chunk is summed by lane 0 with the general recursion.
__global__ void chunk_partials_kernel(const double* __restrict__ rest, int64_t rest_lo,
                                      int64_t rest_hi, int64_t chunk_lo, int64_t chunk_hi,
                                      double* __restrict__ partials) {
  const int lane = threadIdx.x & 31;
  const int64_t c = chunk_lo + (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  if (c >= chunk_hi) return;
  const int64_t lo = c * kReduceChunk;
  int64_t hi = lo + kReduceChunk;
  if (hi > rest_hi) hi = rest_hi;
  const double* a = rest + (lo - rest_lo);
  const int64_t len = hi - lo;
  double res;
  if (len == kReduceChunk) {
    const double* p = a + lane * 128;
    double r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = p[j];
#pragma unroll 4
    for (int i = 8; i < 128; i += 8) {
#pragma unroll
      for (int j = 0; j < 8; ++j) r[j] += p[i + j];
    }
    res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) res += __shfl_xor_sync(0xffffffffu, res, off);
  } else {
    res = lane == 0 ? pairwise_rec(a, len) : 0.0;
  }
  if (lane == 0) partials[c - chunk_lo] = res;
}

// total = block_first + ((0 + p0) + p1) + ...   (vg/vecchia.py:213, :174-177)
__global__ void total_kernel(const double* __restrict__ partials, int64_t nchunks,
                             double* __restrict__ scalars) {
  double s = 0.0;
  for (int64_t c = 0; c < nchunks; ++c) s += partials[c];
  scalars[0] = scalars[1] + s;
}

__global__ void scatter_partials_kernel(const double* __restrict__ partials, int64_t nch,
                                        int64_t chunk_lo, int has_first,
                                        const double* __restrict__ scalars,
                                        const unsigned long long* __restrict__ fail,
                                        double* __restrict__ out) {
  const bool failed = fail[0] != ~0ull || fail[1] != ~0ull;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nch;
       i += (int64_t)gridDim.x * blockDim.x)
    out[1 + chunk_lo + i] = (failed && i == 0) ? __longlong_as_double(0x7ff8000000000000ll)
                                               : partials[i];
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    if (has_first) out[0] = scalars[1];
    if (failed && nch == 0) out[0] = __longlong_as_double(0x7ff8000000000000ll);
  }
}

__global__ void cov_eval_kernel(CovParams cp, const double* __restrict__ d, int64_t count,
                                double* __restrict__ out) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < count) out[i] = cov_ref(cp, d[i]);
}

__global__ void bessel_eval_kernel(CovParams cp, const double* __restrict__ x, int64_t count,
                                   double* __restrict__ out) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < count) out[i] = bessel_k(cp, x[i]);
}

}  // namespace

cudaError_t launch_bessel_eval(const CovParams& cp, const double* d_in, int64_t count,
                               double* d_out, cudaStream_t stream) {
  if (count <= 0) return cudaSuccess;
  bessel_eval_kernel<<<(unsigned)((count + 255) / 256), 256, 0, stream>>>(cp, d_in, count, d_out);
  return cudaGetLastError();
}

cudaError_t launch_permute(const double* d_raw, const int64_t* d_order, int64_t n, double4* d_pts,
                           cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  permute_kernel<<<(unsigned)((n + 255) / 256), 256, 0, stream>>>(d_raw, d_order, n, d_pts);
  return cudaGetLastError();
}

cudaError_t launch_permute_obs(const double* d_obs, const int64_t* d_order, int64_t n, double4* d_pts,
                               cudaStream_t stream) {
  permute_obs_kernel<<<(unsigned)((n + 255) / 256), 256, 0, stream>>>(d_obs, d_order, n, d_pts);
  return cudaGetLastError();
}

cudaError_t launch_reduce(const Plan& p, bool want_total, cudaStream_t stream) {
  int64_t nch = p.chunk_hi - p.chunk_lo;
  if (nch > 0) {
    const int warps = 4;
    unsigned blocks = (unsigned)((nch + warps - 1) / warps);
    chunk_partials_kernel<<<blocks, warps * 32, 0, stream>>>(p.d_rest, p.rest_lo, p.rest_hi,
                                                             p.chunk_lo, p.chunk_hi, p.d_partials);
  }
  if (want_total) total_kernel<<<1, 1, 0, stream>>>(p.d_partials, nch, p.d_scalars);
  return cudaGetLastError();
}

cudaError_t launch_scatter_partials(const Plan& p, double* d_out, cudaStream_t stream) {
  int64_t nch = p.chunk_hi - p.chunk_lo;
  unsigned blocks = (unsigned)((nch + 255) / 256);
  if (blocks < 1) blocks = 1;
  scatter_partials_kernel<<<blocks, 256, 0, stream>>>(p.d_partials, nch, p.chunk_lo,
                                                       p.blk_lo == 0 ? 1 : 0, p.d_scalars,
                                                       p.d_fail, d_out);
  return cudaGetLastError();
}

cudaError_t launch_cov_eval(const CovParams& cp, const double* d_in, int64_t count, double* d_out,
                            cudaStream_t stream) {
  if (count <= 0) return cudaSuccess;
  cov_eval_kernel<<<(unsigned)((count + 255) / 256), 256, 0, stream>>>(cp, d_in, count, d_out);
  return cudaGetLastError();
}

}  // namespace vgp
