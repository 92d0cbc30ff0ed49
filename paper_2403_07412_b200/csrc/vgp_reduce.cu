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

// One 256-thread CTA per 4096-chunk.  A full chunk is a perfect binary tree
// of 32 numpy 128-blocks (vg/vecchia.py:169-177 via numpy's pairwise sum):
// thread (leaf l, accumulator j) runs numpy's j-th of 8 accumulators over
// block l (the same 16 additions in the same order, 8x the parallelism of a
// lane per block), a 3-level xor shuffle combines the 8 as numpy does
// ((r0 + r1) + (r2 + r3)) + ((r4 + r5) + (r6 + r7)), and the leaf tree is
// numpy's split-in-half recursion: xor shuffles inside a warp (4 leaves),
// shared memory across the 8 warps.  A short tail chunk is summed by one
// thread with the general recursion.  With want_total, the last CTA to
// finish adds the partials in chunk order, total = block_first +
// ((0 + p0) + p1) + ... (vg/vecchia.py:213, :174-177), and rearms the ticket.
__global__ void __launch_bounds__(256)
chunk_partials_kernel(const double* __restrict__ rest, int64_t rest_lo, int64_t rest_hi,
                      int64_t chunk_lo, int64_t chunk_hi, double* __restrict__ partials,
                      double* __restrict__ scalars, unsigned long long* __restrict__ ticket) {
  __shared__ double wsum[8];
  __shared__ bool last;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t c = chunk_lo + blockIdx.x;
  const int64_t lo = c * kReduceChunk;
  int64_t hi = lo + kReduceChunk;
  if (hi > rest_hi) hi = rest_hi;
  const double* a = rest + (lo - rest_lo);
  const int64_t len = hi - lo;
  if (len == kReduceChunk) {
    const int leaf = tid >> 3, j = tid & 7;
    const double* pl = a + leaf * 128 + j;
    double r = pl[0];
#pragma unroll
    for (int i = 8; i < 128; i += 8) r += pl[i];
    r += __shfl_xor_sync(0xffffffffu, r, 1);
    r += __shfl_xor_sync(0xffffffffu, r, 2);
    r += __shfl_xor_sync(0xffffffffu, r, 4);
    // leaves 4w .. 4w + 3 sit at lanes 0, 8, 16, 24 of warp w
    r += __shfl_xor_sync(0xffffffffu, r, 8);
    r += __shfl_xor_sync(0xffffffffu, r, 16);
    if (lane == 0) wsum[warp] = r;
    __syncthreads();
    if (tid == 0) {
      const double s01 = wsum[0] + wsum[1], s23 = wsum[2] + wsum[3];
      const double s45 = wsum[4] + wsum[5], s67 = wsum[6] + wsum[7];
      partials[c - chunk_lo] = (s01 + s23) + (s45 + s67);
    }
  } else if (tid == 0) {
    partials[c - chunk_lo] = pairwise_rec(a, len);
  }
  if (!ticket) return;
  if (tid == 0) {
    __threadfence();
    const unsigned long long t = atomicAdd(ticket, 1ull);
    last = t == (unsigned long long)(gridDim.x - 1);
  }
  __syncthreads();
  if (!last) return;
  // the last CTA: stage the partials in shared memory with all threads (one
  // round trip instead of one per chunk), then add them in chunk order
  __shared__ double buf[2048];
  __threadfence();
  const volatile double* pv = partials;
  double sum = 0.0;
  const int64_t nch = gridDim.x;
  for (int64_t b0 = 0; b0 < nch; b0 += 2048) {
    const int cnt = nch - b0 < 2048 ? (int)(nch - b0) : 2048;
    __syncthreads();
    for (int k = tid; k < cnt; k += blockDim.x) buf[k] = pv[b0 + k];
    __syncthreads();
    if (tid == 0)
      for (int k = 0; k < cnt; ++k) sum += buf[k];
  }
  if (tid == 0) {
    scalars[0] = scalars[1] + sum;
    *ticket = 0ull;
  }
}

// total with no chunks (a plan of the joint block only): total = block_first
__global__ void total_kernel(double* __restrict__ scalars) { scalars[0] = scalars[1] + 0.0; }

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
  // d_scalars[3]: the last-CTA ticket (zeroed at plan creation, rearmed by
  // the last CTA)
  unsigned long long* ticket = reinterpret_cast<unsigned long long*>(p.d_scalars + 3);
  if (nch > 0) {
    chunk_partials_kernel<<<(unsigned)nch, 256, 0, stream>>>(p.d_rest, p.rest_lo, p.rest_hi, p.chunk_lo,
                                                             p.chunk_hi, p.d_partials, p.d_scalars,
                                                             want_total ? ticket : nullptr);
  } else if (want_total) {
    total_kernel<<<1, 1, 0, stream>>>(p.d_scalars);
  }
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
