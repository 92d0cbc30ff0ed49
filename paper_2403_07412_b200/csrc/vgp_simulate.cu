// Vecchia forward simulation on the device: draws y from the Gaussian whose
// exact log-density IS the Vecchia likelihood of the plan,
// so likelihood parity fixtures are model-consistent at any n.  Data
// generation for tests and bench.py, not a reference code path: the
// reference's own generator is the dense exact.simulate_grf (vg/exact.py:47-66,
// capped at n <= 20000), which this replaces beyond desk scale.
//
//   y[0:m]  = L0 z[0:m],                   L0 = chol(Sigma_0)
//   y[t]    = b_t . y[J_t] + sqrt(D_t) z_t,  b_t = Sigma_t^-1 v_t,
//                                           D_t = sigma^2 - v_t . b_t,   t = m..n-1
//
// Two kernels.  sim_coef_kernel: one CTA per batch entry (the generic
// kernel's right-looking sweep on the augmented [Sigma; v] matrix, then the
// back substitution b = L^-T w), all entries in parallel.  sim_sweep_kernel:
// the sequential O(n m) recursion, one warp per target taken in increasing
// order from an atomic ticket; a warp spins on its neighbours' ready flags
// (acquire) and publishes y[t] with a release store.  Tickets go only to
// running warps and every wait is on a smaller ticket, so the sweep cannot
// deadlock; it runs at the depth of the neighbour DAG, not at n.
#include "vgp_internal.cuh"
#include "vgp_math.cuh"

namespace vgp {

namespace {

constexpr int kSimThreads = 128;

template <bool kShared>
__global__ void __launch_bounds__(kSimThreads)
sim_coef_kernel(const double4* __restrict__ pts, const int32_t* __restrict__ nbr, int m,
                int64_t count, CovParams cp, int metric, double radius,
                const double* __restrict__ z, double* __restrict__ y, double* __restrict__ coef,
                double* __restrict__ sd, double* __restrict__ work, int ld,
                unsigned long long* __restrict__ fail) {
  extern __shared__ double smem[];
  double* px = smem;
  double* py = px + (m + 1);
  double* A = kShared ? (py + (m + 1)) : (work + (size_t)blockIdx.x * ld * (m + 1));
  __shared__ double s_piv;
  __shared__ int s_bad;
  const int P = m + 1;  // rows 0..m-1 Sigma, row m v

  for (int64_t e = blockIdx.x; e < count; e += gridDim.x) {
    const bool joint = (e == 0);
    for (int a = threadIdx.x; a <= m; a += blockDim.x) {
      int64_t src = joint ? (a < m ? a : 0)
                          : (a < m ? (int64_t)nbr[(e - 1) * (int64_t)m + a] : (m + e - 1));
      const double4 p = pts[src];
      px[a] = p.x;
      py[a] = p.y;
    }
    if (threadIdx.x == 0) s_bad = 0;
    __syncthreads();
    for (int k = 0; k < m; ++k) {
      for (int i = k + threadIdx.x; i < P; i += blockDim.x) {
        double val;
        if (i == k)
          val = cp.s2;
        else if (i < m || !joint)
          val = cov_ref(cp, point_dist(metric, radius, px[i], py[i], px[k], py[k]));
        else
          val = 0.0;
        A[i + (size_t)k * ld] = val;
      }
    }
    __syncthreads();
    // right-looking Cholesky of Sigma; row m rides along: w = L^-1 v
    for (int j = 0; j < m; ++j) {
      if (threadIdx.x == 0) {
        const double piv = A[j + (size_t)j * ld];
        if (!(piv > 0.0)) s_bad = 1;
        s_piv = sqrt(piv);
        A[j + (size_t)j * ld] = s_piv;
      }
      __syncthreads();
      const double d = s_piv;
      for (int i = j + 1 + threadIdx.x; i < P; i += blockDim.x) A[i + (size_t)j * ld] /= d;
      __syncthreads();
      for (int i = j + 1 + threadIdx.x; i < P; i += blockDim.x) {
        const double lij = A[i + (size_t)j * ld];
        const int kmax = i < m ? i : m - 1;
        for (int k = j + 1; k <= kmax; ++k)
          A[i + (size_t)k * ld] = fma(-lij, A[k + (size_t)j * ld], A[i + (size_t)k * ld]);
      }
      __syncthreads();
    }
    if (s_bad) {
      if (threadIdx.x == 0) atomicMin(fail, (unsigned long long)e);
      __syncthreads();
      continue;
    }
    if (joint) {
      // y[0:m] = L0 z[0:m]
      for (int i = threadIdx.x; i < m; i += blockDim.x) {
        double acc = 0.0;
        for (int k = 0; k <= i; ++k) acc = fma(A[i + (size_t)k * ld], z[k], acc);
        y[i] = acc;
      }
    } else {
      if (threadIdx.x == 0) {
        double ww = 0.0;
        for (int k = 0; k < m; ++k) ww = fma(A[m + (size_t)k * ld], A[m + (size_t)k * ld], ww);
        const double dv = cp.s2 - ww;
        sd[e - 1] = sqrt(dv > 0.0 ? dv : 0.0);
      }
      __syncthreads();
      // back substitution b = L^-T w, in place in row m
      for (int a = m - 1; a >= 0; --a) {
        if (threadIdx.x == 0) A[m + (size_t)a * ld] /= A[a + (size_t)a * ld];
        __syncthreads();
        const double ba = A[m + (size_t)a * ld];
        for (int i = threadIdx.x; i < a; i += blockDim.x)
          A[m + (size_t)i * ld] = fma(-A[a + (size_t)i * ld], ba, A[m + (size_t)i * ld]);
        __syncthreads();
      }
      for (int a = threadIdx.x; a < m; a += blockDim.x)
        coef[(e - 1) * (int64_t)m + a] = A[m + (size_t)a * ld];
    }
    __syncthreads();
  }
}

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__global__ void __launch_bounds__(256)
sim_sweep_kernel(const int32_t* __restrict__ nbr, int m, int64_t n, const double* __restrict__ coef,
                 const double* __restrict__ sd, const double* __restrict__ z, double* y,
                 int* ready, unsigned long long* ticket) {
  const int lane = threadIdx.x & 31;
  for (;;) {
    unsigned long long tk = 0;
    if (lane == 0) tk = atomicAdd(ticket, 1ull);
    tk = __shfl_sync(0xffffffffu, tk, 0);
    const int64_t t = m + (int64_t)tk;
    if (t >= n) break;
    const int64_t row = t - m;
    double acc = 0.0;
    for (int a = lane; a < m; a += 32) {
      const int j = nbr[row * m + a];
      if (j >= m)
        while (ld_acquire(ready + j) == 0) {
        }
      acc = fma(coef[row * m + a], __ldcg(y + j), acc);
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    if (lane == 0) {
      __stcg(y + t, fma(sd[row], z[t], acc));
      st_release(ready + t, 1);
    }
  }
}

}  // namespace

cudaError_t launch_simulate(const Plan& p, const CovParams& cp, const double* d_z, double* d_y,
                            unsigned long long* d_fail, cudaStream_t stream) {
  const int m = p.m;
  const int64_t n = p.n;
  const int64_t count = n - m + 1;
  const int ld = (m + 1) | 1;
  double *d_coef = nullptr, *d_sd = nullptr, *d_work = nullptr;
  int* d_ready = nullptr;
  unsigned long long* d_ticket = nullptr;
  cudaError_t e = cudaMalloc(&d_coef, sizeof(double) * (size_t)(n - m) * m);
  if (e == cudaSuccess) e = cudaMalloc(&d_sd, sizeof(double) * (size_t)(n - m));
  if (e == cudaSuccess) e = cudaMalloc(&d_ready, sizeof(int) * (size_t)n);
  if (e == cudaSuccess) e = cudaMalloc(&d_ticket, sizeof(unsigned long long));
  if (e == cudaSuccess) e = cudaMemsetAsync(d_ready, 0, sizeof(int) * (size_t)n, stream);
  if (e == cudaSuccess) e = cudaMemsetAsync(d_ticket, 0, sizeof(unsigned long long), stream);
  const size_t coord_bytes = sizeof(double) * 2 * (m + 1);
  const size_t mat_bytes = sizeof(double) * (size_t)ld * (m + 1);
  if (e == cudaSuccess) {
    if (coord_bytes + mat_bytes <= 160 * 1024) {
      const size_t sm = coord_bytes + mat_bytes;
      e = cudaFuncSetAttribute(sim_coef_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      const int64_t grid = count < (int64_t)p.num_sms * 32 ? count : (int64_t)p.num_sms * 32;
      if (e == cudaSuccess)
        sim_coef_kernel<true><<<(unsigned)grid, kSimThreads, sm, stream>>>(
            p.d_pts, p.d_nbr, m, count, cp, p.metric, p.radius, d_z, d_y, d_coef, d_sd, nullptr, ld, d_fail);
    } else {
      const int64_t grid = count < (int64_t)p.num_sms * 4 ? count : (int64_t)p.num_sms * 4;
      e = cudaMalloc(&d_work, sizeof(double) * (size_t)grid * ld * (m + 1));
      if (e == cudaSuccess)
        e = cudaFuncSetAttribute(sim_coef_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)coord_bytes);
      if (e == cudaSuccess)
        sim_coef_kernel<false><<<(unsigned)grid, kSimThreads, coord_bytes, stream>>>(
            p.d_pts, p.d_nbr, m, count, cp, p.metric, p.radius, d_z, d_y, d_coef, d_sd, d_work, ld, d_fail);
    }
    if (e == cudaSuccess) e = cudaGetLastError();
  }
  if (e == cudaSuccess && n > m) {
    sim_sweep_kernel<<<p.num_sms * 8, 256, 0, stream>>>(p.d_nbr, m, n, d_coef, d_sd, d_z, d_y, d_ready,
                                                         d_ticket);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
  cudaFree(d_coef);
  cudaFree(d_sd);
  cudaFree(d_ready);
  cudaFree(d_ticket);
  cudaFree(d_work);
  return e;
}

}  // namespace vgp
