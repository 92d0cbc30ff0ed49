// Batched small dense linear algebra on strided buffers: the drop-ins for
// batchla.batch_potrf / batch_trsv / batch_dot (vg/batchla.py:141-229), used
// by callers outside the fused likelihood (kriging, vg/fit.py:252-264, and
// the reference's phase-split bench, vg/cli.py:257-270).  Layout: matrix k
// at buffer + k*stride, column-major, entry (i, j) at j*dim + i
// (vg/batchla.py:74-82).  Arithmetic follows the reference sweep (true
// divisions, separately rounded products and sums, ascending dots).
#include <algorithm>
#include <string>

#include "vgp_internal.cuh"

namespace vgp {
namespace {

constexpr int kThreads = 128;

// One CTA per matrix, right-looking sweep, vg/batchla.py:141-156.
__global__ void __launch_bounds__(kThreads)
potrf_kernel(double* __restrict__ buf, int64_t count, int dim, int64_t stride,
             unsigned long long* __restrict__ fail) {
  __shared__ int s_fail;
  __shared__ double s_piv;
  for (int64_t k = blockIdx.x; k < count; k += gridDim.x) {
    double* A = buf + k * stride;
    if (threadIdx.x == 0) s_fail = 0;
    __syncthreads();
    for (int j = 0; j < dim; ++j) {
      if (threadIdx.x == 0) {
        double piv = A[j + (int64_t)j * dim];
        if (!(piv > 0.0)) {
          s_fail = 1 + j;
        } else {
          s_piv = sqrt(piv);
          A[j + (int64_t)j * dim] = s_piv;
        }
      }
      __syncthreads();
      if (s_fail) break;
      const double d = s_piv;
      for (int i = j + 1 + threadIdx.x; i < dim; i += blockDim.x) A[i + (int64_t)j * dim] /= d;
      __syncthreads();
      for (int i = j + 1 + threadIdx.x; i < dim; i += blockDim.x) {
        const double lij = A[i + (int64_t)j * dim];
        for (int c = j + 1; c <= i; ++c)
          A[i + (int64_t)c * dim] = __dsub_rn(A[i + (int64_t)c * dim], __dmul_rn(lij, A[c + (int64_t)j * dim]));
      }
      __syncthreads();
    }
    if (s_fail && threadIdx.x == 0) atomicMin(fail, npd_key(k, s_fail - 1, dim));
    __syncthreads();
  }
}

// One thread per entry: forward substitution, vg/batchla.py:196-207.
__global__ void trsv_kernel(const double* __restrict__ L, int64_t lstride, const double* __restrict__ b,
                            double* __restrict__ x, int64_t count, int dim, int64_t vstride,
                            unsigned long long* __restrict__ fail) {
  int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= count) return;
  const double* A = L + k * lstride;
  double* xs = x + k * vstride;
  const double* bs = b + k * vstride;
  for (int i = 0; i < dim; ++i) xs[i] = bs[i];
  for (int j = 0; j < dim; ++j) {
    double piv = A[j + (int64_t)j * dim];
    if (piv == 0.0) {
      atomicMin(fail, (unsigned long long)k);
      return;
    }
    double xj = xs[j] / piv;
    xs[j] = xj;
    for (int i = j + 1; i < dim; ++i) xs[i] = __dsub_rn(xs[i], __dmul_rn(A[i + (int64_t)j * dim], xj));
  }
}

// One thread per entry, ascending accumulation, vg/batchla.py:223-226.
__global__ void dot_kernel(const double* __restrict__ a, const double* __restrict__ b, int64_t count,
                           int dim, int64_t stride, double* __restrict__ out) {
  int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= count) return;
  double acc = 0.0;
  for (int i = 0; i < dim; ++i) acc = __dadd_rn(acc, __dmul_rn(a[k * stride + i], b[k * stride + i]));
  out[k] = acc;
}

int check_dev(int device) {
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0)
    return fail(VGP_E_CUDA, "no CUDA device available; the B200 path has no CPU fallback");
  if (device < 0 || device >= count) return fail(VGP_E_INVALID, "device ordinal out of range");
  return cudaSetDevice(device) == cudaSuccess ? VGP_OK : fail(VGP_E_CUDA, "cudaSetDevice");
}

}  // namespace
}  // namespace vgp

using namespace vgp;

extern "C" {

int vgp_batch_potrf(int device, double* buffer, int64_t count, int32_t dim, int64_t stride,
                    int64_t* fail_index) {
  if (count < 0 || dim < 1 || stride < (int64_t)dim * dim || (count > 0 && !buffer))
    return fail(VGP_E_INVALID, "bad batch_potrf arguments");
  if (fail_index) *fail_index = -1;
  if (count == 0) return VGP_OK;
  int rc = check_dev(device);
  if (rc) return rc;
  double* d = nullptr;
  unsigned long long* f = nullptr;
  size_t bytes = sizeof(double) * (size_t)count * stride;
  VGP_CUDA_TRY(cudaMalloc(&d, bytes));
  cudaError_t e = cudaMalloc(&f, sizeof(unsigned long long));
  if (e == cudaSuccess) e = cudaMemcpy(d, buffer, bytes, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemset(f, 0xff, sizeof(unsigned long long));
  if (e == cudaSuccess) {
    int grid = (int)std::min<int64_t>(count, 148 * 16);
    potrf_kernel<<<grid, kThreads>>>(d, count, dim, stride, f);
    e = cudaGetLastError();
  }
  unsigned long long key = ~0ull;
  if (e == cudaSuccess) e = cudaMemcpy(buffer, d, bytes, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess) e = cudaMemcpy(&key, f, sizeof(key), cudaMemcpyDeviceToHost);
  cudaFree(d);
  cudaFree(f);
  if (e != cudaSuccess) return fail(VGP_E_CUDA, std::string("batch_potrf: ") + cudaGetErrorString(e));
  if (key != ~0ull) {
    if (fail_index) *fail_index = npd_key_entry(key, dim);
    return VGP_NOT_POSITIVE_DEFINITE;
  }
  return VGP_OK;
}

int vgp_batch_trsv(int device, const double* lbuf, int64_t lstride, const double* b, double* x,
                   int64_t count, int32_t dim, int64_t vstride, int64_t* fail_index) {
  if (count < 0 || dim < 1 || lstride < (int64_t)dim * dim || vstride < dim ||
      (count > 0 && (!lbuf || !b || !x)))
    return fail(VGP_E_INVALID, "bad batch_trsv arguments");
  if (fail_index) *fail_index = -1;
  if (count == 0) return VGP_OK;
  int rc = check_dev(device);
  if (rc) return rc;
  double *dl = nullptr, *db = nullptr, *dx = nullptr;
  unsigned long long* f = nullptr;
  size_t lb = sizeof(double) * (size_t)count * lstride, vb = sizeof(double) * (size_t)count * vstride;
  cudaError_t e = cudaMalloc(&dl, lb);
  if (e == cudaSuccess) e = cudaMalloc(&db, vb);
  if (e == cudaSuccess) e = cudaMalloc(&dx, vb);
  if (e == cudaSuccess) e = cudaMalloc(&f, sizeof(unsigned long long));
  if (e == cudaSuccess) e = cudaMemcpy(dl, lbuf, lb, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(db, b, vb, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemset(dx, 0, vb);
  if (e == cudaSuccess) e = cudaMemset(f, 0xff, sizeof(unsigned long long));
  if (e == cudaSuccess) {
    trsv_kernel<<<(unsigned)((count + 127) / 128), 128>>>(dl, lstride, db, dx, count, dim, vstride, f);
    e = cudaGetLastError();
  }
  unsigned long long key = ~0ull;
  if (e == cudaSuccess) e = cudaMemcpy(x, dx, vb, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess) e = cudaMemcpy(&key, f, sizeof(key), cudaMemcpyDeviceToHost);
  cudaFree(dl);
  cudaFree(db);
  cudaFree(dx);
  cudaFree(f);
  if (e != cudaSuccess) return fail(VGP_E_CUDA, std::string("batch_trsv: ") + cudaGetErrorString(e));
  if (key != ~0ull) {
    if (fail_index) *fail_index = (int64_t)key;
    return VGP_SINGULAR_TRIANGULAR;
  }
  return VGP_OK;
}

int vgp_batch_dot(int device, const double* a, const double* b, int64_t count, int32_t dim,
                  int64_t stride, double* out) {
  if (count < 0 || dim < 1 || stride < dim || (count > 0 && (!a || !b || !out)))
    return fail(VGP_E_INVALID, "bad batch_dot arguments");
  if (count == 0) return VGP_OK;
  int rc = check_dev(device);
  if (rc) return rc;
  double *da = nullptr, *db = nullptr, *dout = nullptr;
  size_t vb = sizeof(double) * (size_t)count * stride;
  cudaError_t e = cudaMalloc(&da, vb);
  if (e == cudaSuccess) e = cudaMalloc(&db, vb);
  if (e == cudaSuccess) e = cudaMalloc(&dout, sizeof(double) * count);
  if (e == cudaSuccess) e = cudaMemcpy(da, a, vb, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(db, b, vb, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) {
    dot_kernel<<<(unsigned)((count + 127) / 128), 128>>>(da, db, count, dim, stride, dout);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaMemcpy(out, dout, sizeof(double) * count, cudaMemcpyDeviceToHost);
  cudaFree(da);
  cudaFree(db);
  cudaFree(dout);
  if (e != cudaSuccess) return fail(VGP_E_CUDA, std::string("batch_dot: ") + cudaGetErrorString(e));
  return VGP_OK;
}

}  // extern "C"
