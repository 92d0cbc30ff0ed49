// Dependent-chain latency of the instructions on the fused kernel's pivot
// chain (DFMA, DMUL, SHFL.64, MUFU.RSQ64H, DMMA, LDS.64), one warp, clock64.
#include <cstdio>
#include <cuda_runtime.h>

#define N 256

__global__ void lat(double* out, long long* cyc, double x0, int srcl) {
  double x = x0 + threadIdx.x * 1e-9;
  __shared__ double sm[64];
  __shared__ int si[64];
  sm[threadIdx.x & 63] = x;
  si[threadIdx.x & 63] = (threadIdx.x * 7 + 3) & 63;
  si[(threadIdx.x + 32) & 63] = (threadIdx.x * 5 + 1) & 63;
  __syncwarp();
  long long t0, t1;
  // DFMA chain
  t0 = clock64();
#pragma unroll
  for (int i = 0; i < N; ++i) asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(x) : "d"(0.999999), "d"(1e-7));
  t1 = clock64();
  cyc[0] = t1 - t0;
  // DMUL chain
  t0 = clock64();
#pragma unroll
  for (int i = 0; i < N; ++i) asm volatile("mul.rn.f64 %0, %0, %1;" : "+d"(x) : "d"(1.0000001));
  t1 = clock64();
  cyc[1] = t1 - t0;
  // DADD chain
  t0 = clock64();
#pragma unroll
  for (int i = 0; i < N; ++i) asm volatile("add.rn.f64 %0, %0, %1;" : "+d"(x) : "d"(1e-9));
  t1 = clock64();
  cyc[2] = t1 - t0;
  // SHFL of a double chain
  t0 = clock64();
#pragma unroll
  for (int i = 0; i < N; ++i) x = __shfl_sync(0xffffffffu, x, (srcl + i) & 31);
  t1 = clock64();
  cyc[3] = t1 - t0;
  // MUFU rsqrt seed chain (+ DADD to keep positive)
  t0 = clock64();
#pragma unroll
  for (int i = 0; i < N; ++i) {
    double y;
    asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    x = y;
  }
  t1 = clock64();
  cyc[4] = t1 - t0;
  // DMMA chain on the same accumulator
  double d0 = x, d1 = x;
  t0 = clock64();
#pragma unroll
  for (int i = 0; i < N; ++i)
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1) : "d"(1e-3), "d"(1e-3));
  t1 = clock64();
  cyc[5] = t1 - t0;
  // DMMA independent (8 accumulators)
  double a[8][2];
  for (int k = 0; k < 8; ++k) a[k][0] = a[k][1] = x + k;
  t0 = clock64();
#pragma unroll
  for (int i = 0; i < N / 8; ++i)
#pragma unroll
    for (int k = 0; k < 8; ++k)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(a[k][0]), "+d"(a[k][1]) : "d"(1e-3), "d"(1e-3));
  t1 = clock64();
  cyc[6] = t1 - t0;
  // LDS.64 pointer chase
  int idx = threadIdx.x & 63;
  t0 = clock64();
#pragma unroll
  for (int i = 0; i < N; ++i) {
    idx = si[idx];
  }
  t1 = clock64();
  cyc[7] = t1 - t0;
  // DFMA independent x8 (throughput, one warp)
  double b[8];
  for (int k = 0; k < 8; ++k) b[k] = x + k;
  t0 = clock64();
#pragma unroll
  for (int i = 0; i < N / 8; ++i)
#pragma unroll
    for (int k = 0; k < 8; ++k) asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(b[k]) : "d"(0.999999), "d"(1e-7));
  t1 = clock64();
  cyc[8] = t1 - t0;
  double s = x + d0 + d1 + idx;
  for (int k = 0; k < 8; ++k) s += a[k][0] + a[k][1] + b[k];
  out[threadIdx.x] = s;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 32 * sizeof(double));
  cudaMallocManaged(&cyc, 16 * sizeof(long long));
  for (int rep = 0; rep < 3; ++rep) lat<<<1, 32>>>(out, cyc, 1.5, 1);
  cudaDeviceSynchronize();
  const char* names[] = {"dfma", "dmul", "dadd", "shfl.f64", "mufu.rsq64h", "dmma_dep", "dmma_indep8", "lds.64_chase", "dfma_indep8"};
  for (int i = 0; i < 9; ++i)
    printf("{\"op\":\"%s\",\"cycles_per_op\":%.2f}\n", names[i], (double)cyc[i] / N);
  return 0;
}
