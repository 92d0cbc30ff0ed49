// Latency of a dependent chain (DFMA, SHFL.64, MUFU) in warp 0 while other
// warps of the same SM sub-partition (warp % 4 == 0) issue background work:
// none / DMMA stream / LDS.128 stream / DFMA stream.  One CTA of 16 warps.
#include <cstdio>
#include <cuda_runtime.h>

#define N 512

__global__ void bench(double* out, long long* cyc, int mode, int nbg) {
  __shared__ double sm[4096];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) sm[i] = 1.0 + i * 1e-6;
  __syncthreads();
  double x = 1.0 + lane * 1e-9;
  volatile __shared__ int stop;
  if (threadIdx.x == 0) stop = 0;
  __syncthreads();
  if (warp == 0) {
    long long t0 = clock64();
    for (int i = 0; i < N; ++i) asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(x) : "d"(0.999999), "d"(1e-7));
    long long t1 = clock64();
    for (int i = 0; i < N; ++i) x = __shfl_sync(0xffffffffu, x, (lane + 1) & 31);
    long long t2 = clock64();
    for (int i = 0; i < N; ++i) {
      double y;
      asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
      x = y + 1.0;
    }
    long long t3 = clock64();
    if (lane == 0) {
      cyc[0] = t1 - t0;
      cyc[1] = t2 - t1;
      cyc[2] = t3 - t2;
    }
    __syncwarp();
    if (lane == 0) stop = 1;
  } else if ((mode < 10 && (warp & 3) == 0 && (warp >> 2) <= nbg) ||
             (mode >= 10 && (warp & 3) == 1 && (warp >> 2) < nbg)) {
    double a[8][2];
    for (int k = 0; k < 8; ++k) a[k][0] = a[k][1] = x + k;
    int it = 0;
    while (!stop && it < 200000) {
      ++it;
      if (mode == 1 || mode == 11) {
#pragma unroll
        for (int k = 0; k < 8; ++k)
          asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                       : "+d"(a[k][0]), "+d"(a[k][1]) : "d"(1e-3), "d"(1e-3));
      } else if (mode == 2) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          double2 v = *reinterpret_cast<double2*>(sm + ((lane * 2 + k * 64 + it) & 4094));
          a[k][0] += v.x;
        }
      } else if (mode == 4) {  // DMMA with an 8-instruction integer gap
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                       : "+d"(a[k][0]), "+d"(a[k][1]) : "d"(1e-3), "d"(1e-3));
          int z = it;
#pragma unroll
          for (int g = 0; g < 8; ++g) asm volatile("add.s32 %0, %0, 1;" : "+r"(z));
          if (z == -5) a[k][0] = 0;
        }
      } else if (mode == 3) {
#pragma unroll
        for (int k = 0; k < 8; ++k)
          asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(a[k][0]) : "d"(0.999999), "d"(1e-7));
      }
    }
    double s = 0;
    for (int k = 0; k < 8; ++k) s += a[k][0] + a[k][1];
    out[threadIdx.x] = s;
  }
  if (warp == 0) out[threadIdx.x] = x;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 1024 * sizeof(double));
  cudaMallocManaged(&cyc, 16 * sizeof(long long));
  const char* names[] = {"idle", "dmma", "lds128", "dfma", "dmma_gap8", "", "", "", "", "", "", "dmma_other_smsp"};
  const int modes[] = {0, 1, 4, 11, 2, 3};
  for (int mi = 0; mi < 6; ++mi)
    for (int nbg = 1; nbg <= 3; ++nbg) {
      const int mode = modes[mi];
      if (mode == 0 && nbg > 1) continue;
      for (int rep = 0; rep < 2; ++rep) bench<<<1, 512>>>(out, cyc, mode, nbg);
      cudaDeviceSynchronize();
      printf("{\"background\":\"%s\",\"bg_warps_same_smsp\":%d,\"dfma_lat\":%.1f,\"shfl64_lat\":%.1f,\"mufu_dadd_lat\":%.1f}\n",
             names[mode], mode ? nbg : 0, (double)cyc[0] / N, (double)cyc[1] / N, (double)cyc[2] / N);
    }
  return 0;
}
