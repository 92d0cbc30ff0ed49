// FP64 peak microbenchmark for B200 (sm_100a): DFMA pipe, DMMA (mma.sync f64)
// and both concurrently. Used to fix the roofline denominator for the fused
// Vecchia kernel (MEASURED_PEAKS.json carries no FP64 figure).
#include <cstdio>
#include <cuda_runtime.h>

#define CHECK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

template <int CHAINS>
__device__ __forceinline__ void dfma_body(double* acc, double a, double b, int iters) {
#pragma unroll 1
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) acc[c] = fma(acc[c], a, b);
  }
}

__global__ void k_dfma(double* out, double a, double b, int iters) {
  double acc[16];
#pragma unroll
  for (int c = 0; c < 16; ++c) acc[c] = threadIdx.x * 1e-3 + c;
  dfma_body<16>(acc, a, b, iters);
  double s = 0;
#pragma unroll
  for (int c = 0; c < 16; ++c) s += acc[c];
  if (s == 12345.678) out[threadIdx.x] = s;
}

// m8n8k4 f64: A 1 reg, B 1 reg, C/D 2 regs per thread. 2*8*8*4 = 512 flop per warp-mma.
__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
// m16n8k16 f64 (sm_90+ PTX): A 8 regs, B 4 regs, C/D 4 regs. 2*16*8*16 = 4096 flop.
__device__ __forceinline__ void dmma16816(double* d, const double* a, const double* b) {
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, "
               "{%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
               : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
               : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                 "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
}

__global__ void k_dmma884(double* out, int iters) {
  double d[8][2];
  double a = 1e-9 * threadIdx.x, b = 1e-9;
#pragma unroll
  for (int c = 0; c < 8; ++c) { d[c][0] = c; d[c][1] = -c; }
#pragma unroll 1
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < 8; ++c) dmma884(d[c][0], d[c][1], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < 8; ++c) s += d[c][0] + d[c][1];
  if (s == 12345.678) out[threadIdx.x] = s;
}

__global__ void k_dmma16816(double* out, int iters) {
  double d[4][4], a[8], b[4];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = 1e-9 * (threadIdx.x + i);
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = 1e-9 * i;
#pragma unroll
  for (int c = 0; c < 4; ++c)
#pragma unroll
    for (int i = 0; i < 4; ++i) d[c][i] = c + i;
#pragma unroll 1
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < 4; ++c) dmma16816(d[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < 4; ++c)
#pragma unroll
    for (int i = 0; i < 4; ++i) s += d[c][i];
  if (s == 12345.678) out[threadIdx.x] = s;
}

// half the warps DFMA, half DMMA 8x8x4
__global__ void k_mixed(double* out, double a0, double b0, int iters) {
  int w = threadIdx.x / 32;
  if (w & 1) {
    double d[8][2];
    double a = 1e-9 * threadIdx.x, b = 1e-9;
#pragma unroll
    for (int c = 0; c < 8; ++c) { d[c][0] = c; d[c][1] = -c; }
#pragma unroll 1
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int c = 0; c < 8; ++c) dmma884(d[c][0], d[c][1], a, b);
    }
    double s = 0;
#pragma unroll
    for (int c = 0; c < 8; ++c) s += d[c][0] + d[c][1];
    if (s == 12345.678) out[threadIdx.x] = s;
  } else {
    double acc[16];
#pragma unroll
    for (int c = 0; c < 16; ++c) acc[c] = threadIdx.x * 1e-3 + c;
    dfma_body<16>(acc, a0, b0, iters * 4);
    double s = 0;
#pragma unroll
    for (int c = 0; c < 16; ++c) s += acc[c];
    if (s == 12345.678) out[threadIdx.x] = s;
  }
}

int main() {
  int sms = 0, clk = 0;
  CHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  CHECK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0));
  double* out; CHECK(cudaMalloc(&out, 1 << 20));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int threads = 256;
  for (int bpsm : {2, 4, 8}) {
    int blocks = sms * bpsm;
    int iters = 20000;
    for (int rep = 0; rep < 2; ++rep) {
      k_dfma<<<blocks, threads>>>(out, 1.0000001, 1e-7, iters);
      cudaEventRecord(e0);
      k_dfma<<<blocks, threads>>>(out, 1.0000001, 1e-7, iters);
      cudaEventRecord(e1); CHECK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double flop = 2.0 * 16 * iters * (double)blocks * threads;
      if (rep) printf("{\"kernel\":\"dfma\",\"blocks_per_sm\":%d,\"ms\":%.3f,\"tflops\":%.3f}\n", bpsm, ms, flop / ms / 1e9);
    }
    for (int rep = 0; rep < 2; ++rep) {
      k_dmma884<<<blocks, threads>>>(out, iters);
      cudaEventRecord(e0);
      k_dmma884<<<blocks, threads>>>(out, iters);
      cudaEventRecord(e1); CHECK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double flop = 512.0 * 8 * iters * (double)blocks * (threads / 32);
      if (rep) printf("{\"kernel\":\"dmma_m8n8k4\",\"blocks_per_sm\":%d,\"ms\":%.3f,\"tflops\":%.3f}\n", bpsm, ms, flop / ms / 1e9);
    }
    for (int rep = 0; rep < 2; ++rep) {
      k_dmma16816<<<blocks, threads>>>(out, iters / 4);
      cudaEventRecord(e0);
      k_dmma16816<<<blocks, threads>>>(out, iters / 4);
      cudaEventRecord(e1); CHECK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double flop = 4096.0 * 4 * (iters / 4) * (double)blocks * (threads / 32);
      if (rep) printf("{\"kernel\":\"dmma_m16n8k16\",\"blocks_per_sm\":%d,\"ms\":%.3f,\"tflops\":%.3f}\n", bpsm, ms, flop / ms / 1e9);
    }
    for (int rep = 0; rep < 2; ++rep) {
      k_mixed<<<blocks, threads>>>(out, 1.0000001, 1e-7, iters);
      cudaEventRecord(e0);
      k_mixed<<<blocks, threads>>>(out, 1.0000001, 1e-7, iters);
      cudaEventRecord(e1); CHECK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double flop = (2.0 * 16 * iters * 4 * 32 + 512.0 * 8 * iters) * (double)blocks * (threads / 64);
      if (rep) printf("{\"kernel\":\"mixed_dfma_dmma\",\"blocks_per_sm\":%d,\"ms\":%.3f,\"tflops\":%.3f}\n", bpsm, ms, flop / ms / 1e9);
    }
  }
  printf("{\"sms\":%d,\"clock_khz\":%d}\n", sms, clk);
  CHECK(cudaGetLastError());
  return 0;
}
