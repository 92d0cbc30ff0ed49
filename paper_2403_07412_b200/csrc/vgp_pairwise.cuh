// numpy's float64 pairwise summation (what ndarray.sum() does on contiguous
// data) restated for the device, so device totals reproduce
// vecchia._ordered_sum (vg/vecchia.py:169-177) and half_log_det
// (vg/batchla.py:232-237) bit for bit given the same summands:
//   n < 8        : sequential from 0.0
//   n <= 128     : 8 strided accumulators, ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)), tail sequential
//   otherwise    : split at n2 = n/2 - (n/2 % 8) and add the two halves
#pragma once
#include <stdint.h>

namespace vgp {

__device__ inline double pairwise_block(const double* p, int64_t n) {
  if (n < 8) {
    double res = 0.0;
    for (int64_t i = 0; i < n; ++i) res += p[i];
    return res;
  }
  double r[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) r[j] = p[j];
  int64_t i;
  for (i = 8; i < n - (n % 8); i += 8) {
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] += p[i + j];
  }
  double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
  for (; i < n; ++i) res += p[i];
  return res;
}

// Iterative form of the recursion (explicit stack, depth <= 64).
__device__ inline double pairwise_rec(const double* a, int64_t n) {
  struct Frame {
    int64_t off, n;
    int state;
    double left;
  };
  Frame st[64];
  int sp = 0;
  st[0] = {0, n, 0, 0.0};
  double ret = 0.0;
  while (sp >= 0) {
    Frame& f = st[sp];
    if (f.n <= 128) {
      ret = pairwise_block(a + f.off, f.n);
      --sp;
      continue;
    }
    int64_t n2 = f.n / 2;
    n2 -= n2 % 8;
    if (f.state == 0) {
      f.state = 1;
      st[++sp] = {f.off, n2, 0, 0.0};
    } else if (f.state == 1) {
      f.left = ret;
      f.state = 2;
      st[++sp] = {f.off + n2, f.n - n2, 0, 0.0};
    } else {
      ret = f.left + ret;
      --sp;
    }
  }
  return ret;
}

}  // namespace vgp
