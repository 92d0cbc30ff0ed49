// Internal declarations shared by the sm_100a translation units of
// libvecchia_b200.so.  Nothing here crosses the C ABI (include/vecchia_b200.h).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <utility>
#include <vector>

#include "vecchia_b200.h"

namespace vgp {

// ---------------------------------------------------------------- errors

void set_error(const std::string& msg);
int fail(int code, const std::string& msg);

#define VGP_CUDA_TRY(expr)                                                          \
  do {                                                                              \
    cudaError_t _e = (expr);                                                        \
    if (_e != cudaSuccess)                                                          \
      return ::vgp::fail(VGP_E_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e)); \
  } while (0)

constexpr double kLog2Pi = 1.8378770664093453;  // math.log(2*pi), vg/vecchia.py:31
constexpr double kPi = 3.141592653589793;

// Reduction chunk of vecchia._ordered_sum (vg/vecchia.py:35).
constexpr int64_t kReduceChunk = 4096;

// ---------------------------------------------------------------- covariance

enum CovKind : int {
  kMatern05 = 0,   // s2 exp(-u)                      vg/kernels.py:69-70
  kMatern15 = 1,   // s2 (1+u) exp(-u)                vg/kernels.py:71-72
  kMatern25 = 2,   // s2 (1+u+u^2/3) exp(-u)          vg/kernels.py:73-74
  kMaternGen = 3,  // s2 2^(1-nu)/G(nu) u^nu K_nu(u)  vg/kernels.py:75-81
  kPowExp = 4,     // s2 exp(-d^nu / beta)            vg/kernels.py:85-91
};

// Per-evaluation covariance constants (everything that depends on theta only
// is folded on the host once per likelihood evaluation).
struct CovParams {
  int kind;
  int nl;          // general nu: number of upward recurrence steps (nu = mu + nl)
  double s2, beta, inv_beta, nu;
  double coef;     // 2^(1-nu) / Gamma(nu)
  double mu;       // nu - nl, in [-0.5, 0.5)
  double gam1, gam2, gampl, gammi, fact;  // Temme series constants (see bessel_k)
};

int make_cov_params(int family, double s2, double beta, double nu, CovParams* out);

// ---------------------------------------------------------------- plan

struct Plan {
  int device = 0;
  int64_t n = 0;
  int32_t m = 0;
  int metric = VGP_METRIC_EUCLIDEAN;
  double radius = 6371.0;
  int64_t blk_lo = 0, blk_hi = 0;  // batch entries [blk_lo, blk_hi); entry 0 = joint block
  int64_t rest_lo = 0, rest_hi = 0;  // block_rest indices k = e - 1 covered by this plan
  cudaStream_t stream = nullptr;
  cudaStream_t side = nullptr;  // joint block and result downloads overlap the main kernel
  cudaStream_t aux = nullptr;   // vgp_loglik_data: location upload + check next to the evaluation
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  cudaEvent_t ev_chunk[8] = {};
  int64_t* d_order = nullptr;   // n, ordered position -> original index
  int32_t* d_nbr = nullptr;     // (rest_hi - rest_lo) x m, row r <-> entry rest_lo + r + 1
  double4* d_pts = nullptr;     // n x (x, y, obs, 0), ordered
  double* d_raw = nullptr;      // n x 3 upload staging (x, y, obs), original order
  double* d_rest = nullptr;     // block_rest / mu_new / sigma_new for the local range
  double* d_mu = nullptr;
  double* d_sig = nullptr;
  double* d_partials = nullptr; // chunk partials for local chunks
  double* d_scalars = nullptr;  // [0] total, [1] block_first
  unsigned long long* d_fail = nullptr;  // [0] NPD key, [1] variance index
  double* d_work = nullptr;     // global workspace for the large-m generic path
  size_t work_doubles = 0;
  int work_slots = 0;
  double* h_stage = nullptr;    // pinned host staging (n x 3 doubles)
  double* h_small = nullptr;    // pinned scalars
  bool has_data = false;
  int num_sms = 148;
  int64_t chunk_lo = 0, chunk_hi = 0;  // global 4096-chunk ids covered (rest range aligned)
  int kernel_variant = -1;      // last kernel used (for introspection)
  int force_variant = -1;       // -1 auto
  int tune = 0;                 // experiment selector (env VGP_TUNE at plan creation)
  double* d_gscratch = nullptr; // large-m kernel: per-CTA tile triangles (L2-resident)
  int gscratch_slots = 0;
  double* d_ktab = nullptr;     // general-nu Matern polynomial table (vgp_ktab.cuh), per evaluation
  bool no_ktab = false;         // env VGP_NO_KTAB: exact Bessel K in every entry (testing aid)
  double* d_dcache = nullptr;   // per-block distance cache (ws:: tile layout)
  int64_t dcache_stride = 0;    // doubles per block (16-byte multiple)
  bool dcache_valid = false;
  double dcache_dmax = 0.0;     // largest cached distance (K_nu table shared-memory window)
  double* d_prev_locs = nullptr;  // locations the cache was built from (n x 2)
  int* d_flag = nullptr;
  bool timing = false;          // record events around the fused kernel
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>>* events = nullptr;  // pending pairs
  std::vector<cudaEvent_t>* event_pool = nullptr;
};

// ---------------------------------------------------------------- kernels (launchers)

// kNN, vg/geo.py:234-263 / :331-358. All pointers are device pointers.
cudaError_t launch_knn(const double2* d_data, int64_t nd, const double2* d_query, int64_t nq,
                       int64_t q_offset, int pred, int32_t m, int64_t* d_out, double* d_keys,
                       int32_t* d_idx, cudaStream_t stream);

// Sphere kNN (vg/geo.py:266-292); points (lambda, phi, cos phi, 0) in radians.
cudaError_t launch_knn_sphere(const double4* d_data, int64_t nd, const double4* d_query, int64_t nq,
                              int64_t q_offset, int pred, int32_t m, int64_t* d_out, double* d_keys,
                              int32_t* d_idx, cudaStream_t stream);

// Predecessor kNN by index batches with a grid over the earlier points
// (vgp_knn.cu), bit-identical to launch_knn; h_locs / h_out on the host.
cudaError_t knn_pred_grid(const double2* d_pts, const double* h_locs, int64_t n, int32_t m, int64_t batch,
                          int64_t* h_out, cudaStream_t st, int64_t row_lo = 0, int64_t row_hi = -1);

// The same for great-circle plans: points (lambda, phi, cos phi, 0) on the device.
cudaError_t knn_pred_grid_sphere(const double4* d_pts, int64_t n, int32_t m, int64_t batch, int64_t* h_out,
                                 cudaStream_t st);

// Thread-per-block kernel for m <= 10, closed-form Matern, Euclidean (vgp_tiny.cu).
bool tiny_supported(int m, int kind);
cudaError_t launch_loglik_tiny(const Plan& p, const CovParams& cp, int64_t e_lo, int64_t e_hi,
                               cudaStream_t stream);

// Exact maxmin ordering (vgp_maxmin.cu): order[t] for t < n, starting at
// `first`; bbox = (x0, x1, y0, y1) of the points; at most maxmin_capacity()
// points (one cluster holds every chunk's metadata in shared memory).
int64_t maxmin_capacity();
cudaError_t launch_maxmin(const double2* d_pts, int64_t n, int64_t first, const double bbox[4],
                          int64_t* d_order, cudaStream_t stream);

// Materialised conditioning batches for entries [e0, e0 + ne) (vgp_assemble.cu).
cudaError_t launch_assemble(const double2* d_pts, const double* d_obs, int m, const int64_t* d_nbr, int64_t e0,
                            int64_t ne, int metric, double radius, const CovParams& cp, double* d_S,
                            double* d_v, double* d_y, int num_sms, cudaStream_t s);

// Permute raw (x, y, obs) rows into ordered double4 points.
cudaError_t launch_permute(const double* d_raw, const int64_t* d_order, int64_t n,
                           double4* d_pts, cudaStream_t stream);

// Vecchia forward simulation of ordered observations (vgp_simulate.cu):
// d_z, d_y ORDERED (n,); needs a full-range plan.  *d_fail gets the first
// non-positive-definite entry (initialise to ~0).
cudaError_t launch_simulate(const Plan& p, const CovParams& cp, const double* d_z, double* d_y,
                            unsigned long long* d_fail, cudaStream_t stream);

// Permute only the observations into pts[i].z (locations unchanged).
cudaError_t launch_permute_obs(const double* d_obs, const int64_t* d_order, int64_t n, double4* d_pts,
                               cudaStream_t stream);

// Generic per-block likelihood kernel (any m; smem- or global-resident block).
cudaError_t launch_loglik_generic(const Plan& p, const CovParams& cp, int64_t e_lo, int64_t e_hi,
                                  cudaStream_t stream);

// Fast warp-per-block DMMA kernel for m + 2 <= 64.  Returns cudaErrorNotSupported
// when the shape is not covered.
cudaError_t launch_loglik_dmma(const Plan& p, const CovParams& cp, int64_t e_lo, int64_t e_hi,
                               cudaStream_t stream);
bool dmma_supported(int m, int kind);
// Warp-specialised DMMA kernel (chain + worker warp per block), same
// coverage; `cache` streams the plan's distance cache (vgp_dcache.cu).
cudaError_t launch_loglik_ws(const Plan& p, const CovParams& cp, int64_t e_lo, int64_t e_hi,
                             cudaStream_t stream, bool cache);
// CTA-per-block DMMA kernel (vgp_big_kernel.cuh): any m, every kernel family
// (general nu via the device Bessel K); tiles in shared memory or, past
// ~200 KB, in d_gscratch.
bool big_supported(int m, int kind);
bool big_needs_scratch(int m);
int64_t big_scratch_doubles(int m);
cudaError_t launch_loglik_big(const Plan& p, const CovParams& cp, int64_t e_lo, int64_t e_hi,
                              cudaStream_t stream, bool cache);
// Scheduler-aware layout: one worker warp per SM sub-partition serving the
// two blocks whose chain warps share that sub-partition (vgp_ws3_kernel.cuh).
// closed forms or general nu (table) with m + 2 <= 64
bool ws3_supported(int m, int kind);
cudaError_t launch_loglik_ws3(const Plan& p, const CovParams& cp, int64_t e_lo, int64_t e_hi,
                              cudaStream_t stream, bool cache);

// Scatter the shard's chunk partials (and block_first) into a global device
// vector for the cross-GPU all-reduce; NaN-poison on failure.
cudaError_t launch_scatter_partials(const Plan& p, double* d_out, cudaStream_t stream);

// Distance cache (vgp_dcache.cu).
int64_t dcache_stride(int m);
cudaError_t launch_build_dcache(const Plan& p, cudaStream_t stream);
cudaError_t launch_diff(const double* a, const double* b, int64_t n, int* flag,
                        cudaStream_t stream);

// numpy-pairwise 4096-chunk partials of d_rest and the ordered total.
cudaError_t launch_reduce(const Plan& p, bool want_total, cudaStream_t stream);

// Covariance evaluation at distances (kernels.cov, vg/kernels.py:94-98).
cudaError_t launch_cov_eval(const CovParams& cp, const double* d_in, int64_t count, double* d_out,
                            cudaStream_t stream);

// K_nu(x) at given points (kernels.bessel_kv, vg/kernels.py:50-56); cp from
// make_cov_params(MATERN, 1, 1, nu) with the general-nu constants filled.
cudaError_t launch_bessel_eval(const CovParams& cp, const double* d_in, int64_t count,
                               double* d_out, cudaStream_t stream);
int make_bessel_params(double nu, CovParams* out);

// NPD key: (chunk(e), pivot column, e) ordered like the reference's first raise
// (vg/batchla.py:146-151 inside parallel.map_chunks, vg/parallel.py:37-43).
__host__ __device__ inline unsigned long long npd_key(int64_t e, int j, int m) {
  if (m > 256) return (unsigned long long)e;  // per-entry LAPACK path, vg/batchla.py:159-164
  int64_t chunk = (int64_t(1) << 21) / (int64_t(m) * m);
  if (chunk < 1) chunk = 1;
  unsigned long long c = (unsigned long long)(e / chunk);
  unsigned long long w = (unsigned long long)(e % chunk);
  return (c << 42) | ((unsigned long long)j << 24) | w;
}
inline int64_t npd_key_entry(unsigned long long key, int m) {
  if (m > 256) return (int64_t)key;
  int64_t chunk = (int64_t(1) << 21) / (int64_t(m) * m);
  if (chunk < 1) chunk = 1;
  return (int64_t)(key >> 42) * chunk + (int64_t)(key & ((1ull << 24) - 1));
}

}  // namespace vgp
