// C ABI of libvecchia_b200.so (include/vecchia_b200.h): argument checking,
// device memory of a plan, host<->device staging and status mapping.  All
// arithmetic happens in the sm_100a kernels of the sibling .cu files; there is
// no host compute path.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "vgp_internal.cuh"
#include "vgp_ktab.cuh"

namespace vgp {

static thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

// Taylor coefficients of 1/Gamma(1+x) about 0 (a_0 .. a_24), mpmath at 50 digits.
static const double kRecipGammaTaylor[25] = {
    0x1.0000000000000p+0,   0x1.2788cfc6fb619p-1,  -0x1.4fcf4026afa2ep-1, -0x1.5815e8fa27048p-5,
    0x1.5512320b43fbep-3,  -0x1.59af103c34092p-5,  -0x1.3b4af28483e21p-7, 0x1.d919c527f60b2p-8,
    -0x1.317112ce3a2a8p-10, -0x1.c364fe6f1563dp-13, 0x1.0c8a78cd9f9d2p-13, -0x1.51ce8af47eabep-16,
    -0x1.4fad41fc34fbbp-20, 0x1.302509dbc0de3p-20, -0x1.b9986666c225dp-23, 0x1.a44b7ba22d629p-28,
    0x1.57bc3fc384334p-28,  -0x1.44b4cedca388fp-30, 0x1.cae7675c18607p-34, 0x1.11d065bfaf067p-37,
    -0x1.0423bac8ca3fbp-38, 0x1.1f20151323cd0p-41, -0x1.72cb88ea5ae6ep-46, -0x1.815f72a05f16fp-48,
    0x1.6198491a83bcdp-50};

void fill_bessel(double nu, CovParams* c);

int make_cov_params(int family, double s2, double beta, double nu, CovParams* c) {
  // KernelParams validation, vg/kernels.py:31-35
  if (!(std::isfinite(s2) && s2 > 0.0) || !(std::isfinite(beta) && beta > 0.0) ||
      !(std::isfinite(nu) && nu > 0.0))
    return fail(VGP_E_INVALID, "sigma_sq, beta and nu must be finite and > 0");
  std::memset(c, 0, sizeof(*c));
  c->s2 = s2;
  c->beta = beta;
  c->inv_beta = 1.0 / beta;
  c->nu = nu;
  if (family == VGP_FAMILY_POWEXP) {
    c->kind = kPowExp;
    return VGP_OK;
  }
  if (family != VGP_FAMILY_MATERN) return fail(VGP_E_INVALID, "unknown kernel family");
  // closed forms by exact equality, vg/kernels.py:69-74
  if (nu == 0.5) {
    c->kind = kMatern05;
  } else if (nu == 1.5) {
    c->kind = kMatern15;
  } else if (nu == 2.5) {
    c->kind = kMatern25;
  } else {
    c->kind = kMaternGen;
    c->coef = std::pow(2.0, 1.0 - nu) / std::tgamma(nu);  // 2^(1-nu)/Gamma(nu), vg/kernels.py:81
    fill_bessel(nu, c);
  }
  return VGP_OK;
}

int make_bessel_params(double nu, CovParams* c) {
  if (!(std::isfinite(nu) && nu >= 0.0)) return fail(VGP_E_INVALID, "nu must be finite and >= 0");
  std::memset(c, 0, sizeof(*c));
  c->kind = kMaternGen;
  c->nu = nu;
  fill_bessel(nu, c);
  return VGP_OK;
}

void fill_bessel(double nu, CovParams* c) {
  {
    int nl = (int)(nu + 0.5);
    double mu = nu - nl;
    c->nl = nl;
    c->mu = mu;
    // f(x) = 1/Gamma(1+x); gampl = f(mu), gammi = f(-mu),
    // gam1 = (f(-mu) - f(mu)) / (2 mu) = -sum_{k odd} a_k mu^(k-1),
    // gam2 = (f(-mu) + f(mu)) / 2     =  sum_{k even} a_k mu^k
    double fp = 0.0, fm = 0.0, g1 = 0.0, g2 = 0.0;
    for (int k = 24; k >= 0; --k) {
      fp = fp * mu + kRecipGammaTaylor[k];
      fm = fm * (-mu) + kRecipGammaTaylor[k];
    }
    for (int k = 23; k >= 1; k -= 2) g1 = g1 * (mu * mu) + kRecipGammaTaylor[k];
    for (int k = 24; k >= 0; k -= 2) g2 = g2 * (mu * mu) + kRecipGammaTaylor[k];
    c->gampl = fp;
    c->gammi = fm;
    c->gam1 = -g1;
    c->gam2 = g2;
    double pimu = kPi * mu;
    c->fact = std::fabs(pimu) < 1e-16 ? 1.0 : pimu / std::sin(pimu);
  }
}

namespace {

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

int check_device(int device) {
  int count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count == 0)
    return fail(VGP_E_CUDA, std::string("no CUDA device available (") +
                                (e == cudaSuccess ? "0 devices" : cudaGetErrorString(e)) +
                                "); the B200 path has no CPU fallback");
  if (device < 0 || device >= count) return fail(VGP_E_INVALID, "device ordinal out of range");
  return VGP_OK;
}

template <typename T>
int dalloc(T** p, size_t count) {
  *p = nullptr;
  if (count == 0) count = 1;
  cudaError_t e = cudaMalloc((void**)p, sizeof(T) * count);
  if (e != cudaSuccess) return fail(VGP_E_NOMEM, std::string("cudaMalloc: ") + cudaGetErrorString(e));
  return VGP_OK;
}

void free_plan(Plan* p) {
  if (!p) return;
  cudaFree(p->d_order);
  cudaFree(p->d_nbr);
  cudaFree(p->d_pts);
  cudaFree(p->d_raw);
  cudaFree(p->d_rest);
  cudaFree(p->d_mu);
  cudaFree(p->d_sig);
  cudaFree(p->d_partials);
  cudaFree(p->d_scalars);
  cudaFree(p->d_fail);
  cudaFree(p->d_work);
  cudaFree(p->d_gscratch);
  cudaFree(p->d_dcache);
  cudaFree(p->d_ktab);
  cudaFree(p->d_prev_locs);
  cudaFree(p->d_flag);
  if (p->h_stage) cudaFreeHost(p->h_stage);
  if (p->h_small) cudaFreeHost(p->h_small);
  if (p->events) {
    for (auto& pr : *p->events) {
      cudaEventDestroy(pr.first);
      cudaEventDestroy(pr.second);
    }
    delete p->events;
  }
  if (p->event_pool) {
    for (auto ev : *p->event_pool) cudaEventDestroy(ev);
    delete p->event_pool;
  }
  if (p->stream) cudaStreamDestroy(p->stream);
  if (p->side) cudaStreamDestroy(p->side);
  if (p->aux) cudaStreamDestroy(p->aux);
  if (p->ev_fork) cudaEventDestroy(p->ev_fork);
  if (p->ev_join) cudaEventDestroy(p->ev_join);
  for (auto ev : p->ev_chunk)
    if (ev) cudaEventDestroy(ev);
  delete p;
}

int take_event(Plan* p, cudaEvent_t* ev) {
  if (!p->event_pool->empty()) {
    *ev = p->event_pool->back();
    p->event_pool->pop_back();
    return VGP_OK;
  }
  VGP_CUDA_TRY(cudaEventCreate(ev));
  return VGP_OK;
}

// Host destinations of the per-block results (vgp_loglik); null = none.
struct HostOut {
  double* rest = nullptr;
  double* mu = nullptr;
  double* sig = nullptr;
};

// Launch the full evaluation sequence on the plan's stream.  The joint block
// (entry 0, generic kernel) runs on the side stream next to the main kernel.
// With host outputs the main kernel is launched in chunks of blocks and each
// chunk's results are downloaded (side stream) while later chunks compute;
// the caller synchronises both streams.
int launch_eval(Plan* p, const CovParams& cp, bool want_total, const HostOut* out = nullptr) {
  cudaStream_t s = p->stream;
  VGP_CUDA_TRY(cudaMemsetAsync(p->d_fail, 0xff, 2 * sizeof(unsigned long long), s));
  int64_t e_lo = p->blk_lo, e_hi = p->blk_hi;
  const bool joint = e_lo == 0;
  // the generic kernel's global workspace slots are per CTA: when the main
  // launch may use them too, the joint block runs first on the main stream
  const bool serial_joint = p->d_work != nullptr;
  if (joint && serial_joint) {
    VGP_CUDA_TRY(launch_loglik_generic(*p, cp, 0, 1, s));
    e_lo = 1;
  } else if (joint) {
    VGP_CUDA_TRY(cudaEventRecord(p->ev_fork, s));
    VGP_CUDA_TRY(cudaStreamWaitEvent(p->side, p->ev_fork, 0));
    VGP_CUDA_TRY(launch_loglik_generic(*p, cp, 0, 1, p->side));
    VGP_CUDA_TRY(cudaEventRecord(p->ev_join, p->side));
    e_lo = 1;
  } else {
    VGP_CUDA_TRY(cudaMemsetAsync(p->d_scalars + 1, 0, sizeof(double), s));
  }
  if (e_hi > e_lo) {
    // variants: -1 auto, 0 generic, 1 all-register warp-DMMA, 2 grouped
    // warp-DMMA, 3 warp-specialised DMMA, 4 warp-specialised + distance cache,
    // (5, 6, 9, 10: retired experiments),
    // 7 scheduler-aware warp-specialised, 8 the same + distance cache,
    // 11 large-m CTA-per-block, 12 the same + distance cache
    // The DMMA kernels only need distances: with the distance cache (built
    // for either metric) they cover great-circle plans too; computing
    // distances on the fly they are Euclidean only.
    const bool eu = p->metric == VGP_METRIC_EUCLIDEAN;
    const bool cached = p->d_dcache && p->dcache_valid;
    const bool fast_c = dmma_supported(p->m, cp.kind) && cached;
    const bool fast_n = dmma_supported(p->m, cp.kind) && eu;
    // general-nu Matern: covariances from a per-evaluation polynomial table
    // (vgp_ktab.cuh), built here once per evaluation, in the scheduler-aware
    // kernel for m + 2 <= 64 and in the large-m kernel
    if (cp.kind == kMaternGen && !p->no_ktab) {
      if (!p->d_ktab) VGP_CUDA_TRY(cudaMalloc(&p->d_ktab, sizeof(double) * kKtabDoubles));
      VGP_CUDA_TRY(launch_ktab_build(cp, p->d_ktab, s));
    }
    const bool gen3 = cp.kind == kMaternGen && p->d_ktab && !p->no_ktab && ws3_supported(p->m, cp.kind);
    const bool ws3_c = (fast_c || gen3) && cached;
    const bool ws3_n = (fast_n || gen3) && eu;
    const bool scratch_ok = !big_needs_scratch(p->m) || p->d_gscratch;
    const bool big_c = big_supported(p->m, cp.kind) && cached && scratch_ok;
    const bool big_n = big_supported(p->m, cp.kind) && eu && scratch_ok;
    int v = p->force_variant;
    // (the CTA-per-block kernel is faster computing Euclidean distances than
    // streaming them for the closed forms, profiles/r01_sweep_c3_n250k.jsonl;
    // for general nu / power exponential, where covariance generation
    // dominates, streaming them is 1.6x faster, profiles/r01_c5_general_nu.txt)
    const bool big_prefer_cache = cp.kind >= kMaternGen;
    // by tile count (profiles/r01_smallm_variants.txt): up to 3 tile columns
    // one warp per block with everything in registers wins; up to 7 the
    // warp-specialised pair streaming the cache; 8 the scheduler-aware layout
    const bool small = p->m + 2 <= 24;
    const bool mid = p->m + 2 <= 56;
    const bool tiny = tiny_supported(p->m, cp.kind) && eu;
    if (v < 0)
      v = tiny ? 13
        : small && fast_n ? 1
        : (small || mid) && fast_c ? 4
        : ws3_c ? 8
        : (ws3_n ? 7
                 : (big_c && big_prefer_cache ? 12 : (big_n ? 11 : (big_c ? 12 : 0))));
    // (2 grouped warp-DMMA and 3 uncached warp-specialised pair: retired in
    // round 2 — never auto-selected)
    const bool ok = v == 0 || (v == 1 && fast_n) || (v == 7 && ws3_n) ||
                    (v == 4 && fast_c) || (v == 8 && ws3_c) || (v == 11 && big_n) || (v == 12 && big_c) ||
                    (v == 13 && tiny);
    if (!ok) return fail(VGP_E_UNSUPPORTED, "kernel variant does not cover this plan (m, kernel, metric, cache)");
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    if (p->timing) {
      int rc = take_event(p, &ev0);
      if (!rc) rc = take_event(p, &ev1);
      if (rc) return rc;
      VGP_CUDA_TRY(cudaEventRecord(ev0, s));
    }
    auto main_kernel = [&](int64_t lo, int64_t hi) -> cudaError_t {
      if (v == 0) return launch_loglik_generic(*p, cp, lo, hi, s);
      if (v == 1) return launch_loglik_dmma(*p, cp, lo, hi, s);
      if (v == 4) return launch_loglik_ws(*p, cp, lo, hi, s, true);
      if (v <= 6 || v >= 9 && v <= 10) return cudaErrorNotSupported;  // retired variants
      if (v <= 8) return launch_loglik_ws3(*p, cp, lo, hi, s, v == 8);
      if (v == 13) return launch_loglik_tiny(*p, cp, lo, hi, s);
      return launch_loglik_big(*p, cp, lo, hi, s, v == 12);
    };
    const int64_t count = e_hi - e_lo;
    // chunks shrinking geometrically (60/25/10/4/1 %): a chunk's 24 bytes per
    // block download ~17x faster than the next chunk computes, so only the
    // last, 1% chunk's download is exposed (4 equal chunks exposed a quarter)
    constexpr int kChunks = 5;
    constexpr int kCut[kChunks + 1] = {0, 60, 85, 95, 99, 100};
    const int nchunk = (out && count >= 65536) ? kChunks : 1;
    auto cut = [&](int k) -> int64_t {
      return e_lo + (nchunk == 1 ? (k ? count : 0) : count * kCut[k] / 100);
    };
    // all chunks are queued before any download: a download into pageable
    // memory blocks the host, the later chunks keep the GPU busy meanwhile
    for (int k = 0; k < nchunk; ++k) {
      VGP_CUDA_TRY(main_kernel(cut(k), cut(k + 1)));
      if (out) VGP_CUDA_TRY(cudaEventRecord(p->ev_chunk[k], s));
    }
    p->kernel_variant = v;
    if (p->timing) {
      VGP_CUDA_TRY(cudaEventRecord(ev1, s));
      p->events->emplace_back(ev0, ev1);
    }
    for (int k = 0; out && k < nchunk; ++k) {
      const int64_t lo = cut(k), hi = cut(k + 1);
      VGP_CUDA_TRY(cudaStreamWaitEvent(p->side, p->ev_chunk[k], 0));
      const int64_t r0 = lo - 1 - p->rest_lo, nr = hi - lo;
      if (out->rest)
        VGP_CUDA_TRY(cudaMemcpyAsync(out->rest + r0, p->d_rest + r0, sizeof(double) * nr,
                                     cudaMemcpyDeviceToHost, p->side));
      if (out->mu)
        VGP_CUDA_TRY(cudaMemcpyAsync(out->mu + r0, p->d_mu + r0, sizeof(double) * nr,
                                     cudaMemcpyDeviceToHost, p->side));
      if (out->sig)
        VGP_CUDA_TRY(cudaMemcpyAsync(out->sig + r0, p->d_sig + r0, sizeof(double) * nr,
                                     cudaMemcpyDeviceToHost, p->side));
    }
  }
  if (joint && !serial_joint) VGP_CUDA_TRY(cudaStreamWaitEvent(s, p->ev_join, 0));
  VGP_CUDA_TRY(launch_reduce(*p, want_total, s));
  return VGP_OK;
}

int decode_status(const Plan* p, const unsigned long long* flags, int64_t* fail_index) {
  if (flags[0] != ~0ull) {
    if (fail_index) *fail_index = npd_key_entry(flags[0], p->m);
    return VGP_NOT_POSITIVE_DEFINITE;
  }
  if (flags[1] != ~0ull) {
    if (fail_index) *fail_index = (int64_t)flags[1];
    return VGP_BAD_CONDITIONAL_VARIANCE;
  }
  if (fail_index) *fail_index = -1;
  return VGP_OK;
}

}  // namespace
}  // namespace vgp

using namespace vgp;

struct vgp_plan {
  Plan p;
};

extern "C" {

const char* vgp_version(void) { return "vecchia_b200 0.1.0 (sm_100a)"; }

const char* vgp_last_error(void) { return g_last_error.c_str(); }

int vgp_device_count(int* count) {
  int c = 0;
  cudaError_t e = cudaGetDeviceCount(&c);
  if (e != cudaSuccess) c = 0;
  if (count) *count = c;
  return VGP_OK;
}

int vgp_knn_predecessors(int device, const double* locations, int64_t n, int32_t m,
                         int64_t* neighbors) {
  if (m < 1 || n <= m) return fail(VGP_E_INVALID, "need 1 <= m < n");
  return vgp_knn_predecessors_range(device, locations, n, m, 0, n - m, neighbors);
}

int vgp_knn_predecessors_range(int device, const double* locations, int64_t n, int32_t m,
                               int64_t row_lo, int64_t row_hi, int64_t* neighbors) {
  if (!locations || !neighbors) return fail(VGP_E_INVALID, "null pointer");
  if (m < 1 || n <= m) return fail(VGP_E_INVALID, "need 1 <= m < n");
  if (n > (int64_t)INT32_MAX) return fail(VGP_E_INVALID, "n exceeds int32 index range");
  if (row_lo < 0 || row_hi > n - m || row_lo > row_hi) return fail(VGP_E_INVALID, "row range outside [0, n - m)");
  if (row_lo == row_hi) return VGP_OK;
  n = m + row_hi;  // later points are never candidates of these targets
  int rc = check_device(device);
  if (rc) return rc;
  DeviceGuard g(device);
  cudaStream_t s;
  VGP_CUDA_TRY(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  double2* d_pts = nullptr;
  int64_t* d_out = nullptr;
  double* d_keys = nullptr;
  int32_t* d_idx = nullptr;
  const int64_t nq = row_hi - row_lo;
  // grid-pruned search past ~200k points (env VGP_KNN_GRID_MIN overrides);
  // both paths produce the same table bit for bit
  int64_t grid_min = 200000;
  if (const char* env = std::getenv("VGP_KNN_GRID_MIN")) grid_min = std::atoll(env);
  if (n >= grid_min) {
    rc = dalloc(&d_pts, n);
    cudaError_t e = cudaSuccess;
    if (!rc) e = cudaMemcpyAsync(d_pts, locations, sizeof(double2) * n, cudaMemcpyHostToDevice, s);
    if (!rc && e == cudaSuccess) e = knn_pred_grid(d_pts, locations, n, m, int64_t(1) << 21, neighbors, s, row_lo, row_hi);
    if (!rc && e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (!rc && e != cudaSuccess) rc = fail(VGP_E_CUDA, std::string("knn (grid): ") + cudaGetErrorString(e));
    cudaFree(d_pts);
    cudaStreamDestroy(s);
    return rc;
  }
  const int64_t batch = std::min<int64_t>(nq, int64_t(1) << 20);
  const int64_t slots = ((batch + 127) / 128) * 128;
  rc = dalloc(&d_pts, n);
  if (!rc) rc = dalloc(&d_out, (size_t)batch * m);
  if (!rc) rc = dalloc(&d_keys, (size_t)slots * m);
  if (!rc) rc = dalloc(&d_idx, (size_t)slots * m);
  cudaError_t e = cudaSuccess;
  if (!rc) e = cudaMemcpyAsync(d_pts, locations, sizeof(double2) * n, cudaMemcpyHostToDevice, s);
  for (int64_t q0 = 0; !rc && e == cudaSuccess && q0 < nq; q0 += batch) {
    int64_t qn = std::min(batch, nq - q0);
    e = launch_knn(d_pts, n, d_pts + m + row_lo + q0, qn, row_lo + q0, 1, m, d_out, d_keys, d_idx, s);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(neighbors + q0 * m, d_out, sizeof(int64_t) * qn * m,
                          cudaMemcpyDeviceToHost, s);
  }
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (!rc && e != cudaSuccess) rc = fail(VGP_E_CUDA, std::string("knn: ") + cudaGetErrorString(e));
  cudaFree(d_pts);
  cudaFree(d_out);
  cudaFree(d_keys);
  cudaFree(d_idx);
  cudaStreamDestroy(s);
  return rc;
}

int vgp_assemble(int device, const double* locations, const double* observations, int64_t n, int32_t m,
                 const int64_t* neighbors, int metric, double radius, int family, double sigma_sq,
                 double beta, double nu, double* sigma, int64_t sigma_stride, double* v, int64_t v_stride,
                 double* yj, int64_t yj_stride) {
  if (!locations || !observations || !sigma || !v || !yj || !neighbors)
    return fail(VGP_E_INVALID, "null pointer");
  if (m < 1 || n <= m) return fail(VGP_E_INVALID, "need 1 <= m < n");
  if (sigma_stride < (int64_t)m * m || v_stride < m || yj_stride < m)
    return fail(VGP_E_INVALID, "stride smaller than the block size");
  if (metric != VGP_METRIC_EUCLIDEAN && metric != VGP_METRIC_GREAT_CIRCLE)
    return fail(VGP_E_INVALID, "unknown metric");
  CovParams cp;
  int rc = make_cov_params(family, sigma_sq, beta, nu, &cp);
  if (rc) return rc;
  const int64_t count = n - m + 1;
  for (int64_t i = 0; i < (n - m) * (int64_t)m; ++i)
    if (neighbors[i] < 0 || neighbors[i] >= n) return fail(VGP_E_INVALID, "neighbour index out of range");
  rc = check_device(device);
  if (rc) return rc;
  DeviceGuard g(device);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  cudaStream_t s;
  VGP_CUDA_TRY(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  // entries per chunk: at most ~256 MB of matrices on the device
  const int64_t mm = (int64_t)m * m;
  const int64_t chunk = std::max<int64_t>(1, std::min<int64_t>(count, (int64_t(32) << 20) / mm));
  double2* d_pts = nullptr;
  double *d_obs = nullptr, *d_S = nullptr, *d_v = nullptr, *d_y = nullptr;
  int64_t* d_nbr = nullptr;
  rc = dalloc(&d_pts, n);
  if (!rc) rc = dalloc(&d_obs, n);
  if (!rc) rc = dalloc(&d_nbr, (size_t)(n - m) * m);
  if (!rc) rc = dalloc(&d_S, (size_t)chunk * mm);
  if (!rc) rc = dalloc(&d_v, (size_t)chunk * m);
  if (!rc) rc = dalloc(&d_y, (size_t)chunk * m);
  cudaError_t e = cudaSuccess;
  if (!rc) e = cudaMemcpyAsync(d_pts, locations, sizeof(double2) * n, cudaMemcpyHostToDevice, s);
  if (!rc && e == cudaSuccess) e = cudaMemcpyAsync(d_obs, observations, sizeof(double) * n, cudaMemcpyHostToDevice, s);
  if (!rc && e == cudaSuccess)
    e = cudaMemcpyAsync(d_nbr, neighbors, sizeof(int64_t) * (n - m) * m, cudaMemcpyHostToDevice, s);
  for (int64_t e0 = 0; !rc && e == cudaSuccess && e0 < count; e0 += chunk) {
    const int64_t ne = std::min(chunk, count - e0);
    e = launch_assemble(d_pts, d_obs, m, d_nbr, e0, ne, metric, metric == VGP_METRIC_GREAT_CIRCLE ? radius : 0.0, cp,
                        d_S, d_v, d_y, sms, s);
    if (e == cudaSuccess)
      e = cudaMemcpy2DAsync(sigma + e0 * sigma_stride, sizeof(double) * sigma_stride, d_S, sizeof(double) * mm,
                            sizeof(double) * mm, ne, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess)
      e = cudaMemcpy2DAsync(v + e0 * v_stride, sizeof(double) * v_stride, d_v, sizeof(double) * m,
                            sizeof(double) * m, ne, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess)
      e = cudaMemcpy2DAsync(yj + e0 * yj_stride, sizeof(double) * yj_stride, d_y, sizeof(double) * m,
                            sizeof(double) * m, ne, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);  // the device chunk is reused
  }
  if (!rc && e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (!rc && e != cudaSuccess) rc = fail(VGP_E_CUDA, std::string("assemble: ") + cudaGetErrorString(e));
  cudaFree(d_pts);
  cudaFree(d_obs);
  cudaFree(d_nbr);
  cudaFree(d_S);
  cudaFree(d_v);
  cudaFree(d_y);
  cudaStreamDestroy(s);
  return rc;
}

int vgp_maxmin_order(int device, const double* locations, int64_t n, int64_t first, int64_t* order) {
  if (!locations || !order) return fail(VGP_E_INVALID, "null pointer");
  if (n < 1) return fail(VGP_E_INVALID, "need n >= 1");
  if (first < 0 || first >= n) return fail(VGP_E_INVALID, "first index out of range");
  int rc = check_device(device);
  if (rc) return rc;
  DeviceGuard g(device);
  if (n > maxmin_capacity())
    return fail(VGP_E_UNSUPPORTED, "maxmin ordering holds at most " + std::to_string(maxmin_capacity()) + " points");
  double bbox[4] = {locations[0], locations[0], locations[1], locations[1]};
  for (int64_t i = 0; i < n; ++i) {
    const double x = locations[2 * i], y = locations[2 * i + 1];
    if (!(x == x) || !(y == y)) return fail(VGP_E_INVALID, "NaN location");
    bbox[0] = std::min(bbox[0], x);
    bbox[1] = std::max(bbox[1], x);
    bbox[2] = std::min(bbox[2], y);
    bbox[3] = std::max(bbox[3], y);
  }
  cudaStream_t s;
  VGP_CUDA_TRY(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  double2* d_pts = nullptr;
  int64_t* d_order = nullptr;
  rc = dalloc(&d_pts, n);
  if (!rc) rc = dalloc(&d_order, n);
  cudaError_t e = cudaSuccess;
  if (!rc) e = cudaMemcpyAsync(d_pts, locations, sizeof(double2) * n, cudaMemcpyHostToDevice, s);
  if (!rc && e == cudaSuccess) e = launch_maxmin(d_pts, n, first, bbox, d_order, s);
  if (!rc && e == cudaSuccess)
    e = cudaMemcpyAsync(order, d_order, sizeof(int64_t) * n, cudaMemcpyDeviceToHost, s);
  if (!rc && e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (!rc && e != cudaSuccess) rc = fail(VGP_E_CUDA, std::string("maxmin: ") + cudaGetErrorString(e));
  cudaFree(d_pts);
  cudaFree(d_order);
  cudaStreamDestroy(s);
  return rc;
}

int vgp_knn_sphere(int device, const double* data3, int64_t nd, const double* query3, int64_t nq,
                   int32_t m, int predecessors, int64_t* neighbors) {
  if (!data3 || !neighbors || (!predecessors && !query3)) return fail(VGP_E_INVALID, "null pointer");
  if (predecessors) {
    if (m < 1 || nd <= m) return fail(VGP_E_INVALID, "need 1 <= m < n");
    nq = nd - m;
  } else if (m < 1 || m > nd) {
    return fail(VGP_E_INVALID, "need 1 <= m <= nd");
  }
  if (nd > (int64_t)INT32_MAX) return fail(VGP_E_INVALID, "n exceeds int32 index range");
  if (nq <= 0) return VGP_OK;
  int rc = check_device(device);
  if (rc) return rc;
  DeviceGuard g(device);
  std::vector<double4> hd((size_t)nd), hq(predecessors ? 0 : (size_t)nq);
  for (int64_t i = 0; i < nd; ++i) hd[i] = make_double4(data3[3 * i], data3[3 * i + 1], data3[3 * i + 2], 0.0);
  for (int64_t i = 0; i < (int64_t)hq.size(); ++i)
    hq[i] = make_double4(query3[3 * i], query3[3 * i + 1], query3[3 * i + 2], 0.0);
  cudaStream_t s;
  VGP_CUDA_TRY(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  int64_t grid_min = 200000;  // as vgp_knn_predecessors
  if (const char* env = std::getenv("VGP_KNN_GRID_MIN")) grid_min = std::atoll(env);
  if (predecessors && nd >= grid_min) {
    double4* d_pts = nullptr;
    rc = dalloc(&d_pts, nd);
    cudaError_t e = cudaSuccess;
    if (!rc) e = cudaMemcpyAsync(d_pts, hd.data(), sizeof(double4) * nd, cudaMemcpyHostToDevice, s);
    if (!rc && e == cudaSuccess) e = knn_pred_grid_sphere(d_pts, nd, m, 32768, neighbors, s);
    if (!rc && e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (!rc && e != cudaSuccess) rc = fail(VGP_E_CUDA, std::string("knn sphere (grid): ") + cudaGetErrorString(e));
    cudaFree(d_pts);
    cudaStreamDestroy(s);
    return rc;
  }
  double4 *d_data = nullptr, *d_q = nullptr;
  int64_t* d_out = nullptr;
  double* d_keys = nullptr;
  int32_t* d_idx = nullptr;
  const int64_t batch = std::min<int64_t>(nq, int64_t(1) << 20);
  const int64_t slots = ((batch + 127) / 128) * 128;
  rc = dalloc(&d_data, nd);
  if (!rc && !predecessors) rc = dalloc(&d_q, nq);
  if (!rc) rc = dalloc(&d_out, (size_t)batch * m);
  if (!rc) rc = dalloc(&d_keys, (size_t)slots * m);
  if (!rc) rc = dalloc(&d_idx, (size_t)slots * m);
  cudaError_t e = cudaSuccess;
  if (!rc) e = cudaMemcpyAsync(d_data, hd.data(), sizeof(double4) * nd, cudaMemcpyHostToDevice, s);
  if (!rc && e == cudaSuccess && !predecessors)
    e = cudaMemcpyAsync(d_q, hq.data(), sizeof(double4) * nq, cudaMemcpyHostToDevice, s);
  for (int64_t q0 = 0; !rc && e == cudaSuccess && q0 < nq; q0 += batch) {
    int64_t qn = std::min(batch, nq - q0);
    e = predecessors ? launch_knn_sphere(d_data, nd, d_data + m + q0, qn, q0, 1, m, d_out, d_keys, d_idx, s)
                     : launch_knn_sphere(d_data, nd, d_q + q0, qn, q0, 0, m, d_out, d_keys, d_idx, s);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(neighbors + q0 * m, d_out, sizeof(int64_t) * qn * m,
                          cudaMemcpyDeviceToHost, s);
  }
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (!rc && e != cudaSuccess) rc = fail(VGP_E_CUDA, std::string("knn sphere: ") + cudaGetErrorString(e));
  cudaFree(d_data);
  cudaFree(d_q);
  cudaFree(d_out);
  cudaFree(d_keys);
  cudaFree(d_idx);
  cudaStreamDestroy(s);
  return rc;
}

int vgp_knn_points(int device, const double* query, int64_t nq, const double* data, int64_t nd,
                   int32_t m, int64_t* neighbors) {
  if (!query || !data || !neighbors) return fail(VGP_E_INVALID, "null pointer");
  if (m < 1 || m > nd) return fail(VGP_E_INVALID, "need 1 <= m <= nd");
  if (nq <= 0) return VGP_OK;
  int rc = check_device(device);
  if (rc) return rc;
  DeviceGuard g(device);
  cudaStream_t s;
  VGP_CUDA_TRY(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  double2 *d_data = nullptr, *d_q = nullptr;
  int64_t* d_out = nullptr;
  double* d_keys = nullptr;
  int32_t* d_idx = nullptr;
  const int64_t batch = std::min<int64_t>(nq, int64_t(1) << 20);
  const int64_t slots = ((batch + 127) / 128) * 128;
  rc = dalloc(&d_data, nd);
  if (!rc) rc = dalloc(&d_q, nq);
  if (!rc) rc = dalloc(&d_out, (size_t)batch * m);
  if (!rc) rc = dalloc(&d_keys, (size_t)slots * m);
  if (!rc) rc = dalloc(&d_idx, (size_t)slots * m);
  cudaError_t e = cudaSuccess;
  if (!rc) e = cudaMemcpyAsync(d_data, data, sizeof(double2) * nd, cudaMemcpyHostToDevice, s);
  if (!rc && e == cudaSuccess)
    e = cudaMemcpyAsync(d_q, query, sizeof(double2) * nq, cudaMemcpyHostToDevice, s);
  for (int64_t q0 = 0; !rc && e == cudaSuccess && q0 < nq; q0 += batch) {
    int64_t qn = std::min(batch, nq - q0);
    e = launch_knn(d_data, nd, d_q + q0, qn, q0, 0, m, d_out, d_keys, d_idx, s);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(neighbors + q0 * m, d_out, sizeof(int64_t) * qn * m,
                          cudaMemcpyDeviceToHost, s);
  }
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (!rc && e != cudaSuccess) rc = fail(VGP_E_CUDA, std::string("knn: ") + cudaGetErrorString(e));
  cudaFree(d_data);
  cudaFree(d_q);
  cudaFree(d_out);
  cudaFree(d_keys);
  cudaFree(d_idx);
  cudaStreamDestroy(s);
  return rc;
}

int vgp_cov(int device, int family, double sigma_sq, double beta, double nu, const double* d,
            int64_t count, double* out) {
  if (count < 0 || (count > 0 && (!d || !out))) return fail(VGP_E_INVALID, "bad arguments");
  CovParams cp;
  int rc = make_cov_params(family, sigma_sq, beta, nu, &cp);
  if (rc) return rc;
  if (count == 0) return VGP_OK;
  rc = check_device(device);
  if (rc) return rc;
  DeviceGuard g(device);
  double *d_in = nullptr, *d_out = nullptr;
  rc = dalloc(&d_in, count);
  if (!rc) rc = dalloc(&d_out, count);
  cudaError_t e = cudaSuccess;
  if (!rc) e = cudaMemcpy(d_in, d, sizeof(double) * count, cudaMemcpyHostToDevice);
  if (!rc && e == cudaSuccess) e = launch_cov_eval(cp, d_in, count, d_out, 0);
  if (!rc && e == cudaSuccess) e = cudaMemcpy(out, d_out, sizeof(double) * count, cudaMemcpyDeviceToHost);
  if (!rc && e != cudaSuccess) rc = fail(VGP_E_CUDA, std::string("cov: ") + cudaGetErrorString(e));
  cudaFree(d_in);
  cudaFree(d_out);
  return rc;
}

int vgp_bessel_kv(int device, double nu, const double* x, int64_t count, double* out) {
  if (count < 0 || (count > 0 && (!x || !out))) return fail(VGP_E_INVALID, "bad arguments");
  CovParams cp;
  int rc = make_bessel_params(nu, &cp);
  if (rc) return rc;
  for (int64_t i = 0; i < count; ++i)
    if (!(x[i] > 0.0)) return fail(VGP_E_INVALID, "bessel_kv requires x > 0");
  if (count == 0) return VGP_OK;
  rc = check_device(device);
  if (rc) return rc;
  DeviceGuard g(device);
  double *d_in = nullptr, *d_out = nullptr;
  rc = dalloc(&d_in, count);
  if (!rc) rc = dalloc(&d_out, count);
  cudaError_t e = cudaSuccess;
  if (!rc) e = cudaMemcpy(d_in, x, sizeof(double) * count, cudaMemcpyHostToDevice);
  if (!rc && e == cudaSuccess) e = launch_bessel_eval(cp, d_in, count, d_out, 0);
  if (!rc && e == cudaSuccess) e = cudaMemcpy(out, d_out, sizeof(double) * count, cudaMemcpyDeviceToHost);
  if (!rc && e != cudaSuccess) rc = fail(VGP_E_CUDA, std::string("bessel_kv: ") + cudaGetErrorString(e));
  cudaFree(d_in);
  cudaFree(d_out);
  return rc;
}

static int plan_create(int device, int64_t n, int32_t m, int metric, double radius,
                       const int64_t* order, const int64_t* shard_rows, int64_t block_lo,
                       int64_t block_hi, vgp_plan** out);

int vgp_plan_create(int device, int64_t n, int32_t m, int metric, double radius,
                    const int64_t* order, const int64_t* neighbors, int64_t block_lo,
                    int64_t block_hi, vgp_plan** out) {
  const int64_t rest_lo = std::max<int64_t>(block_lo, 1) - 1;
  return plan_create(device, n, m, metric, radius, order,
                     neighbors ? neighbors + rest_lo * (int64_t)m : nullptr, block_lo, block_hi, out);
}

int vgp_plan_create_shard(int device, int64_t n, int32_t m, int metric, double radius,
                          const int64_t* order, const int64_t* shard_neighbors, int64_t block_lo,
                          int64_t block_hi, vgp_plan** out) {
  return plan_create(device, n, m, metric, radius, order, shard_neighbors, block_lo, block_hi, out);
}

static int plan_create(int device, int64_t n, int32_t m, int metric, double radius,
                       const int64_t* order, const int64_t* neighbors, int64_t block_lo,
                       int64_t block_hi, vgp_plan** out) {
  if (!out || !order) return fail(VGP_E_INVALID, "null pointer");
  *out = nullptr;
  if (m < 1 || n <= m) return fail(VGP_E_INVALID, "need 1 <= m < n");
  if (n > (int64_t)INT32_MAX) return fail(VGP_E_INVALID, "n exceeds int32 index range");
  const int64_t count = n - m + 1;
  if (block_lo < 0 || block_hi > count || block_lo >= block_hi)
    return fail(VGP_E_INVALID, "block range outside [0, n - m + 1)");
  if (metric != VGP_METRIC_EUCLIDEAN && metric != VGP_METRIC_GREAT_CIRCLE)
    return fail(VGP_E_INVALID, "unknown metric");
  const int64_t rest_lo = std::max<int64_t>(block_lo, 1) - 1;
  const int64_t rest_hi = block_hi - 1;
  if (rest_hi > rest_lo && !neighbors) return fail(VGP_E_INVALID, "null neighbour table");
  if (rest_lo % kReduceChunk != 0)
    return fail(VGP_E_INVALID, "shard must start on a 4096-entry reduction chunk boundary");
  if (rest_hi < count - 1 && rest_hi % kReduceChunk != 0)
    return fail(VGP_E_INVALID, "shard must end on a 4096-entry reduction chunk boundary");
  int rc = check_device(device);
  if (rc) return rc;
  DeviceGuard g(device);
  Plan* p = new Plan();
  p->device = device;
  p->n = n;
  p->m = m;
  p->metric = metric;
  p->radius = radius;
  p->blk_lo = block_lo;
  p->blk_hi = block_hi;
  p->rest_lo = rest_lo;
  p->rest_hi = std::max(rest_hi, rest_lo);
  p->chunk_lo = rest_lo / kReduceChunk;
  p->chunk_hi = (p->rest_hi + kReduceChunk - 1) / kReduceChunk;
  cudaDeviceGetAttribute(&p->num_sms, cudaDevAttrMultiProcessorCount, device);
  if (const char* tv = std::getenv("VGP_TUNE")) p->tune = std::atoi(tv);
  if (const char* nk = std::getenv("VGP_NO_KTAB")) p->no_ktab = std::atoi(nk) != 0;
  p->events = new std::vector<std::pair<cudaEvent_t, cudaEvent_t>>();
  p->event_pool = new std::vector<cudaEvent_t>();
  const int64_t nrest = p->rest_hi - p->rest_lo;
  cudaError_t e = cudaStreamCreateWithFlags(&p->stream, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&p->side, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&p->aux, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&p->ev_fork, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&p->ev_join, cudaEventDisableTiming);
  for (int i = 0; i < 8 && e == cudaSuccess; ++i)
    e = cudaEventCreateWithFlags(&p->ev_chunk[i], cudaEventDisableTiming);
  if (e != cudaSuccess) {
    free_plan(p);
    return fail(VGP_E_CUDA, cudaGetErrorString(e));
  }
  rc = dalloc(&p->d_order, n);
  if (!rc) rc = dalloc(&p->d_nbr, (size_t)nrest * m);
  if (!rc) rc = dalloc(&p->d_pts, n);
  if (!rc) rc = dalloc(&p->d_raw, (size_t)n * 3);
  if (!rc) rc = dalloc(&p->d_rest, nrest);
  if (!rc) rc = dalloc(&p->d_mu, nrest);
  if (!rc) rc = dalloc(&p->d_sig, nrest);
  if (!rc) rc = dalloc(&p->d_partials, std::max<int64_t>(p->chunk_hi - p->chunk_lo, 1));
  if (!rc) rc = dalloc(&p->d_scalars, 4);  // total | block_first | - | reduction ticket
  if (!rc && cudaMemset(p->d_scalars, 0, 4 * sizeof(double)) != cudaSuccess) rc = fail(VGP_E_CUDA, "memset");
  if (!rc) rc = dalloc(&p->d_fail, 2);
  if (!rc) {
    // generic-path global workspace when a block does not fit in shared memory
    const int P = m + 2;
    size_t mat = (size_t)(P | 1) * P;
    if (sizeof(double) * (mat + 3 * (m + 1)) > 200 * 1024) {
      int slots = p->num_sms * 2;
      int64_t need = std::max<int64_t>(nrest, 1);
      if (need < slots) slots = (int)need;
      p->work_slots = slots;
      p->work_doubles = mat * slots;
      rc = dalloc(&p->d_work, p->work_doubles);
    }
  }
  // distance cache where it pays: the warp-specialised kernel (m + 2 <= 64)
  // and great-circle plans (haversine per entry would dominate)
  if (!rc && nrest > 0 && big_supported(m, kMatern15) &&
      (dmma_supported(m, kMatern15) || metric == VGP_METRIC_GREAT_CIRCLE)) {
    // distance cache: on unless VGP_DCACHE=0, and only when it fits in half
    // of the free device memory
    const char* env = std::getenv("VGP_DCACHE");
    const bool want = !(env && env[0] == '0');
    size_t freeb = 0, totalb = 0;
    cudaMemGetInfo(&freeb, &totalb);
    const int64_t stride = dcache_stride(m);
    const size_t bytes = sizeof(double) * (size_t)stride * (size_t)nrest;
    if (want && bytes < freeb / 2) {
      if (cudaMalloc((void**)&p->d_dcache, bytes) == cudaSuccess &&
          cudaMalloc((void**)&p->d_prev_locs, sizeof(double) * 2 * (size_t)n) == cudaSuccess &&
          cudaMalloc((void**)&p->d_flag, 4 * sizeof(int)) == cudaSuccess) {  // flag | pad | max distance (u64)
        p->dcache_stride = stride;
      } else {
        cudaFree(p->d_dcache);
        cudaFree(p->d_prev_locs);
        cudaFree(p->d_flag);
        p->d_dcache = nullptr;
        p->d_prev_locs = nullptr;
        p->d_flag = nullptr;
        cudaGetLastError();
      }
    }
  }
  if (!rc && nrest > 0 && big_supported(m, kMatern15) && big_needs_scratch(m)) {
    // large-m tiles: two CTA slots per SM (the scratch stays mostly in L2)
    const int slots = p->num_sms * 2;
    if (cudaMalloc((void**)&p->d_gscratch, sizeof(double) * (size_t)big_scratch_doubles(m) * slots) ==
        cudaSuccess) {
      p->gscratch_slots = slots;
    } else {
      p->d_gscratch = nullptr;
      cudaGetLastError();
    }
  }
  if (!rc && cudaMallocHost((void**)&p->h_small, 64) != cudaSuccess)
    rc = fail(VGP_E_NOMEM, "cudaMallocHost small");
  if (rc) {
    free_plan(p);
    return rc;
  }
  e = cudaMemcpyAsync(p->d_order, order, sizeof(int64_t) * n, cudaMemcpyHostToDevice, p->stream);
  if (e == cudaSuccess && nrest > 0) {
    // int64 -> int32 neighbour rows of this shard, via the pinned stage
    std::vector<int32_t> tmp((size_t)nrest * m);
    const int64_t* src = neighbors;  // rows [rest_lo, rest_hi)
    for (size_t i = 0; i < tmp.size(); ++i) {
      int64_t v = src[i];
      if (v < 0 || v >= n) {
        free_plan(p);
        return fail(VGP_E_INVALID, "neighbour index out of range");
      }
      tmp[i] = (int32_t)v;
    }
    e = cudaMemcpyAsync(p->d_nbr, tmp.data(), sizeof(int32_t) * tmp.size(), cudaMemcpyHostToDevice,
                        p->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(p->stream);
  }
  if (e == cudaSuccess) e = cudaStreamSynchronize(p->stream);
  if (e != cudaSuccess) {
    free_plan(p);
    return fail(VGP_E_CUDA, std::string("plan upload: ") + cudaGetErrorString(e));
  }
  vgp_plan* h = new vgp_plan();
  h->p = *p;
  delete p;  // ownership of the device buffers moved into h->p
  *out = h;
  return VGP_OK;
}

int vgp_krige(int device, const double* train_locations, const double* train_observations,
              int64_t n_train, const double* test_locations, int64_t n_test, int32_t m,
              const int64_t* neighbors, int metric, double radius, int family, double sigma_sq,
              double beta, double nu, double* predictions, double* variances,
              int64_t* fail_index) {
  if (fail_index) *fail_index = -1;
  if (!train_locations || !train_observations || !test_locations || !neighbors || !predictions ||
      !variances)
    return fail(VGP_E_INVALID, "null pointer");
  if (m < 1 || m > n_train) return fail(VGP_E_INVALID, "need 1 <= m <= n_train");
  if (n_test < 0) return fail(VGP_E_INVALID, "negative test count");
  if (metric != VGP_METRIC_EUCLIDEAN && metric != VGP_METRIC_GREAT_CIRCLE)
    return fail(VGP_E_INVALID, "unknown metric");
  if (n_test == 0) return VGP_OK;
  const int64_t np = (int64_t)m + n_test + n_train;
  if (np > (int64_t)INT32_MAX) return fail(VGP_E_INVALID, "too many points for int32 indices");
  CovParams cp;
  int rc = make_cov_params(family, sigma_sq, beta, nu, &cp);
  if (rc) return rc;
  rc = check_device(device);
  if (rc) return rc;
  DeviceGuard g(device);
  // Point layout [m unused | n_test targets | n_train data]: conditioning
  // block e (1..n_test) then has its target at m + e - 1, exactly where the
  // likelihood kernels look, and its neighbours at n_train-relative index +
  // m + n_test; the per-block mu / sigma_new outputs are the kriging mean and
  // variance (vg/fit.py:252-264: potrf, two trsv, two dots per test point).
  Plan* p = new Plan();
  p->device = device;
  p->n = np;
  p->m = m;
  p->metric = metric;
  p->radius = radius;
  p->blk_lo = 1;
  p->blk_hi = n_test + 1;
  p->rest_lo = 0;
  p->rest_hi = n_test;
  cudaDeviceGetAttribute(&p->num_sms, cudaDevAttrMultiProcessorCount, device);
  p->events = new std::vector<std::pair<cudaEvent_t, cudaEvent_t>>();
  p->event_pool = new std::vector<cudaEvent_t>();
  cudaError_t e = cudaStreamCreateWithFlags(&p->stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) {
    free_plan(p);
    return fail(VGP_E_CUDA, cudaGetErrorString(e));
  }
  rc = dalloc(&p->d_nbr, (size_t)n_test * m);
  if (!rc) rc = dalloc(&p->d_pts, np);
  if (!rc) rc = dalloc(&p->d_rest, n_test);
  if (!rc) rc = dalloc(&p->d_mu, n_test);
  if (!rc) rc = dalloc(&p->d_sig, n_test);
  if (!rc) rc = dalloc(&p->d_fail, 2);
  const bool fast = dmma_supported(m, cp.kind);
  // great-circle: the kernels take haversine distances from a one-shot
  // distance cache (vgp_dcache.cu); Euclidean distances are computed in place
  const bool gcd = metric == VGP_METRIC_GREAT_CIRCLE;
  if (!rc && gcd) {
    p->dcache_stride = dcache_stride(m);
    rc = dalloc(&p->d_dcache, (size_t)p->dcache_stride * n_test);
  }
  if (!rc && !fast && big_needs_scratch(m)) {
    const int slots = p->num_sms * 2;
    if (cudaMalloc((void**)&p->d_gscratch, sizeof(double) * (size_t)big_scratch_doubles(m) * slots) ==
        cudaSuccess)
      p->gscratch_slots = slots;
    else
      rc = fail(VGP_E_NOMEM, "kriging tile scratch");
  }
  if (rc) {
    free_plan(p);
    return rc;
  }
  {
    std::vector<double4> pts((size_t)np, make_double4(0.0, 0.0, 0.0, 0.0));
    for (int64_t q = 0; q < n_test; ++q)
      pts[m + q] = make_double4(test_locations[2 * q], test_locations[2 * q + 1], 0.0, 0.0);
    for (int64_t i = 0; i < n_train; ++i)
      pts[m + n_test + i] = make_double4(train_locations[2 * i], train_locations[2 * i + 1],
                                         train_observations[i], 0.0);
    std::vector<int32_t> nb((size_t)n_test * m);
    for (size_t i = 0; i < nb.size(); ++i) {
      const int64_t v = neighbors[i];
      if (v < 0 || v >= n_train) {
        free_plan(p);
        return fail(VGP_E_INVALID, "neighbour index out of range");
      }
      nb[i] = (int32_t)(v + m + n_test);
    }
    e = cudaMemcpyAsync(p->d_pts, pts.data(), sizeof(double4) * pts.size(), cudaMemcpyHostToDevice,
                        p->stream);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(p->d_nbr, nb.data(), sizeof(int32_t) * nb.size(), cudaMemcpyHostToDevice,
                          p->stream);
    if (e == cudaSuccess) e = cudaMemsetAsync(p->d_fail, 0xff, 2 * sizeof(unsigned long long), p->stream);
    if (e == cudaSuccess && gcd) {
      e = launch_build_dcache(*p, p->stream);
      p->dcache_valid = e == cudaSuccess;
    }
    if (e == cudaSuccess)
      e = fast ? launch_loglik_ws3(*p, cp, 1, n_test + 1, p->stream, gcd)
               : launch_loglik_big(*p, cp, 1, n_test + 1, p->stream, gcd);
    unsigned long long flags[2] = {0, 0};
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(predictions, p->d_mu, sizeof(double) * n_test, cudaMemcpyDeviceToHost, p->stream);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(variances, p->d_sig, sizeof(double) * n_test, cudaMemcpyDeviceToHost, p->stream);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(flags, p->d_fail, sizeof(flags), cudaMemcpyDeviceToHost, p->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(p->stream);
    free_plan(p);
    if (e != cudaSuccess) return fail(VGP_E_CUDA, std::string("krige: ") + cudaGetErrorString(e));
    // a non-positive pivot raises like batch_potrf (vg/batchla.py:146-151);
    // a non-positive variance is returned as is (no check in krige_predict)
    if (flags[0] != ~0ull) {
      if (fail_index) *fail_index = npd_key_entry(flags[0], m) - 1;
      return VGP_NOT_POSITIVE_DEFINITE;
    }
  }
  return VGP_OK;
}

int vgp_host_register(void* ptr, int64_t bytes) {
  if (!ptr || bytes <= 0) return fail(VGP_E_INVALID, "bad host range");
  VGP_CUDA_TRY(cudaHostRegister(ptr, (size_t)bytes, cudaHostRegisterDefault));
  return VGP_OK;
}

int vgp_host_unregister(void* ptr) {
  if (!ptr) return fail(VGP_E_INVALID, "null pointer");
  VGP_CUDA_TRY(cudaHostUnregister(ptr));
  return VGP_OK;
}

int vgp_plan_set_data(vgp_plan* plan, const double* locations, const double* observations) {
  if (!plan || !locations || !observations) return fail(VGP_E_INVALID, "null pointer");
  Plan* p = &plan->p;
  DeviceGuard g(p->device);
  const int64_t n = p->n;
  // (x, y) rows then observations, straight from the caller's arrays
  VGP_CUDA_TRY(cudaMemcpyAsync(p->d_raw, locations, sizeof(double) * 2 * n, cudaMemcpyHostToDevice,
                               p->stream));
  VGP_CUDA_TRY(cudaMemcpyAsync(p->d_raw + 2 * n, observations, sizeof(double) * n,
                               cudaMemcpyHostToDevice, p->stream));
  VGP_CUDA_TRY(launch_permute(p->d_raw, p->d_order, n, p->d_pts, p->stream));
  if (p->d_dcache) {
    // rebuild the distance cache only when the locations changed
    bool rebuild = !p->dcache_valid;
    if (!rebuild) {
      int* hflag = (int*)(p->h_small + 6);
      VGP_CUDA_TRY(cudaMemsetAsync(p->d_flag, 0, sizeof(int), p->stream));
      VGP_CUDA_TRY(launch_diff(p->d_raw, p->d_prev_locs, 2 * n, p->d_flag, p->stream));
      VGP_CUDA_TRY(cudaMemcpyAsync(hflag, p->d_flag, sizeof(int), cudaMemcpyDeviceToHost, p->stream));
      VGP_CUDA_TRY(cudaStreamSynchronize(p->stream));
      rebuild = *hflag != 0;
    }
    if (rebuild) {
      VGP_CUDA_TRY(cudaMemcpyAsync(p->d_prev_locs, p->d_raw, sizeof(double) * 2 * n,
                                   cudaMemcpyDeviceToDevice, p->stream));
      VGP_CUDA_TRY(launch_build_dcache(*p, p->stream));
      p->dcache_valid = true;
      unsigned long long* hmax = (unsigned long long*)(p->h_small + 7);
      VGP_CUDA_TRY(cudaMemcpyAsync(hmax, p->d_flag + 2, sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                                   p->stream));
      VGP_CUDA_TRY(cudaStreamSynchronize(p->stream));
      std::memcpy(&p->dcache_dmax, hmax, sizeof(double));
    }
  }
  VGP_CUDA_TRY(cudaStreamSynchronize(p->stream));
  p->has_data = true;
  return VGP_OK;
}

int vgp_plan_destroy(vgp_plan* plan) {
  if (!plan) return VGP_OK;
  DeviceGuard g(plan->p.device);
  Plan* p = new Plan(plan->p);
  free_plan(p);
  delete plan;
  return VGP_OK;
}

int vgp_plan_info(const vgp_plan* plan, int64_t* info) {
  if (!plan || !info) return fail(VGP_E_INVALID, "null pointer");
  const Plan& p = plan->p;
  info[0] = p.n;
  info[1] = p.m;
  info[2] = p.blk_lo;
  info[3] = p.blk_hi;
  info[4] = p.chunk_lo;
  info[5] = p.chunk_hi - p.chunk_lo;
  info[6] = p.kernel_variant;
  info[7] = p.device;
  info[8] = (p.d_dcache && p.dcache_valid) ? 1 : 0;
  return VGP_OK;
}

int vgp_loglik_partials_device(vgp_plan* plan, int family, double sigma_sq, double beta,
                               double nu, double* out) {
  if (!plan || !out) return fail(VGP_E_INVALID, "null pointer");
  Plan* p = &plan->p;
  if (!p->has_data) return fail(VGP_E_INVALID, "plan has no data (vgp_plan_set_data)");
  CovParams cp;
  int rc = make_cov_params(family, sigma_sq, beta, nu, &cp);
  if (rc) return rc;
  DeviceGuard g(p->device);
  rc = launch_eval(p, cp, false);
  if (rc) return rc;
  VGP_CUDA_TRY(launch_scatter_partials(*p, out, p->stream));
  VGP_CUDA_TRY(cudaStreamSynchronize(p->stream));
  return VGP_OK;
}

int vgp_plan_set_timing(vgp_plan* plan, int enable) {
  if (!plan) return fail(VGP_E_INVALID, "null plan");
  plan->p.timing = enable != 0;
  return VGP_OK;
}

int vgp_plan_kernel_time(vgp_plan* plan, double* ms, int64_t* launches) {
  if (!plan) return fail(VGP_E_INVALID, "null plan");
  Plan* p = &plan->p;
  DeviceGuard g(p->device);
  double total = 0.0;
  int64_t count = 0;
  for (auto& pr : *p->events) {
    VGP_CUDA_TRY(cudaEventSynchronize(pr.second));
    float t = 0.f;
    VGP_CUDA_TRY(cudaEventElapsedTime(&t, pr.first, pr.second));
    total += t;
    ++count;
    p->event_pool->push_back(pr.first);
    p->event_pool->push_back(pr.second);
  }
  p->events->clear();
  if (ms) *ms = total;
  if (launches) *launches = count;
  return VGP_OK;
}

int vgp_plan_set_variant(vgp_plan* plan, int variant) {
  if (!plan || variant < -1 || variant > 13) return fail(VGP_E_INVALID, "bad variant");
  // -1 auto, 0 generic, 1 all-register warp-DMMA, 2 grouped warp-DMMA,
  // 3 warp-specialised DMMA, 4 warp-specialised streaming the distance cache
  plan->p.force_variant = variant;
  return VGP_OK;
}

void* vgp_plan_stream(vgp_plan* plan) { return plan ? (void*)plan->p.stream : nullptr; }

int vgp_loglik_async(vgp_plan* plan, int family, double sigma_sq, double beta, double nu) {
  if (!plan) return fail(VGP_E_INVALID, "null plan");
  Plan* p = &plan->p;
  if (!p->has_data) return fail(VGP_E_INVALID, "plan has no data (vgp_plan_set_data)");
  CovParams cp;
  int rc = make_cov_params(family, sigma_sq, beta, nu, &cp);
  if (rc) return rc;
  DeviceGuard g(p->device);
  const bool full = p->blk_lo == 0 && p->blk_hi == p->n - p->m + 1;
  return launch_eval(p, cp, full);
}

int vgp_plan_fetch(vgp_plan* plan, double* total, int64_t* fail_index, int* status) {
  if (!plan) return fail(VGP_E_INVALID, "null plan");
  Plan* p = &plan->p;
  DeviceGuard g(p->device);
  unsigned long long* flags = (unsigned long long*)p->h_small;
  double* sc = p->h_small + 2;
  VGP_CUDA_TRY(cudaMemcpyAsync(flags, p->d_fail, 2 * sizeof(unsigned long long),
                               cudaMemcpyDeviceToHost, p->stream));
  VGP_CUDA_TRY(cudaMemcpyAsync(sc, p->d_scalars, 2 * sizeof(double), cudaMemcpyDeviceToHost, p->stream));
  VGP_CUDA_TRY(cudaStreamSynchronize(p->stream));
  int st = decode_status(p, flags, fail_index);
  if (status) *status = st;
  if (total) *total = st == VGP_OK ? sc[0] : NAN;
  return VGP_OK;
}

int vgp_loglik(vgp_plan* plan, int family, double sigma_sq, double beta, double nu,
               double* total, int64_t* fail_index, double* block_first, double* block_rest,
               double* mu_new, double* sigma_new) {
  if (!plan) return fail(VGP_E_INVALID, "null plan");
  Plan* p = &plan->p;
  if (!(p->blk_lo == 0 && p->blk_hi == p->n - p->m + 1))
    return fail(VGP_E_INVALID, "vgp_loglik needs a plan over all blocks; use vgp_loglik_partials");
  if (!p->has_data) return fail(VGP_E_INVALID, "plan has no data (vgp_plan_set_data)");
  CovParams cp;
  int rc = make_cov_params(family, sigma_sq, beta, nu, &cp);
  if (rc) return rc;
  DeviceGuard g(p->device);
  HostOut out;
  out.rest = block_rest;
  out.mu = mu_new;
  out.sig = sigma_new;
  const bool any = block_rest || mu_new || sigma_new;
  rc = launch_eval(p, cp, true, any ? &out : nullptr);
  if (rc) return rc;
  unsigned long long* flags = (unsigned long long*)p->h_small;
  double* sc = p->h_small + 2;
  VGP_CUDA_TRY(cudaMemcpyAsync(flags, p->d_fail, 2 * sizeof(unsigned long long),
                               cudaMemcpyDeviceToHost, p->stream));
  VGP_CUDA_TRY(cudaMemcpyAsync(sc, p->d_scalars, 2 * sizeof(double), cudaMemcpyDeviceToHost, p->stream));
  VGP_CUDA_TRY(cudaStreamSynchronize(p->side));
  VGP_CUDA_TRY(cudaStreamSynchronize(p->stream));
  int st = decode_status(p, flags, fail_index);
  if (total) *total = st == VGP_OK ? sc[0] : NAN;
  if (block_first) *block_first = st == VGP_OK ? sc[1] : NAN;
  return st;
}

int vgp_loglik_data(vgp_plan* plan, const double* locations, const double* observations, int family,
                    double sigma_sq, double beta, double nu, double* total, int64_t* fail_index,
                    double* block_first, double* block_rest, double* mu_new, double* sigma_new) {
  if (!plan || !locations || !observations) return fail(VGP_E_INVALID, "null pointer");
  Plan* p = &plan->p;
  if (!(p->blk_lo == 0 && p->blk_hi == p->n - p->m + 1))
    return fail(VGP_E_INVALID, "vgp_loglik_data needs a plan over all blocks");
  CovParams cp;
  int rc = make_cov_params(family, sigma_sq, beta, nu, &cp);
  if (rc) return rc;
  const bool spec = p->has_data && p->d_dcache && p->dcache_valid && p->aux;
  if (!spec) {
    rc = vgp_plan_set_data(plan, locations, observations);
    if (rc) return rc;
    return vgp_loglik(plan, family, sigma_sq, beta, nu, total, fail_index, block_first, block_rest,
                      mu_new, sigma_new);
  }
  DeviceGuard g(p->device);
  const int64_t n = p->n;
  // Speculate that the locations are the ones the distance cache was built
  // from (an MLE loop re-evaluates one dataset): the observations go up and
  // the evaluation starts; the locations go up on another stream and are
  // compared with the cache's next to it.  If they differ, the cache is
  // rebuilt and the evaluation rerun before returning.
  VGP_CUDA_TRY(cudaMemcpyAsync(p->d_raw + 2 * n, observations, sizeof(double) * n,
                               cudaMemcpyHostToDevice, p->stream));
  VGP_CUDA_TRY(launch_permute_obs(p->d_raw + 2 * n, p->d_order, n, p->d_pts, p->stream));
  int* hflag = (int*)(p->h_small + 6);
  VGP_CUDA_TRY(cudaMemcpyAsync(p->d_raw, locations, sizeof(double) * 2 * n, cudaMemcpyHostToDevice, p->aux));
  VGP_CUDA_TRY(cudaMemsetAsync(p->d_flag, 0, sizeof(int), p->aux));
  VGP_CUDA_TRY(launch_diff(p->d_raw, p->d_prev_locs, 2 * n, p->d_flag, p->aux));
  VGP_CUDA_TRY(cudaMemcpyAsync(hflag, p->d_flag, sizeof(int), cudaMemcpyDeviceToHost, p->aux));
  rc = vgp_loglik(plan, family, sigma_sq, beta, nu, total, fail_index, block_first, block_rest, mu_new,
                  sigma_new);
  VGP_CUDA_TRY(cudaStreamSynchronize(p->aux));
  if (*hflag == 0) return rc;
  // the locations changed: the full upload path (permute, rebuild the
  // cache and its d_max), then evaluate again
  rc = vgp_plan_set_data(plan, locations, observations);
  if (rc) return rc;
  return vgp_loglik(plan, family, sigma_sq, beta, nu, total, fail_index, block_first, block_rest, mu_new,
                    sigma_new);
}

int vgp_plan_fail_keys(vgp_plan* plan, uint64_t* keys) {
  if (!plan || !keys) return fail(VGP_E_INVALID, "null pointer");
  Plan* p = &plan->p;
  DeviceGuard g(p->device);
  VGP_CUDA_TRY(cudaStreamSynchronize(p->stream));
  VGP_CUDA_TRY(cudaMemcpy(keys, p->d_fail, 2 * sizeof(uint64_t), cudaMemcpyDeviceToHost));
  return VGP_OK;
}

int vgp_simulate(vgp_plan* plan, int family, double sigma_sq, double beta, double nu,
                 const double* z, double* y, int64_t* fail_index) {
  if (!plan || !z || !y) return fail(VGP_E_INVALID, "null pointer");
  Plan* p = &plan->p;
  if (!(p->blk_lo == 0 && p->blk_hi == p->n - p->m + 1))
    return fail(VGP_E_INVALID, "vgp_simulate needs a plan over all blocks");
  if (!p->has_data) return fail(VGP_E_INVALID, "plan has no data (vgp_plan_set_data)");
  CovParams cp;
  int rc = make_cov_params(family, sigma_sq, beta, nu, &cp);
  if (rc) return rc;
  DeviceGuard g(p->device);
  double *d_z = nullptr, *d_y = nullptr;
  unsigned long long* d_f = nullptr;
  rc = dalloc(&d_z, p->n);
  if (!rc) rc = dalloc(&d_y, p->n);
  if (!rc) rc = dalloc(&d_f, 1);
  cudaError_t e = cudaSuccess;
  if (!rc) e = cudaMemcpyAsync(d_z, z, sizeof(double) * p->n, cudaMemcpyHostToDevice, p->stream);
  if (!rc && e == cudaSuccess) e = cudaMemsetAsync(d_f, 0xff, sizeof(unsigned long long), p->stream);
  if (!rc && e == cudaSuccess) e = launch_simulate(*p, cp, d_z, d_y, d_f, p->stream);
  unsigned long long hf = ~0ull;
  if (!rc && e == cudaSuccess) e = cudaMemcpy(&hf, d_f, sizeof(hf), cudaMemcpyDeviceToHost);
  if (!rc && e == cudaSuccess) e = cudaMemcpy(y, d_y, sizeof(double) * p->n, cudaMemcpyDeviceToHost);
  if (!rc && e != cudaSuccess) rc = fail(VGP_E_CUDA, std::string("simulate: ") + cudaGetErrorString(e));
  cudaFree(d_z);
  cudaFree(d_y);
  cudaFree(d_f);
  if (rc) return rc;
  if (hf != ~0ull) {
    if (fail_index) *fail_index = (int64_t)hf;
    return fail(VGP_NOT_POSITIVE_DEFINITE, "simulate: non-positive pivot");
  }
  if (fail_index) *fail_index = -1;
  return VGP_OK;
}

int vgp_loglik_partials(vgp_plan* plan, int family, double sigma_sq, double beta, double nu,
                        double* partials, double* block_first, int64_t* fail_index) {
  if (!plan) return fail(VGP_E_INVALID, "null plan");
  Plan* p = &plan->p;
  if (!p->has_data) return fail(VGP_E_INVALID, "plan has no data (vgp_plan_set_data)");
  CovParams cp;
  int rc = make_cov_params(family, sigma_sq, beta, nu, &cp);
  if (rc) return rc;
  DeviceGuard g(p->device);
  rc = launch_eval(p, cp, false);
  if (rc) return rc;
  unsigned long long* flags = (unsigned long long*)p->h_small;
  double* sc = p->h_small + 2;
  VGP_CUDA_TRY(cudaMemcpyAsync(flags, p->d_fail, 2 * sizeof(unsigned long long),
                               cudaMemcpyDeviceToHost, p->stream));
  VGP_CUDA_TRY(cudaMemcpyAsync(sc, p->d_scalars, 2 * sizeof(double), cudaMemcpyDeviceToHost, p->stream));
  if (partials)
    VGP_CUDA_TRY(cudaMemcpyAsync(partials, p->d_partials,
                                 sizeof(double) * (p->chunk_hi - p->chunk_lo),
                                 cudaMemcpyDeviceToHost, p->stream));
  VGP_CUDA_TRY(cudaStreamSynchronize(p->stream));
  int st = decode_status(p, flags, fail_index);
  if (block_first) *block_first = p->blk_lo == 0 ? sc[1] : 0.0;
  return st;
}

}  // extern "C"
