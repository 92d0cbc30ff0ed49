/*
 * vecchia_b200.h — C ABI of libvecchia_b200.so, the B200 (sm_100a) hot path
 * for the Vecchia-approximated Gaussian-process log-likelihood
 * (arXiv 2403.07412).
 *
 * The reference (`vecchiagp`, /root/reference/pkg/src/vecchiagp, "vg/" below)
 * is pure Python; its plugin seam is the module-attribute lookup of a few
 * functions (monkeypatched in its own tests, pkg/tests/test_fit.py:112-120).
 * Each entry point below replaces one of those functions; the Python package
 * paper_2403_07412_b200 binds them with ctypes under the reference's names.
 *
 * Conventions (kept from the reference):
 *   - host arrays are float64 C-contiguous, indices int64 (vg/geo.py:123-124, :159, :184);
 *   - coordinates are (n, 2) row-major (x, y) or (lon, lat) in degrees;
 *   - batch entry 0 is the joint block over the first m ordered points,
 *     entry e >= 1 belongs to ordered target m + e - 1 (vg/vecchia.py:127-162);
 *   - every call is synchronous: results are in host memory on return;
 *   - no C++ exceptions cross this boundary; a negative return is an error
 *     whose message is available from vgp_last_error() (thread-local);
 *   - results never depend on launch configuration (vg/parallel.py:1-8).
 *   - there is NO CPU fallback: without a usable CUDA device every compute
 *     entry point returns VGP_E_CUDA.
 */
#ifndef VECCHIA_B200_H
#define VECCHIA_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes ------------------------------------------------------ */
#define VGP_OK 0
/* non-positive Cholesky pivot: errors.NonPositiveDefiniteError(batch_index),
 * re-raised as LikelihoodEvaluationError by _numeric_stage (vg/vecchia.py:182-185) */
#define VGP_NOT_POSITIVE_DEFINITE 1
/* sigma_new <= 0 or NaN: LikelihoodEvaluationError(block_index) (vg/vecchia.py:206-210) */
#define VGP_BAD_CONDITIONAL_VARIANCE 2
/* zero diagonal in a triangular solve: SingularTriangularError (vg/batchla.py:201-204) */
#define VGP_SINGULAR_TRIANGULAR 3
#define VGP_E_INVALID (-1)
#define VGP_E_CUDA (-2)
#define VGP_E_NOMEM (-3)
#define VGP_E_UNSUPPORTED (-4)

/* kernels.FAMILIES (vg/kernels.py:20) */
#define VGP_FAMILY_MATERN 0
#define VGP_FAMILY_POWEXP 1
/* geo.Euclidean / geo.GreatCircle (vg/geo.py:28-48) */
#define VGP_METRIC_EUCLIDEAN 0
#define VGP_METRIC_GREAT_CIRCLE 1

typedef struct vgp_plan vgp_plan;

/* Library version string. */
const char* vgp_version(void);
/* Message of the last failing call on this thread ("" if none). */
const char* vgp_last_error(void);
/* Number of visible CUDA devices (0 on a machine without a GPU). */
int vgp_device_count(int* count);

/* ---- conditioning sets ------------------------------------------------- */

/* Replaces geo.nearest_neighbors (vg/geo.py:331-347) -> _topm_scan ->
 * numba _topm_plane (vg/geo.py:234-263, :295-328).
 * locations: ORDERED (n, 2) Euclidean coordinates; neighbors: (n - m, m)
 * int64 output, row r = ordered target m + r, entries sorted by
 * (dx*dx + dy*dy, index), bit-identical to the reference. */
int vgp_knn_predecessors(int device, const double* locations, int64_t n, int32_t m,
                         int64_t* neighbors);

/* Rows [row_lo, row_hi) of the same table (targets m + row), for a rank
 * that owns only those conditioning blocks (multi-GPU shards, SURVEY.md
 * §8(e); the reference's per-target chunked scan, vg/geo.py:295-328).
 * Only locations[0 : m + row_hi) are read; neighbors: (row_hi - row_lo, m).
 * Bit-identical to the same rows of vgp_knn_predecessors. */
int vgp_knn_predecessors_range(int device, const double* locations, int64_t n, int32_t m,
                               int64_t row_lo, int64_t row_hi, int64_t* neighbors);

/* Great-circle kNN — replaces numba geo._topm_sphere (vg/geo.py:266-292) as
 * called by nearest_neighbors (predecessors != 0: queries are data[m..nd),
 * candidates j < target) and nearest_points (predecessors == 0: queries
 * query3, every candidate).  Points are rows (lambda, phi, cos phi) in
 * radians, computed by the caller exactly as the reference does (numpy
 * radians / cos, vg/geo.py:305-310); the per-pair key is the haversine of
 * the central angle.  Exact up to keys tied within CUDA's 1-ulp sin. */
int vgp_knn_sphere(int device, const double* data3, int64_t nd, const double* query3, int64_t nq,
                   int32_t m, int predecessors, int64_t* neighbors);

/* Replaces vecchia.assemble (vg/vecchia.py:106-166): the materialised
 * conditioning batches of the unfused stage API (assemble -> _numeric_stage
 * -> _reduction_stage, as timed by cli.cmd_bench, vg/cli.py:259-263).
 * locations/observations: ORDERED (n, 2) / (n,); neighbors (n - m, m) int64;
 * outputs for the n - m + 1 entries: sigma column-major m x m matrices at
 * stride sigma_stride (>= m*m), v and yj at strides >= m.  Entry 0 is the
 * joint first block with v = yj = observations[0:m].  Covariances are the
 * reference expressions (vg/kernels.py:59-91) on the device. */
int vgp_assemble(int device, const double* locations, const double* observations, int64_t n, int32_t m,
                 const int64_t* neighbors, int metric, double radius, int family, double sigma_sq,
                 double beta, double nu, double* sigma, int64_t sigma_stride, double* v, int64_t v_stride,
                 double* yj, int64_t yj_stride);

/* Exact maxmin ordering (BASELINE config 5; new — the reference's orderings
 * are random / Morton / identity, vg/vecchia.py:37, vg/geo.py:47-91).
 * order[0] = first (the caller passes the point nearest the centroid); then
 * repeatedly the unselected point with the largest squared Euclidean
 * distance dx*dx + dy*dy (rounded, no FMA) to the selected set, ties to the
 * smallest index.  order: (n,) int64 permutation.  One cooperative launch,
 * n <= 6553600 points (VGP_E_UNSUPPORTED beyond). */
int vgp_maxmin_order(int device, const double* locations, int64_t n, int64_t first, int64_t* order);

/* Replaces geo.nearest_points (vg/geo.py:350-358): unrestricted m nearest
 * data points per query row (kriging). neighbors: (nq, m) int64. */
int vgp_knn_points(int device, const double* query, int64_t nq, const double* data, int64_t nd,
                   int32_t m, int64_t* neighbors);

/* ---- covariance ---------------------------------------------------------- */

/* Replaces kernels.cov / matern_cov / powexp_cov (vg/kernels.py:59-98):
 * out[i] = C(d[i]) for family (VGP_FAMILY_*) and parameters (sigma_sq, beta, nu).
 * Matern closed forms for nu in {0.5, 1.5, 2.5} by exact equality
 * (vg/kernels.py:69-74), a device Bessel K_nu otherwise. */
int vgp_cov(int device, int family, double sigma_sq, double beta, double nu, const double* d,
            int64_t count, double* out);

/* Replaces kernels.bessel_kv (vg/kernels.py:50-56; scipy.special.kv):
 * out[i] = K_nu(x[i]) for x[i] > 0 (VGP_E_INVALID otherwise). */
int vgp_bessel_kv(int device, double nu, const double* x, int64_t count, double* out);

/* ---- likelihood plan ------------------------------------------------------ */

/* Device context for one vecchia.VecchiaPlan (vg/vecchia.py:40-82).
 *   order:     (n,) int64 permutation, order[new_position] = original index
 *              (geo.Permutation, vg/geo.py:152-168);
 *   neighbors: (n - m, m) int64 neighbour table of the ORDERED dataset
 *              (geo.NeighborTable, vg/geo.py:171-188); only rows of the
 *              plan's own block range are read and kept on the device;
 *   [block_lo, block_hi): batch entries this plan evaluates (0 = joint
 *              block; the full problem is [0, n - m + 1)).  Multi-GPU shards
 *              use block ranges whose rest part starts on a 4096 boundary.
 * Only the plan's rows of `neighbors` are read; the pointer is to the full table. */
int vgp_plan_create(int device, int64_t n, int32_t m, int metric, double radius,
                    const int64_t* order, const int64_t* neighbors, int64_t block_lo,
                    int64_t block_hi, vgp_plan** plan);

/* Same, for a multi-GPU shard that holds only its own neighbour rows:
 * shard_neighbors = rows [max(block_lo, 1) - 1, block_hi - 1) of the table
 * (e.g. from vgp_knn_predecessors_range), so no rank ever materialises the
 * full (n - m) x m table. */
int vgp_plan_create_shard(int device, int64_t n, int32_t m, int metric, double radius,
                          const int64_t* order, const int64_t* shard_neighbors, int64_t block_lo,
                          int64_t block_hi, vgp_plan** out);

/* Upload a dataset in ORIGINAL order (geo.Dataset, vg/geo.py:114-149):
 * locations (n, 2), observations (n,).  Permutation by `order` happens on
 * the device (Dataset.permute, vg/geo.py:145-149). */
int vgp_plan_set_data(vgp_plan* plan, const double* locations, const double* observations);

/* Kriging at test locations from m nearest training points — replaces the
 * neighbour branch of fit.krige_predict (vg/fit.py:241-264: batch_potrf, two
 * batch_trsv, two batch_dot per test point) with one fused kernel launch.
 * neighbors: n_test x m training indices (geo.nearest_points, e.g. from
 * vgp_knn_points).  Writes the conditional means (predictions) and variances
 * sigma^2 - v'v'.  Returns VGP_NOT_POSITIVE_DEFINITE with *fail_index = the
 * test point whose conditioning matrix has a non-positive pivot.  metric:
 * VGP_METRIC_EUCLIDEAN or VGP_METRIC_GREAT_CIRCLE (degrees, radius in the
 * distance unit). */
int vgp_krige(int device, const double* train_locations, const double* train_observations,
              int64_t n_train, const double* test_locations, int64_t n_test, int32_t m,
              const int64_t* neighbors, int metric, double radius, int family, double sigma_sq,
              double beta, double nu, double* predictions, double* variances,
              int64_t* fail_index);

/* Page-lock a host range so uploads from it (vgp_plan_set_data) and result
 * downloads into it run as asynchronous DMA (cudaHostRegister); the Python
 * package registers a dataset's arrays on first use and unregisters them when
 * they are freed.  No reference counterpart (host-side transfer plumbing). */
int vgp_host_register(void* ptr, int64_t bytes);
int vgp_host_unregister(void* ptr);

int vgp_plan_destroy(vgp_plan* plan);

/* Replaces vecchia.vecchia_loglik (vg/vecchia.py:217-238) for a plan that
 * covers all blocks.  Writes total and, when non-NULL, block_first and the
 * ordered-space arrays block_rest / mu_new / sigma_new (n - m each,
 * vg/vecchia.py:95-103).  total == block_first + _ordered_sum(block_rest)
 * bit for bit (vg/vecchia.py:169-177, :213).
 * Returns VGP_OK, VGP_NOT_POSITIVE_DEFINITE or VGP_BAD_CONDITIONAL_VARIANCE
 * with *fail_index = failing batch entry (0 = joint block). */
int vgp_loglik(vgp_plan* plan, int family, double sigma_sq, double beta, double nu,
               double* total, int64_t* fail_index, double* block_first, double* block_rest,
               double* mu_new, double* sigma_new);

/* Vecchia forward simulation (data generator for model-consistent parity
 * fixtures; the reference's generator is the dense
 * exact.simulate_grf, vg/exact.py:47-66, capped at n <= 20000):
 * y[0:m] = L0 z[0:m], y[t] = b_t . y[J_t] + sqrt(sigma^2 - v_t . b_t) z_t with
 * b_t = Sigma_t^-1 v_t, for the plan's ordering and neighbour table.
 * z, y: ORDERED (n,) host arrays.  Needs a full-range plan with data set
 * (only its locations are read).  VGP_NOT_POSITIVE_DEFINITE with
 * *fail_index = batch entry on a non-positive pivot. */
int vgp_simulate(vgp_plan* plan, int family, double sigma_sq, double beta, double nu,
                 const double* z, double* y, int64_t* fail_index);

/* vgp_plan_set_data + vgp_loglik in one call (what vecchia_loglik does per
 * evaluation).  When the plan already holds a distance cache, the
 * observations are uploaded and the evaluation starts while the locations
 * upload on another stream and are compared with the cache's; if they
 * differ the cache is rebuilt and the evaluation rerun before returning —
 * the result is always that of the new dataset.  Synchronous. */
int vgp_loglik_data(vgp_plan* plan, const double* locations, const double* observations, int family,
                    double sigma_sq, double beta, double nu, double* total, int64_t* fail_index,
                    double* block_first, double* block_rest, double* mu_new, double* sigma_new);

/* Shard form for multi-GPU evaluation: the plan's fixed 4096-chunk partial
 * sums of block_rest (partials: plan's chunk count, see vgp_plan_info) and,
 * when the plan holds entry 0, block_first (else 0).  Summing every shard's
 * partials in global chunk order reproduces vgp_loglik's total exactly. */
int vgp_loglik_partials(vgp_plan* plan, int family, double sigma_sq, double beta, double nu,
                        double* partials, double* block_first, int64_t* fail_index);

/* Device form of vgp_loglik_partials for the NCCL path: launches the shard's
 * evaluation on the plan's stream and writes into the DEVICE vector `out`
 * (length 1 + total chunk count, zero-initialised by the caller):
 * out[0] = block_first (plan holding entry 0 only), out[1 + c] = partial of
 * global chunk c for the plan's chunks.  A failed shard writes NaN into its
 * first slot so the all-reduced total is NaN; the exact failing index is then
 * available from vgp_plan_fetch.  Synchronises the stream before returning. */
int vgp_loglik_partials_device(vgp_plan* plan, int family, double sigma_sq, double beta,
                               double nu, double* out);

/* Raw failure keys of the plan's last evaluation, for cross-shard agreement
 * (MIN over ranks, then decode): keys[0] = NPD key ordered like the
 * reference's first raise — (potrf chunk of 2^21 / m^2 entries, pivot column,
 * entry) packed as chunk << 42 | column << 24 | entry-in-chunk, or the entry
 * itself for m > 256 (vg/batchla.py:146-164, vg/parallel.py:37-43);
 * keys[1] = first entry with sigma_new <= 0.  UINT64_MAX = none. */
int vgp_plan_fail_keys(vgp_plan* plan, uint64_t* keys);

/* Per-kernel timing of the fused block kernel (CUDA events on the plan's
 * stream around every launch while enabled).  vgp_plan_kernel_time returns
 * the summed milliseconds and launch count since the last call and resets. */
int vgp_plan_set_timing(vgp_plan* plan, int enable);
int vgp_plan_kernel_time(vgp_plan* plan, double* ms, int64_t* launches);

/* Plan geometry: info[0] = n, [1] = m, [2] = block_lo, [3] = block_hi,
 * [4] = first global chunk, [5] = chunk count, [6] = last kernel variant
 * (see vgp_plan_set_variant), [7] = device,
 * [8] = distance cache valid.  info must hold 9 entries. */
int vgp_plan_info(const vgp_plan* plan, int64_t* info);

/* Force a kernel variant — testing / benchmarking aid.  -1 auto (by m, for
 * closed-form Matern: 13 for m <= 12 (Euclidean), 1 for m + 2 <= 24, 4 for
 * m + 2 <= 56, 8 for m + 2 <= 64 — cached variants when the plan has a
 * distance cache; general-nu Matern with m + 2 <= 64: 8 (7 without a cache),
 * covariances from the per-evaluation table; 11 / 12 for larger m and for
 * power exponential; 0 otherwise), 0 generic, 1 all-register warp-DMMA,
 * 4 warp-specialised pair + distance cache, 7/8 scheduler-aware
 * warp-specialised (8: + distance cache), 11/12 the CTA-per-block large-m
 * DMMA kernel (any m, every family; 12: + distance cache), 13
 * thread-per-block (m <= 12, closed-form Matern, Euclidean).  2, 3, 5, 6,
 * 9, 10 are retired experiments (VGP_E_UNSUPPORTED). */
int vgp_plan_set_variant(vgp_plan* plan, int variant);

/* CUDA stream (cudaStream_t) the plan launches on, for event timing. */
void* vgp_plan_stream(vgp_plan* plan);

/* Device-resident evaluation for benchmarking: same work as vgp_loglik but
 * launches only (no host synchronisation, no copies); results stay on the
 * device until vgp_plan_fetch. */
int vgp_loglik_async(vgp_plan* plan, int family, double sigma_sq, double beta, double nu);
int vgp_plan_fetch(vgp_plan* plan, double* total, int64_t* fail_index, int* status);

/* ---- batched small dense linear algebra (vg/batchla.py) ---------------- */

/* Replaces batchla.batch_potrf (vg/batchla.py:167-181): in-place lower
 * Cholesky of `count` column-major dim x dim matrices at buffer + k*stride.
 * VGP_NOT_POSITIVE_DEFINITE with *fail_index on a non-positive pivot. */
int vgp_batch_potrf(int device, double* buffer, int64_t count, int32_t dim, int64_t stride,
                    int64_t* fail_index);

/* Replaces batchla.batch_trsv (vg/batchla.py:184-210): x_k = L_k^-1 b_k. */
int vgp_batch_trsv(int device, const double* lbuf, int64_t lstride, const double* b, double* x,
                   int64_t count, int32_t dim, int64_t vstride, int64_t* fail_index);

/* Replaces batchla.batch_dot (vg/batchla.py:213-229): ascending-index dots. */
int vgp_batch_dot(int device, const double* a, const double* b, int64_t count, int32_t dim,
                  int64_t stride, double* out);

#ifdef __cplusplus
}
#endif

#endif /* VECCHIA_B200_H */
