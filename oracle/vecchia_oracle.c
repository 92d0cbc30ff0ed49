/*
 * TEST INFRASTRUCTURE — NOT PRODUCT CODE.
 *
 * CPU restatement of the reference Vecchia hot path (vecchiagp, arXiv 2403.07412
 * restatement under /root/reference/pkg/src/vecchiagp).  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
 * may load this library, and only as the checker or the timed CPU baseline —
 * never as part of the GPU product path.
 *
 * Each function restates one reference routine with the same arithmetic
 * (same operation order, separate multiply / add roundings: build with
 * -ffp-contract=off) so that it tracks the reference to the last few ulps:
 *
 *   orc_knn_pred      geo._topm_plane + nearest_neighbors   vg/geo.py:234-263, :331-347
 *   orc_knn_points    geo.nearest_points (limits = nd)        vg/geo.py:350-358
 *   orc_cov           kernels.matern_cov closed forms /        vg/kernels.py:59-82, :85-91
 *                     powexp_cov
 *   orc_loglik        vecchia.assemble + _numeric_stage +      vg/vecchia.py:106-214
 *                     _reduction_stage, batchla._potrf_sweep,  vg/batchla.py:141-156,
 *                     batch_trsv, batch_dot, half_log_det      :184-237
 *   orc_pairwise_sum  numpy's pairwise float64 sum, used by    vg/vecchia.py:169-177
 *                     _ordered_sum and half_log_det
 *
 * General-nu Matern needs scipy.special.kv; that case lives in oracle.py.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

/* Minimal static-chunk parallel for over [lo, hi) in fixed chunks (the
 * reference's parallel.map_chunks contract: per-item results never depend on
 * the thread count, vg/parallel.py:1-8). */
typedef void (*orc_body_fn)(void* ctx, int64_t lo, int64_t hi, int tid);
typedef struct {
  orc_body_fn fn; void* ctx; int64_t lo, hi, chunk; int64_t next; pthread_mutex_t mu; int tid;
} orc_pool_t;
typedef struct { orc_pool_t* p; int tid; } orc_worker_t;
static void* orc_worker(void* arg) {
  orc_worker_t* w = (orc_worker_t*)arg;
  orc_pool_t* p = w->p;
  for (;;) {
    pthread_mutex_lock(&p->mu);
    int64_t s = p->next;
    p->next += p->chunk;
    pthread_mutex_unlock(&p->mu);
    if (s >= p->hi) break;
    int64_t e = s + p->chunk < p->hi ? s + p->chunk : p->hi;
    p->fn(p->ctx, s, e, w->tid);
  }
  return NULL;
}
static void orc_parallel_for(orc_body_fn fn, void* ctx, int64_t lo, int64_t hi, int64_t chunk,
                             int threads) {
  if (threads < 1) threads = 1;
  if (threads > 256) threads = 256;
  orc_pool_t p;
  p.fn = fn; p.ctx = ctx; p.lo = lo; p.hi = hi; p.chunk = chunk; p.next = lo;
  pthread_mutex_init(&p.mu, NULL);
  pthread_t th[256];
  orc_worker_t w[256];
  for (int t = 0; t < threads; ++t) {
    w[t].p = &p; w[t].tid = t;
    if (t) pthread_create(&th[t], NULL, orc_worker, &w[t]);
  }
  orc_worker(&w[0]);
  for (int t = 1; t < threads; ++t) pthread_join(th[t], NULL);
  pthread_mutex_destroy(&p.mu);
}

#define ORC_LOG_2PI 1.8378770664093453 /* math.log(2*pi), vg/vecchia.py:31 */

enum { ORC_OK = 0, ORC_NPD = 1, ORC_BAD_VAR = 2, ORC_ARG = -1, ORC_OOM = -3 };
enum { FAM_MATERN = 0, FAM_POWEXP = 1 };

/* ---------------- kNN: vg/geo.py:234-263 ---------------- */

static void topm_one(const double* x, const double* y, double xt, double yt,
                     int64_t limit, int m, double* keys, int64_t* out) {
  int cnt = 0;
  for (int64_t j = 0; j < limit; ++j) {
    double dx = x[j] - xt;
    double dy = y[j] - yt;
    double k = dx * dx + dy * dy; /* no contraction: -ffp-contract=off */
    int p;
    if (cnt == m) {
      if (k >= keys[m - 1]) continue;
      p = m - 1;
    } else {
      p = cnt;
      cnt += 1;
    }
    while (p > 0 && keys[p - 1] > k) {
      keys[p] = keys[p - 1];
      out[p] = out[p - 1];
      p -= 1;
    }
    keys[p] = k;
    out[p] = j;
  }
}

typedef struct {
  const double *x, *y, *qx, *qy; int64_t nd; int m; int pred; int64_t* out; double* keys;
} knn_ctx_t;

static void knn_body(void* vctx, int64_t lo, int64_t hi, int tid) {
  knn_ctx_t* c = (knn_ctx_t*)vctx;
  double* keys = c->keys + (int64_t)tid * c->m;
  for (int64_t t = lo; t < hi; ++t) {
    int64_t limit = c->pred ? t + c->m : c->nd; /* target i = m + t admits j < i */
    topm_one(c->x, c->y, c->qx[t], c->qy[t], limit, c->m, keys, c->out + t * (int64_t)c->m);
  }
}

/* nearest_neighbors, vg/geo.py:331-347: locs n x 2 ordered; out (n-m) x m */
int orc_knn_pred(const double* locs, int64_t n, int m, int64_t* out, int threads) {
  if (m < 1 || n <= m) return ORC_ARG;
  if (threads < 1) threads = 1;
  double* x = (double*)malloc(sizeof(double) * n);
  double* y = (double*)malloc(sizeof(double) * n);
  double* keys = (double*)malloc(sizeof(double) * m * (threads > 256 ? 256 : threads));
  if (!x || !y || !keys) { free(x); free(y); free(keys); return ORC_OOM; }
  for (int64_t i = 0; i < n; ++i) { x[i] = locs[2 * i]; y[i] = locs[2 * i + 1]; }
  knn_ctx_t c = {x, y, x + m, y + m, n, m, 1, out, keys};
  orc_parallel_for(knn_body, &c, 0, n - m, 256, threads);
  free(x); free(y); free(keys);
  return ORC_OK;
}

/* nearest_points, vg/geo.py:350-358 */
int orc_knn_points(const double* q, int64_t nq, const double* d, int64_t nd, int m,
                   int64_t* out, int threads) {
  if (m < 1 || m > nd) return ORC_ARG;
  if (threads < 1) threads = 1;
  double* x = (double*)malloc(sizeof(double) * nd);
  double* y = (double*)malloc(sizeof(double) * nd);
  double* qx = (double*)malloc(sizeof(double) * (nq ? nq : 1));
  double* qy = (double*)malloc(sizeof(double) * (nq ? nq : 1));
  double* keys = (double*)malloc(sizeof(double) * m * (threads > 256 ? 256 : threads));
  if (!x || !y || !qx || !qy || !keys) {
    free(x); free(y); free(qx); free(qy); free(keys); return ORC_OOM;
  }
  for (int64_t i = 0; i < nd; ++i) { x[i] = d[2 * i]; y[i] = d[2 * i + 1]; }
  for (int64_t i = 0; i < nq; ++i) { qx[i] = q[2 * i]; qy[i] = q[2 * i + 1]; }
  knn_ctx_t c = {x, y, qx, qy, nd, m, 0, out, keys};
  orc_parallel_for(knn_body, &c, 0, nq, 64, threads);
  free(x); free(y); free(qx); free(qy); free(keys);
  return ORC_OK;
}

/* ---------------- covariance: vg/kernels.py:59-91 ---------------- */

static inline double cov_closed(double d, int family, double s2, double beta, double nu) {
  if (family == FAM_POWEXP) return s2 * exp(-pow(d, nu) / beta); /* :85-91 */
  double u = d / beta;                                            /* :67 */
  if (nu == 0.5) return s2 * exp(-u);
  if (nu == 1.5) return s2 * (1.0 + u) * exp(-u);
  /* nu == 2.5 (caller guarantees closed-form nu) */
  return s2 * (1.0 + u + u * u / 3.0) * exp(-u);
}

int orc_cov(const double* d, int64_t n, int family, double s2, double beta, double nu, double* out) {
  if (family == FAM_MATERN && !(nu == 0.5 || nu == 1.5 || nu == 2.5)) return ORC_ARG;
  for (int64_t i = 0; i < n; ++i) out[i] = cov_closed(d[i], family, s2, beta, nu);
  return ORC_OK;
}

/* ---------------- numpy pairwise sum (float64, contiguous) ---------------- */

double orc_pairwise_sum(const double* a, int64_t n) {
  if (n < 8) {
    double r = 0.0;
    for (int64_t i = 0; i < n; ++i) r += a[i];
    return r;
  } else if (n <= 128) {
    double r[8];
    int64_t i;
    for (int j = 0; j < 8; ++j) r[j] = a[j];
    for (i = 8; i < n - (n % 8); i += 8)
      for (int j = 0; j < 8; ++j) r[j] += a[i + j];
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; ++i) res += a[i];
    return res;
  } else {
    int64_t n2 = n / 2;
    n2 -= n2 % 8;
    return orc_pairwise_sum(a, n2) + orc_pairwise_sum(a + n2, n - n2);
  }
}

/* vg/vecchia.py:169-177 — 4096-chunk pairwise partials combined in order */
double orc_ordered_sum(const double* a, int64_t n) {
  double total = 0.0;
  for (int64_t lo = 0; lo < n; lo += 4096) {
    int64_t hi = lo + 4096 < n ? lo + 4096 : n;
    total += orc_pairwise_sum(a + lo, hi - lo);
  }
  return total;
}

/* ---------------- one conditioning block ----------------
 * a: dim x dim column-major (lower triangle read), v, yv: dim.
 * Returns 0, or 1 + pivot column on a non-positive pivot (vg/batchla.py:146-151).
 * On success mu = y'.v', sg = v'.v' (vg/vecchia.py:186-189).
 */
static int block_numeric(double* a, int dim, double* v, double* yv, double* mu, double* sg,
                         double* logdiag_sum_buf) {
  /* _potrf_sweep, vg/batchla.py:141-156 */
  for (int j = 0; j < dim; ++j) {
    double piv = a[j * dim + j];
    if (!(piv > 0.0)) return 1 + j;
    piv = sqrt(piv);
    a[j * dim + j] = piv;
    for (int i = j + 1; i < dim; ++i) a[j * dim + i] /= piv;
    for (int c = j + 1; c < dim; ++c) {
      double lc = a[j * dim + c];
      for (int r = c; r < dim; ++r) a[c * dim + r] -= a[j * dim + r] * lc;
    }
  }
  /* batch_trsv twice, vg/batchla.py:184-210 */
  for (int j = 0; j < dim; ++j) {
    double piv = a[j * dim + j];
    v[j] /= piv;
    yv[j] /= piv;
    for (int i = j + 1; i < dim; ++i) {
      v[i] -= a[j * dim + i] * v[j];
      yv[i] -= a[j * dim + i] * yv[j];
    }
  }
  /* batch_dot, vg/batchla.py:213-229: mu' = y'.v', sigma' = v'.v' */
  double accm = 0.0, accs = 0.0;
  for (int i = 0; i < dim; ++i) {
    accm += yv[i] * v[i];
    accs += v[i] * v[i];
  }
  *mu = accm;
  *sg = accs;
  if (logdiag_sum_buf) {
    for (int i = 0; i < dim; ++i) logdiag_sum_buf[i] = log(a[i * dim + i]);
  }
  return 0;
}

typedef struct {
  const double* locs; const double* obs; int m; const int64_t* nbr; int family;
  double s2, beta, nu; int* failcol; double* mus; double* sgs;
} blk_ctx_t;

/* assemble fill() + _numeric_stage for entries [lo, hi), vg/vecchia.py:154-162, :180-190 */
static void blk_body(void* vctx, int64_t lo, int64_t hi, int tid) {
  (void)tid;
  blk_ctx_t* c = (blk_ctx_t*)vctx;
  int m = c->m;
  const double* locs = c->locs;
  double* a = (double*)malloc(sizeof(double) * m * m);
  double* v = (double*)malloc(sizeof(double) * m);
  double* yv = (double*)malloc(sizeof(double) * m);
  for (int64_t e = lo; e < hi; ++e) {
    int64_t t = m + e - 1;
    const int64_t* J = c->nbr + (e - 1) * (int64_t)m;
    for (int cc = 0; cc < m; ++cc) {
      double xc = locs[2 * J[cc]], yc = locs[2 * J[cc] + 1];
      for (int r = 0; r < m; ++r) {
        double d = hypot(locs[2 * J[r]] - xc, locs[2 * J[r] + 1] - yc);
        a[cc * m + r] = cov_closed(d, c->family, c->s2, c->beta, c->nu);
      }
      double dv = hypot(locs[2 * t] - xc, locs[2 * t + 1] - yc);
      v[cc] = cov_closed(dv, c->family, c->s2, c->beta, c->nu);
      yv[cc] = c->obs[J[cc]];
    }
    double mu, sg;
    int f = block_numeric(a, m, v, yv, &mu, &sg, NULL);
    c->failcol[e] = f;
    if (!f) {
      c->mus[e - 1] = mu;
      c->sgs[e - 1] = c->s2 - sg; /* vg/vecchia.py:206 */
    }
  }
  free(a); free(v); free(yv);
}

/*
 * Full Vecchia log-likelihood for an already-ordered dataset
 * (vg/vecchia.py:217-238 after dataset.permute).
 *   locs n x 2, obs n, nbr (n-m) x m.
 * Outputs: total, block_first, block_rest/mu_new/sigma_new (n-m each, may be NULL).
 * Returns ORC_OK, ORC_NPD (fail_index = batch entry) or ORC_BAD_VAR.
 * The NPD index follows the reference's chunk -> column -> entry order
 * (vg/batchla.py:146-151 inside map_chunks of _matrix_chunk(dim) entries).
 */
int orc_loglik(const double* locs, const double* obs, int64_t n, int m, const int64_t* nbr,
               int family, double s2, double beta, double nu, double* total, double* block_first,
               double* block_rest, double* mu_new, double* sigma_new, int64_t* fail_index,
               int threads) {
  if (m < 1 || n <= m) return ORC_ARG;
  int64_t count = n - m + 1;
  double* rest = block_rest ? block_rest : (double*)malloc(sizeof(double) * (count - 1));
  double* mus = mu_new ? mu_new : (double*)malloc(sizeof(double) * (count - 1));
  double* sgs = sigma_new ? sigma_new : (double*)malloc(sizeof(double) * (count - 1));
  /* per-entry failing pivot column (0 = ok) */
  int* failcol = (int*)calloc(count, sizeof(int));
  double mu0 = 0.0, hld = 0.0;
  int status = ORC_OK;
  if (!rest || !mus || !sgs || !failcol) { status = ORC_OOM; goto done; }

  /* entry 0: joint block, vg/vecchia.py:148-150 */
  {
    double* a = (double*)malloc(sizeof(double) * m * m);
    double* v = (double*)malloc(sizeof(double) * m);
    double* yv = (double*)malloc(sizeof(double) * m);
    double* lg = (double*)malloc(sizeof(double) * m);
    for (int c = 0; c < m; ++c)
      for (int r = 0; r < m; ++r) {
        double d = hypot(locs[2 * r] - locs[2 * c], locs[2 * r + 1] - locs[2 * c + 1]);
        a[c * m + r] = cov_closed(d, family, s2, beta, nu);
      }
    for (int i = 0; i < m; ++i) { v[i] = obs[i]; yv[i] = obs[i]; }
    double sg0;
    int f = block_numeric(a, m, v, yv, &mu0, &sg0, lg);
    failcol[0] = f;
    if (!f) hld = orc_pairwise_sum(lg, m); /* half_log_det, vg/batchla.py:232-237 */
    free(a); free(v); free(yv); free(lg);
  }

  {
    blk_ctx_t c = {locs, obs, m, nbr, family, s2, beta, nu, failcol, mus, sgs};
    orc_parallel_for(blk_body, &c, 1, count, 64, threads);
  }

  /* NPD: first failing chunk, then smallest failing column, then entry */
  {
    int64_t chunk = (int64_t)(1 << 21) / ((int64_t)m * m);
    if (chunk < 1) chunk = 1;
    for (int64_t lo = 0; lo < count && status == ORC_OK; lo += chunk) {
      int64_t hi = lo + chunk < count ? lo + chunk : count;
      int bestcol = 0;
      int64_t best = -1;
      for (int64_t e = lo; e < hi; ++e)
        if (failcol[e] && (best < 0 || (m <= 256 && failcol[e] < bestcol))) {
          best = e;
          bestcol = failcol[e];
        }
      if (best >= 0) { status = ORC_NPD; *fail_index = best; }
    }
  }
  if (status != ORC_OK) goto done;
  /* conditional variances, vg/vecchia.py:206-210 */
  for (int64_t k = 0; k < count - 1; ++k)
    if (!(sgs[k] > 0.0)) { status = ORC_BAD_VAR; *fail_index = k + 1; goto done; }
  for (int64_t k = 0; k < count - 1; ++k) {
    double resid = obs[m + k] - mus[k];
    rest[k] = -0.5 * (resid * resid / sgs[k] + ORC_LOG_2PI + log(sgs[k])); /* :211-212 */
  }
  {
    double bf = -hld - 0.5 * mu0 - 0.5 * m * ORC_LOG_2PI; /* :202-204 */
    if (block_first) *block_first = bf;
    *total = bf + orc_ordered_sum(rest, count - 1);
  }
done:
  if (!block_rest) free(rest);
  if (!mu_new) free(mus);
  if (!sigma_new) free(sgs);
  free(failcol);
  return status;
}
