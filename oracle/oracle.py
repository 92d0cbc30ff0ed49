"""TEST INFRASTRUCTURE — CPU oracle for the Vecchia hot path.  NOT PRODUCT CODE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference`` arm) may import this module, and
only as the checker / CPU baseline.  The product package
(``paper_2403_07412_b200``) never imports it.

It restates the reference algorithm (``vecchiagp`` under
``/root/reference/pkg/src/vecchiagp``, abbreviated ``vg/``):

* ``knn_pred`` / ``knn_points``      -> ``geo.nearest_neighbors`` / ``nearest_points``
  (``vg/geo.py:234-263``, ``:331-358``), C restatement in ``vecchia_oracle.c``.
* ``loglik``                          -> ``vecchia.vecchia_loglik`` on an ordered
  dataset (``vg/vecchia.py:106-238``) with ``batchla._potrf_sweep`` /
  ``batch_trsv`` / ``batch_dot`` (``vg/batchla.py:141-237``).  Closed-form
  smoothness runs in C; general nu (``scipy.special.kv``, the third-party
  routine the reference calls at ``vg/kernels.py:81``) runs in the numpy
  restatement ``loglik_numpy``.
* ``matern_cov`` / ``powexp_cov``     -> ``vg/kernels.py:59-91``.
* ``pairwise_sum`` / ``ordered_sum``  -> numpy's float64 pairwise summation and
  ``vecchia._ordered_sum`` (``vg/vecchia.py:169-177``).
* ``nelder_mead_max`` / ``mle``       -> ``fit.nelder_mead_max`` / ``mle_estimate``
  (``vg/fit.py:61-178``).

Pinned against vectors produced by the reference itself: see
``tests/golden/make_golden.py`` and ``tests/test_oracle_golden.py``.
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess
from dataclasses import dataclass

import numpy as np

LOG_2PI = math.log(2.0 * math.pi)
_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "liboracle.so")
_lib = None

STATUS_OK, STATUS_NPD, STATUS_BAD_VAR = 0, 1, 2


def build() -> str:
    """Compile the C restatement (gcc) into oracle/_build/liboracle.so."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        dp = ctypes.POINTER(ctypes.c_double)
        ip = ctypes.POINTER(ctypes.c_int64)
        L.orc_knn_pred.argtypes = [dp, ctypes.c_int64, ctypes.c_int, ip, ctypes.c_int]
        L.orc_knn_points.argtypes = [dp, ctypes.c_int64, dp, ctypes.c_int64, ctypes.c_int, ip, ctypes.c_int]
        L.orc_cov.argtypes = [dp, ctypes.c_int64, ctypes.c_int, ctypes.c_double, ctypes.c_double,
                              ctypes.c_double, dp]
        L.orc_pairwise_sum.argtypes = [dp, ctypes.c_int64]
        L.orc_pairwise_sum.restype = ctypes.c_double
        L.orc_ordered_sum.argtypes = [dp, ctypes.c_int64]
        L.orc_ordered_sum.restype = ctypes.c_double
        L.orc_loglik.argtypes = [dp, dp, ctypes.c_int64, ctypes.c_int, ip, ctypes.c_int,
                                 ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                 dp, dp, dp, dp, dp, ip, ctypes.c_int]
        _lib = L
    return _lib


def _dp(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _ip(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))


def default_threads() -> int:
    return os.cpu_count() or 1


# ---------------------------------------------------------------- kNN

def knn_pred(ordered_locs, m: int, threads: int | None = None) -> np.ndarray:
    """m nearest predecessors of every ordered index i >= m (vg/geo.py:331-347)."""
    locs = np.ascontiguousarray(ordered_locs, dtype=np.float64)
    n = locs.shape[0]
    if m < 1 or n <= m:
        raise ValueError(f"need 1 <= m < n, got m={m}, n={n}")
    out = np.empty((n - m, m), dtype=np.int64)
    rc = lib().orc_knn_pred(_dp(locs), n, m, _ip(out), threads or default_threads())
    if rc:
        raise RuntimeError(f"orc_knn_pred failed: {rc}")
    return out


def knn_points(query, data, m: int, threads: int | None = None) -> np.ndarray:
    """Unrestricted m nearest data points per query (vg/geo.py:350-358)."""
    q = np.ascontiguousarray(query, dtype=np.float64)
    d = np.ascontiguousarray(data, dtype=np.float64)
    out = np.empty((q.shape[0], m), dtype=np.int64)
    rc = lib().orc_knn_points(_dp(q), q.shape[0], _dp(d), d.shape[0], m, _ip(out),
                              threads or default_threads())
    if rc:
        raise RuntimeError(f"orc_knn_points failed: {rc}")
    return out


def knn_pred_bruteforce(locs, m: int) -> np.ndarray:
    """O(n^2) sort-based restatement of the reference test oracle
    (pkg/tests/test_geo.py:17-26) with the kernel's key dx*dx + dy*dy."""
    locs = np.asarray(locs, dtype=np.float64)
    n = locs.shape[0]
    rows = []
    for i in range(m, n):
        dx = locs[:i, 0] - locs[i, 0]
        dy = locs[:i, 1] - locs[i, 1]
        key = dx * dx + dy * dy
        order = np.lexsort((np.arange(i), key))
        rows.append(order[:m])
    return np.asarray(rows, dtype=np.int64).reshape(n - m, m)


# ---------------------------------------------------------------- kernels

def maxmin_order(locs, first: int) -> np.ndarray:
    """Brute-force exact maxmin ordering (checker for vgp_maxmin_order).

    PARITY UNPINNED BY THE REFERENCE: the reference has no maxmin ordering
    (vg/vecchia.py:37 lists random / Morton / identity); this restates the
    definition (Guinness 2018) with the device's arithmetic: squared distance
    (x - cx)**2 + (y - cy)**2 evaluated as rounded dx*dx + dy*dy, argmax with
    ties to the smallest index.  O(n^2); keep n to a few ten thousand.
    """
    locs = np.asarray(locs, dtype=np.float64)
    n = locs.shape[0]
    x, y = locs[:, 0].copy(), locs[:, 1].copy()
    dist = np.full(n, np.inf)
    order = np.empty(n, dtype=np.int64)
    cur = int(first)
    for t in range(n):
        order[t] = cur
        dist[cur] = -1.0
        dx = x - x[cur]
        dy = y - y[cur]
        d = dx * dx + dy * dy
        np.minimum(dist, np.where(dist < 0.0, dist, d), out=dist)
        cur = int(np.argmax(dist))  # first index of the maximum
    return order


def matern_cov(d, sigma_sq: float, beta: float, nu: float) -> np.ndarray:
    """vg/kernels.py:59-82 restated (scipy kv/gamma for general nu)."""
    from scipy.special import gamma as _gamma
    from scipy.special import kv as _kv

    d = np.asarray(d, dtype=np.float64)
    u = np.atleast_1d(d) / beta
    s2 = sigma_sq
    if nu == 0.5:
        out = s2 * np.exp(-u)
    elif nu == 1.5:
        out = s2 * (1.0 + u) * np.exp(-u)
    elif nu == 2.5:
        out = s2 * (1.0 + u + u * u / 3.0) * np.exp(-u)
    else:
        out = np.full(u.shape, s2)
        pos = u > 0.0
        up = u[pos]
        with np.errstate(over="ignore", under="ignore"):
            out[pos] = s2 * (2.0 ** (1.0 - nu) / _gamma(nu)) * up**nu * _kv(nu, up)
    return out.reshape(d.shape)


def powexp_cov(d, sigma_sq: float, beta: float, nu: float) -> np.ndarray:
    """vg/kernels.py:85-91."""
    d = np.asarray(d, dtype=np.float64)
    with np.errstate(under="ignore"):
        return sigma_sq * np.exp(-np.atleast_1d(d) ** nu / beta).reshape(d.shape)


def cov(d, family: str, sigma_sq: float, beta: float, nu: float) -> np.ndarray:
    if family == "matern":
        return matern_cov(d, sigma_sq, beta, nu)
    return powexp_cov(d, sigma_sq, beta, nu)


# ---------------------------------------------------------------- sums

def pairwise_sum(a) -> float:
    """numpy float64 pairwise sum (what ndarray.sum() does on contiguous data)."""
    a = np.ascontiguousarray(a, dtype=np.float64)
    return float(lib().orc_pairwise_sum(_dp(a), a.shape[0]))


def ordered_sum(a) -> float:
    """vecchia._ordered_sum: 4096-chunk pairwise partials summed in order."""
    a = np.ascontiguousarray(a, dtype=np.float64)
    return float(lib().orc_ordered_sum(_dp(a), a.shape[0]))


# ---------------------------------------------------------------- log-likelihood

@dataclass
class OracleResult:
    status: int
    fail_index: int
    total: float
    block_first: float
    block_rest: np.ndarray
    mu_new: np.ndarray
    sigma_new: np.ndarray


def is_closed_form(family: str, nu: float) -> bool:
    return family == "power_exponential" or nu in (0.5, 1.5, 2.5)


def _haversine(lon1, lat1, lon2, lat2, radius):
    # vg/geo.py:70-79, the same numpy expression
    p1 = np.radians(lat1)
    p2 = np.radians(lat2)
    l1 = np.radians(lon1)
    l2 = np.radians(lon2)
    h = np.sin((p2 - p1) / 2.0) ** 2 + np.cos(p1) * np.cos(p2) * np.sin((l2 - l1) / 2.0) ** 2
    return 2.0 * radius * np.arcsin(np.sqrt(np.clip(h, 0.0, 1.0)))


def _pdist(a, b, metric, radius):
    """geo.pairwise_distance (vg/geo.py:92-98) on broadcast (..., 2) arrays."""
    if metric == "great_circle":
        return _haversine(a[..., 0], a[..., 1], b[..., 0], b[..., 1], radius)
    return np.hypot(a[..., 0] - b[..., 0], a[..., 1] - b[..., 1])


def loglik(ordered_locs, ordered_obs, m: int, neighbors, family: str, sigma_sq: float,
           beta: float, nu: float, threads: int | None = None, metric: str = "euclidean",
           radius: float = 6371.0) -> OracleResult:
    """Vecchia log-likelihood of an ORDERED dataset (vg/vecchia.py:217-238).

    Closed-form kernels on the plane run in the C restatement; general nu and
    the great-circle metric in numpy+scipy.
    """
    if not is_closed_form(family, nu) or metric != "euclidean":
        return loglik_numpy(ordered_locs, ordered_obs, m, neighbors, family, sigma_sq, beta, nu,
                            metric=metric, radius=radius)
    locs = np.ascontiguousarray(ordered_locs, dtype=np.float64)
    obs = np.ascontiguousarray(ordered_obs, dtype=np.float64)
    nbr = np.ascontiguousarray(neighbors, dtype=np.int64)
    n = locs.shape[0]
    k = n - m
    rest = np.empty(k)
    mu = np.empty(k)
    sg = np.empty(k)
    total = np.zeros(1)
    bf = np.zeros(1)
    fail = np.zeros(1, dtype=np.int64)
    fam = 0 if family == "matern" else 1
    rc = lib().orc_loglik(_dp(locs), _dp(obs), n, m, _ip(nbr), fam, sigma_sq, beta, nu,
                          _dp(total), _dp(bf), _dp(rest), _dp(mu), _dp(sg), _ip(fail),
                          threads or default_threads())
    if rc < 0:
        raise RuntimeError(f"orc_loglik failed: {rc}")
    return OracleResult(int(rc), int(fail[0]), float(total[0]), float(bf[0]), rest, mu, sg)


def _potrf_sweep(mats):
    # vg/batchla.py:141-156 (raises via return value instead of exception)
    dim = mats.shape[1]
    for j in range(dim):
        piv = mats[:, j, j]
        bad = ~(piv > 0.0)
        if np.any(bad):
            return int(np.argmax(bad)), j
        np.sqrt(piv, out=piv)
        if j + 1 < dim:
            col = mats[:, j + 1:, j]
            col /= piv[:, None]
            mats[:, j + 1:, j + 1:] -= col[:, :, None] * col[:, None, :]
    return None


def _trsv(mats, b):
    x = b.copy()
    dim = mats.shape[1]
    for j in range(dim):
        x[:, j] /= mats[:, j, j]
        if j + 1 < dim:
            x[:, j + 1:] -= mats[:, j + 1:, j] * x[:, j, None]
    return x


def _dot(a, b):
    out = np.zeros(a.shape[0])
    for i in range(a.shape[1]):
        out += a[:, i] * b[:, i]
    return out


def loglik_numpy(ordered_locs, ordered_obs, m, neighbors, family, sigma_sq, beta, nu,
                 chunk: int | None = None, metric: str = "euclidean",
                 radius: float = 6371.0) -> OracleResult:
    """Vectorised numpy restatement of assemble/_numeric_stage/_reduction_stage."""
    locs = np.asarray(ordered_locs, dtype=np.float64)
    y = np.asarray(ordered_obs, dtype=np.float64)
    nbr = np.asarray(neighbors, dtype=np.int64)
    n = locs.shape[0]
    count = n - m + 1
    mats = np.empty((count, m, m))
    vv = np.empty((count, m))
    yv = np.empty((count, m))
    d0 = _pdist(locs[:m, None, :], locs[None, :m, :], metric, radius)
    mats[0] = cov(d0, family, sigma_sq, beta, nu)
    vv[0] = y[:m]
    yv[0] = y[:m]
    if count > 1:
        nl = locs[nbr]  # (count-1, m, 2)
        dm = _pdist(nl[:, :, None, :], nl[:, None, :, :], metric, radius)
        mats[1:] = cov(dm, family, sigma_sq, beta, nu)
        dv = _pdist(locs[m:, None, :], nl, metric, radius)
        vv[1:] = cov(dv, family, sigma_sq, beta, nu)
        yv[1:] = y[nbr]
    # column-major semantics do not matter for symmetric input; work on (k, i, j)
    csz = chunk or max(1, (1 << 21) // (m * m))
    for lo in range(0, count, csz):
        hi = min(lo + csz, count)
        bad = _potrf_sweep(mats[lo:hi])
        if bad is not None:
            k = n - m
            return OracleResult(STATUS_NPD, lo + bad[0], float("nan"), float("nan"),
                                np.empty(k), np.empty(k), np.empty(k))
    vp = _trsv(mats, vv)
    ypr = _trsv(mats, yv)
    mu_p = _dot(ypr, vp)
    sg_p = _dot(vp, vp)
    hld = pairwise_sum(np.log(np.diagonal(mats[0])))
    block_first = -hld - 0.5 * mu_p[0] - 0.5 * m * LOG_2PI
    mu_new = mu_p[1:]
    sigma_new = sigma_sq - sg_p[1:]
    bad = ~(sigma_new > 0.0)
    if np.any(bad):
        k = n - m
        return OracleResult(STATUS_BAD_VAR, 1 + int(np.argmax(bad)), float("nan"), float("nan"),
                            np.empty(k), mu_new, sigma_new)
    resid = y[m:] - mu_new
    block_rest = -0.5 * (resid * resid / sigma_new + LOG_2PI + np.log(sigma_new))
    total = block_first + ordered_sum(block_rest)
    return OracleResult(STATUS_OK, -1, total, block_first, block_rest, mu_new, sigma_new)


def simulate_vecchia(ordered_locs, m, neighbors, family, sigma_sq, beta, nu, seed):
    """Draw y from the Vecchia-implied Gaussian: the model
    whose exact log-density the Vecchia likelihood is, so parity fixtures are
    model-consistent at any n.  y[:m] = L0 z[:m];
    y_i = b_i . y[J_i] + sqrt(D_i) z_i with b_i = Sigma_i^-1 v_i and
    D_i = sigma^2 - v_i . b_i, for ordered i = m..n-1.  Returns ORDERED y."""
    locs = np.asarray(ordered_locs, dtype=np.float64)
    nbr = np.asarray(neighbors, dtype=np.int64)
    n = locs.shape[0]
    z = np.random.default_rng(seed).standard_normal(n)
    d0 = np.hypot(locs[:m, None, 0] - locs[None, :m, 0], locs[:m, None, 1] - locs[None, :m, 1])
    y = np.empty(n)
    y[:m] = np.linalg.cholesky(cov(d0, family, sigma_sq, beta, nu)) @ z[:m]
    b = np.empty((n - m, m))
    dvar = np.empty(n - m)
    for lo in range(0, n - m, 4096):
        hi = min(lo + 4096, n - m)
        nl = locs[nbr[lo:hi]]
        dm = np.hypot(nl[:, :, None, 0] - nl[:, None, :, 0], nl[:, :, None, 1] - nl[:, None, :, 1])
        sig = cov(dm, family, sigma_sq, beta, nu)
        tl = locs[m + lo:m + hi]
        dv = np.hypot(tl[:, None, 0] - nl[:, :, 0], tl[:, None, 1] - nl[:, :, 1])
        v = cov(dv, family, sigma_sq, beta, nu)
        bb = np.linalg.solve(sig, v[:, :, None])[:, :, 0]
        b[lo:hi] = bb
        dvar[lo:hi] = sigma_sq - np.einsum("ij,ij->i", v, bb)
    sd = np.sqrt(np.maximum(dvar, 0.0))
    for i in range(m, n):
        r = i - m
        y[i] = b[r] @ y[nbr[r]] + sd[r] * z[i]
    return y


def exact_loglik(locs, obs, family, sigma_sq, beta, nu) -> float:
    """Dense exact log-likelihood (vg/exact.py:34-44)."""
    from scipy.linalg import solve_triangular

    locs = np.asarray(locs, dtype=np.float64)
    n = locs.shape[0]
    d = np.hypot(locs[:, None, 0] - locs[None, :, 0], locs[:, None, 1] - locs[None, :, 1])
    sig = cov(d, family, sigma_sq, beta, nu)
    low = np.linalg.cholesky(sig)
    alpha = solve_triangular(low, obs, lower=True, check_finite=False)
    return -0.5 * n * LOG_2PI - float(np.log(np.diagonal(low)).sum()) - 0.5 * float(alpha @ alpha)


# ---------------------------------------------------------------- optimizer

def nelder_mead_max(f, x0, bounds, tol=1e-5, max_evals=500):
    """Clamped Nelder-Mead maximiser, vg/fit.py:61-137 restated."""
    x0 = np.asarray(x0, dtype=np.float64)
    lo = np.array([b[0] for b in bounds], dtype=np.float64)
    hi = np.array([b[1] for b in bounds], dtype=np.float64)
    ndim = x0.shape[0]
    state = {"evals": 0, "best_x": None, "best_f": -math.inf}

    def neg(x):
        state["evals"] += 1
        val = f(x)
        if val > state["best_f"]:
            state["best_f"] = val
            state["best_x"] = x.copy()
        return -val

    def clamp(x):
        return np.minimum(np.maximum(x, lo), hi)

    simplex = [x0.copy()]
    for i in range(ndim):
        step = 0.1 * (hi[i] - lo[i])
        v = x0.copy()
        v[i] = x0[i] + step if x0[i] + step <= hi[i] else x0[i] - step
        simplex.append(v)
    values = [neg(v) for v in simplex]
    if not np.any(np.isfinite(values)):
        raise RuntimeError("no feasible point in the initial simplex")
    converged = False
    while state["evals"] < max_evals:
        order = np.argsort(values, kind="stable")
        simplex = [simplex[i] for i in order]
        values = [values[i] for i in order]
        f_best, f_worst = values[0], values[-1]
        if math.isfinite(f_worst) and f_worst - f_best <= tol * max(1.0, abs(f_best)):
            converged = True
            break
        centroid = np.mean(simplex[:-1], axis=0)
        refl = clamp(centroid + 1.0 * (centroid - simplex[-1]))
        f_r = neg(refl)
        if values[0] <= f_r < values[-2]:
            simplex[-1], values[-1] = refl, f_r
        elif f_r < values[0]:
            exp_ = clamp(centroid + 2.0 * (refl - centroid))
            f_e = neg(exp_)
            if f_e < f_r:
                simplex[-1], values[-1] = exp_, f_e
            else:
                simplex[-1], values[-1] = refl, f_r
        else:
            con = clamp(centroid + 0.5 * (simplex[-1] - centroid))
            f_c = neg(con)
            if f_c < values[-1]:
                simplex[-1], values[-1] = con, f_c
            else:
                for i in range(1, len(simplex)):
                    simplex[i] = clamp(simplex[0] + 0.5 * (simplex[i] - simplex[0]))
                    values[i] = neg(simplex[i])
    return state["best_x"], state["best_f"], state["evals"], converged


def mle(ordered_locs, ordered_obs, m, neighbors, init=(1.0, 0.1, 0.5), family="matern",
        bounds=((1e-4, 1e4), (1e-4, 1e4)), tol=1e-5, max_evals=500, threads=None):
    """mle_estimate with the Vecchia objective and fixed nu (vg/fit.py:140-178)."""
    nu = init[2]

    def objective(x):
        s2, beta = float(x[0]), float(x[1])
        if not (np.isfinite(s2) and s2 > 0 and np.isfinite(beta) and beta > 0):
            return -math.inf
        r = loglik(ordered_locs, ordered_obs, m, neighbors, family, s2, beta, nu, threads)
        return r.total if r.status == STATUS_OK else -math.inf

    return nelder_mead_max(objective, np.array(init[:2]), list(bounds), tol, max_evals)
