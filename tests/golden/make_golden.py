"""Generate golden vectors by running the REFERENCE implementation itself.

Run in the build container (the only place /root/reference exists):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py [--with-mle]

It imports ``vecchiagp`` from /root/reference/pkg/src (read-only; numba's
on-disk cache is redirected to NUMBA_CACHE_DIR), evaluates the reference's
own public API on seeded inputs and writes one compressed ``.npz`` per case
into tests/golden/.  Inputs are saved alongside outputs (numpy ``Generator``
streams are not promised stable across numpy versions), together with the
library versions in ``versions.json``.  Nothing on the GPU box reads
/root/reference: the tests only read these files.
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
REF_SRC = "/root/reference/pkg/src"
sys.path.insert(0, REF_SRC)

import numpy as np  # noqa: E402

import vecchiagp  # noqa: E402
from vecchiagp import exact, fit, geo, kernels, parallel, vecchia  # noqa: E402
from vecchiagp.errors import LikelihoodEvaluationError  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def table_digest(table: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(table, dtype=np.int64).tobytes()).hexdigest()


def save(name: str, **arrays):
    path = os.path.join(OUT, f"{name}.npz")
    np.savez_compressed(path, **arrays)
    print(f"wrote {path} ({os.path.getsize(path) / 1024:.1f} KiB)")


def knn_cases():
    # vg tests: pkg/tests/test_geo.py:168-250
    rng = np.random.default_rng(11)
    locs = rng.random((200, 2))
    t = geo.nearest_neighbors(geo.Dataset(locs, np.zeros(200)), 10).neighbors
    save("knn_random_200_10", locs=locs, m=10, table=t)

    g = np.arange(12.0)
    locs = np.stack(np.meshgrid(g, g), axis=-1).reshape(-1, 2)
    t = geo.nearest_neighbors(geo.Dataset(locs, np.zeros(len(locs))), 8).neighbors
    save("knn_grid12_8", locs=locs, m=8, table=t)

    locs = np.array([[0.0, 0.0], [1.0, 0.0], [2.0, 0.0], [3.0, 0.0]])
    t = geo.nearest_neighbors(geo.Dataset(locs, np.zeros(4)), 2).neighbors
    save("knn_collinear", locs=locs, m=2, table=t)

    # coarse integer lattice with many exact duplicates: ties + zero keys
    rng = np.random.default_rng(21)
    locs = rng.integers(0, 6, size=(400, 2)).astype(np.float64)
    t = geo.nearest_neighbors(geo.Dataset(locs, np.zeros(400)), 12).neighbors
    save("knn_dupgrid_400_12", locs=locs, m=12, table=t)

    # random ordering of a uniform cloud, m = 30 and m = 60
    rng = np.random.default_rng(22)
    raw = rng.random((3000, 2))
    perm = geo.random_ordering(3000, 0)
    ordered = geo.Dataset(raw, np.zeros(3000)).permute(perm)
    for m in (30, 60):
        t = geo.nearest_neighbors(ordered, m).neighbors
        save(f"knn_random_3000_{m}", locs=ordered.locations, m=m, table=t)

    # large m relative to n (full-conditioning regime)
    rng = np.random.default_rng(23)
    locs = rng.random((300, 2))
    t = geo.nearest_neighbors(geo.Dataset(locs, np.zeros(300)), 150).neighbors
    save("knn_random_300_150", locs=locs, m=150, table=t)

    # unrestricted search (kriging), pkg/tests/test_geo.py:240-250
    rng = np.random.default_rng(15)
    train = rng.random((90, 2))
    query = rng.random((25, 2))
    t = geo.nearest_points(query, train, geo.Euclidean(), 6)
    save("knn_points_25_90_6", query=query, train=train, m=6, table=t)


def ll_case(name, n, m, family, s2, beta, nu, seed, ordering="random", data_nu=None,
            locs=None, y=None, plan_seed=0, metric=None):
    spec = kernels.KernelSpec(family, kernels.KernelParams(s2, beta, nu))
    if locs is None:
        rng = np.random.default_rng(seed)
        locs = rng.random((n, 2))
    if y is None:
        gspec = kernels.KernelSpec(family, kernels.KernelParams(s2, beta, data_nu or nu))
        y = exact.simulate_grf(locs, gspec, seed + 1, metric or geo.Euclidean())
    data = geo.Dataset(locs, y, metric or geo.Euclidean())
    plan = vecchia.make_plan(data, m, ordering, seed=plan_seed)
    ordered = data.permute(plan.permutation)
    out = dict(locs=locs, obs=y, perm=plan.permutation.order, ordered_locs=ordered.locations,
               ordered_obs=ordered.observations, m=m, table=plan.neighbors.neighbors,
               family=family, theta=np.array([s2, beta, nu]), ordering=ordering,
               metric="great_circle" if isinstance(metric, geo.GreatCircle) else "euclidean")
    try:
        res = vecchia.vecchia_loglik(data, plan, spec)
        out.update(status=0, fail_index=-1, total=res.total, block_first=res.block_first,
                   block_rest=res.block_rest, mu_new=res.mu_new, sigma_new=res.sigma_new)
    except LikelihoodEvaluationError as exc:
        out.update(status=1, fail_index=exc.block_index, total=np.nan)
    if n <= 600 and m == n - 1:
        out["exact"] = exact.exact_loglik(data, spec)
    save(name, **out)


def loglik_cases():
    ll_case("ll_n300_m10_nu05", 300, 10, "matern", 1.0, 0.1, 0.5, seed=100)
    ll_case("ll_n2000_m30_nu15", 2000, 30, "matern", 1.0, 0.052537, 1.5, seed=101)
    ll_case("ll_n1000_m20_nu25", 1000, 20, "matern", 1.0, 0.05, 2.5, seed=102)
    ll_case("ll_n3000_m60_nu15", 3000, 60, "matern", 1.0, 0.052537, 1.5, seed=103)
    ll_case("ll_n2000_m40_nu05_s2", 2000, 40, "matern", 2.7, 0.078809, 0.5, seed=104)
    ll_case("ll_n500_m15_nu08", 500, 15, "matern", 1.0, 0.1, 0.8, seed=105)
    ll_case("ll_n500_m15_nu23", 500, 15, "matern", 1.0, 0.05, 2.3, seed=106, data_nu=2.5)
    ll_case("ll_n400_m12_powexp", 400, 12, "power_exponential", 1.3, 0.2, 1.2, seed=107)
    ll_case("ll_n800_m24_morton", 800, 24, "matern", 1.0, 0.1, 1.5, seed=108, ordering="morton")
    ll_case("ll_n600_m17_identity", 600, 17, "matern", 1.0, 0.1, 0.5, seed=109, ordering="identity")
    ll_case("ll_n1500_m100_nu15", 1500, 100, "matern", 1.0, 0.052537, 1.5, seed=110)
    ll_case("ll_n2500_m120_nu05", 2500, 120, "matern", 1.0, 0.078809, 0.5, seed=111)
    # full conditioning m = n - 1 (pkg/tests/test_vecchia.py:110-116)
    ll_case("ll_full_n300_nu05", 300, 299, "matern", 1.0, 0.1, 0.5, seed=4, plan_seed=5)
    ll_case("ll_full_n200_nu15_morton", 200, 199, "matern", 1.0, 0.1, 1.5, seed=112,
            ordering="morton")
    # duplicate point -> LikelihoodEvaluationError (pkg/tests/test_vecchia.py:149-156)
    locs = np.array([[0.0, 0.0], [1.0, 0.0], [1.0, 0.0]])
    ll_case("ll_fail_duplicate", 3, 1, "matern", 1.0, 0.1, 0.5, seed=0, locs=locs,
            y=np.array([0.1, 0.2, 0.3]), ordering="identity")
    # a dense cloud with duplicates inside conditioning sets -> NPD
    rng = np.random.default_rng(113)
    locs = rng.random((400, 2))
    locs[200:210] = locs[100:110]
    ll_case("ll_fail_npd_dups", 400, 12, "matern", 1.0, 0.1, 1.5, seed=113, locs=locs,
            y=rng.standard_normal(400), ordering="identity")


def c1_case(with_mle: bool):
    """BASELINE config 1: n=20,000, m=30, Matern nu=0.5, beta=0.078809 (c1)."""
    spec = kernels.KernelSpec("matern", kernels.KernelParams(1.0, 0.078809, 0.5))
    locs = np.random.default_rng(500).random((20000, 2))
    t0 = time.perf_counter()
    y = exact.simulate_grf(locs, spec, 501)
    print(f"c1 simulate_grf {time.perf_counter() - t0:.1f}s")
    data = geo.Dataset(locs, y)
    parallel.set_num_threads(os.cpu_count() or 1)
    plan = vecchia.make_plan(data, 30, "random", seed=0)
    res = vecchia.vecchia_loglik(data, plan, spec)
    out = dict(locs=locs, obs=y, perm=plan.permutation.order, m=30,
               table_sha256=table_digest(plan.neighbors.neighbors),
               table_head=plan.neighbors.neighbors[:200], theta=np.array([1.0, 0.078809, 0.5]),
               total=res.total, block_first=res.block_first, block_rest=res.block_rest,
               mu_new=res.mu_new, sigma_new=res.sigma_new)
    if with_mle:
        cfg = fit.FitConfig(objective="vecchia", m=30, ordering="random", seed=0,
                            init=kernels.KernelParams(0.5, 0.05, 0.5))
        t0 = time.perf_counter()
        fr = fit.mle_estimate(data, cfg)
        print(f"c1 MLE {time.perf_counter() - t0:.1f}s evals={fr.evaluations}")
        out.update(mle_theta=np.array([fr.theta_hat.sigma_sq, fr.theta_hat.beta, fr.theta_hat.nu]),
                   mle_loglik=fr.loglik, mle_evals=fr.evaluations, mle_converged=fr.converged)
    save("c1_n20000_m30_nu05", **out)


def mle_free_nu_case(name, n, m, nu_true, beta_true, init, seed, clustered=False):
    """Free-nu MLE of (sigma^2, beta, nu) (vg/fit.py:140-178, free nu at :153-157):
    BASELINE config 5's estimator at desk scale, y from the dense simulate_grf."""
    rng = np.random.default_rng(seed)
    if clustered:
        centers = rng.random((20, 2))
        k = int(0.8 * n)
        locs = np.concatenate([centers[rng.integers(0, 20, k)] + 0.02 * rng.standard_normal((k, 2)),
                               rng.random((n - k, 2))])
    else:
        locs = rng.random((n, 2))
    spec = kernels.KernelSpec("matern", kernels.KernelParams(1.0, beta_true, nu_true))
    y = exact.simulate_grf(locs, spec, seed + 1)
    data = geo.Dataset(locs, y)
    parallel.set_num_threads(os.cpu_count() or 1)
    cfg = fit.FitConfig(objective="vecchia", m=m, ordering="random", seed=0,
                        init=kernels.KernelParams(*init), free_nu=True)
    t0 = time.perf_counter()
    fr = fit.mle_estimate(data, cfg)
    dt = time.perf_counter() - t0
    print(f"{name}: MLE {dt:.1f}s evals={fr.evaluations} theta={fr.theta_hat}")
    save(name, locs=locs, obs=y, m=m, init=np.array(init),
         mle_theta=np.array([fr.theta_hat.sigma_sq, fr.theta_hat.beta, fr.theta_hat.nu]),
         mle_loglik=fr.loglik, mle_evals=fr.evaluations, mle_converged=fr.converged,
         mle_seconds=dt)


def sphere_large_cases():
    """Great-circle kNN at scale (glibc-sin keys, vg/geo.py:266-292): the table
    digest of the reference on 40,000 global points and on 30,000 points in
    a 2-degree patch (dense, many near-ties), random ordering."""
    gc = geo.GreatCircle()
    parallel.set_num_threads(os.cpu_count() or 1)
    cases = [("knn_sphere_big_global", 40000, 30, (-180, 180), (-80, 80), 51),
             ("knn_sphere_big_patch", 30000, 20, (10, 12), (45, 47), 52)]
    if os.environ.get("GOLDEN_SPHERE_100K"):
        # the glibc-vs-CUDA sin tie bound at n >= 100k;
        # a 4-degree patch holds 100k points ~1.4 km apart (dense near-ties)
        cases = [("knn_sphere_big_100k_patch", 100000, 30, (20, 24), (-2, 2), 53)]
    for name, n, m, lon, lat, seed in cases:
        rng = np.random.default_rng(seed)
        locs = np.column_stack([rng.uniform(*lon, n), rng.uniform(*lat, n)])
        ordered = geo.Dataset(locs, np.zeros(n), gc).permute(geo.random_ordering(n, 0))
        t0 = time.perf_counter()
        t = geo.nearest_neighbors(ordered, m).neighbors
        print(f"{name}: {time.perf_counter() - t0:.1f}s")
        save(name, locs=ordered.locations, m=m, table_sha256=table_digest(t), table_head=t[:500])


def mle_cases():
    mle_free_nu_case("mle_freenu_n2000_m20_clustered", 2000, 20, 0.8, 0.05, (0.5, 0.1, 1.0), 601,
                     clustered=True)
    mle_free_nu_case("mle_freenu_n5000_m30", 5000, 30, 1.2, 0.05, (1.0, 0.1, 0.5), 611)


def sphere_cases():
    """Great-circle metric (vg/geo.py:70-79, :266-292): kNN of the reference
    (pkg/tests/test_geo.py:196-204 shape and larger), log-likelihoods with
    haversine covariance, kriging."""
    from vecchiagp import fit

    gc = geo.GreatCircle()
    rng = np.random.default_rng(40)
    locs = np.column_stack([rng.uniform(-30, 30, 120), rng.uniform(-40, 40, 120)])
    t = geo.nearest_neighbors(geo.Dataset(locs, np.zeros(120), gc), 7).neighbors
    save("knn_sphere_120_7", locs=locs, m=7, table=t)
    rng = np.random.default_rng(41)
    locs = np.column_stack([rng.uniform(-180, 180, 2000), rng.uniform(-70, 70, 2000)])
    perm = geo.random_ordering(2000, 0)
    ordered = geo.Dataset(locs, np.zeros(2000), gc).permute(perm)
    t = geo.nearest_neighbors(ordered, 30).neighbors
    save("knn_sphere_2000_30", locs=ordered.locations, m=30, table=t)
    q = np.column_stack([rng.uniform(-180, 180, 50), rng.uniform(-70, 70, 50)])
    t = geo.nearest_points(q, locs, gc, 12)
    save("knn_sphere_points_50_2000_12", query=q, train=locs, m=12, table=t)

    rng = np.random.default_rng(42)
    locs = np.column_stack([rng.uniform(30, 50, 900), rng.uniform(20, 40, 900)])
    ll_case("ll_gcd_n900_m20_nu05", 900, 20, "matern", 1.0, 300.0, 0.5, seed=420, locs=locs,
            metric=gc)
    ll_case("ll_gcd_n900_m60_nu15", 900, 60, "matern", 1.0, 200.0, 1.5, seed=421, locs=locs,
            metric=gc)
    ll_case("ll_gcd_n900_m90_nu08", 900, 90, "matern", 1.0, 250.0, 0.8, seed=422, locs=locs,
            metric=gc)
    spec = kernels.KernelSpec("matern", kernels.KernelParams(1.0, 300.0, 0.5))
    y = exact.simulate_grf(locs, spec, 430, gc)
    data = geo.Dataset(locs[:850], y[:850], gc)
    r = fit.krige_predict(data, spec.params, "matern", locs[850:], 30, y[850:])
    save("krige_gcd_n850_m30_nu05", train=locs[:850], y=y[:850], test=locs[850:], truth=y[850:],
         m=30, family="matern", theta=np.array([1.0, 300.0, 0.5]), pred=r.predictions,
         var=r.variances, mse=r.mse, metric="great_circle")


def krige_cases():
    """fit.krige_predict (vg/fit.py:221-275) on the reference's own kriging
    setup (pkg/tests/test_fit.py:82-88) and acceptance criterion 6's split
    (pkg/tests/test_acceptance.py:150-186, smaller here)."""
    from vecchiagp import exact, fit
    from vecchiagp.kernels import KernelParams, KernelSpec

    spec = KernelSpec("matern", KernelParams(1.0, 0.078809, 0.5))
    rng = np.random.default_rng(200)
    locs = rng.random((320, 2))
    y = exact.simulate_grf(locs, spec, seed=201)
    train, test, truth = locs[:300], locs[300:], y[300:]
    data = vecchiagp.Dataset(train, y[:300])
    for m in (1, 25, 40, 90, 300):
        r = fit.krige_predict(data, spec.params, "matern", test, m, truth)
        save(f"krige_n300_m{m}_nu05", train=train, y=y[:300], test=test, truth=truth, m=m,
             family="matern", theta=np.array([1.0, 0.078809, 0.5]),
             pred=r.predictions, var=r.variances, mse=r.mse)
    spec2 = KernelSpec("matern", KernelParams(1.3, 0.06, 1.5))
    rng = np.random.default_rng(700)
    locs = rng.random((1500, 2))
    y = exact.simulate_grf(locs, spec2, seed=701)
    data = vecchiagp.Dataset(locs[:1400], y[:1400])
    for m, fam, th in ((60, "matern", (1.3, 0.06, 1.5)), (30, "matern", (1.3, 0.06, 0.8)),
                       (20, "power_exponential", (1.3, 0.06, 1.2))):
        r = fit.krige_predict(data, KernelParams(*th), fam, locs[1400:], m, y[1400:])
        save(f"krige_n1400_m{m}_{fam[:6]}", train=locs[:1400], y=y[:1400], test=locs[1400:],
             truth=y[1400:], m=m, family=fam, theta=np.array(th), pred=r.predictions,
             var=r.variances, mse=r.mse)


def kl_cases():
    """exact.exact_loglik / kl_vecchia / simulate_grf / kl_gaussian
    (vg/exact.py) on the reference's own KL setups (pkg/tests/test_exact.py
    TestKLVecchia, pkg/tests/test_acceptance.py criteria 3 and 4, smaller)."""
    from vecchiagp.kernels import KernelParams, KernelSpec

    spec = KernelSpec("matern", KernelParams(1.0, 0.026270, 0.5))
    locs = np.random.default_rng(8).random((400, 2))
    data = vecchiagp.Dataset(locs, np.zeros(400))
    for m in (5, 20, 60, 399):
        plan = vecchia.make_plan(data, m, "random", seed=3)
        r = exact.kl_vecchia(locs, plan, spec)
        save(f"kl_n400_m{m}_random", locs=locs, m=m, ordering="random", plan_seed=3,
             family="matern", theta=np.array([1.0, 0.026270, 0.5]), kl=r.kl,
             exact_ll0=r.exact_ll0, vecchia_ll0=r.vecchia_ll0)
    spec2 = KernelSpec("matern", KernelParams(1.0, 0.078809, 0.5))
    locs = np.random.default_rng(2024).random((1024, 2))
    data = vecchiagp.Dataset(locs, np.zeros(1024))
    for ordering in ("random", "morton"):
        plan = vecchia.make_plan(data, 30, ordering, seed=1)
        r = exact.kl_vecchia(locs, plan, spec2)
        save(f"kl_n1024_m30_{ordering}", locs=locs, m=30, ordering=ordering, plan_seed=1,
             family="matern", theta=np.array([1.0, 0.078809, 0.5]), kl=r.kl,
             exact_ll0=r.exact_ll0, vecchia_ll0=r.vecchia_ll0)
    # exact log-likelihood of simulated fields, general nu and power exponential
    rng = np.random.default_rng(31)
    locs = rng.random((700, 2))
    for fam, th in (("matern", (1.3, 0.06, 1.5)), ("matern", (0.8, 0.05, 0.8)),
                    ("power_exponential", (1.1, 0.07, 1.2))):
        sp = KernelSpec(fam, KernelParams(*th))
        y = exact.simulate_grf(locs, sp, seed=32)
        ll = exact.exact_loglik(vecchiagp.Dataset(locs, y), sp)
        save(f"exact_n700_{fam[:6]}_nu{str(th[2]).replace('.', '')}", locs=locs, y=y, family=fam,
             theta=np.array(th), exact_ll=ll)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--with-mle", action="store_true")
    ap.add_argument("--only", default="")
    args = ap.parse_args()
    import numba
    import scipy

    versions = {"vecchiagp": vecchiagp.__version__, "numpy": np.__version__,
                "scipy": scipy.__version__, "numba": numba.__version__,
                "python": sys.version.split()[0]}
    with open(os.path.join(OUT, "versions.json"), "w") as f:
        json.dump(versions, f, indent=1)
    if args.only in ("", "knn"):
        knn_cases()
    if args.only in ("", "ll"):
        loglik_cases()
    if args.only in ("", "krige"):
        krige_cases()
    if args.only in ("", "sphere"):
        sphere_cases()
    if args.only in ("", "kl"):
        kl_cases()
    if args.only == "mle":
        mle_cases()
    if args.only == "sphere_large":
        sphere_large_cases()
    if args.only in ("", "c1"):
        c1_case(args.with_mle)


if __name__ == "__main__":
    main()
