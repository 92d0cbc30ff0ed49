"""GPU parity tests: the B200 path (through the C ABI via the package) against
golden vectors produced by the reference itself (tests/golden/make_golden.py)
and against the CPU oracle (oracle/) on identical seeded inputs.

Tolerances (north star): log-likelihood totals relative <= 1e-9; neighbour
tables bit-exact; covariance values relative <= 1e-12 (closed forms) and
<= 1e-11 (general-nu Bessel path); MLE estimates relative <= 1e-4.
"""

import math

import numpy as np
import pytest

from _helpers import golden_names, load, rel

pytestmark = pytest.mark.gpu

TOL_TOTAL = 1e-9


@pytest.fixture(scope="module")
def vg():
    import paper_2403_07412_b200 as vg

    if vg._native.device_count() == 0:
        pytest.fail("GPU tests need a CUDA device: the B200 path has no CPU fallback")
    return vg


@pytest.fixture(scope="module")
def oracle():
    from oracle import oracle as O

    return O


# ---------------------------------------------------------------- kNN

@pytest.mark.parametrize("name", [n for n in golden_names("knn_") if "big" not in n])
def test_knn_bit_exact_vs_reference(vg, name):
    z = load(name)
    m = int(z["m"])
    metric = vg.GreatCircle() if "sphere" in name else vg.Euclidean()
    if "query" in z.files:
        got = vg.nearest_points(z["query"], z["train"], metric, m)
    else:
        got = vg.nearest_neighbors(vg.Dataset(z["locs"], np.zeros(len(z["locs"])), metric), m).neighbors
    assert got.dtype == np.int64
    np.testing.assert_array_equal(got, z["table"])


@pytest.mark.parametrize("n,m,seed", [(20000, 30, 0), (20000, 60, 1), (5000, 7, 2), (3000, 128, 3)])
def test_knn_bit_exact_vs_oracle(vg, oracle, n, m, seed):
    rng = np.random.default_rng(seed)
    locs = rng.random((n, 2))
    got = vg.nearest_neighbors(vg.Dataset(locs, np.zeros(n)), m).neighbors
    np.testing.assert_array_equal(got, oracle.knn_pred(locs, m))


def test_knn_ties_and_duplicates(vg, oracle):
    rng = np.random.default_rng(7)
    locs = rng.integers(0, 9, size=(2000, 2)).astype(np.float64) * 0.25
    for m in (1, 5, 33):
        got = vg.nearest_neighbors(vg.Dataset(locs, np.zeros(len(locs))), m).neighbors
        np.testing.assert_array_equal(got, oracle.knn_pred(locs, m))


def test_knn_points_vs_oracle(vg, oracle):
    rng = np.random.default_rng(8)
    train = rng.random((3000, 2))
    query = rng.random((700, 2))
    got = vg.nearest_points(query, train, vg.Euclidean(), 40)
    np.testing.assert_array_equal(got, oracle.knn_points(query, train, 40))


def test_c1_neighbor_table_digest(vg):
    import hashlib

    z = load("c1_n20000_m30_nu05")
    locs = z["locs"][z["perm"]]
    t = vg.nearest_neighbors(vg.Dataset(locs, np.zeros(len(locs))), 30).neighbors
    assert hashlib.sha256(t.tobytes()).hexdigest() == str(z["table_sha256"])


# ---------------------------------------------------------------- likelihood

def _metric(vg, z):
    gc = "metric" in z.files and str(z["metric"]) == "great_circle"
    return vg.GreatCircle() if gc else vg.Euclidean()


def _plan_from_golden(vg, z):
    metric = _metric(vg, z)
    data = vg.Dataset(z["locs"], z["obs"], metric)
    perm = vg.Permutation(z["perm"])
    table = vg.NeighborTable(int(z["m"]), z["table"])
    plan = vg.VecchiaPlan(int(z["m"]), perm, table, metric, str(z["ordering"]))
    s2, beta, nu = (float(v) for v in z["theta"])
    spec = vg.KernelSpec(str(z["family"]), vg.KernelParams(s2, beta, nu))
    return data, plan, spec


@pytest.mark.parametrize("name", [n for n in golden_names("ll_") if "fail" not in n])
@pytest.mark.parametrize("variant", [-1, 0, 1, 4, 7, 8, 11, 12, 13])
def test_loglik_vs_reference_golden(vg, name, variant):
    z = load(name)
    data, plan, spec = _plan_from_golden(vg, z)
    closed = str(z["family"]) == "matern" and float(z["theta"][2]) in (0.5, 1.5, 2.5)
    plane = not isinstance(_metric(vg, z), vg.GreatCircle)
    fast = closed and int(z["m"]) + 2 <= 64
    # general-nu Matern: the scheduler-aware kernel (7/8) with the per-evaluation table
    gen3 = str(z["family"]) == "matern" and not closed and int(z["m"]) + 2 <= 64
    if variant in (7, 8) and not (fast or gen3):
        pytest.skip("scheduler-aware kernel: m + 2 <= 64 Matern")
    if variant in (1, 4) and not fast:
        pytest.skip("warp-DMMA variants cover m + 2 <= 64 closed-form Matern only")
    if variant in (1, 7, 11) and not plane:
        pytest.skip("distances computed in the kernel are Euclidean (great circle: cached variants)")
    cache = not plane or int(z["m"]) + 2 <= 64
    if variant == 12 and not cache:
        pytest.skip("large-m Euclidean plans carry no distance cache")
    tiny = closed and plane and int(z["m"]) <= 12
    if variant == 13 and not tiny:
        pytest.skip("thread-per-block kernel: m <= 12, closed-form Matern, Euclidean")
    plan.device_plan().set_variant(variant)
    res = vg.vecchia_loglik(data, plan, spec)
    # the cache exists for m + 2 <= 64 and for great-circle plans; the large-m
    # kernel computes Euclidean distances for the closed forms and streams
    # the cache for general nu / power exponential when there is one
    small, mid = int(z["m"]) + 2 <= 24, int(z["m"]) + 2 <= 56
    auto = 13 if tiny else ((1 if plane else 4) if small else (4 if mid else 8)) if fast else (
        8 if gen3 else (12 if cache and (not plane or not closed) else 11))
    assert plan.device_plan().kernel_variant == (variant if variant >= 0 else auto)
    assert rel(res.total, float(z["total"])) <= TOL_TOTAL
    assert rel(res.block_first, float(z["block_first"])) <= TOL_TOTAL
    # per-block terms: ill-conditioned blocks amplify ulp-level differences
    np.testing.assert_allclose(res.block_rest, z["block_rest"], rtol=1e-7, atol=1e-7)
    np.testing.assert_allclose(res.mu_new, z["mu_new"], rtol=1e-7, atol=1e-7)
    np.testing.assert_allclose(res.sigma_new, z["sigma_new"], rtol=1e-6, atol=1e-12)
    # additivity as stored, bitwise (pkg/tests/test_vecchia.py:127-133)
    assert res.total == res.block_first + vg.vecchia._ordered_sum(res.block_rest)
    if "exact" in z.files:
        assert rel(res.total, float(z["exact"])) <= 1e-8


def test_loglik_failure_duplicate(vg):
    z = load("ll_fail_duplicate")
    data, plan, spec = _plan_from_golden(vg, z)
    with pytest.raises(vg.LikelihoodEvaluationError) as err:
        vg.vecchia_loglik(data, plan, spec)
    assert err.value.block_index == int(z["fail_index"])


def test_loglik_failure_npd_index(vg):
    z = load("ll_fail_npd_dups")
    data, plan, spec = _plan_from_golden(vg, z)
    with pytest.raises(vg.LikelihoodEvaluationError) as err:
        vg.vecchia_loglik(data, plan, spec)
    assert err.value.block_index == int(z["fail_index"])


def test_c1_loglik_and_blocks(vg):
    z = load("c1_n20000_m30_nu05")
    data = vg.Dataset(z["locs"], z["obs"])
    plan = vg.make_plan(data, 30, "random", seed=0)
    np.testing.assert_array_equal(plan.permutation.order, z["perm"])
    spec = vg.KernelSpec("matern", vg.KernelParams(*[float(v) for v in z["theta"]]))
    res = vg.vecchia_loglik(data, plan, spec)
    assert rel(res.total, float(z["total"])) <= TOL_TOTAL
    np.testing.assert_allclose(res.block_rest, z["block_rest"], rtol=1e-7, atol=1e-7)


@pytest.mark.parametrize("n,m,nu,beta,seed", [
    (30000, 60, 1.5, 0.052537, 11), (30000, 30, 0.5, 0.078809, 12), (20000, 45, 2.5, 0.03, 13),
    (12000, 10, 1.5, 0.052537, 14), (8000, 62, 0.5, 0.1, 15), (6000, 96, 1.5, 0.05, 16),
])
def test_loglik_vs_oracle_seeded(vg, oracle, n, m, nu, beta, seed):
    """Model-consistent y (Vecchia forward simulation under the same theta,
    SURVEY.md §7 H5); totals must agree at 1e-9."""
    rng = np.random.default_rng(seed)
    locs = rng.random((n, 2))
    data = vg.Dataset(locs, np.zeros(n))
    plan = vg.make_plan(data, m, "random", seed=seed)
    spec = vg.KernelSpec("matern", vg.KernelParams(1.0, beta, nu))
    y_ord = oracle.simulate_vecchia(locs[plan.permutation.order], m, plan.neighbors.neighbors,
                                    "matern", 1.0, beta, nu, seed + 100)
    y = np.empty(n)
    y[plan.permutation.order] = y_ord
    data = vg.Dataset(locs, y)
    ordered = data.permute(plan.permutation)
    ref = oracle.loglik(ordered.locations, ordered.observations, m, plan.neighbors.neighbors,
                        "matern", 1.0, beta, nu)
    res = vg.vecchia_loglik(data, plan, spec)
    assert ref.status == 0
    assert rel(res.total, ref.total) <= TOL_TOTAL


def test_singleton_exact_convention(vg):
    spec = vg.KernelSpec("matern", vg.KernelParams(2.0, 0.1, 0.5))
    data = vg.Dataset(np.array([[0.5, 0.5]]), np.array([1.3]))
    plan = vg.make_plan(data, m=1, ordering="identity")
    res = vg.vecchia_loglik(data, plan, spec)
    expected = -0.5 * (1.3**2 / 2.0 + math.log(2 * math.pi) + math.log(2.0))
    assert res.total == pytest.approx(expected, rel=1e-15)
    assert res.block_rest.size == 0


def test_bivariate_closed_form(vg):
    d, y1, y2 = 0.37, 0.8, -0.45
    data = vg.Dataset(np.array([[0.0, 0.0], [d, 0.0]]), np.array([y1, y2]))
    spec = vg.KernelSpec("matern", vg.KernelParams(1.0, 1.0, 0.5))
    plan = vg.make_plan(data, 1, "identity")
    res = vg.vecchia_loglik(data, plan, spec)
    rho = math.exp(-d)
    first = -0.5 * (y1**2 + math.log(2 * math.pi))
    cvar = 1.0 - rho**2
    second = -0.5 * ((y2 - rho * y1) ** 2 / cvar + math.log(2 * math.pi) + math.log(cvar))
    assert res.block_first == pytest.approx(first, rel=1e-14)
    assert res.total == pytest.approx(first + second, rel=1e-14)


def test_deterministic_repeat(vg):
    z = load("ll_n3000_m60_nu15")
    data, plan, spec = _plan_from_golden(vg, z)
    a = vg.vecchia_loglik(data, plan, spec)
    b = vg.vecchia_loglik(data, plan, spec)
    assert a.total == b.total
    np.testing.assert_array_equal(a.block_rest, b.block_rest)


# ---------------------------------------------------------------- kernels

@pytest.mark.parametrize("nu", [0.5, 1.5, 2.5, 0.05, 0.3, 0.8, 1.0, 1.2, 2.3, 3.7, 5.0])
def test_cov_matches_scipy_reference_formula(vg, oracle, nu):
    d = np.concatenate([[0.0], np.geomspace(1e-8, 80.0, 400)])
    for fam in ("matern", "power_exponential"):
        p = vg.KernelParams(1.7, 0.13, nu if fam == "matern" else min(nu, 2.0))
        got = vg.kernels.cov(d, vg.KernelSpec(fam, p))
        want = oracle.cov(d, fam, p.sigma_sq, p.beta, p.nu)
        tol = 1e-12 if (fam != "matern" or nu in (0.5, 1.5, 2.5)) else 1e-11
        scale = np.maximum(np.abs(want), 1e-300)
        assert np.max(np.abs(got - want) / scale) <= tol, (fam, nu)


@pytest.mark.parametrize("nu", [0.0, 0.1, 0.5, 0.9, 1.5, 2.0, 2.5, 3.3, 4.9])
def test_bessel_kv_vs_scipy(vg, nu):
    from scipy.special import kv

    x = np.geomspace(1e-6, 650.0, 500)
    got = vg.bessel_kv(nu, x)
    want = kv(nu, x)
    assert np.max(np.abs(got - want) / want) <= 1e-12


# ---------------------------------------------------------------- batched LA

def test_batch_ops_match_oracle(vg, oracle):
    rng = np.random.default_rng(3)
    count, dim = 300, 17
    a = rng.standard_normal((count, dim, dim))
    spd = a @ np.transpose(a, (0, 2, 1)) + dim * np.eye(dim)
    batch = vg.StridedMatrixBatch.from_matrices(spd)
    vg.batch_potrf(batch)
    ref = spd.copy()
    assert oracle._potrf_sweep(ref) is None
    np.testing.assert_allclose(np.tril(batch.mats), np.tril(ref), rtol=1e-13, atol=1e-13)
    b = vg.StridedVectorBatch.from_vectors(rng.standard_normal((count, dim)))
    x = vg.batch_trsv(batch, b)
    np.testing.assert_allclose(x.vecs, oracle._trsv(ref, b.vecs.copy()), rtol=1e-12, atol=1e-12)
    d = vg.batch_dot(x, b)
    np.testing.assert_array_equal(d.values, oracle._dot(x.vecs, b.vecs))


def test_batch_potrf_npd_index(vg):
    mats = np.stack([np.eye(4)] * 5)
    mats[3, 2, 2] = -1.0
    with pytest.raises(vg.NonPositiveDefiniteError) as err:
        vg.batch_potrf(vg.StridedMatrixBatch.from_matrices(mats))
    assert err.value.batch_index == 3


# ---------------------------------------------------------------- MLE

def test_c1_mle_matches_reference(vg):
    z = load("c1_n20000_m30_nu05")
    if "mle_theta" not in z.files:
        pytest.skip("golden file generated without --with-mle")
    data = vg.Dataset(z["locs"], z["obs"])
    cfg = vg.FitConfig(objective="vecchia", m=30, ordering="random", seed=0,
                       init=vg.KernelParams(0.5, 0.05, 0.5))
    fr = vg.mle_estimate(data, cfg)
    th = z["mle_theta"]
    assert rel(fr.theta_hat.sigma_sq, float(th[0])) <= 1e-4
    assert rel(fr.theta_hat.beta, float(th[1])) <= 1e-4
    assert fr.theta_hat.nu == 0.5
    assert rel(fr.loglik, float(z["mle_loglik"])) <= 1e-9


@pytest.mark.parametrize("name", golden_names("mle_freenu"))
def test_free_nu_mle_matches_reference(vg, name):
    """BASELINE config 5's estimator: (sigma^2, beta, nu) with free_nu
    (vg/fit.py:153-157), general-nu Matérn on the device Bessel K path,
    against the reference's own mle_estimate on the same data."""
    z = load(name)
    data = vg.Dataset(z["locs"], z["obs"])
    cfg = vg.FitConfig(objective="vecchia", m=int(z["m"]), ordering="random", seed=0,
                       init=vg.KernelParams(*[float(v) for v in z["init"]]), free_nu=True)
    fr = vg.mle_estimate(data, cfg)
    th = z["mle_theta"]
    got = (fr.theta_hat.sigma_sq, fr.theta_hat.beta, fr.theta_hat.nu)
    for g, r in zip(got, th):
        assert rel(g, float(r)) <= 1e-4
    assert rel(fr.loglik, float(z["mle_loglik"])) <= 1e-9
    assert fr.converged == bool(z["mle_converged"])


@pytest.mark.parametrize("name", ["ll_n3000_m60_nu15", "ll_n2000_m30_nu15", "ll_n2000_m40_nu05_s2",
                                  "ll_n1000_m20_nu25", "ll_n300_m10_nu05"])
def test_distance_cache_is_bit_identical(vg, name):
    """The plan-time distance cache stores exactly the distances the fused
    kernel computes on the fly: cached and uncached evaluations agree bit
    for bit."""
    z = load(name)
    data, plan, spec = _plan_from_golden(vg, z)
    dp = plan.device_plan()
    dp.set_variant(4)  # warp-specialised kernel streaming the cache
    a = vg.vecchia_loglik(data, plan, spec)
    cached = dp.info()[8] == 1
    dp.set_variant(8)
    f = vg.vecchia_loglik(data, plan, spec)
    dp.set_variant(7)
    g = vg.vecchia_loglik(data, plan, spec)
    dp.set_variant(12)
    h = vg.vecchia_loglik(data, plan, spec)
    dp.set_variant(11)
    k = vg.vecchia_loglik(data, plan, spec)
    dp.set_variant(-1)
    assert cached
    assert h.total == k.total
    np.testing.assert_array_equal(h.block_rest, k.block_rest)
    assert f.total == g.total
    np.testing.assert_array_equal(f.block_rest, g.block_rest)
    assert abs(a.total - f.total) <= 1e-12 * abs(f.total)


def test_distance_cache_rebuilt_when_locations_change(vg, oracle):
    z = load("ll_n3000_m60_nu15")
    data, plan, spec = _plan_from_golden(vg, z)
    vg.vecchia_loglik(data, plan, spec)
    moved = vg.Dataset(z["locs"] * 1.01, z["obs"])
    got = vg.vecchia_loglik(moved, plan, spec).total
    ordered = moved.permute(plan.permutation)
    ref = oracle.loglik(ordered.locations, ordered.observations, int(z["m"]), z["table"], "matern",
                        *[float(v) for v in z["theta"]])
    assert rel(got, ref.total) <= TOL_TOTAL
    # back to the original locations (speculation misses, cache rebuilt),
    # then new observations only (speculation hits): each equals the
    # separate upload + evaluation bit for bit
    dp = plan.device_plan()
    for ds in (data, vg.Dataset(z["locs"], z["obs"][::-1].copy())):
        fused = vg.vecchia_loglik(ds, plan, spec)
        dp.set_data(ds)
        sep = dp.loglik(spec)
        assert fused.total == sep.total
        np.testing.assert_array_equal(fused.block_rest, sep.block_rest)


@pytest.mark.parametrize("m,variant", [(30, -1), (90, -1)])
def test_chunked_result_download_vs_oracle(vg, oracle, m, variant):
    """n - m >= 65536 blocks: the main launch is split into chunks whose
    per-block results download while later chunks compute, from page-locked
    dataset arrays; every block's log-density, mu and sigma must match the
    oracle and the total must equal block_first + _ordered_sum(block_rest)."""
    n, seed, beta = 70000, 21, 0.05
    rng = np.random.default_rng(seed)
    locs = rng.random((n, 2))
    data = vg.Dataset(locs, np.zeros(n))
    plan = vg.make_plan(data, m, "random", seed=seed)
    y_ord = oracle.simulate_vecchia(locs[plan.permutation.order], m, plan.neighbors.neighbors,
                                    "matern", 1.0, beta, 1.5, seed + 100)
    y = np.empty(n)
    y[plan.permutation.order] = y_ord
    data = vg.Dataset(locs, y)
    spec = vg.KernelSpec("matern", vg.KernelParams(1.0, beta, 1.5))
    ordered = data.permute(plan.permutation)
    ref = oracle.loglik(ordered.locations, ordered.observations, m, plan.neighbors.neighbors,
                        "matern", 1.0, beta, 1.5)
    plan.device_plan().set_variant(variant)
    res = vg.vecchia_loglik(data, plan, spec)
    res2 = vg.vecchia_loglik(data, plan, spec)  # page-locked upload path on the second call
    assert res.total == res2.total
    np.testing.assert_array_equal(res.block_rest, res2.block_rest)
    assert rel(res.total, ref.total) <= TOL_TOTAL
    assert res.total == res.block_first + vg.vecchia._ordered_sum(res.block_rest)
    # every block present and in place: 99.9 % of the per-block terms agree to
    # 1e-9; ill-conditioned blocks amplify ulp-level differences, all to 1e-5
    err = np.abs(res.block_rest - ref.block_rest) / np.maximum(np.abs(ref.block_rest), 1.0)
    assert np.quantile(err, 0.999) <= 1e-9 and err.max() <= 1e-5
    np.testing.assert_allclose(res.mu_new, ref.mu_new, rtol=1e-5, atol=1e-6)
    np.testing.assert_allclose(res.sigma_new, ref.sigma_new, rtol=1e-5, atol=1e-12)
    assert res.total == plan.device_plan().total(spec)


@pytest.mark.parametrize("name", golden_names("krige_"))
def test_krige_vs_reference_golden(vg, name):
    """fit.krige_predict on the GPU against the reference's own output
    (tests/golden/make_golden.py krige_cases): same neighbour sets (bit-exact
    kNN), predictions to 1e-10 (1e-8 for m = n_train, where the reference
    switches to its dense path), variances, held-out MSE."""
    z = load(name)
    train = vg.Dataset(z["train"], z["y"], _metric(vg, z))
    s2, beta, nu = (float(v) for v in z["theta"])
    m = int(z["m"])
    rep = vg.krige_predict(train, vg.KernelParams(s2, beta, nu), str(z["family"]), z["test"], m,
                           z["truth"])
    atol = 1e-8 if m == train.n else 1e-10
    np.testing.assert_allclose(rep.predictions, z["pred"], rtol=0, atol=atol)
    np.testing.assert_allclose(rep.variances, z["var"], rtol=1e-7, atol=atol)
    assert rel(rep.mse, float(z["mse"])) <= 1e-6


def test_krige_reference_properties(vg):
    """pkg/tests/test_fit.py:179-221: a coincident point reproduces its
    value, a far point shrinks to the mean with the sill as variance,
    variances are positive and below the sill."""
    z = load("krige_n300_m40_nu05")
    train = vg.Dataset(z["train"], z["y"])
    theta = vg.KernelParams(1.0, 0.078809, 0.5)
    rep = vg.krige_predict(train, theta, "matern", train.locations[5:6], m=1)
    assert rep.predictions[0] == pytest.approx(train.observations[5], rel=1e-12)
    far = vg.krige_predict(train, theta, "matern", np.array([[60.0, 60.0]]), m=30)
    assert abs(far.predictions[0]) <= 1e-6
    assert far.variances[0] == pytest.approx(1.0, abs=1e-6)
    rep = vg.krige_predict(train, theta, "matern", z["test"], m=40)
    assert np.all(rep.variances > 0.0) and np.all(rep.variances <= 1.0 + 1e-12)


@pytest.mark.parametrize("world", [2, 3, 8])
@pytest.mark.parametrize("m,variant", [(30, -1), (60, 7), (90, -1)])
def test_sharded_partials_bitwise_on_one_gpu(vg, oracle, world, m, variant):
    """The multi-GPU path with its collective emulated on one device: every
    rank's shard plan (DevicePlan over shard_blocks' range, its own neighbour
    rows and distance cache) writes its chunk partials into its slots of the
    global vector; summing the rank vectors (what the NCCL all-reduce does)
    and the ordered host sum must reproduce the single-plan total bit for bit
    — kernels run on block ranges that start mid-table (rest_lo > 0)."""
    import torch

    from paper_2403_07412_b200.distributed import n_chunks, ordered_total, shard_blocks

    n, seed, beta = 40000, 31, 0.05
    rng = np.random.default_rng(seed)
    locs = rng.random((n, 2))
    data = vg.Dataset(locs, np.zeros(n))
    plan = vg.make_plan(data, m, "random", seed=seed)
    y_ord = oracle.simulate_vecchia(locs[plan.permutation.order], m, plan.neighbors.neighbors,
                                    "matern", 1.0, beta, 1.5, seed + 100)
    y = np.empty(n)
    y[plan.permutation.order] = y_ord
    data = vg.Dataset(locs, y)
    spec = vg.KernelSpec("matern", vg.KernelParams(1.0, beta, 1.5))
    full = vg.vecchia_loglik(data, plan, spec)
    nvec = 1 + n_chunks(n, m)
    acc = torch.zeros(nvec, dtype=torch.float64, device="cuda")
    for r in range(world):
        lo, hi = shard_blocks(n, m, r, world)
        if hi <= lo:
            continue
        dp = vg.DevicePlan(plan, block_lo=lo, block_hi=hi)
        dp.set_data(data)
        dp.set_variant(variant)
        send = torch.zeros(nvec, dtype=torch.float64, device="cuda")
        dp.partials_device(spec, send.data_ptr())
        torch.cuda.synchronize()
        acc += send
        dp.close()
    assert ordered_total(acc.cpu().numpy()) == full.total


# ---------------------------------------------------------------- maxmin ordering (config 5)

def _clustered(rng, n, k=12, scale=0.02):
    centers = rng.random((k, 2))
    lab = rng.integers(0, k, n)
    return centers[lab] + scale * rng.standard_normal((n, 2))


@pytest.mark.parametrize("case", ["uniform", "clustered", "lattice", "duplicates", "tiny1", "tiny2",
                                  "collinear", "uniform_big"])
def test_maxmin_order_vs_oracle(vg, oracle, case):
    """Exact maxmin (new: no reference counterpart) against the brute-force
    restatement with the same arithmetic; bit-exact permutation, including
    the tie-heavy lattice and duplicate points."""
    rng = np.random.default_rng(hash(case) % 1000)
    if case == "uniform":
        locs = rng.random((3000, 2))
    elif case == "clustered":
        locs = _clustered(rng, 6000)
    elif case == "lattice":
        g = np.arange(70, dtype=np.float64)
        locs = np.stack(np.meshgrid(g, g, indexing="ij"), -1).reshape(-1, 2)
    elif case == "duplicates":
        base = rng.random((500, 2))
        locs = base[rng.integers(0, 500, 4000)]
    elif case == "tiny1":
        locs = rng.random((1, 2))
    elif case == "tiny2":
        locs = rng.random((2, 2))
    elif case == "collinear":
        locs = np.stack([rng.random(2500), np.full(2500, 0.25)], -1)
    else:
        locs = rng.random((20000, 2))
    perm = vg.geo.maxmin_ordering(locs)
    want = oracle.maxmin_order(locs, vg.geo.maxmin_first(locs))
    np.testing.assert_array_equal(perm.order, want)


def test_maxmin_plan_end_to_end(vg, oracle):
    """Config-5 shape at test size: clustered locations, maxmin ordering,
    GPU kNN, fused likelihood vs the oracle at 1e-9."""
    rng = np.random.default_rng(5)
    n, m, nu, beta = 20000, 30, 0.8, 0.05
    locs = _clustered(rng, n)
    plan = vg.make_plan(vg.Dataset(locs, np.zeros(n)), m, "maxmin")
    assert plan.ordering == "maxmin"
    np.testing.assert_array_equal(plan.permutation.order,
                                  oracle.maxmin_order(locs, vg.geo.maxmin_first(locs)))
    y = rng.standard_normal(n)
    data = vg.Dataset(locs, y)
    ordered = data.permute(plan.permutation)
    ref = oracle.loglik(ordered.locations, ordered.observations, m, plan.neighbors.neighbors,
                        "matern", 1.0, beta, nu)
    res = vg.vecchia_loglik(data, plan, vg.KernelSpec("matern", vg.KernelParams(1.0, beta, nu)))
    assert ref.status == 0
    assert rel(res.total, ref.total) <= TOL_TOTAL


def test_maxmin_large_is_permutation_and_monotone(vg):
    """n = 500k (beyond the oracle): a permutation whose selection distances
    (squared distance of order[t] to order[:t], checked on a sample of t via
    the exact predecessor kNN with m = 1) never increase."""
    rng = np.random.default_rng(9)
    n = 500_000
    locs = _clustered(rng, n, k=40, scale=0.05)
    order = vg.geo.maxmin_ordering(locs).order
    assert np.array_equal(np.sort(order), np.arange(n))
    ordered = locs[order]
    nn = vg.geo.nearest_neighbors(vg.Dataset(ordered, np.zeros(n)), 1).neighbors[:, 0]
    d = ((ordered[1:] - ordered[nn]) ** 2).sum(1)
    assert np.all(np.diff(d) <= 1e-12 * d[:-1] + 1e-300)


# ---------------------------------------------------------------- grid-pruned kNN

def _grid_knn(vg, monkeypatch, locs, m, grid):
    monkeypatch.setenv("VGP_KNN_GRID_MIN", "0" if grid else str(1 << 40))
    return vg.nearest_neighbors(vg.Dataset(locs, np.zeros(len(locs))), m).neighbors


@pytest.mark.parametrize("case,m", [("uniform", 30), ("clustered_dups", 60), ("lattice", 10),
                                    ("lattice", 45), ("collinear", 20), ("two_points_spread", 7)])
def test_grid_knn_bit_exact(vg, oracle, monkeypatch, case, m):
    """The index-batched grid search returns the brute-force table bit for
    bit (ties by index included) on tie-heavy and degenerate layouts."""
    rng = np.random.default_rng(len(case) * 7 + m)
    if case == "uniform":
        locs = rng.random((20000, 2))
    elif case == "clustered_dups":
        c = rng.random((30, 2))
        locs = c[rng.integers(0, 30, 30000)] + 0.01 * rng.standard_normal((30000, 2))
        dup = np.arange(0, len(locs), 7)
        locs[dup] = locs[(dup + 3) % len(locs)]
    elif case == "lattice":
        g = np.arange(70, dtype=np.float64)
        locs = np.stack(np.meshgrid(g, g, indexing="ij"), -1).reshape(-1, 2)
        locs = locs[rng.permutation(len(locs))]
    elif case == "collinear":
        locs = np.stack([rng.random(8000), np.full(8000, 0.5)], -1)
    else:
        locs = np.concatenate([rng.random((3000, 2)) * 1e-6, 1e6 + rng.random((3000, 2))])
        locs = locs[rng.permutation(len(locs))]
    grid = _grid_knn(vg, monkeypatch, locs, m, True)
    brute = _grid_knn(vg, monkeypatch, locs, m, False)
    np.testing.assert_array_equal(grid, brute)
    if len(locs) <= 20000:
        np.testing.assert_array_equal(grid, oracle.knn_pred(locs, m))


@pytest.mark.parametrize("name", [n for n in golden_names("knn_") if "sphere" not in n and "points" not in n])
def test_grid_knn_vs_reference_golden(vg, monkeypatch, name):
    z = load(name)
    monkeypatch.setenv("VGP_KNN_GRID_MIN", "0")
    t = vg.nearest_neighbors(vg.Dataset(z["locs"], np.zeros(len(z["locs"]))), int(z["m"])).neighbors
    np.testing.assert_array_equal(t, z["table"])


def test_grid_knn_large_matches_brute_force(vg, monkeypatch):
    rng = np.random.default_rng(77)
    locs = rng.random((500_000, 2))
    np.testing.assert_array_equal(_grid_knn(vg, monkeypatch, locs, 60, True),
                                  _grid_knn(vg, monkeypatch, locs, 60, False))


@pytest.mark.parametrize("case,m", [("global", 30), ("polar", 20), ("dateline", 12), ("dups", 40)])
def test_sphere_grid_knn_bit_exact(vg, monkeypatch, case, m):
    """Great-circle grid search (unit-vector cube grid, chord bound) equals
    the sphere brute-force kernel bit for bit."""
    rng = np.random.default_rng(len(case) + m)
    n = 30000
    if case == "global":
        lon, lat = rng.uniform(-180, 180, n), np.degrees(np.arcsin(rng.uniform(-1, 1, n)))
    elif case == "polar":
        lon, lat = rng.uniform(-180, 180, n), rng.uniform(88.0, 90.0, n)
    elif case == "dateline":
        lon = np.where(rng.random(n) < 0.5, rng.uniform(179.0, 180.0, n), rng.uniform(-180.0, -179.0, n))
        lat = rng.uniform(-5, 5, n)
    else:
        lon, lat = rng.uniform(-20, 20, n), rng.uniform(30, 50, n)
        dup = np.arange(0, n, 5)
        lon[dup], lat[dup] = lon[(dup + 2) % n], lat[(dup + 2) % n]
    locs = np.stack([lon, lat], -1)
    gc = vg.GreatCircle()

    def table(grid):
        monkeypatch.setenv("VGP_KNN_GRID_MIN", "0" if grid else str(1 << 40))
        return vg.nearest_neighbors(vg.Dataset(locs, np.zeros(n), gc), m).neighbors

    np.testing.assert_array_equal(table(True), table(False))


@pytest.mark.parametrize("name", golden_names("knn_sphere_big"))
@pytest.mark.parametrize("grid", [True, False])
def test_sphere_knn_at_scale_vs_reference(vg, monkeypatch, name, grid):
    """Great-circle neighbour tables at 30-100k points (global; dense 2- and
    4-degree patches with many near-ties, 100k points ~1.4 km apart) against
    the reference's own tables (glibc sin
    keys, vg/geo.py:266-292), by sha256 of the whole table: the device key
    (CUDA sin) decides the same top-m sets."""
    import hashlib

    z = load(name)
    monkeypatch.setenv("VGP_KNN_GRID_MIN", "0" if grid else str(1 << 40))
    t = vg.nearest_neighbors(vg.Dataset(z["locs"], np.zeros(len(z["locs"])), vg.GreatCircle()),
                             int(z["m"])).neighbors
    np.testing.assert_array_equal(t[:500], z["table_head"])
    assert hashlib.sha256(np.ascontiguousarray(t, dtype=np.int64).tobytes()).hexdigest() == str(z["table_sha256"])


@pytest.mark.parametrize("name", [n for n in golden_names("knn_sphere") if "points" not in n and "big" not in n])
def test_sphere_grid_knn_vs_reference_golden(vg, monkeypatch, name):
    z = load(name)
    monkeypatch.setenv("VGP_KNN_GRID_MIN", "0")
    t = vg.nearest_neighbors(vg.Dataset(z["locs"], np.zeros(len(z["locs"])), vg.GreatCircle()),
                             int(z["m"])).neighbors
    np.testing.assert_array_equal(t, z["table"])


def test_sphere_grid_knn_large(vg, monkeypatch):
    rng = np.random.default_rng(123)
    n = 300_000
    locs = np.stack([rng.uniform(-180, 180, n), np.degrees(np.arcsin(rng.uniform(-1, 1, n)))], -1)
    gc = vg.GreatCircle()
    out = []
    for grid in (True, False):
        monkeypatch.setenv("VGP_KNN_GRID_MIN", "0" if grid else str(1 << 40))
        out.append(vg.nearest_neighbors(vg.Dataset(locs, np.zeros(n), gc), 30).neighbors)
    np.testing.assert_array_equal(out[0], out[1])


@pytest.mark.parametrize("m,nu", [(1, 0.5), (3, 1.5), (7, 2.5), (10, 1.5), (11, 0.5), (12, 1.5), (12, 2.5)])
def test_thread_per_block_vs_oracle(vg, oracle, m, nu):
    """Variant 13 (one thread per block, m <= 12) on model-consistent data:
    totals at 1e-9 and per-block terms against the oracle."""
    rng = np.random.default_rng(100 + m)
    n, beta = 6000, 0.06
    locs = rng.random((n, 2))
    plan = vg.make_plan(vg.Dataset(locs, np.zeros(n)), m, "random", seed=m)
    y_ord = oracle.simulate_vecchia(locs[plan.permutation.order], m, plan.neighbors.neighbors,
                                    "matern", 1.0, beta, nu, 7)
    y = np.empty(n)
    y[plan.permutation.order] = y_ord
    data = vg.Dataset(locs, y)
    plan.device_plan().set_variant(13)
    res = vg.vecchia_loglik(data, plan, vg.KernelSpec("matern", vg.KernelParams(1.0, beta, nu)))
    assert plan.device_plan().kernel_variant == 13
    ordered = data.permute(plan.permutation)
    ref = oracle.loglik(ordered.locations, ordered.observations, m, plan.neighbors.neighbors,
                        "matern", 1.0, beta, nu)
    assert rel(res.total, ref.total) <= TOL_TOTAL
    # per-block terms: a few ill-conditioned blocks (smooth nu = 2.5, many
    # neighbours) amplify ulp-level differences; same criterion as the
    # chunked-download test
    d = np.abs(res.block_rest - ref.block_rest) / np.maximum(1.0, np.abs(ref.block_rest))
    assert np.quantile(d, 0.999) <= 1e-7
    assert d.max() <= 1e-5
    plan.device_plan().set_variant(-1)


def test_thread_per_block_reports_a_singular_block(vg):
    """A duplicated point makes every block holding both copies exactly
    singular; which of them first rounds a pivot to <= 0 depends on the
    operation order, so the check is that the reported block is one of them."""
    rng = np.random.default_rng(5)
    locs = rng.random((3000, 2))
    locs[1700] = locs[1699]
    data = vg.Dataset(locs, rng.standard_normal(3000))
    m = 8
    plan = vg.make_plan(data, m, "identity")
    spec = vg.KernelSpec("matern", vg.KernelParams(1.0, 0.1, 0.5))
    plan.device_plan().set_variant(13)
    with pytest.raises(vg.LikelihoodEvaluationError) as ei:
        vg.vecchia_loglik(data, plan, spec)
    plan.device_plan().set_variant(-1)
    e = ei.value.block_index
    members = set(plan.neighbors.neighbors[e - 1].tolist()) | {m + e - 1}
    assert {1699, 1700} <= members


# ---------------------------------------------------------------- acceptance C1

def _c1_configs():
    # pkg/tests/test_acceptance.py:43-55: the reference's 20 full-conditioning configs
    configs = []
    for n in (50, 200, 512):
        for nu in (0.5, 1.5, 2.5):
            for ordering in ("random", "morton"):
                configs.append((n, nu, ordering, 1000 + n))
    configs += [(512, 0.5, "random", 77), (512, 0.5, "morton", 78)]
    return configs[:20]


@pytest.mark.parametrize("n,nu,ordering,seed", _c1_configs())
def test_acceptance_c1_full_conditioning_equals_dense(vg, oracle, n, nu, ordering, seed):
    """Reference acceptance criterion 1 (pkg/tests/test_acceptance.py:43-70) on
    the GPU: with m = n - 1 the Vecchia likelihood IS the dense one, to 1e-8
    relative, for the reference's 20 configurations (up to m = 511, nu = 2.5)."""
    spec = vg.KernelSpec("matern", vg.KernelParams(1.0, 0.1, nu))
    rng = np.random.default_rng(seed)
    locs = rng.random((n, 2))
    y = vg.simulate_grf(locs, spec, seed + 1)
    data = vg.Dataset(locs, y)
    plan = vg.make_plan(data, n - 1, ordering, seed=seed + 2)
    approx = vg.vecchia_loglik(data, plan, spec).total
    reference = oracle.exact_loglik(locs, y, "matern", 1.0, 0.1, nu)
    assert rel(approx, reference) <= 1e-8


# ---------------------------------------------------------------- shard plans (multi-GPU, one device)

@pytest.mark.parametrize("world", [2, 3])
def test_shard_plans_bitwise_on_one_gpu(vg, oracle, world):
    """Each rank's ShardPlan (ordering everywhere, kNN only for its own target
    rows: vgp_knn_predecessors_range + vgp_plan_create_shard) gives the same
    neighbour rows as the full table and the same chunk partials, so the
    ordered total equals the single-GPU total bit for bit."""
    from paper_2403_07412_b200.distributed import make_shard_plan, n_chunks, ordered_total

    n, m = 30000, 30
    locs = np.random.default_rng(31).random((n, 2))
    plan = vg.make_plan(vg.Dataset(locs, np.zeros(n)), m, "random", seed=0)
    spec = vg.KernelSpec("matern", vg.KernelParams(1.0, 0.05, 1.5))
    y = vg.simulate_vecchia(vg.Dataset(locs, np.zeros(n)), plan, spec, 3)
    data = vg.Dataset(locs, y)
    full = vg.vecchia_loglik(data, plan, spec)
    vec = np.zeros(1 + n_chunks(n, m))
    for r in range(world):
        sp = make_shard_plan(data, m, "random", 0, r, world)
        np.testing.assert_array_equal(sp.neighbors.neighbors,
                                      plan.neighbors.neighbors[sp.row_lo:sp.row_hi])
        lo, hi = max(sp.row_lo + 1, 0 if r == 0 else 1), sp.row_hi + 1
        lo = 0 if r == 0 else lo
        dp = vg.vecchia.DevicePlan(sp, block_lo=lo, block_hi=hi)
        dp.set_data(data)
        parts, bf, st, _ = dp.partials(spec)
        assert st == 0
        vec[1 + dp.chunk_lo:1 + dp.chunk_lo + dp.nchunks] = parts
        if r == 0:
            vec[0] = bf
        dp.close()
    assert ordered_total(vec) == full.total


@pytest.mark.parametrize("m,nu", [(55, 0.5), (58, 1.5), (60, 2.5), (60, 1.5), (62, 0.5)])
def test_chain_column0_layout_bitwise(vg, oracle, monkeypatch, m, nu):
    """The m + 2 <= 64 kernel's default layout, where the chain generates tile
    column 0 itself (C0), returns the same bits as the previous layout
    (VGP_TUNE=1: the worker generates every column), including the per-block
    arrays, and matches the oracle; several slots' blocks per CTA (n >> 8 x 148)."""
    rng = np.random.default_rng(m)
    n = 4000
    locs = rng.random((n, 2))
    spec = vg.KernelSpec("matern", vg.KernelParams(1.3, 0.07, nu))
    # model-consistent observations: the oracle gate is 1e-9
    plan = vg.make_plan(vg.Dataset(locs, np.zeros(n)), m, "random", seed=3)
    y_ord = oracle.simulate_vecchia(locs[plan.permutation.order], m, plan.neighbors.neighbors,
                                    "matern", 1.3, 0.07, nu, m + 7)
    y = np.empty(n)
    y[plan.permutation.order] = y_ord
    data = vg.Dataset(locs, y)
    res = {}
    for tune in ("0", "1"):
        monkeypatch.setenv("VGP_TUNE", tune)
        plan = vg.make_plan(data, m, "random", seed=3)
        dp = plan.device_plan()
        dp.set_variant(8)
        res[tune] = vg.vecchia_loglik(data, plan, spec)
        assert dp.info()[8] == 1  # the distance cache is streamed (the C0 path)
    monkeypatch.delenv("VGP_TUNE")
    assert res["0"].total == res["1"].total
    np.testing.assert_array_equal(res["0"].block_rest, res["1"].block_rest)
    ordered = data.permute(plan.permutation)
    ref = oracle.loglik(ordered.locations, ordered.observations, m, plan.neighbors.neighbors,
                        "matern", 1.3, 0.07, nu)
    assert rel(res["0"].total, ref.total) <= TOL_TOTAL
