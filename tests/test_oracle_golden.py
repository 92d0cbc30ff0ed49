"""CPU: pin the oracle (oracle/) against golden vectors produced by the
reference itself (tests/golden/make_golden.py runs /root/reference's
vecchiagp), before the oracle is trusted as the GPU parity checker."""

import hashlib

import numpy as np
import pytest

from _helpers import golden_names, load, rel
from oracle import oracle as O


@pytest.mark.parametrize("name", [n for n in golden_names("knn_") if "sphere" not in n])
def test_oracle_knn_matches_reference(name):
    # great-circle neighbour sets (knn_sphere_*) are pinned directly against
    # the reference's golden on the GPU (tests/test_gpu_parity.py)
    z = load(name)
    m = int(z["m"])
    if "query" in z.files:
        got = O.knn_points(z["query"], z["train"], m)
    else:
        got = O.knn_pred(z["locs"], m)
    np.testing.assert_array_equal(got, z["table"])


def test_oracle_knn_bruteforce_restatement_agrees():
    z = load("knn_grid12_8")
    np.testing.assert_array_equal(O.knn_pred_bruteforce(z["locs"], 8), z["table"])
    z = load("knn_dupgrid_400_12")
    np.testing.assert_array_equal(O.knn_pred_bruteforce(z["locs"], 12), z["table"])


def test_oracle_knn_thread_count_independent():
    z = load("knn_random_3000_60")
    a = O.knn_pred(z["locs"], 60, threads=1)
    b = O.knn_pred(z["locs"], 60, threads=7)
    np.testing.assert_array_equal(a, b)


def test_oracle_c1_table_digest():
    z = load("c1_n20000_m30_nu05")
    t = O.knn_pred(z["locs"][z["perm"]], 30)
    assert hashlib.sha256(t.tobytes()).hexdigest() == str(z["table_sha256"])
    np.testing.assert_array_equal(t[:200], z["table_head"])


@pytest.mark.parametrize("name", golden_names("ll_"))
def test_oracle_loglik_matches_reference(name):
    z = load(name)
    s2, beta, nu = (float(v) for v in z["theta"])
    metric = str(z["metric"]) if "metric" in z.files else "euclidean"
    r = O.loglik(z["ordered_locs"], z["ordered_obs"], int(z["m"]), z["table"], str(z["family"]),
                 s2, beta, nu, metric=metric)
    if int(z["status"]) != 0:
        assert r.status != 0
        assert r.fail_index == int(z["fail_index"])
        return
    assert r.status == 0
    assert rel(r.total, float(z["total"])) <= 1e-12
    assert rel(r.block_first, float(z["block_first"])) <= 1e-12
    np.testing.assert_allclose(r.block_rest, z["block_rest"], rtol=1e-9, atol=1e-9)
    # the oracle keeps the reference's additivity contract bit for bit
    assert r.total == r.block_first + O.ordered_sum(r.block_rest)


@pytest.mark.parametrize("name", ["ll_n300_m10_nu05", "ll_n500_m15_nu08", "ll_n400_m12_powexp",
                                  "ll_n1000_m20_nu25"])
def test_oracle_numpy_restatement_matches_reference(name):
    z = load(name)
    s2, beta, nu = (float(v) for v in z["theta"])
    r = O.loglik_numpy(z["ordered_locs"], z["ordered_obs"], int(z["m"]), z["table"],
                       str(z["family"]), s2, beta, nu)
    assert rel(r.total, float(z["total"])) <= 1e-12


def test_oracle_full_conditioning_equals_dense():
    z = load("ll_full_n300_nu05")
    assert rel(float(z["total"]), float(z["exact"])) <= 1e-8
    s2, beta, nu = (float(v) for v in z["theta"])
    dense = O.exact_loglik(z["locs"], z["obs"], "matern", s2, beta, nu)
    assert rel(dense, float(z["exact"])) <= 1e-12


def test_pairwise_sum_is_numpys():
    rng = np.random.default_rng(5)
    for n in [0, 1, 7, 8, 9, 127, 128, 129, 1000, 4095, 4096, 4097, 10001]:
        a = rng.standard_normal(n) * 10.0 ** rng.integers(-6, 6, n)
        assert O.pairwise_sum(a) == float(np.sum(a))


def test_ordered_sum_is_reference_rule():
    rng = np.random.default_rng(6)
    a = rng.standard_normal(20000)
    partials = [float(a[lo:lo + 4096].sum()) for lo in range(0, a.size, 4096)]
    total = 0.0
    for p in partials:
        total += p
    assert O.ordered_sum(a) == total


def test_oracle_mle_c1_matches_reference():
    z = load("c1_n20000_m30_nu05")
    if "mle_theta" not in z.files:
        pytest.skip("golden file generated without --with-mle")
    perm = z["perm"]
    ol, oy = z["locs"][perm], z["obs"][perm]
    table = O.knn_pred(ol, 30)
    x, f, evals, conv = O.mle(ol, oy, 30, table, init=(0.5, 0.05, 0.5))
    th = z["mle_theta"]
    assert rel(x[0], float(th[0])) <= 1e-4 and rel(x[1], float(th[1])) <= 1e-4
    assert rel(f, float(z["mle_loglik"])) <= 1e-9
    assert evals == int(z["mle_evals"])


def test_simulate_vecchia_is_model_consistent():
    """The Vecchia forward simulation (parity fixture generator) draws from the
    Vecchia-implied Gaussian: standardized residuals are ~N(0, 1)."""
    rng = np.random.default_rng(9)
    n, m = 3000, 20
    locs = rng.random((n, 2))
    table = O.knn_pred(locs, m)
    y = O.simulate_vecchia(locs, m, table, "matern", 1.0, 0.05, 1.5, seed=3)
    r = O.loglik(locs, y, m, table, "matern", 1.0, 0.05, 1.5)
    assert r.status == 0
    z = (y[m:] - r.mu_new) / np.sqrt(r.sigma_new)
    assert abs(z.mean()) < 0.1 and abs(z.std() - 1.0) < 0.05
