"""GPU: the unfused stage API (vecchia.assemble -> _numeric_stage ->
_reduction_stage, vg/vecchia.py:85-214) that cli.cmd_bench drives — the
reference's own assemble tests (pkg/tests/test_vecchia.py TestAssemble)
restated, the staged total against the reference golden vectors (<= 1e-9)
and against the fused kernel."""

import math

import numpy as np
import pytest

from _helpers import golden_names, load, rel

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def vg():
    import paper_2403_07412_b200 as vg

    if vg._native.device_count() == 0:
        pytest.fail("GPU tests need a CUDA device: the B200 path has no CPU fallback")
    return vg


def _m05(vg):
    return vg.KernelSpec("matern", vg.KernelParams(1.0, 0.1, 0.5))


def _random_dataset(vg, n, seed):
    rng = np.random.default_rng(seed)
    locs = rng.random((n, 2))
    return vg.Dataset(locs, vg.simulate_grf(locs, _m05(vg), seed + 1))


def _identity_plan(vg, data, m):
    perm = vg.Permutation(np.arange(data.n))
    return vg.VecchiaPlan(m, perm, vg.nearest_neighbors(data, m), data.metric, ordering="identity")


class TestAssemble:
    def test_forced_shapes_n_equals_m_plus_one(self, vg):
        data = _random_dataset(vg, 6, 0)
        plan = _identity_plan(vg, data, 5)
        ws = vg.vecchia.assemble(data, plan, _m05(vg))
        assert ws.Sigma.count == 2 and ws.Sigma.dim == 5
        order = np.argsort(plan.neighbors.neighbors[0])
        np.testing.assert_allclose(ws.Sigma.matrix(1)[np.ix_(order, order)], ws.Sigma.matrix(0), rtol=1e-15)

    def test_entries_match_scalar_kernel(self, vg):
        data = _random_dataset(vg, 5, 1)
        plan = _identity_plan(vg, data, 2)
        ws = vg.vecchia.assemble(data, plan, _m05(vg))
        locs, y = data.locations, data.observations
        np.testing.assert_array_equal(ws.v.vector(0), y[:2])
        np.testing.assert_array_equal(ws.yJ.vector(0), y[:2])
        d01 = vg.euclidean_distance(locs[0], locs[1])
        np.testing.assert_allclose(ws.Sigma.matrix(0), [[1.0, math.exp(-d01 / 0.1)], [math.exp(-d01 / 0.1), 1.0]],
                                   rtol=1e-14)
        for e in range(1, 4):
            target = 2 + e - 1
            nbrs = plan.neighbors.neighbors[e - 1]
            for a in range(2):
                d = vg.euclidean_distance(locs[target], locs[nbrs[a]])
                assert ws.v.vector(e)[a] == pytest.approx(math.exp(-d / 0.1), rel=1e-14)
                for b in range(2):
                    d_ab = vg.euclidean_distance(locs[nbrs[a]], locs[nbrs[b]])
                    assert ws.Sigma.matrix(e)[a, b] == pytest.approx(math.exp(-d_ab / 0.1), rel=1e-14)
            np.testing.assert_array_equal(ws.yJ.vector(e), y[nbrs])

    def test_sigma_diag_is_variance(self, vg):
        spec = vg.KernelSpec("matern", vg.KernelParams(3.3, 0.2, 1.5))
        data = _random_dataset(vg, 20, 2)
        ws = vg.vecchia.assemble(data, _identity_plan(vg, data, 4), spec)
        np.testing.assert_array_equal(ws.sigma_diag.values, np.full(17, 3.3))
        np.testing.assert_array_equal(np.diagonal(ws.Sigma.mats, axis1=1, axis2=2), 3.3)

    def test_size_mismatch_and_refill(self, vg):
        data = _random_dataset(vg, 10, 3)
        plan = _identity_plan(vg, data, 3)
        smaller = vg.Dataset(data.locations[:8], data.observations[:8])
        with pytest.raises(ValueError):
            vg.vecchia.assemble(smaller, plan, _m05(vg))
        ws = vg.vecchia.assemble(data, plan, _m05(vg))
        ws2 = vg.vecchia.assemble(data, plan, vg.KernelSpec("matern", vg.KernelParams(2.0, 0.1, 0.5)), out=ws)
        assert ws2 is ws
        np.testing.assert_array_equal(ws.sigma_diag.values, 2.0)


@pytest.mark.parametrize("name", [n for n in golden_names("ll_") if "fail" not in n and "full" not in n][:12])
def test_staged_total_vs_reference_golden(vg, name):
    """assemble -> _numeric_stage -> _reduction_stage on the ordered dataset
    reproduces the reference's total (<= 1e-9) and the fused kernel's."""
    z = load(name)
    gc = "metric" in z.files and str(z["metric"]) == "great_circle"
    metric = vg.GreatCircle() if gc else vg.Euclidean()
    data = vg.Dataset(z["locs"], z["obs"], metric)
    plan = vg.VecchiaPlan(int(z["m"]), vg.Permutation(z["perm"]), vg.NeighborTable(int(z["m"]), z["table"]),
                          metric, str(z["ordering"]))
    spec = vg.KernelSpec(str(z["family"]), vg.KernelParams(*[float(t) for t in z["theta"]]))
    ordered = data.permute(plan.permutation)
    ws = vg.vecchia.assemble(ordered, plan, spec)
    lower, mu_p, sig_p = vg.vecchia._numeric_stage(ws)
    res = vg.vecchia._reduction_stage(ws, ordered.observations, plan.m, lower, mu_p, sig_p)
    assert rel(res.total, float(z["total"])) <= 1e-9
    fused = vg.vecchia_loglik(data, plan, spec)
    assert rel(res.total, fused.total) <= 1e-9
    np.testing.assert_allclose(res.block_rest, fused.block_rest, rtol=1e-7, atol=1e-7)


def test_staged_npd_maps_to_likelihood_error(vg):
    locs = np.array([[0.1, 0.1], [0.1, 0.1], [0.5, 0.2], [0.3, 0.9]])
    data = vg.Dataset(locs, np.zeros(4))
    plan = _identity_plan(vg, data, 2)
    ws = vg.vecchia.assemble(data, plan, _m05(vg))
    with pytest.raises(vg.LikelihoodEvaluationError):
        vg.vecchia._numeric_stage(ws)
