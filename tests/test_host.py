"""CPU: host-side logic of the drop-in package (containers, orderings, the
unchanged Nelder-Mead loop, flop model), restating the reference's own unit
tests (pkg/tests/test_geo.py, test_fit.py, test_vecchia.py)."""

import math

import numpy as np
import pytest

import paper_2403_07412_b200 as vg
from paper_2403_07412_b200 import fit, geo, vecchia


class TestContainers:
    def test_dataset_validation(self):
        with pytest.raises(ValueError):
            vg.Dataset(np.zeros((3, 3)), np.zeros(3))
        with pytest.raises(ValueError):
            vg.Dataset(np.zeros((3, 2)), np.zeros(2))
        with pytest.raises(ValueError):
            vg.Dataset(np.array([[np.nan, 0.0]]), np.zeros(1))
        with pytest.raises(ValueError):
            vg.Dataset(np.array([[0.0, 95.0]]), np.zeros(1), vg.GreatCircle())

    def test_permutation_bijection(self):
        with pytest.raises(ValueError):
            vg.Permutation(np.array([0, 0, 1]))
        p = vg.Permutation(np.array([2, 0, 1]))
        assert p.n == 3 and p.order.dtype == np.int64

    def test_plan_shape_check(self):
        perm = vg.Permutation(np.arange(5))
        with pytest.raises(ValueError):
            vg.VecchiaPlan(2, perm, vg.NeighborTable(2, np.zeros((2, 2), dtype=np.int64)), vg.Euclidean())

    def test_kernel_params_validation(self):
        with pytest.raises(ValueError):
            vg.KernelParams(0.0, 1.0, 0.5)
        with pytest.raises(ValueError):
            vg.KernelSpec("gaussian", vg.KernelParams(1.0, 1.0, 0.5))

    def test_beta_table_verbatim(self):
        assert vg.beta_from_effective_range(0.3, 1.5) == 0.052537
        assert vg.EFFECTIVE_RANGE_BETA[(0.3, 2.5)] == vg.EFFECTIVE_RANGE_BETA[(0.1, 2.5)]
        with pytest.raises(KeyError):
            vg.beta_from_effective_range(0.5, 0.5)


class TestOrderings:
    def test_random_ordering_is_numpy_permutation(self):
        assert np.array_equal(vg.random_ordering(1000, 7).order,
                              np.random.default_rng(7).permutation(1000))

    def test_morton_bit_convention(self):
        # x on even bits, y on odd bits (vg/geo.py:199-225)
        locs = np.array([[0.0, 0.0], [1.0, 0.0], [0.0, 1.0], [1.0, 1.0]])
        codes = geo.morton_codes(locs)
        top = (1 << 16) - 1
        assert codes[1] == geo._part1by1(np.array([top]))[0]
        assert codes[2] == geo._part1by1(np.array([top]))[0] << np.uint64(1)
        assert list(vg.morton_ordering(locs).order) == [0, 1, 2, 3]

    def test_morton_stable_ties(self):
        locs = np.array([[0.5, 0.5]] * 4 + [[0.0, 0.0]])
        assert list(vg.morton_ordering(locs).order) == [4, 0, 1, 2, 3]


class TestFlopModel:
    def test_formula(self):
        assert vg.flop_count(101, 1) == pytest.approx(101 * (1.0 / 3.0 + 2.0 + 4.0))

    def test_paper_point(self):
        lead = (100000 - 60 + 1) * 60**3 / 3.0
        assert lead == pytest.approx(7.2e9, rel=1e-3)
        assert vg.flop_count(1_000_000, 60) == pytest.approx(7.9435e10, rel=1e-4)

    def test_domain(self):
        with pytest.raises(ValueError):
            vg.flop_count(10, 10)


class TestNelderMead:
    # restated from pkg/tests/test_fit.py:12-69
    def test_quadratic_maximum(self):
        f = lambda x: -((x[0] - 2.0) ** 2) - 3.0 * (x[1] + 1.0) ** 2
        x, fb, evals, conv = vg.nelder_mead_max(f, [0.0, 0.0], [(-5, 5), (-5, 5)], tol=1e-12,
                                                max_evals=2000)
        assert conv and abs(x[0] - 2.0) < 1e-4 and abs(x[1] + 1.0) < 1e-4

    def test_bounds_respected(self):
        f = lambda x: x[0] + x[1]
        x, fb, _, _ = vg.nelder_mead_max(f, [0.5, 0.5], [(0, 1), (0, 2)], max_evals=300)
        assert 0 <= x[0] <= 1 and 0 <= x[1] <= 2
        assert fb == pytest.approx(3.0, abs=1e-3)

    def test_infeasible_start(self):
        with pytest.raises(vg.EstimationError):
            vg.nelder_mead_max(lambda x: -math.inf, [0.5], [(0, 1)])

    def test_start_outside_bounds(self):
        with pytest.raises(vg.EstimationError):
            vg.nelder_mead_max(lambda x: 0.0, [2.0], [(0, 1)])

    def test_same_trajectory_as_oracle_restatement(self):
        from oracle import oracle as O

        f = lambda x: -((x[0] - 0.3) ** 2) - 2.0 * (x[1] - 0.7) ** 4 + 0.1 * x[0] * x[1]
        a = vg.nelder_mead_max(f, [0.1, 0.1], [(0, 1), (0, 1)], tol=1e-9, max_evals=300)
        b = O.nelder_mead_max(f, [0.1, 0.1], [(0, 1), (0, 1)], tol=1e-9, max_evals=300)
        assert np.array_equal(a[0], b[0]) and a[1:] == b[1:]

    def test_fit_config_validation(self):
        with pytest.raises(ValueError):
            vg.FitConfig(objective="bayes")
        with pytest.raises(ValueError):
            vg.FitConfig(bounds={"beta": (1.0, 0.5)})

    def test_m_too_large(self):
        data = vg.Dataset(np.random.default_rng(0).random((30, 2)), np.zeros(30))
        with pytest.raises(vg.EstimationError):
            vg.mle_estimate(data, vg.FitConfig(m=30))

    def test_infeasible_objective_seam(self, monkeypatch):
        # pkg/tests/test_fit.py:112-120: the module attribute is the seam; a
        # replacement that always fails must surface as EstimationError.  The
        # plan/session need a GPU, so stub them too.
        class FakeSession:
            def __init__(self, *a, **k):
                pass

            def total(self, spec):
                raise AssertionError("must not be used when the seam is patched")

            def close(self):
                pass

        def always_infeasible(*args, **kwargs):
            raise vg.LikelihoodEvaluationError(0, "forced failure")

        data = vg.Dataset(np.random.default_rng(0).random((40, 2)), np.zeros(40))
        fake_plan = object()
        monkeypatch.setattr(fit.vecchia, "make_plan", lambda *a, **k: fake_plan)
        monkeypatch.setattr(fit.vecchia, "LikelihoodSession", FakeSession)
        monkeypatch.setattr(fit.vecchia, "vecchia_loglik", always_infeasible)
        with pytest.raises(vg.EstimationError):
            vg.mle_estimate(data, vg.FitConfig(objective="vecchia", m=10))


def test_ordered_sum_matches_oracle():
    from oracle import oracle as O

    a = np.random.default_rng(2).standard_normal(50000)
    assert vecchia._ordered_sum(a) == O.ordered_sum(a)


def test_exact_objective_guard_before_device():
    """The dense objective (vg/fit.py:165-166) keeps the reference's guard:
    ValueError past max_dense_n, raised before any device work."""
    data = vg.Dataset(np.random.default_rng(0).random((40, 2)), np.zeros(40))
    with pytest.raises(ValueError):
        vg.mle_estimate(data, vg.FitConfig(objective="exact", max_dense_n=39))
    from paper_2403_07412_b200 import exact

    with pytest.raises(ValueError):
        exact.kl_gaussian(np.eye(3), np.eye(4))
    with pytest.raises(ValueError):
        exact.exact_loglik(data, vg.KernelSpec("matern", vg.KernelParams(1.0, 0.1, 0.5)), max_n=10)


def test_pin_skips_views_and_small_arrays():
    """Only arrays that own at least 1 MiB of data are page-locked (views and
    small arrays keep the pageable upload), and nothing is registered twice."""
    V = vecchia
    before = dict(V._PINNED)
    small = np.zeros(100)
    V._pin(small)
    view = np.zeros((300000, 2))[:, :1]
    V._pin(view)
    assert V._PINNED == before


class TestDetrendSqrt:
    """Restates pkg/tests/test_fit.py:126-175 (host-side data preparation)."""

    def test_plane_removed(self):
        rng = np.random.default_rng(0)
        locs = rng.random((40, 2))
        values = 1.5 - 2.0 * locs[:, 0] + 0.25 * locs[:, 1]
        res = fit.ols_detrend(geo.Dataset(locs, values))
        assert np.max(np.abs(res.observations)) <= 1e-10

    def test_residuals_orthogonal_to_design(self):
        rng = np.random.default_rng(2)
        locs = rng.random((120, 2))
        res = fit.ols_detrend(geo.Dataset(locs, rng.standard_normal(120)))
        design = np.column_stack([np.ones(120), locs[:, 0], locs[:, 1]])
        assert np.max(np.abs(design.T @ res.observations)) <= 1e-8

    def test_collinear_error(self):
        locs = np.column_stack([np.arange(5.0), 2.0 * np.arange(5.0)])
        with pytest.raises(ValueError):
            fit.ols_detrend(geo.Dataset(locs, np.arange(5.0)))

    def test_sqrt_values_and_negative(self):
        data = geo.Dataset(np.array([[0.0, 0.0], [1.0, 0.0], [0.0, 1.0]]), np.array([4.0, 0.0, 2.25]))
        np.testing.assert_allclose(fit.sqrt_transform(data).observations, [2.0, 0.0, 1.5], rtol=1e-15)
        with pytest.raises(ValueError):
            fit.sqrt_transform(geo.Dataset(np.zeros((1, 2)), np.array([-0.1])))

    def test_krige_validation_before_device(self):
        data = geo.Dataset(np.random.default_rng(1).random((10, 2)), np.zeros(10))
        theta = vg.KernelParams(1.0, 0.1, 0.5)
        with pytest.raises(ValueError):
            fit.krige_predict(data, theta, "matern", np.zeros((3, 2)), m=0)
        with pytest.raises(ValueError):
            fit.krige_predict(data, theta, "matern", np.zeros((3, 2)), m=11)
        with pytest.raises(ValueError):
            fit.krige_predict(data, theta, "matern", np.zeros((3, 3)), m=2)


class TestMaxminHost:
    """The maxmin checker (oracle) against a literal restatement of the
    definition, and the host-side pieces of the device ordering."""

    @staticmethod
    def _literal(locs, first):
        n = len(locs)
        chosen = [first]
        rest = set(range(n)) - {first}
        while rest:
            best, bi = -1.0, None
            for i in sorted(rest):
                d = min((locs[i, 0] - locs[j, 0]) * (locs[i, 0] - locs[j, 0])
                        + (locs[i, 1] - locs[j, 1]) * (locs[i, 1] - locs[j, 1]) for j in chosen)
                if d > best:
                    best, bi = d, i
            chosen.append(bi)
            rest.remove(bi)
        return np.array(chosen)

    @pytest.mark.parametrize("seed", [0, 1, 2])
    def test_oracle_matches_definition(self, seed):
        from oracle import oracle as O

        rng = np.random.default_rng(seed)
        locs = rng.random((60, 2))
        if seed == 2:  # lattice with ties and a duplicate
            g = np.arange(7.0)
            locs = np.stack(np.meshgrid(g, g, indexing="ij"), -1).reshape(-1, 2)
            locs = np.vstack([locs, locs[:3]])
        first = geo.maxmin_first(locs)
        np.testing.assert_array_equal(O.maxmin_order(locs, first), self._literal(locs, first))

    def test_first_is_nearest_centroid(self):
        locs = np.array([[0.0, 0.0], [1.0, 1.0], [0.4, 0.6], [0.6, 0.4]])
        assert geo.maxmin_first(locs) == 2  # tie between 2 and 3 -> smallest index

    def test_validation_before_device(self):
        with pytest.raises(ValueError):
            geo.maxmin_ordering(np.zeros((3, 3)))
        with pytest.raises(ValueError):
            geo.maxmin_ordering(np.array([[0.0, np.nan]]))
        with pytest.raises(ValueError):
            vecchia.make_plan(geo.Dataset(np.zeros((3, 2)), np.zeros(3), geo.GreatCircle()), 1, "maxmin")
        assert "maxmin" in vecchia.ORDERINGS


def test_result_pool_reuses_only_dead_buffers():
    """Per-block results come from a page-locked pool: a buffer is reused
    only after every array / view over it is gone."""
    import gc

    pool = vecchia._ResultPool(keep=2)
    a = pool.take(1000)
    a[:] = 1.0
    addr = a.ctypes.data
    view = a[10:]
    del a
    gc.collect()
    b = pool.take(1000)
    assert b.ctypes.data != addr  # the view still pins the first buffer
    del view
    gc.collect()
    c = pool.take(1000)
    assert c.ctypes.data == addr  # now recycled
    assert c.shape == (1000,) and c.dtype == np.float64
    assert pool.take(0).shape == (0,)


def test_plan_copy_and_pickle_drop_device_contexts():
    """the device-context cache is not part of the plan's value."""
    import copy
    import dataclasses
    import pickle

    import paper_2403_07412_b200 as vg

    n, m = 50, 5
    perm = vg.Permutation(np.arange(n))
    table = vg.NeighborTable(m=m, neighbors=np.tile(np.arange(m, dtype=np.int64), (n - m, 1)))
    plan = vg.VecchiaPlan(m, perm, table, vg.Euclidean(), "identity")
    plan._device_plans["sentinel"] = object()
    for other in (pickle.loads(pickle.dumps(plan)), copy.deepcopy(plan),
                  dataclasses.replace(plan, m=m)):
        assert other._device_plans == {}
        assert other.m == m and np.array_equal(other.neighbors.neighbors, table.neighbors)
    assert "sentinel" in plan._device_plans
