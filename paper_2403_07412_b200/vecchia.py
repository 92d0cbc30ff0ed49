"""Vecchia plans and the B200 log-likelihood (mirrors ``vecchiagp.vecchia``).

``make_plan`` builds the ordering on the host and the conditioning sets on
the GPU (``geo.nearest_neighbors``).  ``vecchia_loglik`` evaluates the
ordered product of conditionals with one fused sm_100a kernel per call
(gather -> Matérn generation -> POTRF/TRSV/dots -> per-block log-density)
followed by the reference's deterministic 4096-chunk ordered reduction, so
``total == block_first + _ordered_sum(block_rest)`` holds bit for bit
(vg/vecchia.py:169-177, :213).

Device state lives in :class:`DevicePlan` (a ``vgp_plan`` handle holding the
permutation and the neighbour rows of a block range) cached on the plan
object, and :class:`LikelihoodSession` (a DevicePlan with a resident
dataset), which is what the MLE loop evaluates against.
"""

from __future__ import annotations

import ctypes
import math
import weakref
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from . import geo, kernels

LOG_2PI = math.log(2.0 * math.pi)
_REDUCE_CHUNK = 4096
ORDERINGS = ("random", "morton", "identity", "maxmin")  # maxmin: new (BASELINE config 5)


@dataclass
class VecchiaPlan:
    """Conditioning size, ordering, and neighbor table for one dataset (vg/vecchia.py:40-56)."""

    m: int
    permutation: geo.Permutation
    neighbors: geo.NeighborTable
    metric: geo.Metric
    ordering: str = "custom"
    # device contexts built from this plan, keyed by (device, metric); not
    # part of the plan's value: dropped by copy/pickle and re-validated
    # against the plan's arrays before every reuse
    _device_plans: dict = field(default_factory=dict, init=False, repr=False, compare=False)

    def __post_init__(self):
        n = self.permutation.n
        if self.m >= 1 and self.neighbors.neighbors.shape != (n - self.m, self.m):
            raise ValueError(
                f"neighbor table shape {self.neighbors.neighbors.shape} inconsistent "
                f"with n={n}, m={self.m}"
            )

    def __getstate__(self):
        state = dict(self.__dict__)
        state["_device_plans"] = {}
        return state

    def __setstate__(self, state):
        self.__dict__.update(state)
        self._device_plans = {}

    def device_plan(self, device: int | None = None, metric: geo.Metric | None = None) -> "DevicePlan":
        """Full-range device context on `device` (created once, then reused
        while m, the permutation and the neighbour table are the very objects
        it was built from).  `metric` (default: the plan's) sets the distance
        used by the likelihood kernels; the reference takes it from the
        dataset (vg/vecchia.py:143)."""
        dev = N.current_device() if device is None else int(device)
        metric = self.metric if metric is None else metric
        key = (dev,) + _metric_code(metric)
        dp = self._device_plans.get(key)
        if dp is None or dp.closed or not dp.built_from(self):
            # a stale context is released when its last reference goes
            dp = DevicePlan(self, device=dev, metric=metric)
            self._device_plans[key] = dp
        return dp


def make_ordering(dataset: geo.Dataset, ordering: str = "random", seed: int = 0) -> geo.Permutation:
    """The ordering step of make_plan (vg/vecchia.py:62-75)."""
    n = dataset.n
    if ordering not in ORDERINGS:
        raise ValueError(f"unknown ordering {ordering!r}; expected one of {ORDERINGS}")
    if ordering == "random":
        perm = geo.random_ordering(n, seed)
    elif ordering == "morton":
        perm = geo.morton_ordering(dataset.locations)
    elif ordering == "maxmin":
        if isinstance(dataset.metric, geo.GreatCircle):
            raise ValueError("maxmin ordering is Euclidean only")
        perm = geo.maxmin_ordering(dataset.locations)
    else:
        perm = geo.Permutation(np.arange(n))
    return perm


def make_plan(dataset: geo.Dataset, m: int, ordering: str = "random", seed: int = 0) -> VecchiaPlan:
    """Build the ordering and preceding-neighbor table for a dataset (vg/vecchia.py:59-82)."""
    n = dataset.n
    perm = make_ordering(dataset, ordering, seed)
    if n == 1:
        table = geo.NeighborTable(m=0, neighbors=np.empty((0, 0), dtype=np.int64))
        return VecchiaPlan(0, perm, table, dataset.metric, ordering)
    if not (1 <= m < n):
        raise ValueError(f"need 1 <= m < n, got m={m}, n={n}")
    table = geo.nearest_neighbors(dataset.permute(perm), m)
    return VecchiaPlan(m, perm, table, dataset.metric, ordering)


@dataclass
class LogLikResult:
    """Total log-likelihood plus its per-block decomposition (vg/vecchia.py:95-103)."""

    total: float
    block_first: float
    block_rest: np.ndarray
    mu_new: np.ndarray
    sigma_new: np.ndarray


def _metric_code(metric) -> tuple[int, float]:
    if isinstance(metric, geo.GreatCircle):
        return N.METRIC_GREAT_CIRCLE, float(metric.radius)
    return N.METRIC_EUCLIDEAN, geo.EARTH_RADIUS_KM


def _release(handle: int) -> None:
    if handle:
        N.lib.vgp_plan_destroy(ctypes.c_void_p(handle))


class DevicePlan:
    """A ``vgp_plan``: permutation + neighbour rows of batch entries
    [block_lo, block_hi) resident on one GPU (entry 0 = joint block)."""

    def __init__(self, plan: VecchiaPlan, device: int | None = None, block_lo: int = 0,
                 block_hi: int | None = None, metric: geo.Metric | None = None):
        n = plan.permutation.n
        m = plan.m
        if not (1 <= m < n):
            raise ValueError(f"need 1 <= m < n, got m={m}, n={n}")
        count = n - m + 1
        block_hi = count if block_hi is None else int(block_hi)
        self.device = N.current_device() if device is None else int(device)
        self.n, self.m = n, m
        self.block_lo, self.block_hi = int(block_lo), block_hi
        self.full = self.block_lo == 0 and self.block_hi == count
        metric, radius = _metric_code(plan.metric if metric is None else metric)
        # the objects this context was built from (identity, not value: a
        # plan whose arrays are replaced gets a fresh context)
        self._source = (plan.m, plan.permutation.order, plan.neighbors.neighbors)
        order = np.ascontiguousarray(plan.permutation.order, dtype=np.int64)
        table = np.ascontiguousarray(plan.neighbors.neighbors, dtype=np.int64)
        h = ctypes.c_void_p()
        rows = getattr(plan, "row_lo", None)
        if rows is not None:
            # a ShardPlan holds only the neighbour rows of its own blocks
            if (max(self.block_lo, 1) - 1, self.block_hi - 1) != (plan.row_lo, plan.row_hi):
                raise ValueError("shard plan rows do not match the block range")
            N.check(N.lib.vgp_plan_create_shard(self.device, n, m, metric, radius, N.iptr(order),
                                                N.iptr(table), self.block_lo, self.block_hi,
                                                ctypes.byref(h)))
        else:
            N.check(N.lib.vgp_plan_create(self.device, n, m, metric, radius, N.iptr(order),
                                          N.iptr(table), self.block_lo, self.block_hi,
                                          ctypes.byref(h)))
        self._h = h
        self._finalizer = weakref.finalize(self, _release, h.value)
        info = self.info()
        self.chunk_lo, self.nchunks = int(info[4]), int(info[5])
        self._data_key = None

    @property
    def closed(self) -> bool:
        return not self._finalizer.alive

    def built_from(self, plan: VecchiaPlan) -> bool:
        m, order, table = self._source
        return (m == plan.m and order is plan.permutation.order
                and table is plan.neighbors.neighbors)

    def close(self) -> None:
        self._finalizer()

    @property
    def handle(self) -> ctypes.c_void_p:
        if self.closed:
            raise ValueError("device plan is closed")
        return self._h

    def info(self) -> np.ndarray:
        out = np.zeros(9, dtype=np.int64)
        N.check(N.lib.vgp_plan_info(self._h, N.iptr(out)))
        return out

    @property
    def kernel_variant(self) -> int:
        return int(self.info()[6])

    def set_variant(self, variant: int) -> None:
        """Force a kernel variant (testing aid; see vgp_plan_set_variant in
        include/vecchia_b200.h): -1 auto, 0 generic, 1 all-register warp-DMMA,
        4 warp-specialised + distance cache, 7/8 scheduler-aware, 11/12
        CTA-per-block, 13 thread-per-block."""
        N.check(N.lib.vgp_plan_set_variant(self.handle, int(variant)))

    def _host_arrays(self, dataset: geo.Dataset):
        if dataset.n != self.n:
            raise ValueError(f"plan built for n={self.n}, dataset has n={dataset.n}")
        locs = np.ascontiguousarray(dataset.locations, dtype=np.float64)
        obs = np.ascontiguousarray(dataset.observations, dtype=np.float64)
        if locs is dataset.locations and obs is dataset.observations:
            _pin(locs)
            _pin(obs)
        return locs, obs

    def set_data(self, dataset: geo.Dataset) -> None:
        """Upload a dataset in original order; the device applies the permutation."""
        locs, obs = self._host_arrays(dataset)
        N.check(N.lib.vgp_plan_set_data(self.handle, N.dptr(locs), N.dptr(obs)))

    @property
    def stream(self) -> int:
        return int(N.lib.vgp_plan_stream(self.handle) or 0)

    def loglik(self, spec: kernels.KernelSpec, full_result: bool = True,
               dataset: geo.Dataset | None = None) -> LogLikResult:
        """Evaluate at `spec`; with `dataset`, upload it first in the same
        call (vgp_loglik_data: the location upload and check overlap the
        evaluation when the plan's distance cache already holds them)."""
        if not self.full:
            raise ValueError("loglik needs a full-range plan; use partials() on shards")
        host = self._host_arrays(dataset) if dataset is not None else None
        p = spec.params
        k = self.n - self.m
        total = np.zeros(1)
        bf = np.zeros(1)
        fail = np.full(1, -1, dtype=np.int64)
        if full_result:
            rest, mu, sg = _RESULTS.take(k), _RESULTS.take(k), _RESULTS.take(k)
            ptrs = (N.dptr(rest), N.dptr(mu), N.dptr(sg))
        else:
            rest = mu = sg = None
            ptrs = (N.null_d(), N.null_d(), N.null_d())
        args = (N.FAMILY_CODES[spec.family], float(p.sigma_sq), float(p.beta), float(p.nu),
                N.dptr(total), N.iptr(fail), N.dptr(bf), *ptrs)
        if host is not None:
            rc = N.lib.vgp_loglik_data(self.handle, N.dptr(host[0]), N.dptr(host[1]), *args)
        else:
            rc = N.lib.vgp_loglik(self.handle, *args)
        N.raise_for_status(rc, int(fail[0]))
        if not full_result:
            rest = mu = sg = np.empty(0)
        return LogLikResult(float(total[0]), float(bf[0]), rest, mu, sg)

    def total(self, spec: kernels.KernelSpec) -> float:
        return self.loglik(spec, full_result=False).total

    def partials(self, spec: kernels.KernelSpec):
        """(chunk partials, block_first, status, fail_index) of this shard."""
        p = spec.params
        parts = np.zeros(max(self.nchunks, 1))
        bf = np.zeros(1)
        fail = np.full(1, -1, dtype=np.int64)
        rc = N.lib.vgp_loglik_partials(self.handle, N.FAMILY_CODES[spec.family], float(p.sigma_sq),
                                       float(p.beta), float(p.nu), N.dptr(parts), N.dptr(bf),
                                       N.iptr(fail))
        N.check(rc)
        return parts[: self.nchunks], float(bf[0]), int(rc), int(fail[0])

    def partials_device(self, spec: kernels.KernelSpec, out_ptr: int) -> None:
        """Write block_first / this shard's chunk partials into a device vector
        (see vgp_loglik_partials_device) for a cross-GPU all-reduce."""
        p = spec.params
        N.check(N.lib.vgp_loglik_partials_device(self.handle, N.FAMILY_CODES[spec.family],
                                                 float(p.sigma_sq), float(p.beta), float(p.nu),
                                                 ctypes.c_void_p(out_ptr)))

    def set_timing(self, enable: bool) -> None:
        N.check(N.lib.vgp_plan_set_timing(self.handle, 1 if enable else 0))

    def kernel_time(self):
        """(summed ms, launches) of the fused block kernel since the last call."""
        ms = np.zeros(1)
        cnt = np.zeros(1, dtype=np.int64)
        N.check(N.lib.vgp_plan_kernel_time(self.handle, N.dptr(ms), N.iptr(cnt)))
        return float(ms[0]), int(cnt[0])

    # -- launch-only interface for device-timed benchmarking
    def launch(self, spec: kernels.KernelSpec) -> None:
        p = spec.params
        N.check(N.lib.vgp_loglik_async(self.handle, N.FAMILY_CODES[spec.family],
                                       float(p.sigma_sq), float(p.beta), float(p.nu)))

    def fetch(self):
        total = np.zeros(1)
        fail = np.full(1, -1, dtype=np.int64)
        st = ctypes.c_int(0)
        N.check(N.lib.vgp_plan_fetch(self.handle, N.dptr(total), N.iptr(fail), ctypes.byref(st)))
        return float(total[0]), int(st.value), int(fail[0])


_PINNED: dict = {}  # data pointer -> bytes of page-locked dataset arrays


def _pin(arr: np.ndarray) -> None:
    """Page-lock a dataset array in place the first time it is uploaded, so
    the per-evaluation upload runs as DMA; unregistered when the array is
    freed.  Registration failure leaves the (slower) pageable upload."""
    if not arr.flags.owndata or arr.nbytes < (1 << 20):
        return
    ptr = arr.ctypes.data
    if ptr in _PINNED:
        return
    if N.lib.vgp_host_register(ctypes.c_void_p(ptr), arr.nbytes) != 0:
        return
    _PINNED[ptr] = arr.nbytes
    weakref.finalize(arr, _unpin, ptr)


def _unpin(ptr: int) -> None:
    if _PINNED.pop(ptr, None) is not None:
        N.lib.vgp_host_unregister(ctypes.c_void_p(ptr))


class _ResultPool:
    """Page-locked buffers for the per-block results of ``vecchia_loglik``.

    Every call still returns fresh arrays (the reference's contract), but
    their memory comes from a pool of registered (page-locked) buffers, so
    the chunked device->host result download runs as DMA instead of through
    the driver's pageable bounce buffer.  A buffer returns to the pool when
    the last array (or view) over it is garbage collected: the handed-out
    array is built over a per-call ctypes object whose finalizer does the
    return, and numpy views keep that object alive.
    """

    def __init__(self, keep: int = 6):
        self.keep = keep
        self.free: dict = {}  # length -> [raw arrays]
        self.busy: dict = {}  # id(ctypes holder) -> raw array

    def take(self, k: int) -> np.ndarray:
        lst = self.free.get(k)
        if lst:
            raw = lst.pop()
        else:
            raw = np.empty(max(k, 1))
            if raw.nbytes >= (1 << 20):
                _pin(raw)
        holder = (ctypes.c_double * k).from_address(raw.ctypes.data)
        out = np.ctypeslib.as_array(holder) if k else np.empty(0)
        self.busy[id(holder)] = raw
        weakref.finalize(holder, self._give, id(holder), k)
        return out

    def _give(self, key: int, k: int) -> None:
        raw = self.busy.pop(key, None)
        if raw is None:
            return
        lst = self.free.setdefault(k, [])
        if len(lst) < self.keep:
            lst.append(raw)


_RESULTS = _ResultPool()


class LikelihoodSession:
    """A dataset resident on the GPU next to its plan: the MLE objective.

    Equivalent to calling ``vecchia_loglik(dataset, plan, spec)`` repeatedly
    with the same dataset, without re-uploading it each time.
    """

    def __init__(self, dataset: geo.Dataset, plan: VecchiaPlan, device: int | None = None):
        if plan.permutation.n != dataset.n:
            raise ValueError(f"plan built for n={plan.permutation.n}, dataset has n={dataset.n}")
        self.dataset = dataset
        self.plan = plan
        self.single = dataset.n == 1
        if not self.single:
            self.dplan = DevicePlan(plan, device=device)
            self.dplan.set_data(dataset)

    def loglik(self, spec: kernels.KernelSpec) -> LogLikResult:
        if self.single:
            return _singleton(self.dataset, spec)
        return self.dplan.loglik(spec)

    def total(self, spec: kernels.KernelSpec) -> float:
        if self.single:
            return _singleton(self.dataset, spec).total
        return self.dplan.total(spec)

    def close(self) -> None:
        if not self.single:
            self.dplan.close()


def _singleton(dataset: geo.Dataset, spec: kernels.KernelSpec) -> LogLikResult:
    # exact univariate density for n == 1 (vg/vecchia.py:229-233)
    s2 = spec.params.sigma_sq
    y0 = float(dataset.observations[0])
    ll = -0.5 * (y0 * y0 / s2 + LOG_2PI + math.log(s2))
    return LogLikResult(ll, ll, np.empty(0), np.empty(0), np.empty(0))


def vecchia_loglik(dataset: geo.Dataset, plan: VecchiaPlan, spec: kernels.KernelSpec) -> LogLikResult:
    """Vecchia-approximated Gaussian log-likelihood of a dataset (vg/vecchia.py:217-238).

    The dataset (original order) is uploaded and permuted on the device each
    call; the plan's permutation and neighbour table stay resident.  Raises
    LikelihoodEvaluationError with the failing block index when a
    conditioning matrix is not positive definite or a conditional variance is
    non-positive.
    """
    if dataset.n == 1:
        return _singleton(dataset, spec)
    if plan.permutation.n != dataset.n:
        raise ValueError(f"plan built for n={plan.permutation.n}, dataset has n={dataset.n}")
    dp = plan.device_plan(metric=dataset.metric)
    return dp.loglik(spec, dataset=dataset)


def simulate_vecchia(dataset: geo.Dataset, plan: VecchiaPlan, spec: kernels.KernelSpec,
                     seed) -> np.ndarray:
    """Draw observations (ORIGINAL order) from the Gaussian whose exact
    log-density is the Vecchia likelihood of `plan`:
    y[:m] = L0 z[:m], y_t = b_t . y[J_t] + sqrt(sigma^2 - v_t . b_t) z_t in the
    plan's order, z = numpy default_rng(seed).standard_normal(n) (ordered).

    The device-scale counterpart of the reference's dense generator
    ``exact.simulate_grf`` (vg/exact.py:47-66, capped at n <= 20000): only
    ``dataset.locations`` are read.  Model-consistent fields keep the
    CPU/GPU likelihood comparison well conditioned; white noise does not
    (SURVEY.md H5)."""
    n = dataset.n
    if plan.permutation.n != n:
        raise ValueError(f"plan built for n={plan.permutation.n}, dataset has n={n}")
    z = np.random.default_rng(seed).standard_normal(n)
    if n == 1:
        return np.sqrt(spec.params.sigma_sq) * z
    dp = plan.device_plan(metric=dataset.metric)
    dp.set_data(dataset)
    p = spec.params
    y_ord = np.empty(n)
    fail = np.full(1, -1, dtype=np.int64)
    rc = N.lib.vgp_simulate(dp.handle, N.FAMILY_CODES[spec.family], float(p.sigma_sq),
                            float(p.beta), float(p.nu), N.dptr(z), N.dptr(y_ord), N.iptr(fail))
    N.raise_for_status(rc, int(fail[0]))
    y = np.empty(n)
    y[plan.permutation.order] = y_ord
    return y


# The package's own implementation, so callers can tell whether the module
# attribute (the reference's plugin seam, vg/fit.py:165) has been replaced.
NATIVE_VECCHIA_LOGLIK = vecchia_loglik


def _ordered_sum(values: np.ndarray) -> float:
    """4096-chunk pairwise partials combined in index order (vg/vecchia.py:169-177)."""
    partials = [float(values[lo:lo + _REDUCE_CHUNK].sum())
                for lo in range(0, values.shape[0], _REDUCE_CHUNK)]
    total = 0.0
    for p in partials:
        total += p
    return total


def flop_count(n: int, m: int) -> float:
    """(n - m + 1)(m^3/3 + 2 m^2 + 4 m), vg/vecchia.py:241-251."""
    if not (1 <= m < n):
        raise ValueError(f"need 1 <= m < n, got m={m}, n={n}")
    blocks = float(n - m + 1)
    fm = float(m)
    return blocks * (fm**3 / 3.0 + 2.0 * fm**2 + 4.0 * fm)


# ---------------------------------------------------------------- staged API
# The reference's three-stage evaluation (vg/vecchia.py:85-214), kept for
# callers that drive the stages themselves (cli.cmd_bench, vg/cli.py:259-263,
# and the reference's assemble tests).  Unlike vecchia_loglik, which runs the
# fused kernel and never materialises a block, this path stores every
# conditioning block (28.8 GB at n = 1M, m = 60, as the reference does): the
# blocks are generated on the device (vgp_assemble) and factored / solved by
# the device batched kernels (batchla, vgp_batch_*).


@dataclass
class BatchWorkspace:
    """Strided storage for the n - m + 1 conditioning blocks (vg/vecchia.py:85-92)."""

    Sigma: "batchla.StridedMatrixBatch"
    v: "batchla.StridedVectorBatch"
    yJ: "batchla.StridedVectorBatch"
    sigma_diag: "batchla.BatchScalars"


def assemble(dataset: geo.Dataset, plan: VecchiaPlan, spec: kernels.KernelSpec,
             out: BatchWorkspace | None = None) -> BatchWorkspace:
    """Populate the conditioning batches of an already-permuted dataset
    (vg/vecchia.py:106-166) with ``vgp_assemble`` on the GPU.  Passing a
    previous workspace as ``out`` refills it in place."""
    from . import batchla

    n, m = dataset.n, plan.m
    if plan.permutation.n != n:
        raise ValueError(f"plan built for n={plan.permutation.n}, dataset has n={n}")
    if not (1 <= m < n):
        raise ValueError(f"need 1 <= m < n, got m={m}, n={n}")
    count = n - m + 1
    if out is None:
        ws = BatchWorkspace(
            Sigma=batchla.StridedMatrixBatch.zeros(count, m),
            v=batchla.StridedVectorBatch.zeros(count, m),
            yJ=batchla.StridedVectorBatch.zeros(count, m),
            sigma_diag=batchla.BatchScalars(np.empty(count)),
        )
    else:
        ws = out
        if ws.Sigma.count != count or ws.Sigma.dim != m:
            raise ValueError(f"workspace shaped ({ws.Sigma.count}, {ws.Sigma.dim}), need ({count}, {m})")
    ws.sigma_diag.values[:] = spec.params.sigma_sq
    metric, radius = _metric_code(dataset.metric)
    locs = np.ascontiguousarray(dataset.locations, dtype=np.float64)
    obs = np.ascontiguousarray(dataset.observations, dtype=np.float64)
    nbr = np.ascontiguousarray(plan.neighbors.neighbors, dtype=np.int64)
    p = spec.params
    N.check(N.lib.vgp_assemble(N.current_device(), N.dptr(locs), N.dptr(obs), n, m, N.iptr(nbr), metric,
                               radius, N.FAMILY_CODES[spec.family], float(p.sigma_sq), float(p.beta),
                               float(p.nu), N.dptr(ws.Sigma.buffer), ws.Sigma.stride,
                               N.dptr(ws.v.buffer), ws.v.stride, N.dptr(ws.yJ.buffer), ws.yJ.stride))
    return ws


def _numeric_stage(ws: BatchWorkspace):
    """Factor, solve and dot every block on the GPU; Sigma is overwritten by
    its factor (vg/vecchia.py:180-190)."""
    from . import batchla
    from .errors import LikelihoodEvaluationError, NonPositiveDefiniteError

    try:
        lower = batchla.batch_potrf(ws.Sigma)
    except NonPositiveDefiniteError as exc:
        raise LikelihoodEvaluationError(exc.batch_index, str(exc)) from exc
    v_prime = batchla.batch_trsv(lower, ws.v)
    y_prime = batchla.batch_trsv(lower, ws.yJ)
    mu_prime = batchla.batch_dot(y_prime, v_prime).values
    sigma_prime = batchla.batch_dot(v_prime, v_prime).values
    return lower, mu_prime, sigma_prime


def _reduction_stage(ws: BatchWorkspace, ordered_obs: np.ndarray, m: int, lower, mu_prime: np.ndarray,
                     sigma_prime: np.ndarray) -> LogLikResult:
    """Per-block log-densities and the ordered total (vg/vecchia.py:193-214),
    the same O(n) arithmetic the fused kernel's epilogue performs."""
    from . import batchla
    from .errors import LikelihoodEvaluationError

    block_first = -batchla.half_log_det(lower.matrix(0)) - 0.5 * mu_prime[0] - 0.5 * m * LOG_2PI
    mu_new = mu_prime[1:]
    sigma_new = ws.sigma_diag.values[1:] - sigma_prime[1:]
    bad = ~(sigma_new > 0.0)
    if np.any(bad):
        k = 1 + int(np.argmax(bad))
        raise LikelihoodEvaluationError(k, f"conditional variance {sigma_new[k - 1]!r} <= 0")
    resid = np.asarray(ordered_obs, dtype=np.float64)[m:] - mu_new
    block_rest = -0.5 * (resid * resid / sigma_new + LOG_2PI + np.log(sigma_new))
    total = block_first + _ordered_sum(block_rest)
    return LogLikResult(total, block_first, block_rest, mu_new, sigma_new)
