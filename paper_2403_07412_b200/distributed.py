"""Multi-GPU Vecchia log-likelihood: blocks sharded over ranks, one collective.

One process per GPU (torchrun).  The n - m + 1 conditioning blocks are cut
into the reference's fixed 4096-entry reduction chunks (vg/vecchia.py:35,
:169-177); rank r owns a contiguous chunk range (and rank 0 the joint block
0).  Each rank evaluates its blocks with the fused kernel and writes its chunk
partials into its own slots of a zero vector of length 1 + n_chunks; one
all-reduce (SUM) of that vector — every slot has exactly one non-zero
contributor, so the sum is exact — gives every rank all partials, and the
ordered host sum  block_first + ((0 + p0) + p1) + ...  reproduces the
single-GPU total bit for bit for any world size.  Infeasibility propagates as
NaN; only then a second all-reduce (MIN) of the failure keys recovers the
reference's error index.

Locations, observations and the permutation are replicated (24 B/point);
neighbour rows are kept only for the rank's own blocks.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np

from . import _native as N
from . import geo, vecchia
from .errors import LikelihoodEvaluationError

CHUNK = vecchia._REDUCE_CHUNK


def n_chunks(n: int, m: int) -> int:
    return (n - m + CHUNK - 1) // CHUNK


def shard_blocks(n: int, m: int, rank: int, world: int) -> tuple[int, int]:
    """Batch-entry range [lo, hi) of `rank`: contiguous 4096-chunk ranges,
    balanced by chunk count (blocks are uniform in cost at fixed m); rank 0
    also owns the joint block 0."""
    if not (0 <= rank < world):
        raise ValueError("rank out of range")
    nrest = n - m
    c = n_chunks(n, m)
    c_lo = (c * rank) // world
    c_hi = (c * (rank + 1)) // world
    lo = 1 + c_lo * CHUNK
    hi = 1 + min(c_hi * CHUNK, nrest)
    if rank == 0:
        lo = 0
    if c_hi <= c_lo and rank != 0:
        return (hi, hi)  # empty shard
    return (lo, hi)


def ordered_total(vec: np.ndarray) -> float:
    """block_first + ((0 + p0) + p1) + ... (vg/vecchia.py:174-177, :213)."""
    s = 0.0
    for p in vec[1:]:
        s += float(p)
    return float(vec[0]) + s


def combine_partials(send, buf, dist, group=None) -> np.ndarray:
    """The one collective of an evaluation: every rank's `send` holds its own
    slots (block_first at 0 for rank 0, its chunk partials at 1 + c) and zeros
    elsewhere; SUM-all-reduce into `buf` and return it on the host.  Device
    agnostic (NCCL on CUDA tensors, gloo on CPU tensors in the tests)."""
    buf.copy_(send)
    dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=group)
    return buf.cpu().numpy()


@dataclass
class ShardPlan:
    """One rank's slice of a VecchiaPlan: the full ordering, the neighbour
    rows of its own blocks only (rows [row_lo, row_hi) of the table)."""

    m: int
    permutation: object
    neighbors: object  # geo.NeighborTable of the shard's rows
    metric: object
    ordering: str
    row_lo: int
    row_hi: int


def make_shard_plan(dataset, m: int, ordering: str, seed: int, rank: int, world: int) -> ShardPlan:
    """make_plan for one rank (vg/vecchia.py:59-82 restricted to a shard): the
    ordering is computed identically on every rank, the kNN only for the
    rank's targets (vgp_knn_predecessors_range), so the O(n^2)-class search
    is split across GPUs instead of replicated."""
    n = dataset.n
    perm = vecchia.make_ordering(dataset, ordering, seed)
    lo, hi = shard_blocks(n, m, rank, world)
    row_lo, row_hi = max(lo, 1) - 1, max(hi - 1, max(lo, 1) - 1)
    rows = geo.nearest_neighbor_rows(dataset.permute(perm), m, row_lo, row_hi)
    return ShardPlan(m, perm, geo.NeighborTable(m=m, neighbors=rows), dataset.metric, ordering,
                     row_lo, row_hi)


NO_FAILURE = np.iinfo(np.int64).max


def npd_key_entry(key: int, m: int) -> int:
    """Batch entry of a packed NPD key (include/vecchia_b200.h vgp_plan_fail_keys)."""
    if m > 256:
        return int(key)
    chunk = max(1, (1 << 21) // (m * m))
    return (key >> 42) * chunk + (key & ((1 << 24) - 1))


class ShardObjective:
    """Host side of a sharded evaluation, device-agnostic: fill this rank's
    slots of the global vector, all-reduce it (the one collective), take the
    ordered total; on a NaN total agree on the reference's failure index with
    a second all-reduce (MIN over packed keys, so the index is the one the
    reference would raise, whichever shard holds it).  Subclasses provide
    _fill(spec) and _failure_keys()."""

    def __init__(self, n, m, group, dist, torch, device):
        self.n, self.m = n, m
        self.group, self.dist, self.torch = group, dist, torch
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.block_lo, self.block_hi = shard_blocks(n, m, self.rank, self.world)
        self.dev = device
        self.send = torch.zeros(1 + n_chunks(n, m), dtype=torch.float64, device=device)
        self.buf = torch.empty_like(self.send)

    def _fill(self, spec) -> None:
        raise NotImplementedError

    def _failure_keys(self) -> tuple[int, int]:
        return NO_FAILURE, NO_FAILURE

    def reduce_vector(self, spec) -> np.ndarray:
        self._fill(spec)
        return combine_partials(self.send, self.buf, self.dist, self.group)

    def total(self, spec) -> float:
        total = ordered_total(self.reduce_vector(spec))
        if math.isnan(total):
            t = self.torch.tensor(list(self._failure_keys()), dtype=self.torch.int64, device=self.dev)
            self.dist.all_reduce(t, op=self.dist.ReduceOp.MIN, group=self.group)
            npd, var = (int(v) for v in t.cpu().tolist())
            if npd != NO_FAILURE:
                raise LikelihoodEvaluationError(npd_key_entry(npd, self.m), "sharded evaluation failed")
            if var != NO_FAILURE:
                raise LikelihoodEvaluationError(var, "sharded evaluation failed")
            # NaN without a failure flag: returned as is, like the single-GPU path
        return total

    def close(self) -> None:
        pass


class ShardedVecchia(ShardObjective):
    """The MLE objective on this rank's GPU shard: `total(spec)` is collective.
    `plan` is a full VecchiaPlan or this rank's ShardPlan."""

    def __init__(self, dataset, plan, group=None, device=None):
        import torch
        import torch.distributed as dist

        dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        super().__init__(dataset.n, plan.m, group, dist, torch, dev)
        lo, hi = self.block_lo, self.block_hi
        self.dplan = None
        if hi > lo:
            self.dplan = vecchia.DevicePlan(plan, device=dev.index, block_lo=lo, block_hi=hi)
            self.dplan.set_data(dataset)

    def set_data(self, dataset) -> None:
        if self.dplan is not None:
            self.dplan.set_data(dataset)

    def _fill(self, spec) -> None:
        if self.dplan is not None:
            self.dplan.partials_device(spec, self.send.data_ptr())

    def _failure_keys(self) -> tuple[int, int]:
        if self.dplan is None:
            return NO_FAILURE, NO_FAILURE
        keys = (ctypes.c_uint64 * 2)()
        N.check(N.lib.vgp_plan_fail_keys(self.dplan.handle, keys))
        return tuple(NO_FAILURE if k == 2**64 - 1 else int(k) for k in keys)

    def close(self):
        if self.dplan is not None:
            self.dplan.close()


def mle_estimate_sharded(train, config, family: str = "matern", group=None, device=None,
                         evaluator=None):
    """fit.mle_estimate (vg/fit.py:140-178) with the objective evaluated across
    all ranks of `group`: every rank runs the same host Nelder-Mead, each
    evaluation is one sharded likelihood (its blocks on this GPU + one
    all-reduce), so every rank follows the identical trajectory and returns
    the single-process estimate bit for bit.  Collective: call on every rank.
    `evaluator` (an object with total(spec) and close()) replaces the GPU
    shard — the CPU tests pass an oracle-backed one."""
    from . import fit

    if config.objective != "vecchia":
        raise ValueError("the sharded objective is the Vecchia likelihood")
    if evaluator is None:
        import torch.distributed as dist

        rank, world = dist.get_rank(group), dist.get_world_size(group)
        sp = make_shard_plan(train, config.m, config.ordering, config.seed, rank, world)
        evaluator = ShardedVecchia(train, sp, group=group, device=device)
    try:
        return fit.mle_estimate(train, config, family, objective_fn=evaluator.total)
    finally:
        evaluator.close()
