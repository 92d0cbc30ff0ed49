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

import math

import numpy as np

from . import vecchia
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


class ShardedVecchia:
    """The MLE objective on this rank's shard: `total(spec)` is collective."""

    def __init__(self, dataset, plan, group=None, device=None):
        import torch
        import torch.distributed as dist

        self.torch, self.dist, self.group = torch, dist, group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.n, self.m = dataset.n, plan.m
        lo, hi = shard_blocks(self.n, self.m, self.rank, self.world)
        self.block_lo, self.block_hi = lo, hi
        self.dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        self.dplan = None
        if hi > lo:
            self.dplan = vecchia.DevicePlan(plan, device=self.dev.index, block_lo=lo, block_hi=hi)
            self.dplan.set_data(dataset)
        nvec = 1 + n_chunks(self.n, self.m)
        self.send = torch.zeros(nvec, dtype=torch.float64, device=self.dev)
        self.buf = torch.empty_like(self.send)

    def set_data(self, dataset) -> None:
        if self.dplan is not None:
            self.dplan.set_data(dataset)

    def reduce_vector(self, spec) -> np.ndarray:
        if self.dplan is not None:
            self.dplan.partials_device(spec, self.send.data_ptr())
        return combine_partials(self.send, self.buf, self.dist, self.group)

    def total(self, spec) -> float:
        vec = self.reduce_vector(spec)
        total = ordered_total(vec)
        if math.isnan(total):
            self._raise_failure()
        return total

    def _raise_failure(self):
        torch = self.torch
        big = np.iinfo(np.int64).max
        keys = [big, big]
        if self.dplan is not None:
            _, st, idx = self.dplan.fetch()
            if st == 1:
                keys[0] = idx
            elif st == 2:
                keys[1] = idx
        t = torch.tensor(keys, dtype=torch.int64, device=self.dev)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MIN, group=self.group)
        npd, var = (int(v) for v in t.cpu().tolist())
        idx = npd if npd != big else var
        raise LikelihoodEvaluationError(idx, "sharded evaluation failed")

    def close(self):
        if self.dplan is not None:
            self.dplan.close()
