"""CPU: the multi-GPU path's host logic on world_size 2 with the gloo backend.

Each rank evaluates its own shard of blocks (shard_blocks), turns its
block_rest slice into fixed 4096-chunk partials, writes them into its slots
of the global vector and runs the same collective (combine_partials) and
ordered total the GPU ranks run.  The CPU oracle stands in for the fused
kernel here (test infrastructure only); the result must equal the
single-process total bit for bit, for every world size."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2403_07412_b200.distributed import (
    CHUNK,
    combine_partials,
    n_chunks,
    ordered_total,
    shard_blocks,
)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _problem(n=13000, m=12, seed=4):
    from oracle import oracle as O

    rng = np.random.default_rng(seed)
    locs = rng.random((n, 2))
    table = O.knn_pred(locs, m)
    y = O.simulate_vecchia(locs, m, table, "matern", 1.0, 0.08, 0.5, seed=seed)
    return locs, y, table


def _worker(rank, world, port, n, m, out_path):
    from oracle import oracle as O

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    locs, y, table = _problem(n, m)
    ref = O.loglik(locs, y, m, table, "matern", 1.0, 0.08, 0.5, threads=1)
    lo, hi = shard_blocks(n, m, rank, world)
    send = torch.zeros(1 + n_chunks(n, m), dtype=torch.float64)
    if lo == 0:
        send[0] = ref.block_first
    k_lo, k_hi = max(lo, 1) - 1, hi - 1
    for c in range(k_lo // CHUNK, (k_hi + CHUNK - 1) // CHUNK):
        a, b = c * CHUNK, min((c + 1) * CHUNK, n - m)
        send[1 + c] = O.pairwise_sum(ref.block_rest[a:b])
    vec = combine_partials(send, torch.empty_like(send), dist)
    total = ordered_total(vec)
    if rank == 0:
        np.save(out_path, np.array([total, ref.total]))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_total_bit_identical(tmp_path, world):
    n, m = 13000, 12
    out = str(tmp_path / "tot.npy")
    mp.spawn(_worker, args=(world, _free_port(), n, m, out), nprocs=world, join=True)
    total, single = np.load(out)
    assert total == single


def test_shards_partition_blocks_on_chunk_boundaries():
    for n, m in [(1_000_000, 60), (4_000_000, 120), (13000, 12), (5000, 4999), (4200, 100)]:
        count = n - m + 1
        for world in (1, 2, 3, 4, 8):
            covered = []
            for r in range(world):
                lo, hi = shard_blocks(n, m, r, world)
                if hi > lo:
                    covered.append((lo, hi))
                    if lo > 0:
                        assert (lo - 1) % CHUNK == 0
                    if hi < count:
                        assert (hi - 1) % CHUNK == 0
            assert covered[0][0] == 0 and covered[-1][1] == count
            for (a, b), (c, d) in zip(covered, covered[1:]):
                assert b == c


def test_ordered_total_matches_reference_rule():
    rng = np.random.default_rng(1)
    vec = rng.standard_normal(300)
    s = 0.0
    for p in vec[1:]:
        s += p
    assert ordered_total(vec) == vec[0] + s
