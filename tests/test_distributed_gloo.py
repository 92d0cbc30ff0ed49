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


# ---------------------------------------------------------------- sharded MLE

class _OracleShard:
    """A ShardObjective whose per-rank fill is the CPU oracle over this rank's
    blocks (test infrastructure standing in for the GPU shard): the package's
    own collective, ordered total and failure agreement run unchanged."""

    def __new__(cls, locs, y, m, table, dist_mod, torch_mod):
        from paper_2403_07412_b200.distributed import ShardObjective

        class Impl(ShardObjective):
            def __init__(self):
                super().__init__(locs.shape[0], m, None, dist_mod, torch_mod, "cpu")
                self.last = None

            def _fill(self, spec):
                from oracle import oracle as O

                p = spec.params
                r = O.loglik(locs, y, m, table, spec.family, p.sigma_sq, p.beta, p.nu, threads=1)
                self.last = r
                self.send.zero_()
                lo, hi = self.block_lo, self.block_hi
                if r.status != 0:
                    if hi > lo:
                        self.send[1 + (max(lo, 1) - 1) // CHUNK] = float("nan")
                    return
                if lo == 0:
                    self.send[0] = r.block_first
                k_lo, k_hi = max(lo, 1) - 1, hi - 1
                for c in range(k_lo // CHUNK, (k_hi + CHUNK - 1) // CHUNK):
                    a, b = c * CHUNK, min((c + 1) * CHUNK, self.n - m)
                    self.send[1 + c] = O.pairwise_sum(r.block_rest[a:b])

            def _failure_keys(self):
                from paper_2403_07412_b200.distributed import NO_FAILURE

                r = self.last
                lo, hi = self.block_lo, self.block_hi
                if r is None or r.status == 0 or not (lo <= r.fail_index < hi):
                    return NO_FAILURE, NO_FAILURE
                if r.status == 2:
                    return NO_FAILURE, r.fail_index
                chunk = max(1, (1 << 21) // (m * m))  # pivot column unknown here: 0
                e = r.fail_index
                return ((e // chunk) << 42) | (e % chunk), NO_FAILURE

        return Impl()


def _mle_worker(rank, world, port, n, m, out_path):
    import paper_2403_07412_b200 as vg
    from paper_2403_07412_b200.distributed import mle_estimate_sharded

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    locs, y, table = _problem(n, m)
    data = vg.Dataset(locs, y)
    cfg = vg.FitConfig(objective="vecchia", m=m, ordering="identity", seed=0,
                       init=vg.KernelParams(0.5, 0.05, 0.5), max_evals=120)
    ev = _OracleShard(locs, y, m, table, dist, torch)
    fr = mle_estimate_sharded(data, cfg, evaluator=ev)
    np.save(out_path + f".{rank}.npy", np.array([fr.theta_hat.sigma_sq, fr.theta_hat.beta,
                                                  fr.loglik, fr.evaluations]))
    dist.destroy_process_group()


def test_sharded_mle_matches_single_process(tmp_path):
    """mle_estimate_sharded at world size 2: every rank follows the single-
    process Nelder-Mead trajectory (vg/fit.py:61-137) bit for bit, because
    every sharded total equals the single-process total bit for bit."""
    import paper_2403_07412_b200 as vg
    from oracle import oracle as O

    n, m, world = 9000, 10, 2
    out = str(tmp_path / "mle")
    mp.spawn(_mle_worker, args=(world, _free_port(), n, m, out), nprocs=world, join=True)
    locs, y, table = _problem(n, m)
    data = vg.Dataset(locs, y)
    cfg = vg.FitConfig(objective="vecchia", m=m, ordering="identity", seed=0,
                       init=vg.KernelParams(0.5, 0.05, 0.5), max_evals=120)

    def single(spec):
        p = spec.params
        r = O.loglik(locs, y, m, table, spec.family, p.sigma_sq, p.beta, p.nu, threads=1)
        if r.status != 0:
            raise vg.LikelihoodEvaluationError(r.fail_index)
        return r.total

    fr = vg.mle_estimate(data, cfg, objective_fn=single)
    ref = np.array([fr.theta_hat.sigma_sq, fr.theta_hat.beta, fr.loglik, fr.evaluations])
    for r in range(world):
        np.testing.assert_array_equal(np.load(out + f".{r}.npy"), ref)


def _fail_worker(rank, world, port, out_path):
    import paper_2403_07412_b200 as vg

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    # duplicated point at ordered index 9000 > the first shard: the failure
    # sits on rank 1 and every rank must raise the same index
    n, m = 13000, 12
    locs, y, table = _problem(n, m)
    spec = vg.KernelSpec("matern", vg.KernelParams(1.0, 0.08, 0.5))
    locs[9000] = locs[int(table[9000 - m][0])]  # the target duplicates its nearest neighbour
    ev = _OracleShard(locs, y, m, table, dist, torch)
    try:
        ev.total(spec)
        res = -1
    except vg.LikelihoodEvaluationError as exc:
        res = exc.block_index if hasattr(exc, "block_index") else exc.args[0]
    np.save(out_path + f".{rank}.npy", np.array([res]))
    dist.destroy_process_group()


def test_sharded_failure_raises_on_every_rank(tmp_path):
    out = str(tmp_path / "fail")
    mp.spawn(_fail_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    got = [int(np.load(out + f".{r}.npy")[0]) for r in range(2)]
    assert got[0] == got[1] and got[0] > 0
