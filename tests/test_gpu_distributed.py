"""GPU: the multi-GPU objective over a real NCCL communicator (one rank on
this one-GPU box): the shard plan's split kNN, the device partials, the
all-reduce and the sharded MLE driver give the single-GPU results."""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def nccl():
    import torch
    import torch.distributed as dist

    import paper_2403_07412_b200 as vg

    if vg._native.device_count() == 0:
        pytest.fail("GPU tests need a CUDA device: the B200 path has no CPU fallback")
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    yield dist
    dist.destroy_process_group()


def test_sharded_mle_over_nccl_matches_single_gpu(nccl):
    import paper_2403_07412_b200 as vg
    from paper_2403_07412_b200.distributed import ShardedVecchia, make_shard_plan, mle_estimate_sharded

    n, m = 20000, 30
    locs = np.random.default_rng(21).random((n, 2))
    plan = vg.make_plan(vg.Dataset(locs, np.zeros(n)), m, "random", seed=0)
    spec = vg.KernelSpec("matern", vg.KernelParams(1.0, 0.078809, 0.5))
    data = vg.Dataset(locs, vg.simulate_vecchia(vg.Dataset(locs, np.zeros(n)), plan, spec, 4))
    sp = make_shard_plan(data, m, "random", 0, 0, 1)
    np.testing.assert_array_equal(sp.neighbors.neighbors, plan.neighbors.neighbors)
    sh = ShardedVecchia(data, sp, device=0)
    assert sh.total(spec) == vg.vecchia_loglik(data, plan, spec).total
    sh.close()
    cfg = vg.FitConfig(objective="vecchia", m=m, ordering="random", seed=0,
                       init=vg.KernelParams(0.5, 0.05, 0.5))
    a = mle_estimate_sharded(data, cfg)
    b = vg.mle_estimate(data, cfg)
    assert (a.theta_hat.sigma_sq, a.theta_hat.beta, a.loglik, a.evaluations) == \
        (b.theta_hat.sigma_sq, b.theta_hat.beta, b.loglik, b.evaluations)
