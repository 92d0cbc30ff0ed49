"""One invocation of a non-headline kernel, for `ncu -k regex:<kernel> -c 1`
(tools/gpu/prof_aux.sh): the kNN grid query and the distance-cache build of
config 2, the maxmin ordering of config 5, the small-m likelihood kernels of
the config-3 sweep.

  python tools/prof_aux.py knn|dcache|maxmin|m10|m20|m30|m45"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402  (synthetic locations of the bench workloads)
import paper_2403_07412_b200 as vg  # noqa: E402

mode = sys.argv[1]
if mode == "maxmin":
    locs = bench.synthetic(2_000_000, 0, "clustered")
    vg.geo.maxmin_ordering(locs)
elif mode in ("knn", "dcache"):
    locs = bench.synthetic(1_000_000, 0)
    data = vg.Dataset(locs, np.zeros(len(locs)))
    plan = vg.make_plan(data, 60, "random", seed=0)
    if mode == "dcache":
        plan.device_plan().set_data(data)
else:
    m = int(mode[1:])
    locs = bench.synthetic(250_000, 0)
    data = vg.Dataset(locs, np.random.default_rng(1).standard_normal(len(locs)))
    plan = vg.make_plan(data, m, "random", seed=0)
    dp = plan.device_plan()
    dp.set_data(data)
    dp.total(vg.KernelSpec("matern", vg.KernelParams(1.0, 0.052537, 1.5)))
print("done", mode)
