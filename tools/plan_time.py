"""Plan-time breakdown (ordering, kNN, device plan + distance cache) for the
BASELINE shapes: python tools/plan_time.py [c2|c4|c5]..."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2403_07412_b200 as vg  # noqa: E402

SHAPES = {"c2": (1_000_000, 60, "uniform", "random"), "c4": (4_000_000, 120, "uniform", "random"),
          "c5": (2_000_000, 60, "clustered", "maxmin")}
for name in sys.argv[1:] or ["c2"]:
    n, m, kind, ordering = SHAPES[name]
    locs = bench.synthetic(n, 0, kind)
    data = vg.Dataset(locs, np.zeros(n))
    t0 = time.perf_counter()
    perm = vg.vecchia.make_ordering(data, ordering, 0)
    t1 = time.perf_counter()
    ordered = data.permute(perm)
    t2 = time.perf_counter()
    table = vg.geo.nearest_neighbors(ordered, m)
    t3 = time.perf_counter()
    plan = vg.VecchiaPlan(m, perm, table, data.metric, ordering)
    dp = plan.device_plan()
    t4 = time.perf_counter()
    dp.set_data(data)
    t5 = time.perf_counter()
    print(name, {"ordering_s": round(t1 - t0, 3), "permute_s": round(t2 - t1, 3), "knn_s": round(t3 - t2, 3),
                 "device_plan_s": round(t4 - t3, 3), "set_data_s": round(t5 - t4, 3)}, flush=True)
