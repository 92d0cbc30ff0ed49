"""Time the device maxmin ordering (config 5 plan-time step) on clustered
and uniform locations; one JSON line per size to stdout."""
import json
import sys
import time

import numpy as np

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))

import paper_2403_07412_b200 as vg

sizes = [int(s) for s in sys.argv[1:]] or [250_000, 1_000_000, 2_000_000]
for n in sizes:
    for kind in (("uniform",) if __import__("os").environ.get("MM_UNIFORM") else ("clustered", "uniform")):
        rng = np.random.default_rng(n)
        if kind == "uniform":
            locs = rng.random((n, 2))
        else:
            c = rng.random((50, 2))
            locs = c[rng.integers(0, 50, n)] + 0.03 * rng.standard_normal((n, 2))
        vg.geo.maxmin_ordering(locs[:1000])  # warm-up (context, module load)
        t0 = time.perf_counter()
        perm = vg.geo.maxmin_ordering(locs)
        t1 = time.perf_counter()
        t2 = time.perf_counter()
        vg.geo.nearest_neighbors(vg.Dataset(locs[perm.order], np.zeros(n)), 60)
        t3 = time.perf_counter()
        print(json.dumps({"n": n, "locations": kind, "maxmin_s": round(t1 - t0, 3),
                          "us_per_point": round((t1 - t0) / n * 1e6, 3),
                          "knn_m60_s": round(t3 - t2, 3)}), flush=True)
