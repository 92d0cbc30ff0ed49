#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "sphere" --timeout 800 2>&1 | tail -3
timeout 600 python - <<'PY'
import json, os, sys, time
sys.path.insert(0, ".")
import numpy as np
import paper_2403_07412_b200 as vg
vg.nearest_neighbors(vg.Dataset(np.random.default_rng(1).random((1000, 2)), np.zeros(1000)), 5)
for n in (1_000_000, 2_000_000):
    rng = np.random.default_rng(n)
    locs = np.stack([rng.uniform(-180, 180, n), np.degrees(np.arcsin(rng.uniform(-1, 1, n)))], -1)
    data = vg.Dataset(locs, np.zeros(n), vg.GreatCircle())
    for grid in (True, False):
        if not grid and n > 1_000_000:
            continue
        os.environ["VGP_KNN_GRID_MIN"] = "0" if grid else str(1 << 40)
        t0 = time.perf_counter()
        t = vg.nearest_neighbors(data, 60).neighbors
        print(json.dumps({"n": n, "m": 60, "metric": "great_circle", "grid": grid,
                          "knn_s": round(time.perf_counter() - t0, 3),
                          "digest": int(np.bitwise_xor.reduce(t[::997].ravel()))}), flush=True)
PY
