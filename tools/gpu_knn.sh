#!/bin/bash
# grid kNN: parity and plan-time timing
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "grid_knn or knn_bit" --timeout 800 2>&1 | tail -4
timeout 900 python - <<'PY'
import json, os, sys, time
sys.path.insert(0, ".")
import numpy as np
import paper_2403_07412_b200 as vg
for n, m in ((1_000_000, 60), (4_000_000, 120), (2_000_000, 60)):
    locs = np.random.default_rng(0).random((n, 2))
    data = vg.Dataset(locs, np.zeros(n))
    for grid in (True, False):
        if not grid and n > 1_000_000:
            continue
        os.environ["VGP_KNN_GRID_MIN"] = "0" if grid else str(1 << 40)
        t0 = time.perf_counter()
        t = vg.nearest_neighbors(data, m).neighbors
        dt = time.perf_counter() - t0
        print(json.dumps({"n": n, "m": m, "grid": grid, "knn_s": round(dt, 3),
                          "digest": int(np.bitwise_xor.reduce(t[::997].ravel()))}), flush=True)
PY
