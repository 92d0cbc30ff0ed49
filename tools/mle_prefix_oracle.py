"""Build-container side of the c5 prefix MLE check (tools/mle_runs.py c5):
the oracle's free-nu Nelder-Mead (vg/fit.py:61-178 restated, numpy + scipy
Bessel K) on the ordered prefix the GPU box saved, compared with the GPU's
estimate.  TEST INFRASTRUCTURE: runs the oracle, never the product.

  python tools/mle_prefix_oracle.py gpurun_out/r02_c5_prefix.npz >> profiles/r02_mle.jsonl
"""
import json
import math
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as O  # noqa: E402

z = np.load(sys.argv[1])
locs, obs, m, table = z["locs"], z["obs"], int(z["m"]), z["table"]
init = [float(v) for v in z["init"]]
bounds = [(1e-4, 1e4), (1e-4, 1e4), (0.05, 5.0)]  # vg/fit.py:21-25


def objective(x):
    s2, beta, nu = (float(v) for v in x)
    if not all(math.isfinite(v) and v > 0 for v in (s2, beta, nu)):
        return -math.inf
    r = O.loglik(locs, obs, m, table, "matern", s2, beta, nu)
    return r.total if r.status == 0 else -math.inf


t0 = time.perf_counter()
x, f, ev, conv = O.nelder_mead_max(objective, np.array(init), bounds)
gpu = [float(v) for v in z["gpu_theta"]]
rel = max(abs(a - b) / abs(b) for a, b in zip(gpu, x))
print(json.dumps({"config": "c5-prefix", "n_prefix": int(locs.shape[0]), "m": m,
                  "oracle_theta": [float(v) for v in x], "oracle_loglik": f, "oracle_evals": ev,
                  "oracle_converged": bool(conv), "oracle_s": time.perf_counter() - t0,
                  "gpu_theta": gpu, "gpu_loglik": float(z["gpu_loglik"]),
                  "gpu_evals": int(z["gpu_evals"]), "theta_max_rel_err": rel}))
