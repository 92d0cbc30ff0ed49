"""Where the end-to-end vecchia_loglik time goes (n = 1M, m = 60)."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2403_07412_b200 as vg

n, m = 1_000_000, 60
rng = np.random.default_rng(0)
locs, y = rng.random((n, 2)), rng.standard_normal(n)
data = vg.Dataset(locs, y)
plan = vg.make_plan(data, m, "random", seed=0)
spec = vg.KernelSpec("matern", vg.KernelParams(1.0, 0.052537, 1.5))
dp = plan.device_plan()
dp.set_data(data)
for _ in range(3):
    vg.vecchia_loglik(data, plan, spec)

def t(f, k=5):
    f()
    t0 = time.perf_counter()
    for _ in range(k):
        f()
    return (time.perf_counter() - t0) / k * 1e3

print("set_data        ms", round(t(lambda: dp.set_data(data)), 3))
print("loglik total    ms", round(t(lambda: dp.total(spec)), 3))
print("loglik full     ms", round(t(lambda: dp.loglik(spec)), 3))
print("vecchia_loglik  ms", round(t(lambda: vg.vecchia_loglik(data, plan, spec)), 3))
a = np.empty(n - m)
b = np.empty(n - m)
print("numpy 8MB copy  ms", round(t(lambda: np.copyto(a, b)), 3))
