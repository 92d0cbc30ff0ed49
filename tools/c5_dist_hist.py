import sys, os, numpy as np
sys.path.insert(0, os.getcwd())
import bench, paper_2403_07412_b200 as vg
n, m = 2_000_000, 60
locs = bench.synthetic(n, 0, "clustered")
data = vg.Dataset(locs, np.zeros(n))
plan = vg.make_plan(data, m, "maxmin", 0)
L = locs[plan.permutation.order]
T = plan.neighbors.neighbors
rng = np.random.default_rng(0)
rows = np.concatenate([np.arange(2000), rng.choice(len(T), 20000, replace=False)])
tri = np.tril_indices(m + 1, -1)
hs = []
for r in rows:
    idx = np.concatenate([T[r], [m + r]])
    P = L[idx]
    d = np.sqrt(((P[:, None, :] - P[None, :, :]) ** 2).sum(-1))[tri]
    hs.append(d)
h = np.concatenate(hs)
print("dmax sample", h.max())
for beta in (0.052537, 0.389, 0.1):
    b = np.floor(np.log2(h[h > 0] / beta)).astype(int)
    vals, cnt = np.unique(b, return_counts=True)
    print("beta", beta, dict(zip(vals.tolist(), (cnt / cnt.sum()).round(4).tolist())))
    top = int(np.floor(np.log2(h.max() / beta)))
    lo = top - 13
    print("  window [%d, %d] covers %.4f" % (lo, top, ((b >= lo) & (b <= top)).mean()))
