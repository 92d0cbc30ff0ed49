"""Summarise the maxmin kernel's phase trace (VGP_MM_TRACE=<file>)."""
import sys
import numpy as np

a = np.loadtxt(sys.argv[1], dtype=np.int64).reshape(-1, 8, 256, 8)[-1]  # last run: cta, step, ev
names = ["chunks", "cta_bar", "cta_red", "cluster", "dsmem"]
d = np.stack([a[..., 1] - a[..., 0], a[..., 2] - a[..., 1], a[..., 3] - a[..., 2],
              a[..., 4] - a[..., 3], a[..., 5] - a[..., 4]], -1)
step = a[:, 1:, 0] - a[:, :-1, 0]
print("mean cycles per phase (over CTAs, steps):", dict(zip(names, d.mean((0, 1)).round())))
print("step period per CTA:", step.mean(1).round())
print("hits per step (sum over CTAs): mean", a[..., 6].sum(0).mean(), "max", a[..., 6].sum(0).max())
hit = a[..., 6] > 0
print("chunk phase with hits:", d[..., 0][hit].mean().round(), " without:", d[..., 0][~hit].mean().round())
ld = a[..., 7]
m = hit & (ld > 0)
print("hit CTAs: start->loads consumed", (ld - a[..., 0])[m].mean().round(),
      " loads consumed->chunks done", (a[..., 1] - ld)[m].mean().round())
