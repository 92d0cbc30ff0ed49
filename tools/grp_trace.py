"""Summarise the lock-step group kernel's clock64 trace (VGP_TRACEG=<file>):
rows group x round, events 0 round start, 1 staged, per column c:
2+3c tiles done, 3+3c diagonal done, 4+3c panel rows done."""
import sys

import numpy as np

G, R, E, NC = 2, 6, 32, 8
a = np.loadtxt(sys.argv[1], dtype=np.int64)[-G * R:].reshape(G, R, E)
stage, tiles, diag, rows = [], [], [], []
for g in range(G):
    for rd in range(1, R - 1):
        ev = a[g, rd]
        stage.append(ev[1] - ev[0])
        prev = ev[1]
        for c in range(NC):
            tiles.append(ev[2 + 3 * c] - prev)
            diag.append(ev[3 + 3 * c] - ev[2 + 3 * c])
            rows.append(ev[4 + 3 * c] - ev[3 + 3 * c])
            prev = ev[4 + 3 * c]
r = lambda v: np.array(v).reshape(-1, NC).mean(0).round()
print(f"staging {np.mean(stage):.0f}")
print(f"tiles  {np.mean(tiles):6.0f} by column {r(tiles)}")
print(f"diag   {np.mean(diag):6.0f} by column {r(diag)}")
print(f"rows   {np.mean(rows):6.0f} by column {r(rows)}")
per = [a[g, rd + 1, 0] - a[g, rd, 0] for g in range(G) for rd in range(1, R - 2)]
print(f"round (4 blocks per group) {np.mean(per):.0f} cycles")
