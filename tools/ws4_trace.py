"""Summarise the split-scheduler kernel's clock64 trace (VGP_TRACE4=<file>).
Rows: slot x role (0 chain, 1 worker) x block, 24 events each.
chain: 2+2c column c available, 3+2c panel c done
worker: 1 dist landed, 2c generation + lookahead of column c done (c >= 1),
2c+1 L(c-1) arrived, 16+c column c handed over"""
import sys

import numpy as np

S, B, E, NC = 8, 8, 24, 8
a = np.loadtxt(sys.argv[1], dtype=np.int64)
a = a[-S * 2 * B:].reshape(S, 2, B, E)
cw, cp, gen0, dist, wl, wlast = [], [], [], [], [], []
for s in range(S):
    for b in range(1, B - 1):
        ch, wk = a[s, 0, b], a[s, 1, b]
        if ch[2] == 0:
            continue
        gen0.append(wk[16] - wk[1])
        for c in range(NC):
            cp.append(ch[3 + 2 * c] - ch[2 + 2 * c])
            if c >= 1:
                cw.append(ch[2 + 2 * c] - ch[1 + 2 * c])  # chain idle: panel c-1 done -> column c in
                wl.append(wk[2 * c + 1] - wk[2 * c])      # worker idle waiting for L(c-1)
                wlast.append(wk[16 + c] - wk[2 * c + 1])  # worker: L(c-1) in -> column c out
        if b == 3 and s == 0:
            t0 = wk[1]
            print("chain  ev:", [int(x - t0) for x in ch[:2 + 2 * NC]])
            print("worker ev:", [int(x - t0) for x in wk[2:16]], [int(x - t0) for x in wk[17:24]])
r = lambda v, k: np.array(v).reshape(-1, k).mean(0).round()
print(f"worker gen(0) {np.mean(gen0):.0f}")
print(f"chain panel     mean {np.mean(cp):6.0f} by column {r(cp, NC)}")
print(f"chain idle      mean {np.mean(cw):6.0f} by column {r(cw, NC - 1)}")
print(f"worker idle(L)  mean {np.mean(wl):6.0f} by column {r(wl, NC - 1)}")
print(f"worker L->col   mean {np.mean(wlast):6.0f} by column {r(wlast, NC - 1)}")
c2 = a[:, 0, 1:B - 1, :]
print("panel 2 split: loads %.0f  pivots %.0f  ballot+stores %.0f  arrive %.0f" % (
    (c2[..., 18] - c2[..., 6]).mean(), (c2[..., 19] - c2[..., 18]).mean(),
    (c2[..., 20] - c2[..., 19]).mean(), (c2[..., 7] - c2[..., 20]).mean()))
blk = [a[s, 0, b + 1, 2] - a[s, 0, b, 2] for s in range(S) for b in range(1, B - 2)]
print(f"block period mean {np.mean(blk):.0f} cycles")
