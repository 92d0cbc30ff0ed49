"""Summarise the warp-specialised kernel's clock64 trace (VGP_TRACE=<file>).
Rows: pair x role (0 chain, 1 worker) x block, 24 events each."""
import sys
import numpy as np

import os
P, B, E = int(os.environ.get("SLOTS", 4)), 8, 24
a = np.loadtxt(sys.argv[1], dtype=np.int64)
a = a[-P * 2 * B:].reshape(P, 2, B, E)
NC = 8
cw, cp, ww, wb = [], [], [], []
for p in range(P):
    for b in range(1, B - 1):  # skip the first block (cold start)
        ch, wk = a[p, 0, b], a[p, 1, b]
        if ch[1] == 0 or wk[0] == 0:
            continue
        for c in range(NC):
            cw.append(ch[2 * c + 1] - ch[2 * c])  # chain waiting for column c
            end = ch[2 * c + 2] if c + 1 < NC else ch[20]
            cp.append(end - ch[2 * c + 1])  # chain panel c (incl. L write)
        for c in range(1, NC):
            ww.append(wk[3 + 2 * c] - wk[2 + 2 * c])  # worker waiting for L(c-1)
        wb.append(wk[1] - wk[0])  # worker block start (O stage + TMA wait)
        if b == 3 and p == 0:
            t0 = wk[0]
            print("worker ev:", [int(x - t0) for x in wk[:18]])
            print("chain  ev:", [int(x - t0) for x in ch[:17]] + [int(ch[20] - t0)])
cw, cp, ww, wb = map(np.array, (cw, cp, ww, wb))
print(f"chain wait per column  mean {cw.mean():7.0f}  by column {np.array(cw).reshape(-1, NC).mean(0).round()}")
print(f"chain panel per column mean {cp.mean():7.0f}  by column {np.array(cp).reshape(-1, NC).mean(0).round()}")
print(f"worker wait for L      mean {ww.mean():7.0f}  by column {np.array(ww).reshape(-1, NC - 1).mean(0).round()}")
print(f"worker block start     mean {wb.mean():7.0f}")
blk = [a[p, 0, b + 1, 20] - a[p, 0, b, 20] for p in range(P) for b in range(1, B - 2)]
print(f"block period (chain epilogue to epilogue) mean {np.mean(blk):.0f} cycles")
