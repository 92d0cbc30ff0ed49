"""Summarise the short-critical-path kernel's clock64 trace (VGP_TRACE2=<file>)."""
import sys
import numpy as np

P, B, E = 4, 8, 24
a = np.loadtxt(sys.argv[1], dtype=np.int64)
a = a[-P * 2 * B:].reshape(P, 2, B, E)
NC = 8
cw, cp, ww = [], [], []
for p in range(P):
    for b in range(1, B - 1):
        ch, wk = a[p, 0, b], a[p, 1, b]
        if ch[1] == 0 or wk[0] == 0:
            continue
        for c in range(NC):
            cw.append(ch[2 * c + 1] - ch[2 * c])
            end = ch[2 * c + 2] if c + 1 < NC else ch[20]
            cp.append(end - ch[2 * c + 1])
        for c in range(NC - 1):
            ww.append(wk[3 + 2 * c] - wk[2 + 2 * c])
cw, cp, ww = map(np.array, (cw, cp, ww))
print(f"chain wait per column  mean {cw.mean():7.0f}  by column {cw.reshape(-1, NC).mean(0).round()}")
print(f"chain panel per column mean {cp.mean():7.0f}  by column {cp.reshape(-1, NC).mean(0).round()}")
print(f"worker wait for L      mean {ww.mean():7.0f}  by column {ww.reshape(-1, NC - 1).mean(0).round()}")
blk = [a[p, 0, b + 1, 20] - a[p, 0, b, 20] for p in range(P) for b in range(1, B - 2)]
print(f"block period (chain epilogue to epilogue) mean {np.mean(blk):.0f} cycles")
