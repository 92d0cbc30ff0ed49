"""Split an ncu source-page (SASS) CSV into warp-role regions and sum stall
samples per reason: worker region = span of DMMA instructions, chain region =
span of MUFU.RSQ64H; usage: python tools/ncu_regions.py src.csv"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
data = [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr)]
idx = {k: i for i, k in enumerate(hdr)}
addrs = [int(d["Address"], 16) for d in data]
src = [d["Source"].strip() for d in data]
dm = [a for a, s in zip(addrs, src) if s.startswith("DMMA")]
mu = [a for a, s in zip(addrs, src) if "MUFU.RSQ64H" in s]
regions = {"worker": (min(dm), max(dm)), "chain": (min(mu), max(mu))}
stall_cols = [k for k in hdr if k.startswith("stall_") and "Not Issued" not in k]
agg = defaultdict(lambda: defaultdict(float))
inst = defaultdict(float)
ops = defaultdict(lambda: defaultdict(float))
for a, s, d in zip(addrs, src, data):
    reg = "other"
    for name, (lo, hi) in regions.items():
        if lo - 4096 <= a <= hi + 4096:
            reg = name
    for k in stall_cols:
        agg[reg][k] += float(d[k] or 0)
    n = float(d["Instructions Executed"] or 0)
    inst[reg] += n
    ops[reg][s.split()[0].split(".")[0] if s else "?"] += n
for reg in agg:
    tot = sum(agg[reg].values())
    print(f"== {reg}: samples {tot:.0f}, warp-instructions {inst[reg]:.3e}")
    for k, v in sorted(agg[reg].items(), key=lambda kv: -kv[1])[:8]:
        print(f"   {k:24s} {v / max(tot, 1):.3f}")
    top = sorted(ops[reg].items(), key=lambda kv: -kv[1])[:14]
    print("   ops:", ", ".join(f"{k} {v:.2e}" for k, v in top))
