"""Attribute ncu per-SASS-instruction stall samples to CUDA source lines.

  python tools/ncu_lines.py <object.o> <kernel-mangled-substring> <ncu source csv> [top]

The ncu source page (--page source --csv --print-source sass) carries
runtime addresses; nvdisasm -g on the object's cubin gives offset -> line.
"""
import csv
import os
import re
import subprocess
import sys
import tempfile
from collections import defaultdict

obj, kname, csvp = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=tmp, check=True,
               capture_output=True)
cubin = [f for f in os.listdir(tmp) if f.endswith(".cubin")][0]
dis = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(tmp, cubin)], capture_output=True,
                     text=True).stdout.splitlines()
line_of = {}
inside = False
cur = None
for ln in dis:
    if ln.startswith("//----") and ".text." in ln:
        inside = kname in ln
        continue
    if not inside:
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
    if m:
        cur = (os.path.basename(m.group(1)), int(m.group(2)))
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/", ln)
    if m and cur:
        line_of[int(m.group(1), 16)] = cur
rows = list(csv.reader(open(csvp)))
hdr = rows[1]
data = [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr)]
base = int(data[0]["Address"], 16)
key = "Warp Stall Sampling (All Samples)"
stall_cols = [k for k in hdr if k.startswith("stall_") and "Not Issued" not in k]
agg = defaultdict(float)
inst = defaultdict(float)
reasons = defaultdict(lambda: defaultdict(float))
for d in data:
    off = int(d["Address"], 16) - base
    loc = line_of.get(off, ("?", 0))
    agg[loc] += float(d[key] or 0)
    inst[loc] += float(d["Instructions Executed"] or 0)
    for k in stall_cols:
        reasons[loc][k] += float(d[k] or 0)
tot = sum(agg.values())
srcs = {}
for loc, v in sorted(agg.items(), key=lambda kv: -kv[1])[:top]:
    f, l = loc
    if f not in srcs:
        path = next((os.path.join(dp, f) for dp, _, fs in os.walk("paper_2403_07412_b200") if f in fs), None)
        srcs[f] = open(path).read().splitlines() if path else []
    text = srcs[f][l - 1].strip()[:70] if 0 < l <= len(srcs[f]) else ""
    rs = sorted(reasons[loc].items(), key=lambda kv: -kv[1])[:2]
    rtxt = " ".join(f"{k[6:]}:{v / max(agg[loc], 1):.2f}" for k, v in rs)
    print(f"{v / tot:6.3f} {inst[loc]:9.2e} {f}:{l:<5} {rtxt:32s} {text}")
