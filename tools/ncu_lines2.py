"""Per-SASS-instruction stall breakdown for the hottest instructions.
usage: ncu_lines2.py REP [topN]"""
import csv, io, subprocess, sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
iS, iW = h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
stalls = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
idx = [h.index(k) for k in stalls]
data = []
for i, r in enumerate(rows[2:]):
    if len(r) <= iW or not r[iW].isdigit():
        continue
    w = int(r[iW])
    br = sorted(((int(r[j]) if r[j].isdigit() else 0, k[6:]) for j, k in zip(idx, stalls)), reverse=True)[:3]
    data.append((w, i, r[iS].strip()[:60], br))
tot = sum(d[0] for d in data) or 1
for w, i, src, br in sorted(data, reverse=True)[:top]:
    print(f"{100*w/tot:5.1f}% #{i:5d} {src:60s} " + " ".join(f"{k}={100*v/max(w,1):.0f}%" for v, k in br))
