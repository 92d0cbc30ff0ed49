"""Per-source-line stall samples / executed instructions from an ncu report
(cuda,sass source view).  usage: ncu_lines.py REP [topN]"""
import csv, io, subprocess, sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
f = None
rows = []
hdr = None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if r[0] and r[0].isdigit() and hdr:
        try:
            samp = int(r[4]); inst = int(r[7])
        except ValueError:
            continue
        rows.append((samp, inst, f, int(r[0]), r[1].strip()[:70]))
tot = sum(x[0] for x in rows) or 1
rows.sort(reverse=True)
for s, i, f, ln, src in rows[:top]:
    print(f"{100*s/tot:5.1f}%  inst={i:>12}  {f}:{ln}  {src}")
