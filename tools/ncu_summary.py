"""Summarise an ncu report: headline metrics, per-opcode executed instructions
and stall samples from the SASS source page (run where ncu is installed)."""
import collections
import csv
import io
import json
import re
import subprocess
import sys


def page(rep, name, extra=()):
    out = subprocess.run(["ncu", "-i", rep, "--page", name, "--csv", *extra],
                         capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main(rep, blocks=None, out_json=None):
    rows = page(rep, "raw")
    hdr, units, vals = rows[0], rows[1], rows[2]
    raw = {k: (f"{v} {u}".strip() if u else v) for k, u, v in zip(hdr, units, vals)}
    keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "sm__inst_executed_pipe_fp64.sum", "smsp__inst_executed.sum",
            "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
            "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct"]
    summary = {k: raw.get(k) for k in keys if k in raw}
    for k in hdr:
        if "pipe_fp64" in k and "pct" in k:
            summary[k] = raw[k]
    src = page(rep, "source", ["--print-source", "sass"])
    h = src[1]
    iS, iE = h.index("Source"), h.index("Instructions Executed")
    iW = h.index("Warp Stall Sampling (All Samples)")
    ops, stalls = collections.Counter(), collections.Counter()
    tot = totw = 0
    for r in src[2:]:
        if len(r) <= iE:
            continue
        m = re.match(r"(@!?U?P\w+\s+)?([A-Z0-9_]+)(\.[A-Z0-9_.]+)?", r[iS].strip())
        if not m:
            continue
        op = m.group(2)
        n = int(r[iE] or 0)
        w = int(r[iW] or 0)
        ops[op] += n
        stalls[op] += w
        tot += n
        totw += w
    summary["sass_instructions_total"] = tot
    if blocks:
        summary["sass_instructions_per_block"] = tot / blocks
        summary["opcodes_per_block"] = {k: round(v / blocks, 1) for k, v in ops.most_common(30)}
    summary["stall_share_by_opcode"] = {k: round(v / max(totw, 1), 3) for k, v in stalls.most_common(15)}
    stall = {}
    for k in hdr:
        if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
            try:
                stall[k.replace("smsp__pcsamp_warps_issue_stalled_", "")] = int(raw[k].split()[0].replace(",", ""))
            except ValueError:
                pass
    st = sum(stall.values()) or 1
    summary["stall_reasons"] = {k: round(v / st, 3) for k, v in sorted(stall.items(), key=lambda x: -x[1]) if v}
    print(json.dumps(summary, indent=1))
    if out_json:
        json.dump(summary, open(out_json, "w"), indent=1)


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else None,
         sys.argv[3] if len(sys.argv) > 3 else None)
