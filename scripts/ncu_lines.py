"""Summarise an ncu source page (cuda,sass CSV) by source line: stall samples and
executed warp instructions. Usage: python scripts/ncu_lines.py report.ncu-rep [top]"""
import csv
import subprocess
import sys

import os

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
by = 1 if os.environ.get("NCU_BY") == "inst" else 0   # NCU_BY=inst: sort by executed instructions
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(txt.splitlines()))
agg = {}
cur_file = "?"
hdr = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] in ("Function Name",):
        continue
    if r[0]:  # source line row (aggregated metrics for the line)
        d = dict(zip(hdr[2:], r[2:]))
        key = (cur_file, int(r[0]))
        try:
            samp = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
            inst = int(d.get("Instructions Executed", "0") or 0)
        except ValueError:
            continue
        a = agg.setdefault(key, [0, 0, r[1][:70]])
        a[0] += samp
        a[1] += inst
tot_s = sum(v[0] for v in agg.values()) or 1
tot_i = sum(v[1] for v in agg.values()) or 1
print(f"total samples {tot_s}  total warp-instr {tot_i}")
for (f, ln), (s, i, src) in sorted(agg.items(), key=lambda kv: -kv[1][by])[:top]:
    print(f"{100*s/tot_s:5.1f}% smp {100*i/tot_i:5.1f}% inst  {f}:{ln:<4d} {src}")

if len(sys.argv) > 3:
    # phase breakdown: name=file:lo-hi,...
    phases = {}
    for spec in sys.argv[3].split(","):
        name, rng = spec.split("=")
        f, lohi = rng.split(":")
        lo, hi = (int(x) for x in lohi.split("-"))
        phases[name] = (f, lo, hi)
    out = {k: [0, 0] for k in phases}
    out["other"] = [0, 0]
    for (f, ln), (s, i, _) in agg.items():
        for name, (pf, lo, hi) in phases.items():
            if f == pf and lo <= ln <= hi:
                out[name][0] += s
                out[name][1] += i
                break
        else:
            out["other"][0] += s
            out["other"][1] += i
    for k, (s, i) in out.items():
        print(f"{k:12s} {100*s/tot_s:5.1f}% samples {100*i/tot_i:5.1f}% inst ({i} warp-instr)")
