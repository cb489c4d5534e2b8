"""Print the SASS of a source-line range with per-instruction execution counts.
Usage: python scripts/ncu_sass.py report.ncu-rep file.cuh LO HI [min_count]"""
import csv
import subprocess
import sys

rep, fname, lo, hi = sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4])
mn = int(sys.argv[5]) if len(sys.argv) > 5 else 1
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
cur_file, line = "?", None
for r in csv.reader(txt.splitlines()):
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No" or r[0] == "Function Name":
        continue
    if r[0].isdigit():
        line = int(r[0])
        if cur_file == fname and lo <= line <= hi:
            print(f"--- {line}: {r[1][:90]}")
        continue
    if len(r) > 10 and r[2].startswith("0x") and cur_file == fname and line and lo <= line <= hi:
        n = int(r[7] or 0)
        if n >= mn:
            print(f"    {n:9d} {r[10]:>5s}  {r[3].strip()[:80]}")
