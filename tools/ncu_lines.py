#!/usr/bin/env python
"""Per-source-line instruction counts and stall samples of an ncu report (source page, cuda+sass).

usage: python tools/ncu_lines.py REPORT.ncu-rep [top]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
res, fname, hdr = [], None, None
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8 or r[0] == "" or r[0] == "Function Name":
        continue
    try:
        inst = int(r[hdr.index("Instructions Executed")] or 0)
        samp = int(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
    except ValueError:
        continue
    res.append((inst, samp, f"{fname}:{r[0]}", r[1].strip()[:90]))
tot_i = sum(x[0] for x in res) or 1
tot_s = sum(x[1] for x in res) or 1
print(f"total warp instructions {tot_i}, stall samples {tot_s}")
for inst, samp, loc, src in sorted(res, reverse=True)[:top]:
    print(f"{100*inst/tot_i:5.1f}% inst {100*samp/tot_s:5.1f}% samp  {loc:24s} {src}")
