#!/usr/bin/env python
"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list into a markdown table.

usage: python tools/launch_list.py LAUNCHES.csv OUT.md "title"
"""
import collections
import csv
import sys

src, out, title = sys.argv[1], sys.argv[2], sys.argv[3]
rows = [r for r in csv.reader(open(src)) if len(r) > 14 and r[12] == "gpu__time_duration.sum"]
agg = collections.OrderedDict()
for r in rows:
    agg.setdefault(r[4], []).append(float(r[14]) / 1000)
tot = sum(sum(v) for v in agg.values()) or 1.0
lines = [f"# {title}", "",
         "`ncu --metrics gpu__time_duration.sum --clock-control none -c 400` (cold-cache, serialised: compare shares).", "",
         "| kernel | launches | mean us | share of GPU time |", "|---|---|---|---|"]
for k, v in sorted(agg.items(), key=lambda t: -sum(t[1])):
    lines.append(f"| {k} | {len(v)} | {sum(v) / len(v):.1f} | {100 * sum(v) / tot:.1f}% |")
open(out, "w").write("\n".join(lines) + "\n")
print("\n".join(lines))
