#!/usr/bin/env python3
"""Warp-stall samples of an ncu report aggregated by CUDA source line
(ncu --page source --print-source cuda,sass), top N.
usage: python tools/ncu_lines.py report.ncu-rep [N]"""
import collections
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True, check=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = next(r for r in rows if r and r[0] == "Line No")
i_s = hdr.index("Warp Stall Sampling (All Samples)")
agg, src, cur, fname = collections.Counter(), {}, None, ""
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
    if not r or r[0] in ("File Path", "Function Name", "Line No") or len(r) <= i_s:
        continue
    if r[0]:
        cur = (fname, int(r[0]))
        src[cur] = r[1].strip()
    if r[i_s].isdigit() and cur:
        agg[cur] += int(r[i_s])
tot = sum(agg.values())
print(f"total samples {tot}")
for (f, ln), n in agg.most_common(top):
    print(f"{n:7d} {100 * n / tot:5.1f}%  {f}:{ln:<5d} {src[(f, ln)][:90]}")
