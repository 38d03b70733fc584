#!/usr/bin/env python
"""Top stalled SASS lines of an ncu report:  python scripts/ncu_hot.py report.ncu-rep [N]"""
import csv
import subprocess
import sys

rep, top = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 16
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout.splitlines()
rows = list(csv.reader(out[1:]))
h = rows[0]
i_src, i_st = h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
body = [r for r in rows[1:] if len(r) > i_st]
tot = sum(float(r[i_st] or 0) for r in body)
for r in sorted(body, key=lambda r: -float(r[i_st] or 0))[:top]:
    print(f"{float(r[i_st]) / tot * 100:5.1f}%  {r[i_src].strip()[:100]}")
