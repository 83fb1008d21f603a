"""Summarise an ncu --page source (SASS) export: top stall sites with the preceding
SYNCS/barrier instruction for context.  Usage: ncu_src_summary.py report.ncu-rep"""
import csv
import io
import re
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
data = [dict(zip(hdr, r)) for r in rows[2:]]
col = "Warp Stall Sampling (All Samples)"
tot = sum(float(d[col] or 0) for d in data)
print(f"total samples {tot:.0f}")
for i, d in sorted(enumerate(data), key=lambda p: -float(p[1][col] or 0))[:int(sys.argv[2]) if len(sys.argv) > 2 else 20]:
    ctx = ""
    for j in range(i, max(0, i - 8), -1):
        if "SYNCS" in data[j]["Source"] or "BAR" in data[j]["Source"] or "LDTM" in data[j]["Source"]:
            ctx = data[j]["Source"].strip()[:70]
            break
    print(f"{float(d[col] or 0)/tot*100:5.1f}% {d['Instructions Executed']:>8} {d['Source'].strip()[:60]:60s} | {ctx}")
