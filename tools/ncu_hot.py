"""Print the hottest SASS lines (warp-stall samples) of one kernel in an ncu report."""
import csv
import re
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                      "--print-source", "sass"], capture_output=True, text=True).stdout
lines = out.splitlines()
r = csv.reader(lines[1:])
h = next(r)
rows = [x for x in r if len(x) > 3 and re.match(r'^[0-9.]+$', x[3] or '')]
si = h.index("Warp Stall Sampling (All Samples)")
tot = sum(float(x[si] or 0) for x in rows)
for k, row in enumerate(rows):
    row.append(k)
for row in sorted(rows, key=lambda x: -float(x[si] or 0))[:top]:
    print(f"{row[-1]:5d} {float(row[si]) / tot * 100:5.1f}%  {row[1].strip()[:90]}")
