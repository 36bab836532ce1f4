"""Top source lines of one kernel in an ncu --set full report (--import-source on, built
with -lineinfo): warp instructions executed and stall samples per CUDA source line.
  python tools/ncu_source_top.py <report.ncu-rep> <kernel-regex> [top] > out.md"""
import csv
import io
import subprocess
import sys

rep, rx = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{rx}",
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
cur, hdr, lines = None, None, []
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if len(r) >= 2 and r[0] == "Line No":
        hdr = r
        continue
    if hdr and r and r[0] not in ("", "Function Name"):
        try:
            ln = int(r[0])
            ie = int(r[hdr.index("Instructions Executed")] or 0)
            st = int(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
        except ValueError:
            continue
        lines.append((cur, ln, ie, st, r[1].strip()[:100]))
ti = sum(x[2] for x in lines) or 1
ts = sum(x[3] for x in lines) or 1
print(f"# {rx}: top source lines ({rep})\n")
print(f"warp instructions executed: {ti}, stall samples: {ts}\n")
print("| file:line | instructions | stall samples | source |")
print("|---|---|---|---|")
for x in sorted(lines, key=lambda t: -t[2])[:top]:
    src = x[4].replace("|", "\\\\|")
    print(f"| {x[0]}:{x[1]} | {x[2] / ti * 100:.1f}% | {x[3] / ts * 100:.1f}% | `{src}` |")
