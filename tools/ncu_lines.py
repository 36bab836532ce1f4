"""Per-CUDA-source-line warp-stall samples and executed instructions of one kernel in an
ncu report:  python tools/ncu_lines.py <report> <kernel-regex> [top]"""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows, hdr, fname = [], None, ""
for ln in csv.reader(out.splitlines()):
    if len(ln) == 2 and ln[0] == "File Path":
        fname = ln[1].split("/")[-1]
        continue
    if ln and ln[0] == "Line No":
        hdr = ln
        continue
    if hdr and ln and ln[0] not in ("",) and ln[0].isdigit():
        try:
            rows.append((float(ln[4] or 0), float(ln[7] or 0), fname, ln[0], ln[1]))
        except ValueError:
            pass
tot = sum(r[0] for r in rows) or 1
itot = sum(r[1] for r in rows) or 1
print(f"total samples {tot:.0f}, warp instructions {itot:.0f}")
for s, i, f, l, src in sorted(rows, reverse=True)[:top]:
    print(f"{s / tot * 100:5.1f}% smp {i / itot * 100:5.1f}% ins  {f}:{l}: {src.strip()[:90]}")
