"""Summarise an ncu launch list (gpu__time_duration + dram bytes per launch, CSV) into a
markdown table and the per-kernel traffic file bench.py reads:
  python tools/summarize_launches.py <launches.csv> <out.md> [profiles/ncu_traffic.json]"""
import csv
import json
import sys
from collections import OrderedDict, defaultdict

src, out_md = sys.argv[1], sys.argv[2]
out_json = sys.argv[3] if len(sys.argv) > 3 else None
rows = list(csv.DictReader(l for l in open(src) if not l.startswith("==")))
per = OrderedDict()
for r in rows:
    k = (r["ID"], r["Kernel Name"].split("(")[0].replace("am::", ""))
    per.setdefault(k, {})[r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
agg = defaultdict(lambda: {"n": 0, "us": 0.0, "rd": 0.0, "wr": 0.0})
for (_, name), m in per.items():
    a = agg[name]
    a["n"] += 1
    a["us"] += m.get("gpu__time_duration.sum", 0.0) / 1000.0   # ns -> us
    a["rd"] += m.get("dram__bytes_read.sum", 0.0)
    a["wr"] += m.get("dram__bytes_write.sum", 0.0)
rounds = max(a["n"] for a in agg.values())
tot = sum(a["us"] for a in agg.values()) / rounds
lines = ["| kernel | launches/round | ncu us / launch | share of serialised round | DRAM read MB / launch | DRAM write MB / launch |",
         "|---|---|---|---|---|---|"]
for name, a in sorted(agg.items(), key=lambda kv: -kv[1]["us"]):
    n = a["n"]
    lines.append(f"| {name} | {n / rounds:.0f} | {a['us'] / n:.1f} | {a['us'] / rounds / tot * 100:.1f}% | "
                 f"{a['rd'] / n / 1e6:.2f} | {a['wr'] / n / 1e6:.2f} |")
lines.append(f"| **serialised round** | | {tot:.1f} | | | |")
open(out_md, "w").write("\n".join(lines) + "\n")
print("\n".join(lines))
if out_json:
    tj = {"source": f"ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
                    f"--clock-control none (cache control all: cold-cache DRAM bytes) on tools/profile_round.py C5, "
                    f"{rounds} steady-state replay rounds ({src})"}
    for name, a in agg.items():
        n = a["n"]
        tj[name] = {"dram_bytes_per_launch": (a["rd"] + a["wr"]) / n, "launches": n / rounds, "us": a["us"] / n}
    if "k_scan_hw" in tj:
        tj["k_scan"] = dict(tj["k_scan_hw"], note="k_scan_hw (timed as k_scan by bench.py)")
    if "k_efilter" in tj:
        tj["k_near"] = dict(tj["k_efilter"], note="k_efilter (timed as k_near by bench.py)")
    json.dump(tj, open(out_json, "w"), indent=1)
