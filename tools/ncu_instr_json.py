"""Per-kernel warp instructions, duration, issue-active and DRAM bytes from an
`ncu --set full` capture (exported with `ncu -i rep --page raw --csv`) merged into
profiles/ncu_instr.json (the issue roofline bench.py reports reads it).
  python tools/ncu_instr_json.py <raw.csv> <source-note> [profiles/ncu_instr.json]"""
import csv
import json
import sys

src, note = sys.argv[1], sys.argv[2]
out = sys.argv[3] if len(sys.argv) > 3 else "profiles/ncu_instr.json"
rows = list(csv.reader(open(src)))
h, units, data = rows[0], rows[1], rows[2:]
col = {c: h.index(c) for c in h}
SCALE = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "second": 1e6,                 # -> us
         "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def val(d, name):
    """The metric in base units (us for times, bytes for sizes) from the units row."""
    try:
        v = float(d[col[name]].replace(",", ""))
    except (KeyError, ValueError):
        return None
    return v * SCALE.get(units[col[name]], 1.0)


try:
    cur = json.load(open(out))
except FileNotFoundError:
    cur = {}
acc = {}
for d in data:
    k = d[col["Kernel Name"]].split("(")[0].replace("am::", "").split("<")[0]
    a = acc.setdefault(k, {"n": 0, "instr": 0.0, "us": 0.0, "act": 0.0, "dram": 0.0})
    a["n"] += 1
    a["instr"] += val(d, "smsp__inst_executed.sum") or 0.0
    a["us"] += val(d, "gpu__time_duration.sum") or 0.0
    a["act"] += (val(d, "sm__issue_active.avg.pct_of_peak_sustained_elapsed")
                 or val(d, "smsp__issue_active.avg.pct_of_peak_sustained_active") or 0.0)
    a["dram"] += ((val(d, "dram__bytes_read.sum") or 0.0) + (val(d, "dram__bytes_write.sum") or 0.0))
for k, a in acc.items():
    n = a["n"]
    cur[k] = {"warp_instructions_per_launch": a["instr"] / n, "ncu_us": a["us"] / n,
              "issue_active_pct": a["act"] / n, "dram_mb": a["dram"] / n / 1e6, "launches_captured": n}
if "k_scan_hw" in acc:
    cur["k_scan"] = dict(cur["k_scan_hw"], note="k_scan_hw (timed as k_scan by bench.py)")
cur["source"] = note
json.dump(cur, open(out, "w"), indent=0)
print({k: (round(v["warp_instructions_per_launch"]), round(v["ncu_us"], 1), round(v.get("dram_mb", 0.0), 1))
       for k, v in cur.items() if isinstance(v, dict) and "warp_instructions_per_launch" in v})
