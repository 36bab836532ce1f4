"""Per-kernel key metrics of an `ncu --set full` capture exported with
`ncu -i rep --page raw --csv` -> markdown table.
  python tools/ncu_full_summary.py <raw.csv> > profiles/<name>.md"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h, data = rows[0], rows[2:]
cols = [("gpu__time_duration.sum", "us", 1.0),
        ("dram__bytes_read.sum", "DRAM rd MB", 1.0),
        ("dram__bytes_write.sum", "DRAM wr MB", 1.0),
        ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % peak", 1.0),
        ("lts__t_sector_hit_rate.pct", "L2 hit %", 1.0),
        ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM % peak", 1.0),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %", 1.0),
        ("launch__grid_size", "grid", 1.0),
        ("launch__registers_per_thread", "regs", 1.0),
        ("smsp__inst_executed.sum", "warp instr (k)", 1e-3)]
idx = [(h.index(c), name, sc) for c, name, sc in cols if c in h]
print("| kernel | " + " | ".join(n for _, n, _ in idx) + " |")
print("|---" * (len(idx) + 1) + "|")
for d in data:
    name = d[h.index("Kernel Name")].split("(")[0]
    vals = []
    for i, _, sc in idx:
        try:
            v = float(d[i].replace(",", "")) * sc
            vals.append(f"{v:.1f}" if abs(v) < 1e4 else f"{v:.0f}")
        except ValueError:
            vals.append(d[i])
    print(f"| {name} | " + " | ".join(vals) + " |")
