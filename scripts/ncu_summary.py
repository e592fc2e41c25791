"""Markdown table of the key counters of `ncu --page raw --csv` exports:
kernel, duration, DRAM read / write, dram cycles active avg / max / min.
  python scripts/ncu_summary.py profiles/round2/ncu3/*_raw.csv"""
import csv
import os
import sys

COLS = [("gpu__time_duration.sum", "time"), ("dram__bytes_read.sum", "DRAM read"),
        ("dram__bytes_write.sum", "DRAM write"),
        ("dram__cycles_active.avg.pct_of_peak_sustained_elapsed", "active avg %"),
        ("dram__cycles_active.max.pct_of_peak_sustained_elapsed", "max %"),
        ("dram__cycles_active.min.pct_of_peak_sustained_elapsed", "min %")]
print("| capture | kernel | " + " | ".join(c[1] for c in COLS) + " |")
print("|" + "---|" * (len(COLS) + 2))
for path in sys.argv[1:]:
    rows = list(csv.reader(open(path)))
    if len(rows) < 3:
        continue
    h, u = rows[0], rows[1]
    for r in rows[2:]:
        cells = []
        for c, _ in COLS:
            i = h.index(c)
            unit = u[i] if u[i] != "%" else ""
            cells.append(f"{r[i]} {unit}".strip())
        k = r[h.index("Kernel Name")].split("(")[0]
        print(f"| {os.path.basename(path).replace('_raw.csv', '')} | `{k}` | " + " | ".join(cells) + " |")
