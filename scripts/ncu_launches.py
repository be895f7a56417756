"""Summarise an ncu --csv launch list (one row per launch and metric) into
one line per launch: id, kernel, grid, time (us), DRAM read/write (MB), L2 sectors (M)."""
import csv
import sys
from collections import OrderedDict

rows = OrderedDict()
with open(sys.argv[1]) as f:
    lines = [l for l in f if l.startswith('"')]
for r in csv.DictReader(lines):
    k = (r["ID"], r["Kernel Name"].split("(")[0], r["Grid Size"])
    rows.setdefault(k, {})[r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
tot = 0.0
for (i, name, grid), m in rows.items():
    t = m.get("gpu__time_duration.sum", 0) / 1e3
    tot += t
    print(f"{i:>4} {name[:40]:40s} {grid:>14s} {t:9.1f} us  rd {m.get('dram__bytes_read.sum', 0)/1e6:9.1f} MB"
          f"  wr {m.get('dram__bytes_write.sum', 0)/1e6:8.1f} MB  l2 {m.get('lts__t_sectors.sum', 0)/1e6:8.1f} M")
print(f"total {tot:.1f} us over {len(rows)} launches")
