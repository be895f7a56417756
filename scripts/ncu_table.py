"""Summarise ncu --set full reports (gpurun_out/full_*.ncu-rep) as a markdown
table: duration, DRAM bytes and throughput, occupancy, issue activity and the
top stall reasons per kernel."""
import csv
import io
import subprocess
import sys
from pathlib import Path

out = Path(__file__).resolve().parents[1] / "gpurun_out"
rows = []
reps = [Path(a) for a in sys.argv[1:]] or sorted(out.glob("full_*.ncu-rep"))
for rep, h, u, v in ((rep, *hdr, v) for rep in reps
                     for hdr, vals in [(lambda r: ((r[0], r[1]), r[2:]))(list(csv.reader(io.StringIO(
                         subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True,
                                        text=True).stdout))))] for v in vals):
    m = dict(zip(h, v))
    unit = dict(zip(h, u))

    def g(name, scale=1.0):
        x = m.get(name, "")
        try:
            return float(x.replace(",", "")) * scale
        except ValueError:
            return float("nan")
    dur_us = g("gpu__time_duration.sum") * {"ns": 1e-3, "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3,
                                             "s": 1e6, "second": 1e6}.get(unit.get("gpu__time_duration.sum"), 1.0)
    def mb(name):
        s = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}.get(unit.get(name, ""), float("nan"))
        return g(name) * s
    rd, wr = mb("dram__bytes_read.sum"), mb("dram__bytes_write.sum")
    stalls = sorted(((g(k), k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""))
                     for k in h if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")
                     and "not_issued" not in k and "selected" not in k), reverse=True)[:2]
    rows.append((m.get("Kernel Name", rep.stem)[:48], dur_us, rd, wr, (rd + wr) / dur_us if dur_us else 0,
                 g("launch__registers_per_thread"), g("sm__warps_active.avg.pct_of_peak_sustained_active"),
                 g("smsp__issue_active.avg.pct_of_peak_sustained_active"),
                 ", ".join(f"{n} {x:.1f}" for x, n in stalls)))
print("| kernel | us | DRAM rd MB | DRAM wr MB | DRAM TB/s | regs | warps active % | issue active % | top stalls (cycles/issue) |")
print("|---|---:|---:|---:|---:|---:|---:|---:|---|")
for k in rows:
    print(f"| {k[0]} | {k[1]:.1f} | {k[2]:.1f} | {k[3]:.1f} | {k[4]:.2f} | {k[5]:.0f} | {k[6]:.1f} | {k[7]:.1f} | {k[8]} |")
