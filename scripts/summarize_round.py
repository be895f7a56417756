"""Regenerate the measured summary of a round from a round check
(scripts/round_gpu.sh): the bench line and the ncu launch list.

    python scripts/summarize_round.py [r2]

r1 rewrites profiles/r1_summary.md keeping its hand-written sections from
"## ncu --set full" on; r2 writes profiles/r2/summary.md (bench line, launch
list, per-kernel table) and points at the per-kernel notes in profiles/r2/."""
import collections
import csv
import json
import shutil
import sys
from pathlib import Path

root = Path(__file__).resolve().parents[1]
out = root / "gpurun_out"
rnd = sys.argv[1] if len(sys.argv) > 1 else "r1"
prof = root / "profiles" if rnd == "r1" else root / "profiles" / rnd
names = {"bench": "r1_bench_line.json", "launches": "r1_launches.csv", "summary": "r1_summary.md"} if rnd == "r1" \
    else {"bench": "bench_line.json", "launches": "launches.csv", "summary": "summary.md"}
bench = json.loads((out / "bench.json").read_text().strip().splitlines()[-1])
shutil.copy(out / "bench.json", prof / names["bench"])
shutil.copy(out / "launches.csv", prof / names["launches"])
tests = (out / "gputests.log").read_text().strip().splitlines()[-1] if (out / "gputests.log").exists() else "?"

rows = [r for r in csv.reader(open(out / "launches.csv")) if len(r) > 10]
h = rows[0]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[1:]:
    name = r[ki].split("(")[0].replace("void ", "")
    agg[name][0] += 1
    agg[name][1] += float(r[vi].replace(",", ""))
total = sum(v[1] for v in agg.values())

rf, e2e = bench["roofline"], bench["e2e"]
rel = "profiles/" if rnd == "r1" else f"profiles/{rnd}/"
L = [f"# Round {rnd[1:]} profile summary (B200, sm_100a)", "",
     "Sources (all N = 1, one B200):",
     f"* `{rel}{names['bench']}` — the default `python bench.py` line of the",
     f"  last round check (`pytest -m gpu` in the same call: {tests}).",
     f"* `{rel}{names['launches']}` — ncu `--metrics gpu__time_duration.sum",
     "  --clock-control none` launch list of `python bench.py --no-cpu --steps 2",
     f"  --warmup 1` ({len(rows) - 1} launches; cold-cache and serialised: compare shares).",
     "* per-kernel `ncu --set full` captures (reports in gpurun_out/, metrics",
     "  below); `profiles/hotspot_traffic.json` for the headline kernel.", "",
     "## Headline (hotspot 8192^2 f32, 100 launches per step through Runtime.launch)", "",
     "| | value |", "|---|---|",
     f"| value (device, CUDA events on the worker stream) | {bench['value']} GB/s ({bench['ms_per_step']} ms per 100 iterations) |",
     f"| roofline | {rf['kernel']} avg launch {rf['avg_launch_us']} us, {rf['achieved']} GB/s of {rf['peak']} measured = {rf['frac']} |",
     f"| DRAM traffic per launch (ncu) | {rf['traffic']} B (algorithmic 805,306,368) |",
     f"| e2e (pinned host buffers, H2D + 100 launches + D2H per step) | {e2e['value']} GB/s pipelined, {e2e.get('serial_value')} GB/s serial |",
     f"| fused driver (bf_hotspot_run, register-wavefront temporal blocking) | {bench.get('hotspot_fused', {}).get('value', bench.get('hotspot_fused'))} GB/s algorithmic |",
     f"| CPU port (oracle.c, OpenMP, host cores) | {bench['cpu_baseline']['value']} {bench['cpu_baseline']['unit']} |",
     f"| clocks | {bench['clocks']} |", "",
     f"## Launch list shares (`{rel}{names['launches']}`)", "",
     "| kernel | launches | avg us (ncu) | share |", "|---|---:|---:|---:|"]
for name, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:16]:
    L.append(f"| {name[:90]} | {n} | {t / n / 1e3:.1f} | {100 * t / total:.1f} % |")
L += ["", f"Inside the headline's timed region only {rf['kernel']} runs (100 launches per",
      "step, share 100 %).", "",
      "## Per-kernel table (CUDA events, N = 1, fraction of the measured HBM peak)", "",
      "| case | GB/s | frac | elements/s | ms/step | full-size check |", "|---|---:|---:|---|---:|---|"]
for k, v in bench["kernels"].items():
    eps = next((f"{x:.3g} {key[:-6].replace('_', ' ')}/s" for key, x in v.items() if key.endswith("_per_s")), "")
    L.append(f"| {k} | {v['gbs']} | {v['frac_hbm']} | {eps} | {v['ms_per_step']} | {v['checked']} |")
if rnd == "r1":
    old = (prof / "r1_summary.md").read_text()
    keep = old[old.index("## ncu --set full, per kernel"):]
else:
    keep = ("## ncu --set full, per kernel\n\n"
            "* `hotspot.md` — the headline kernel (hotspot_rows) and its variants.\n"
            "* `bfs.md`, `bfs_do_launches.txt` — the direction-optimizing traversal level by level.\n"
            "* `kmeans.md`, `kmeans_tg_sass.txt`, `umma_sw128_probe.log`, `umma_bf16_probe.log`, `umma_rate.log` — kmeans_tg (tcgen05) and its probes.\n"
            "* `sanitizer_summary.md` — compute-sanitizer memcheck / racecheck / synccheck / initcheck.\n"
            "* `grain_host_vs_device_fetch.json` — the fetch-grain study with host-issued and device-side fetching.\n")
(prof / names["summary"]).write_text("\n".join(L) + "\n\n" + keep)
print("ok")
