"""bench.py — B200 throughput of the launch runtime's hot path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload hotspot] [--size 8192] [--iters 100]

Default workload (BASELINE.json configs[1]): hotspot 2D thermal stencil,
8192 x 8192 f32 cells, 100 iterations per step, each iteration one launch of
the `hotspot` kernel through the reference-shaped API (Runtime.launch ->
C ABI -> sm_100a kernel).  Metric: algorithmic HBM GB/s at 12 B per cell and
iteration (read src + power, write dst), plus elements/s.

value  = algorithmic bytes of the K timed steps / device time (CUDA events on
         the worker stream, inputs resident in HBM, max over ranks)
e2e    = the same metric through the public API with host buffers: pinned
         host -> device upload of temp + power, 100 launches, download of the
         final grid, every step
roofline / cpu_baseline / clocks: see DESIGN.md.

`--impl reference` times the CPU reference path (the oracle restatement in
oracle/oracle.c, all host threads) on a bounded sample of the same workload.
Multi-GPU: launched by torchrun, one process per GPU; rows are partitioned in
contiguous bands (the average grain law over ranks) with ghost-zone halos
exchanged over NCCL every `--halo` iterations (paper_2206_07896_b200.parallel).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

BYTES_PER_CELL_ITER = 12  # read src f32 + power f32, write dst f32


def _peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"hbm_gbs": float(d["hbm_gbs"]), "source": "measured (MEASURED_PEAKS.json)"}
    return {"hbm_gbs": 6650.0, "source": "fallback (B200_PROFILING.md)"}


class ClockSampler:
    """SM clocks and clock-event (throttle) reasons sampled during the timed
    region through NVML every ~5 ms (nvidia-smi's -lms polling cannot sample
    a ~100 ms region); falls back to nvidia-smi when NVML is unavailable."""

    REASONS = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"),
               ("hw_power_brake", "nvmlClocksEventReasonHwPowerBrakeSlowdown"))

    def __init__(self, index: int = 0):
        self.index = index
        self.sm: list = []
        self.reasons: set = set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None

    def _run(self, nv, h):
        masks = [(n, getattr(nv, a)) for n, a in self.REASONS if hasattr(nv, a)]
        while not self._stop.is_set():
            try:
                self.sm.append(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                for n, m in masks:
                    if r & m:
                        self.reasons.add(n)
            except Exception:
                pass
            self._stop.wait(0.005)

    def __enter__(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            h = nv.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
            self._t = threading.Thread(target=self._run, args=(nv, h), daemon=True)
            self._t.start()
        except Exception:
            self._t = None
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._t is not None:
            self._t.join(timeout=2)

    def summary(self) -> dict:
        sm = self.sm
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(sm), "source": "nvml"}


# ---------------------------------------------------------------------------
# distributed plumbing
# ---------------------------------------------------------------------------

def dist_env() -> tuple[int, int, int]:
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def max_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world: int) -> None:
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


# ---------------------------------------------------------------------------
# hotspot workload
# ---------------------------------------------------------------------------

def cpu_baseline_hotspot(size: int, iters_full: int, budget_s: float, threads: int) -> dict:
    """The oracle port (oracle/oracle.c, OpenMP over blocks) on a bounded
    sample: the full 8192^2 grid for as many iterations as fit the budget."""
    sys.path.insert(0, str(ROOT / "oracle"))
    import instances as I
    import oracle
    temp, power = I.hotspot_inputs(size, size, 0)
    params = I.hotspot_params(size, size)
    t0 = time.perf_counter()
    oracle.hotspot_iterate(temp, power, size, size, params, 1, nthreads=threads)
    one = time.perf_counter() - t0
    iters = max(1, min(iters_full, int(budget_s / max(one, 1e-6))))
    t0 = time.perf_counter()
    oracle.hotspot_iterate(temp, power, size, size, params, iters, nthreads=threads)
    dt = time.perf_counter() - t0
    gbs = BYTES_PER_CELL_ITER * size * size * iters / dt / 1e9
    return {"value": round(gbs, 4), "unit": "GB/s", "cores": threads, "kind": "port",
            "sample": f"hotspot {size}x{size}, {iters} iteration(s) of {iters_full}, "
                      f"{dt:.2f} s, oracle/oracle.c OpenMP",
            "elem_per_s": size * size * iters / dt}


def run_reference_arm(args) -> None:
    rank, world, _ = dist_env()
    if rank != 0:
        return
    threads = len(os.sched_getaffinity(0))
    steps_t = []
    base = None
    for _ in range(args.warmup):
        cpu_baseline_hotspot(args.size, args.iters, args.cpu_budget / 4, threads)
    for _ in range(args.steps):
        base = cpu_baseline_hotspot(args.size, args.iters, args.cpu_budget, threads)
        steps_t.append(base["value"])
    value = statistics.median(steps_t)
    cells_iter = args.size * args.size * args.iters
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "GB/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": BYTES_PER_CELL_ITER * cells_iter / (value * 1e9) * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": f"hotspot {args.size}x{args.size} f32, {args.iters} iterations",
                   "bytes_per_cell_iter": BYTES_PER_CELL_ITER},
        "cpu_baseline": base,
        "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


METRIC = "per-kernel GB/s & elem/s vs HBM roofline at 1/2/4/8 B200; speedup vs CPU runtime"


def run_ours(args) -> None:
    import torch

    from paper_2206_07896_b200 import ArgSlot, DeviceArena, Dim3, PackedArgs, Runtime, routines
    from paper_2206_07896_b200.parallel import HotspotBands

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    sys.path.insert(0, str(ROOT / "oracle"))
    import instances as I

    size, iters = args.size, args.iters
    params = I.hotspot_params(size, size)
    temp, power = I.hotspot_inputs(size, size, 0)
    bands = HotspotBands(size, size, world, rank, halo=args.halo if world > 1 else 0)
    r0, r1 = bands.local_rows  # global rows held locally (incl. ghost rows)
    lrows = r1 - r0
    arena = DeviceArena(local)
    cells = lrows * size
    routine = routines.get("hotspot")
    bx, by = 16, 16
    grid = Dim3(-(-size // bx), -(-lrows // by))
    block = Dim3(bx, by)
    rt = Runtime(arena, pool_size=1)
    stream = torch.cuda.ExternalStream(rt.worker_stream(0), device=torch.device("cuda", local))

    class BufferSet:
        """src / power / dst of one resident copy of the grid."""

        def __init__(self):
            self.src, self.pow, self.dst = (arena.alloc("f32", cells) for _ in range(3))
            self.packs = [self.slots(self.src, self.dst), self.slots(self.dst, self.src)]
            self.exch = bands.exchanger(arena, stream) if world > 1 else None

        def slots(self, src, dst):
            return PackedArgs([ArgSlot("handle", src), ArgSlot("handle", self.pow), ArgSlot("handle", dst),
                               ArgSlot("i32", lrows), ArgSlot("i32", size), ArgSlot("f32", params["sdc"]),
                               ArgSlot("f32", params["rx1"]), ArgSlot("f32", params["ry1"]),
                               ArgSlot("f32", params["rz1"]), ArgSlot("f32", params["amb"])])

        def step(self, events=None) -> int:
            """One full run: `iters` ping-pong launches (+ halo exchanges);
            returns the handle holding the result."""
            cur = 0
            for it in range(iters):
                if events is not None:
                    events[it][0].record(stream)
                rt.launch(routine, grid, block, 0, self.packs[cur])
                if events is not None:
                    events[it][1].record(stream)
                cur ^= 1
                if self.exch is not None and (it + 1) % bands.halo == 0 and it + 1 < iters:
                    self.exch.exchange(self.dst if cur == 1 else self.src)
            return self.src if cur == 0 else self.dst

    sets = [BufferSet()]
    h_src, h_pow, h_dst = sets[0].src, sets[0].pow, sets[0].dst
    arena.upload_numpy(h_src, temp[r0 * size:r1 * size])
    arena.upload_numpy(h_pow, power[r0 * size:r1 * size])

    def step(events=None):
        return sets[0].step(events)

    # warm-up
    for _ in range(args.warmup):
        step()
    rt.device_synchronize()
    barrier(world)

    # timed region: K steps, inputs resident (3 x 256 MiB > 126 MB L2)
    per_launch = None if not args.launch_events else \
        [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(iters)] for _ in range(args.steps)]
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    barrier(world)
    with ClockSampler(local) as clocks:
        start.record(stream)
        for k in range(args.steps):
            step(per_launch[k] if per_launch else None)
        stop.record(stream)
        rt.device_synchronize()
        torch.cuda.synchronize()
    barrier(world)
    dev_ms = max_over_ranks(start.elapsed_time(stop), world)
    if per_launch:
        launch_ms = [a.elapsed_time(b) for ev in per_launch for a, b in ev]
        avg_launch_ms = statistics.mean(launch_ms)
    else:
        avg_launch_ms = dev_ms / (args.steps * iters)

    total_cells = size * size * iters * args.steps  # whole job (strong scaling)
    value = BYTES_PER_CELL_ITER * total_cells / (dev_ms * 1e-3) / 1e9
    peaks = _peaks()
    local_bytes = BYTES_PER_CELL_ITER * lrows * size  # per launch, this rank
    achieved = local_bytes / (avg_launch_ms * 1e-3) / 1e9

    # the same workload through the fused host-loop driver (temporal blocking)
    fused = None
    if world == 1 and not args.no_fused:
        from paper_2206_07896_b200 import stencil
        for _ in range(args.warmup):
            stencil.hotspot_run(rt, h_src, h_pow, h_dst, lrows, size, params, iters, args.tsteps)
        rt.device_synchronize()
        torch.cuda.synchronize()
        fa, fb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        fa.record(stream)
        for _ in range(args.steps):
            stencil.hotspot_run(rt, h_src, h_pow, h_dst, lrows, size, params, iters, args.tsteps)
        fb.record(stream)
        rt.device_synchronize()
        torch.cuda.synchronize()
        fms = fa.elapsed_time(fb) / args.steps
        fgbs = BYTES_PER_CELL_ITER * size * size * iters / (fms * 1e-3) / 1e9
        fused = {"value": round(fgbs, 2), "unit": "GB/s (algorithmic 12 B/cell/iter)",
                 "ms_per_step": round(fms, 4), "x_per_launch_path": round(dev_ms / args.steps / fms, 3),
                 "tsteps": args.tsteps or 4,
                 "kernel": "hotspot_wave<4>",
                 "note": "stencil.hotspot_run (bf_hotspot_run): the 100-launch host loop fused "
                         "on the device; register-wavefront temporal blocking, 4 iterations per "
                         "pass through HBM (~3.2 B/cell/iter of DRAM traffic), so the algorithmic "
                         "12 B/cell/iter rate exceeds the HBM copy roofline; FP64-bound; "
                         "bit-identical to the per-launch loop"}

    # end-to-end through the public API with host buffers (pinned): every
    # step uploads its inputs (temp + power) and downloads its result.
    # serial: upload, 100 launches, sync, download — nothing overlaps.
    # pipelined (the reported e2e): three resident buffer sets; launches are
    # asynchronous (Runtime.launch returns at issue), so while step k runs on
    # set k%3 the host downloads step k-1's result from set (k-1)%3 and
    # uploads step k+1's inputs into set (k+1)%3 (uploads on the arena's copy
    # stream, the download concurrently on its D2H stream from a helper
    # thread).  Three sets keep the download source, the upload target and
    # the running step disjoint.  Every step's copies are inside the timed
    # region, and every step's downloaded grid is compared bit for bit with
    # the resident-path result after the region.
    h_temp = torch.from_numpy(temp[r0 * size:r1 * size].copy()).pin_memory().numpy()
    h_power = torch.from_numpy(power[r0 * size:r1 * size].copy()).pin_memory().numpy()
    arena.upload_numpy(h_src, h_temp)  # the timed steps above evolved the resident grid
    arena.upload_numpy(h_pow, h_power)
    res = step()
    rt.device_synchronize()
    expect = arena.to_numpy(res)  # the resident path's result on the step's inputs
    n_outs = min(args.steps, 16)
    h_outs = [torch.empty(cells, dtype=torch.float32).pin_memory().numpy() for _ in range(n_outs)]
    h_out = h_outs[0]
    serial = []
    for k in range(args.warmup + args.steps):
        barrier(world)
        t0 = time.perf_counter()
        arena.upload_numpy(h_src, h_temp)
        arena.upload_numpy(h_pow, h_power)
        res = step()
        rt.device_synchronize()
        arena.download_into(res, h_out)
        dt = time.perf_counter() - t0
        if k >= args.warmup:
            serial.append(max_over_ranks(dt, world))
    serial_s = statistics.median(serial)
    e2e_checked = bool(np.array_equal(h_out.view(np.uint32), expect.view(np.uint32)))

    while len(sets) < 3:
        sets.append(BufferSet())

    trace = os.environ.get("BENCH_E2E_TRACE")

    def pipelined(nsteps: int) -> float:
        barrier(world)
        t0 = time.perf_counter()
        arena.upload_numpy(sets[0].src, h_temp)
        arena.upload_numpy(sets[0].pow, h_power)
        prev = None
        for k in range(nsteps):
            ts = [time.perf_counter()]
            res = sets[k % 3].step()
            ts.append(time.perf_counter())
            pending = None
            if prev is not None:  # D2H of step k-1 on its own stream, from a helper thread
                pending = copier.submit(arena.download_into, prev, h_outs[(k - 1) % n_outs])
            if k + 1 < nsteps:
                nxt = sets[(k + 1) % 3]
                arena.upload_numpy(nxt.src, h_temp)
                arena.upload_numpy(nxt.pow, h_power)
            ts.append(time.perf_counter())
            if pending is not None:
                pending.result()
            ts.append(time.perf_counter())
            rt.device_synchronize()
            ts.append(time.perf_counter())
            if trace:
                print("e2e step", k, " ".join(f"{(b - a) * 1e3:.2f}" for a, b in zip(ts, ts[1:])),
                      file=sys.stderr, flush=True)
            prev = res
        arena.download_into(prev, h_outs[(nsteps - 1) % n_outs])
        return max_over_ranks(time.perf_counter() - t0, world)

    import concurrent.futures as cf
    copier = cf.ThreadPoolExecutor(max_workers=1)

    pipelined(max(2, args.warmup))
    for h in h_outs:
        h.fill(np.nan)
    e2e_s = pipelined(args.steps) / args.steps
    e2e_value = BYTES_PER_CELL_ITER * size * size * iters / e2e_s / 1e9
    copier.shutdown()
    for h in h_outs:  # every timed step's delivered result (the last 16 if steps > 16)
        e2e_checked &= bool(np.array_equal(h.view(np.uint32), expect.view(np.uint32)))
    e2e_checked = bool(max_over_ranks(0.0 if e2e_checked else 1.0, world) == 0.0)
    del h_outs, h_out
    launch = launch_latency(arena, rt, torch, stream) if rank == 0 else None

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline_hotspot(size, iters, args.cpu_budget, len(os.sched_getaffinity(0)))
        import benchkit
        ref = benchkit.reference_runtime_pair("hotspot", benchkit.REF_LOG_BENCH, len(os.sched_getaffinity(0)))
        cpu["reference_runtime"] = ref  # the unmodified blockfuse.Runtime on a sample of the same kernel
        best = max((v["elem_per_s"] for v in ref.values() if isinstance(v, dict)), default=None)
        if best:
            cpu["speedup_vs_reference_runtime"] = round(total_cells / (dev_ms * 1e-3) / best, 1)

    kernels = None
    kernel_launches = 0
    if rank == 0 and world == 1 and not args.no_kernels:
        kernels, kernel_launches = per_kernel_table(arena, rt, torch, stream, args)

    traffic = None
    prof = ROOT / "profiles" / "hotspot_traffic.json"
    if prof.exists():
        traffic = json.loads(prof.read_text()).get("dram_bytes_per_launch")

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 2), "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(dev_ms / args.steps, 4),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": f"hotspot {size}x{size} f32, {iters} iterations per step",
                       "grid_launch": f"{grid.x}x{grid.y} blocks of {bx}x{by}",
                       "bytes_per_cell_iter": BYTES_PER_CELL_ITER,
                       "l2": "inputs larger than L2 (3 x 256 MiB vs 126 MB)",
                       "parallelism": f"row bands x{world}" + (f", ghost halo {bands.halo}" if world > 1 else ""),
                       "elem_per_s": total_cells / (dev_ms * 1e-3)},
            "roofline": {"bound": "hbm", "achieved": round(achieved, 2), "peak": peaks["hbm_gbs"],
                         "unit": "GB/s", "frac": round(achieved / peaks["hbm_gbs"], 4),
                         "traffic": traffic, "peak_source": peaks["source"],
                         "kernel": "hotspot_rows", "avg_launch_us": round(avg_launch_ms * 1e3, 3)},
            "e2e": {"value": round(e2e_value, 3), "unit": "GB/s",
                    "h2d_bytes_per_step": 2 * cells * 4 * world, "d2h_bytes_per_step": cells * 4 * world,
                    "ms_per_step": round(e2e_s * 1e3, 3), "mode": "pipelined (3 buffer sets)",
                    "checked": e2e_checked,
                    "check": "every timed step's downloaded grid == the resident-path result, bit for bit",
                    "serial_value": round(BYTES_PER_CELL_ITER * size * size * iters / serial_s / 1e9, 3),
                    "serial_ms_per_step": round(serial_s * 1e3, 3)},
            "gpu_launches": iters * args.steps,
            "launch_latency": launch,
            "clocks": clocks.summary(),
        }
        if cpu is not None:
            line["cpu_baseline"] = cpu
        if fused is not None:
            line["hotspot_fused"] = fused
        if kernels is not None:
            line["kernels"] = kernels
            line["kernel_table_launches"] = kernel_launches
        print(json.dumps(line), flush=True)
        if kernels is not None:
            out = ROOT / "profiles" / "last_bench_kernels.json"
            try:
                out.parent.mkdir(exist_ok=True)
                out.write_text(json.dumps(kernels, indent=1) + "\n")
            except OSError:
                pass
    rt.shutdown()
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def run_sweep(args) -> None:
    """BASELINE configs[4]: vecadd / nn bandwidth sweep, footprint 1 MB ...
    16 GB doubling, split over the ranks (contiguous logical-block ranges =
    the average grain with ranks as workers); one JSON line with the table."""
    import torch

    from paper_2206_07896_b200 import ArgSlot, DeviceArena, Dim3, PackedArgs, Runtime, routines
    from paper_2206_07896_b200.parallel import rank_range

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    device = torch.device("cuda", local)
    peaks = _peaks()
    rows = []
    for kernel in ("vecadd", "nn"):
        for e in range(15):
            footprint = (1 << 20) << e  # 1 MB .. 16 GB
            n = (footprint // 12) // 256 * 256
            blocks = n // 256
            lo_b, hi_b = rank_range(blocks, world, rank)
            ent = {"kernel": kernel, "footprint_bytes": footprint, "n": n}
            if kernel == "nn" and 2 * (n - 1) + 1 > 2**31 - 1:
                ent["skipped"] = "ll[2*id] index beyond i32 in kernels/nn.kn (the reference traps)"
                rows.append(ent)
                continue
            arena = DeviceArena(local)
            rt = Runtime(arena)
            stream = torch.cuda.ExternalStream(rt.worker_stream(0), device=device)
            ln = (hi_b - lo_b) * 256  # local elements (local arrays, global ids offset)
            if kernel == "vecadd":
                hs = [arena.alloc("f32", max(ln, 1)) for _ in range(3)]
                for h in hs[:2]:
                    torch.as_tensor(arena.cuda_array(h), device=device).uniform_(-1, 1)
                pk = PackedArgs([ArgSlot("handle", hs[0]), ArgSlot("handle", hs[1]),
                                 ArgSlot("handle", hs[2]), ArgSlot("i32", ln)])
                routine = routines.get("vecadd")
            else:
                hl, hd = arena.alloc("f32", max(2 * ln, 2)), arena.alloc("f32", max(ln, 1))
                t = torch.as_tensor(arena.cuda_array(hl), device=device)
                t.uniform_(-90, 90)
                pk = PackedArgs([ArgSlot("handle", hl), ArgSlot("handle", hd), ArgSlot("i32", ln),
                                 ArgSlot("f32", 30.0), ArgSlot("f32", 90.0)])
                routine = routines.get("nn")
            torch.cuda.synchronize()
            grid = Dim3(max(1, hi_b - lo_b))
            for _ in range(args.warmup):
                rt.launch(routine, grid, Dim3(256), 0, pk)
            rt.device_synchronize()
            barrier(world)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            for _ in range(args.steps):
                rt.launch(routine, grid, Dim3(256), 0, pk)
            b.record(stream)
            rt.device_synchronize()
            b.synchronize()
            ms = max_over_ranks(a.elapsed_time(b) / args.steps, world)
            gbs = 12 * n / (ms * 1e-3) / 1e9
            ent.update({"gbs": round(gbs, 2), "elem_per_s": n / (ms * 1e-3), "us_per_launch": round(ms * 1e3, 3),
                        "frac_roofline": round(gbs / (world * peaks["hbm_gbs"]), 4),
                        "l2_resident": footprint / world < 126e6})
            rows.append(ent)
            rt.shutdown()
            del rt, arena
            torch.cuda.synchronize()
    if rank == 0:
        big = [r for r in rows if r.get("gbs") and r["footprint_bytes"] >= (1 << 30)]
        best = max((r["gbs"] for r in big), default=None)
        print(json.dumps({
            "metric": METRIC, "value": best, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f32/f64", "data": "synthetic",
            "config": {"workload": "vecadd/nn sweep 1 MB..16 GB footprint (12 B/elem), split over ranks",
                       "value": "best GB/s over points >= 1 GiB"},
            "sweep": rows}), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def run_kmeans(args) -> None:
    """BASELINE configs[2] across ranks: Rodinia's kmeans host loop (16M
    points x 32 features, k = 16) for --passes passes per step.  Each rank
    assigns its contiguous range of logical blocks (rank_range: the average
    grain with ranks as workers) through Runtime.launch_range; per pass the
    k x nf sums and k counts are all-reduced over NCCL (~2.1 KB) and every
    rank applies the same centroid update (cluster.KmeansDriver).  value =
    points assigned per second over the whole job (strong scaling)."""
    import torch

    from paper_2206_07896_b200 import DeviceArena, Runtime
    from paper_2206_07896_b200.cluster import KmeansDriver
    from paper_2206_07896_b200.parallel import nccl_allreduce

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=device)
    npts, nf, k, passes = args.kmeans_points, 32, 16, args.passes
    arena = DeviceArena(local)
    rt = Runtime(arena)
    stream = torch.cuda.ExternalStream(rt.worker_stream(0), device=device)
    f, cent, member = arena.alloc("f32", npts * nf), arena.alloc("f32", k * nf), arena.alloc("i32", npts)
    g = torch.Generator(device=device)
    g.manual_seed(0)  # the same points on every rank
    tf = torch.as_tensor(arena.cuda_array(f), device=device)
    tf.uniform_(0, 1, generator=g)
    tc = torch.as_tensor(arena.cuda_array(cent), device=device)
    c0 = tf.view(nf, npts)[:, :k].t().contiguous().view(-1).clone()
    allreduce = nccl_allreduce(arena, device) if world > 1 else None
    drv = KmeansDriver(rt, arena, f, cent, member, npts, nf, k, world, rank)

    def step():
        tc.copy_(c0)
        arena.fill_value(drv.prev, -1)
        torch.cuda.synchronize()
        for _ in range(passes):
            drv.assign()
            if world > 1:
                allreduce([drv.sums, drv.counts])
            d = drv.update()
            if world > 1:
                allreduce(d)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    barrier(world)
    with ClockSampler(local) as clocks:
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(args.steps):
            step()
        b.record(stream)
        rt.device_synchronize()
        torch.cuda.synchronize()
    barrier(world)
    ms = max_over_ranks(a.elapsed_time(b) / args.steps, world)
    cent_sum = float(tc.double().sum().item())
    # e2e: the same step through the public API from pinned host memory: the
    # points are uploaded every step, the memberships and centroids read back
    # and compared with the resident run's (every rank holds all points)
    import numpy as np
    expect_member, expect_cent = arena.to_numpy(member), arena.to_numpy(cent)
    h_f = torch.empty(npts * nf, dtype=torch.float32).pin_memory().numpy()
    arena.download_into(f, h_f)
    h_member = torch.empty(npts, dtype=torch.int32).pin_memory().numpy()
    h_cent = torch.empty(k * nf, dtype=torch.float32).pin_memory().numpy()
    e2e_s = []
    for i in range(args.warmup + args.steps):
        barrier(world)
        t0 = time.perf_counter()
        arena.upload_numpy(f, h_f)
        step()
        rt.device_synchronize()
        torch.cuda.synchronize()
        arena.download_into(member, h_member)
        arena.download_into(cent, h_cent)
        dt = time.perf_counter() - t0
        if i >= args.warmup:
            e2e_s.append(max_over_ranks(dt, world))
    # the centroid sums are f32 atomics (order-dependent, as in the reference),
    # so a later pass may differ in the last bits: centroids within 1e-4, and
    # memberships equal up to the points the rounding moves across a tie
    mismatch = float(np.mean(h_member != expect_member))
    e2e_checked = bool(np.allclose(h_cent, expect_cent, rtol=1e-4, atol=1e-6) and mismatch <= 1e-3)
    if rank == 0:
        pts = npts * passes
        e2e_t = statistics.median(e2e_s)
        print(json.dumps({
            "metric": METRIC, "value": round(pts * (4 * nf + 4) / (ms * 1e-3) / 1e9, 2), "unit": "GB/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32/f64",
            "data": "synthetic",
            "config": {"workload": f"kmeans {npts} x {nf} f32, k={k}, {passes} passes per step (Rodinia host loop)",
                       "parallelism": f"point ranges x{world}, per-pass all-reduce of sums/counts",
                       "bytes_per_point_pass": 4 * nf + 4},
            "elem_per_s": pts / (ms * 1e-3), "centroid_checksum": cent_sum,
            "e2e": {"value": round(pts * (4 * nf + 4) / e2e_t / 1e9, 2), "unit": "GB/s",
                    "h2d_bytes_per_step": npts * nf * 4, "d2h_bytes_per_step": npts * 4 + k * nf * 4,
                    "ms_per_step": round(e2e_t * 1e3, 3), "checked": e2e_checked,
                    "member_mismatch": mismatch},
            "clocks": clocks.summary()}), flush=True)
    rt.shutdown()
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def run_cpu_runtime(args) -> None:
    """SURVEY §8d "CPU timing (reference path)": the unmodified reference
    runtime (blockfuse.Runtime) per kernel at the survey's sizes, pool =
    host cores and pool = 1, each result checked against the oracle; beside
    it the C port (oracle/oracle.c) on all host cores.  Host-only (no GPU)."""
    import benchkit
    threads = len(os.sched_getaffinity(0))
    rows = {}
    for name, log_n in benchkit.REF_LOG_SURVEY.items():
        ent = benchkit.reference_runtime_pair(name, benchkit.REF_LOG_SURVEY, threads)
        try:
            ent = dict(ent, port=benchkit.cpu_sample(name, threads))
        except Exception as e:
            ent = dict(ent, port={"error": repr(e)})
        rows[name] = ent
        print(json.dumps({"kernel": name, **ent}), file=sys.stderr, flush=True)
    print(json.dumps({"metric": "reference CPU runtime per kernel (blockfuse.Runtime) and the C port",
                      "value": None, "unit": "elem/s", "n_gpus": 0, "host_threads": threads,
                      "config": {"workload": "SURVEY §8d CPU sample sizes (log2)", "sizes": benchkit.REF_LOG_SURVEY},
                      "kernels": rows}), flush=True)


def run_reorder(args) -> None:
    """the reference's grid-stride reordering study
    (bench.run_reorder_experiment, transform.reorder_grid_stride) on the B200.
    The reference rewrites `base + j*blockDim.x` into `base*K + j` so that a
    CPU thread walks a contiguous chunk (fewer simulated LLC misses); on the
    GPU the same rewrite turns every warp access into 32 scattered sectors.
    Both versions of hist_stride and fir run through the JIT (codegen + NVRTC,
    one CTA per logical block, exactly the DSL semantics) on the same inputs;
    the outputs must agree; reported: device time per launch, and the sectors
    per warp request when run under ncu (profiles/r1_reorder_sectors.csv)."""
    import torch

    ref = ROOT / "baseline" / "_ref"
    if not (ref / "blockfuse").exists():
        ref = Path("/root/reference/pkg/src")
    sys.path.append(str(ref))
    from blockfuse.bench import CORPUS
    from blockfuse.transform import reorder_grid_stride

    from paper_2206_07896_b200 import ArgSlot, DeviceArena, Dim3, PackedArgs, Runtime, routines
    torch.cuda.set_device(0)
    device = torch.device("cuda", 0)
    arena = DeviceArena(0)
    rows = []
    routines.FORCE_JIT = True
    try:
        for name in ("hist_stride", "fir"):
            orig = CORPUS[name].compiled()
            reord = reorder_grid_stride(orig)
            bx, k = 256, args.reorder_k
            if name == "hist_stride":
                n = bx * k
                x, out = arena.alloc("i32", n), arena.alloc("i32", 16)
                torch.as_tensor(arena.cuda_array(x), device=device).random_(0, 1 << 16)
                pk = PackedArgs([ArgSlot("handle", x), ArgSlot("handle", out), ArgSlot("i32", k), ArgSlot("i32", 16)])
                nbytes = 4 * n
            else:
                n, taps = bx * k, 4
                x, out, w = arena.alloc("f32", n + taps), arena.alloc("f32", n), arena.alloc("f32", taps)
                torch.as_tensor(arena.cuda_array(x), device=device).uniform_(-1, 1)
                torch.as_tensor(arena.cuda_array(w), device=device).uniform_(-1, 1)
                pk = PackedArgs([ArgSlot("handle", x), ArgSlot("handle", out), ArgSlot("handle", w),
                                 ArgSlot("i32", taps), ArgSlot("i32", k)])
                nbytes = 8 * n
            res = {}
            for label, mk in (("original", orig), ("reordered", reord)):
                with Runtime(arena) as rt:
                    ot = torch.as_tensor(arena.cuda_array(out), device=device)
                    stream = torch.cuda.ExternalStream(rt.worker_stream(0))
                    ts = []
                    for rep in range(args.warmup + args.steps):
                        ot.zero_()
                        torch.cuda.synchronize()
                        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                        a.record(stream)
                        rt.launch(mk, Dim3(1), Dim3(bx), 0, pk)
                        b.record(stream)
                        rt.device_synchronize()
                        b.synchronize()
                        if rep >= args.warmup:
                            ts.append(a.elapsed_time(b) * 1e-3)
                    res[label] = (statistics.median(ts), ot.clone())
            same = bool(torch.equal(res["original"][1], res["reordered"][1]))
            rows.append({"kernel": name, "elements": n, "grid": "1 x 256 (one logical block: one CTA)",
                         "original_ms": round(res["original"][0] * 1e3, 4),
                         "reordered_ms": round(res["reordered"][0] * 1e3, 4),
                         "original_gbs": round(nbytes / res["original"][0] / 1e9, 2),
                         "reordered_gbs": round(nbytes / res["reordered"][0] / 1e9, 2),
                         "slowdown_x": round(res["reordered"][0] / res["original"][0], 2),
                         "outputs_equal": same})
    finally:
        routines.FORCE_JIT = False
    print(json.dumps({"metric": "grid-stride reordering study on the GPU (reference transform.reorder_grid_stride)",
                      "value": None, "unit": "ms", "n_gpus": 1,
                      "config": {"workload": f"hist_stride / fir, 256 threads x {args.reorder_k} strides, JIT"},
                      "reorder": rows}), flush=True)


def run_grain(args) -> None:
    """the paper's grain-size study on the GPU runtime.
    fetch="device": the CTAs of one persistent grid claim block_per_fetch
    blocks per atomic on a device counter, so the grain trades claim count
    (atomic traffic on one address) against load balance as block_per_fetch
    does on the CPU pool; fetch="host": each fetch is one
    grid launch (the grain trades launch count instead).  Reports fetches and
    wall time per launch+sync for vecadd and hist at pool sizes 1/4/8."""
    import torch

    from paper_2206_07896_b200 import (ArgSlot, Average, DeviceArena, Dim3, Fixed, PackedArgs,
                                       Runtime, routines)
    torch.cuda.set_device(0)
    device = torch.device("cuda", 0)
    n = 1 << 24
    blocks = n // 256
    arena = DeviceArena(0)
    a, b, c = (arena.alloc("f32", n) for _ in range(3))
    pix, cnt = arena.alloc("i32", n), arena.alloc("i32", 16)
    for h in (a, b):
        torch.as_tensor(arena.cuda_array(h), device=device).uniform_(-1, 1)
    torch.as_tensor(arena.cuda_array(pix), device=device).random_(0, 1 << 16)
    torch.cuda.synchronize()
    cases = {
        "vecadd": (routines.get("vecadd"), PackedArgs([ArgSlot("handle", a), ArgSlot("handle", b),
                                                        ArgSlot("handle", c), ArgSlot("i32", n)]), 12 * n),
        "hist": (routines.get("hist"), PackedArgs([ArgSlot("handle", pix), ArgSlot("handle", cnt),
                                                    ArgSlot("i32", n), ArgSlot("i32", 16)]), 4 * n),
    }
    rows = []
    for name, (routine, pk, nbytes) in cases.items():
        for fetch in ("device", "host"):
            for pool in (1, 4, 8):
                for grain in (1, 4, 16, 256, 4096, "average"):
                    policy = Average() if grain == "average" else Fixed(grain)
                    rt = Runtime(arena, pool_size=pool, policy=policy, fetch=fetch)
                    rt.launch(routine, Dim3(blocks), Dim3(256), 0, pk)
                    rt.device_synchronize()
                    reps = 3 if fetch == "host" and grain in (1, 4) else 20
                    t0 = time.perf_counter()
                    for _ in range(reps):
                        task = rt.launch(routine, Dim3(blocks), Dim3(256), 0, pk)
                        rt.device_synchronize()
                    wall = (time.perf_counter() - t0) / reps
                    rows.append({"kernel": name, "fetch": fetch, "pool": pool, "grain": grain,
                                 "block_per_fetch": task.block_per_fetch, "fetches": task.fetches,
                                 "wall_ms": round(wall * 1e3, 4), "gbs": round(nbytes / wall / 1e9, 2)})
                    rt.shutdown()
    print(json.dumps({"metric": "grain-size study (fetches vs launch+sync wall time)", "value": None,
                      "unit": "GB/s", "n_gpus": 1,
                      "config": {"workload": "vecadd/hist 2^24, 65536 blocks x 256",
                                 "fetch": "device: one persistent grid claims block_per_fetch blocks per atomic "
                                          "(Runtime(fetch='device')); host: one grid launch per fetched range"},
                      "grain": rows}), flush=True)


def launch_latency(arena, rt, torch, stream, reps: int = 2000) -> dict:
    """BASELINE configs[0] / SURVEY §8d C1: vecAdd 2^20 f32, grid 4096 x 256
    (PR1), through Runtime.launch.  launch_us: host time of one
    Runtime.launch call (non-blocking); launch_sync_us: one launch followed
    by device_synchronize, wall clock (the reference measures 59.5 us for
    this pair on its thread pool, runtime.py:255-278); device_us: device time
    per launch back to back (CUDA events on the worker stream)."""
    from paper_2206_07896_b200 import ArgSlot, Dim3, PackedArgs, routines
    n = 1 << 20
    hs = [arena.alloc("f32", n) for _ in range(3)]
    dev = torch.device("cuda", arena.device)
    for h in hs[:2]:
        torch.as_tensor(arena.cuda_array(h), device=dev).uniform_(-1, 1)
    torch.cuda.synchronize()
    pk = PackedArgs([ArgSlot("handle", hs[0]), ArgSlot("handle", hs[1]), ArgSlot("handle", hs[2]),
                     ArgSlot("i32", n)])
    va, g, b = routines.get("vecadd"), Dim3(4096), Dim3(256)
    for _ in range(100):
        rt.launch(va, g, b, 0, pk)
    rt.device_synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        rt.launch(va, g, b, 0, pk)
    launch_us = (time.perf_counter() - t0) / reps * 1e6
    rt.device_synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        rt.launch(va, g, b, 0, pk)
        rt.device_synchronize()
    sync_us = (time.perf_counter() - t0) / reps * 1e6
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(reps):
        rt.launch(va, g, b, 0, pk)
    e1.record(stream)
    rt.device_synchronize()
    e1.synchronize()
    dev_us = e0.elapsed_time(e1) * 1e3 / reps
    for h in hs:
        arena.free(h)
    return {"workload": "vecadd 2^20 f32, grid 4096 x 256 (PR1)", "launch_us": round(launch_us, 3),
            "launch_sync_us": round(sync_us, 3), "device_us_per_launch": round(dev_us, 3),
            "device_gbs": round(12 * n / (dev_us * 1e-6) / 1e9, 1), "reps": reps,
            "reference_launch_sync_us": 59.5}


def per_kernel_table(arena, rt, torch, stream, args) -> tuple[dict, int]:
    """Every other kernel of the path at full size (benchkit.py), N=1."""
    import benchkit
    device = torch.device("cuda", arena.device)
    peaks = _peaks()
    cases = benchkit.build_cases(arena, torch, device, scale=args.kernel_scale)
    if not args.no_bfs:
        cases.extend(benchkit.bfs_case(arena, torch, device, log_v=args.bfs_log_v))
    torch.cuda.synchronize()
    threads = len(os.sched_getaffinity(0))
    table, launches = {}, 0
    if args.cases:
        keep = set(args.cases.split(","))
        cases = [c for c in cases if c.name in keep]
    for c in cases:
        r = benchkit.time_case(c, rt, torch, stream, reps=args.steps, warmup=args.warmup)
        launches += r["launches"] * args.steps
        gbs = c.bytes_per_step / r["dev_s"] / 1e9
        ent = {"kernel": c.kernel, "gbs": round(gbs, 2), "frac_hbm": round(gbs / peaks["hbm_gbs"], 4),
               f"{c.unit_elem}_per_s": c.elems_per_step / r["dev_s"],
               "ms_per_step": round(r["dev_s"] * 1e3, 4), "wall_ms_per_step": round(r["wall_s"] * 1e3, 4),
               "launches_per_step": r["launches"], "bytes_per_step": c.bytes_per_step,
               "checked": r["checked"]}
        if c.note:
            ent["note"] = c.note
        if hasattr(c, "levels"):
            ent["levels"] = c.levels["n"]
        if getattr(c, "extra", None) and "build_ms" in c.extra:
            ent["transpose_build_ms"] = round(c.extra["build_ms"], 3)
        if not args.no_cpu:
            try:
                cpu = benchkit.cpu_sample(c.name, threads)
            except Exception as e:
                cpu = {"error": repr(e)}
            if cpu is not None:
                ent["cpu_baseline"] = cpu
                if "elem_per_s" in cpu:
                    ent["speedup_vs_cpu_port"] = round(c.elems_per_step / r["dev_s"] / cpu["elem_per_s"], 1)
            ref = benchkit.reference_runtime_pair(c.name, benchkit.REF_LOG_BENCH, threads)
            if ref is not None:
                ent["reference_runtime"] = ref
                best = max((v["elem_per_s"] for v in ref.values() if isinstance(v, dict)), default=None)
                if best:
                    ent["speedup_vs_reference_runtime"] = round(c.elems_per_step / r["dev_s"] / best, 1)
        table[c.name] = ent
    return table, launches


def spawn_ranks(args) -> int:
    """`--gpus N` without a launcher: re-exec this script under torchrun, one
    process per GPU (RANK / LOCAL_RANK / WORLD_SIZE from the environment),
    rendezvous on 127.0.0.1.  Fails loudly when fewer than N GPUs are
    visible (the reference arm needs no GPU: its ranks > 0 exit at once)."""
    if args.impl == "ours":
        import torch
        have = torch.cuda.device_count()
        if have < args.gpus:
            print(f"bench.py: --gpus {args.gpus} requested but only {have} CUDA device(s) visible",
                  file=sys.stderr, flush=True)
            return 1
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(Path(__file__).resolve()),
           *sys.argv[1:]]
    return subprocess.call(cmd)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=["hotspot", "sweep", "grain", "reorder", "kmeans", "cpu-runtime"], default="hotspot")
    ap.add_argument("--reorder-k", type=int, default=1 << 16, help="strides per thread (reorder study)")
    ap.add_argument("--size", type=int, default=8192)
    ap.add_argument("--kmeans-points", type=int, default=1 << 24)
    ap.add_argument("--passes", type=int, default=10, help="kmeans host-loop passes per step")
    ap.add_argument("--iters", type=int, default=100)
    ap.add_argument("--halo", type=int, default=8)
    ap.add_argument("--cpu-budget", type=float, default=10.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-kernels", action="store_true", help="skip the per-kernel table")
    ap.add_argument("--no-fused", action="store_true", help="skip the fused hotspot driver")
    ap.add_argument("--tsteps", type=int, default=0, help="temporal-blocking depth (0 = default)")
    ap.add_argument("--no-bfs", action="store_true")
    ap.add_argument("--launch-events", action="store_true",
                    help="bracket every launch with its own event pair (the default times each step with one "
                         "pair and divides by the launches: per-launch events cost ~3 us each)")
    ap.add_argument("--kernel-scale", type=int, default=28, help="log2 elements per kernel case")
    ap.add_argument("--bfs-log-v", type=int, default=26)
    ap.add_argument("--cases", default="", help="comma list: only these per-kernel cases")
    args = ap.parse_args()
    if args.gpus < 1:
        ap.error("--gpus must be >= 1")
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(spawn_ranks(args))
    world = int(os.environ.get("WORLD_SIZE", 1))
    if world != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}: one process per GPU expected")
    if args.impl == "reference":
        run_reference_arm(args)
    elif args.workload == "sweep":
        run_sweep(args)
    elif args.workload == "reorder":
        run_reorder(args)
    elif args.workload == "kmeans":
        run_kmeans(args)
    elif args.workload == "cpu-runtime":
        run_cpu_runtime(args)
    elif args.workload == "grain":
        run_grain(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
