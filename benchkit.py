"""Per-kernel measurement cases for bench.py (one B200, inputs resident).

Each case issues its launches through the reference-shaped API
(Runtime.launch -> C ABI -> sm_100a kernel) on worker stream 0 and is timed
with CUDA events on that stream.  Algorithmic bytes per launch follow
SURVEY.md §8(d) / DESIGN.md; sizes put every working set well above the
126 MB L2 (except the latency cases, which are labelled).  Synthetic inputs
are generated on the device with torch (plumbing) directly into the arena's
buffers.  A light full-size check against a plain PyTorch computation runs
once per case where one is cheap (exact for these kernels); full parity is
the job of tests/.
"""

from __future__ import annotations

import os
import statistics
import sys
import time
from dataclasses import dataclass, field
from pathlib import Path
from typing import Callable, Optional

ROOT = Path(__file__).resolve().parent


@dataclass
class Case:
    name: str
    kernel: str                 # device kernel measured (ncu name)
    bytes_per_step: float       # algorithmic bytes of one step
    elems_per_step: float
    unit_elem: str
    launches: list              # [(routine, grid, block, shmem, packed)]
    note: str = ""
    check: Optional[Callable[[], bool]] = None
    host_loop: Optional[Callable] = None  # custom step (bfs), returns launches issued
    reset: Optional[Callable[[], None]] = None


def _t(arena, h, torch, device):
    return torch.as_tensor(arena.cuda_array(h), device=device)


def build_cases(arena, torch, device, scale: int = 28) -> list:
    """Cases at 2^scale elements (default 2^28: 1-3 GiB per array)."""
    from paper_2206_07896_b200 import ArgSlot, Dim3, PackedArgs, routines

    g = torch.Generator(device=device)
    g.manual_seed(1234)
    n = 1 << scale
    cases = []

    def alloc(scalar, length):
        return arena.alloc(scalar, length)

    # --- vecadd, PR1 config (2^20, grid 4096 x 256): latency-bound ---------
    h = [alloc("f32", 1 << 20) for _ in range(3)]
    for x in h[:2]:
        _t(arena, x, torch, device).uniform_(-1, 1, generator=g)
    pk = PackedArgs([ArgSlot("handle", h[0]), ArgSlot("handle", h[1]), ArgSlot("handle", h[2]),
                     ArgSlot("i32", 1 << 20)])
    cases.append(Case("vecadd_pr1", "vecadd_stream", 12 * (1 << 20), 1 << 20, "elem",
                      [(routines.get("vecadd"), Dim3(4096), Dim3(256), 0, pk)],
                      note="PR1: 2^20 f32, grid 4096x256; 12.6 MB fits L2 (latency case)"))

    # --- vecadd, 2^28 -----------------------------------------------------
    va = [alloc("f32", n) for _ in range(3)]
    ta = [_t(arena, x, torch, device) for x in va]
    ta[0].uniform_(-1, 1, generator=g)
    ta[1].uniform_(-1, 1, generator=g)
    pk = PackedArgs([ArgSlot("handle", va[0]), ArgSlot("handle", va[1]), ArgSlot("handle", va[2]),
                     ArgSlot("i32", n)])
    cases.append(Case("vecadd", "vecadd_stream", 12 * n, n, "elem",
                      [(routines.get("vecadd"), Dim3(n // 256), Dim3(256), 0, pk)],
                      check=lambda: bool(torch.equal(ta[2], ta[0] + ta[1]))))

    # --- nn, 2^28 records -------------------------------------------------
    ll = alloc("f32", 2 * n)
    d = alloc("f32", n)
    tl = _t(arena, ll, torch, device)
    tl[0::2].uniform_(-90, 90, generator=g)
    tl[1::2].uniform_(-180, 180, generator=g)
    td = _t(arena, d, torch, device)
    pk = PackedArgs([ArgSlot("handle", ll), ArgSlot("handle", d), ArgSlot("i32", n),
                     ArgSlot("f32", 30.0), ArgSlot("f32", 90.0)])

    def nn_check():
        k = 1 << 22
        a = tl[0:2 * k:2].double() - 30.0
        b = tl[1:2 * k:2].double() - 90.0
        return bool(torch.equal(td[:k], torch.sqrt(a * a + b * b).float()))
    cases.append(Case("nn", "nn_stream", 12 * n, n, "record",
                      [(routines.get("nn"), Dim3(n // 256), Dim3(256), 0, pk)], check=nn_check))

    # --- nn top-k indices: the 5 nearest of the 2^28 distances --------------
    tk = 5
    ti, tdist = alloc("i32", tk), alloc("f32", tk)
    pk = PackedArgs([ArgSlot("handle", d), ArgSlot("handle", ti), ArgSlot("handle", tdist),
                     ArgSlot("i32", n), ArgSlot("i32", tk)])

    def topk_check():
        order = torch.sort(td, stable=True).indices[:tk]
        return bool(torch.equal(_t(arena, ti, torch, device).long(), order))
    cases.append(Case("nn_topk", "nn_topk_pass", 4 * n, n, "record",
                      [(routines.get("nn_topk"), Dim3(1), Dim3(1), 0, pk)], check=topk_check,
                      note="Rodinia nn's k-nearest selection (k=5) over the nn case's 2^28 distances; "
                           "4 B per record; indices checked against a stable sort"))

    # --- hist, 2^28 pixels, 16 bins -----------------------------------------
    pix = alloc("i32", n)
    cnt = alloc("i32", 16)
    tp = _t(arena, pix, torch, device)
    tp.random_(0, 1 << 16, generator=g)
    tc = _t(arena, cnt, torch, device)
    pk = PackedArgs([ArgSlot("handle", pix), ArgSlot("handle", cnt), ArgSlot("i32", n), ArgSlot("i32", 16)])

    def hist_check():
        want = torch.bincount((tp % 16).long(), minlength=16)
        return bool(torch.equal(tc.long(), want))
    cases.append(Case("hist", "hist_range", 4 * n, n, "pixel",
                      [(routines.get("hist"), Dim3(n // 256), Dim3(256), 0, pk)], check=hist_check,
                      reset=lambda: tc.zero_()))

    # --- hist_stride: one block of 256 threads, k = n / 256 strides ------------
    pk = PackedArgs([ArgSlot("handle", pix), ArgSlot("handle", cnt), ArgSlot("i32", n // 256),
                     ArgSlot("i32", 16)])
    cases.append(Case("hist_stride", "hist_range", 4 * n, n, "pixel",
                      [(routines.get("hist_stride"), Dim3(1), Dim3(256), 0, pk)], check=hist_check,
                      reset=lambda: tc.zero_(),
                      note="grid 1 x 256 threads: the single logical block is spread over all SMs"))

    # --- reduce: per-block sums, block 256 ------------------------------------
    rout = alloc("i32", n // 256)
    to = _t(arena, rout, torch, device)
    pk = PackedArgs([ArgSlot("handle", pix), ArgSlot("handle", rout), ArgSlot("i32", n)])

    def reduce_check():
        want = tp.view(-1, 256).long().sum(1)
        want = ((want + 2**31) % 2**32 - 2**31).int()
        return bool(torch.equal(to, want))
    cases.append(Case("reduce", "reduce_warp", 4 * n + 4 * (n // 256), n, "elem",
                      [(routines.get("reduce"), Dim3(n // 256), Dim3(256), 0, pk)], check=reduce_check))

    # --- wreduce (warp mode, warp 32), block 256 ------------------------------
    wout = alloc("i32", 1)
    tw = _t(arena, wout, torch, device)
    pk = PackedArgs([ArgSlot("handle", pix), ArgSlot("handle", wout), ArgSlot("i32", n)])

    def wreduce_check():
        s = int(tp.long().sum().item())
        return int(tw.item()) == ((s + 2**31) % 2**32 - 2**31)
    cases.append(Case("wreduce", "wreduce_blocks", 4 * n, n, "elem",
                      [(routines.get("wreduce", warp_size=32), Dim3(n // 256), Dim3(256), 0, pk)],
                      check=wreduce_check, reset=lambda: tw.zero_()))

    # --- fir: 1 block x 256 threads, m = n/256 strides, 8 taps ----------------
    taps = 8
    fx = alloc("f32", n + taps)
    fy = alloc("f32", n)
    fw = alloc("f32", taps)
    tfx = _t(arena, fx, torch, device)
    tfx.uniform_(-1, 1, generator=g)
    tfw = _t(arena, fw, torch, device)
    tfw.uniform_(-1, 1, generator=g)
    tfy = _t(arena, fy, torch, device)
    pk = PackedArgs([ArgSlot("handle", fx), ArgSlot("handle", fy), ArgSlot("handle", fw),
                     ArgSlot("i32", taps), ArgSlot("i32", n // 256)])

    def fir_check():
        k = 1 << 20
        acc = torch.zeros(k, dtype=torch.float64, device=device)
        for i in range(taps):
            acc = acc + tfw[i].double() * tfx[i:i + k].double()
        return bool(torch.equal(tfy[:k], acc.float()))
    cases.append(Case("fir", "fir_reg<8>", 8 * n + 4 * (taps - 1), n, "output",
                      [(routines.get("fir"), Dim3(1), Dim3(256), 0, pk)], check=fir_check,
                      note="grid 1 x 256 threads, 8 taps"))

    # --- kmeans: 16M points x 32 features, k = 16 -----------------------------
    npts, nf, k = 1 << 24, 32, 16
    kf = alloc("f32", npts * nf)
    kc = alloc("f32", k * nf)
    km = alloc("i32", npts)
    ks = alloc("f32", k * nf)
    kn = alloc("i32", k)
    tkf = _t(arena, kf, torch, device)
    tkf.uniform_(0, 1, generator=g)
    tkc = _t(arena, kc, torch, device)
    tkc.copy_(tkf.view(nf, npts)[:, :k].t().contiguous().view(-1))
    tks, tkn = _t(arena, ks, torch, device), _t(arena, kn, torch, device)
    pk = PackedArgs([ArgSlot("handle", kf), ArgSlot("handle", kc), ArgSlot("handle", km),
                     ArgSlot("handle", ks), ArgSlot("handle", kn), ArgSlot("i32", npts),
                     ArgSlot("i32", nf), ArgSlot("i32", k)])

    def km_reset():
        tks.zero_()
        tkn.zero_()
    cases.append(Case("kmeans", "kmeans_tg", npts * (4 * nf + 4), npts, "point",
                      [(routines.get("kmeans"), Dim3(npts // 256), Dim3(256), 0, pk)],
                      check=lambda: int(tkn.long().sum().item()) == npts, reset=km_reset,
                      note="16M x 32 f32, k=16: one assignment + accumulation pass; f64 distances"))

    # --- kmeans host loop: 10 passes of assignment + centroid update (cluster.py)
    from paper_2206_07896_b200.cluster import KmeansDriver
    kc2 = alloc("f32", k * nf)
    km2 = alloc("i32", npts)
    tkc2 = _t(arena, kc2, torch, device)
    passes = 10
    state = {}

    def km_loop(rt, stream):
        if "drv" not in state:
            state["drv"] = KmeansDriver(rt, arena, kf, kc2, km2, npts, nf, k)
        d = state["drv"]
        for _ in range(passes):
            d.assign()
            d.update()
        return 2 * passes

    def km_loop_reset():
        tkc2.copy_(tkc)
        if "drv" in state:
            arena.fill_value(state["drv"].prev, -1)
    cases.append(Case("kmeans_loop", "kmeans_tg+kmeans_update", passes * npts * (4 * nf + 4), passes * npts, "point",
                      [], host_loop=km_loop, reset=km_loop_reset,
                      check=lambda: bool(torch.isfinite(tkc2).all().item()),
                      note=f"Rodinia kmeans host loop, {passes} passes (assignment + centroid update + delta "
                           "through cluster.KmeansDriver); per pass one host sync (delta)"))

    # --- backprop: Rodinia's two device kernels, 2^(scale-4) input units x 16 hidden
    nin, hid = 1 << (scale - 4), 16
    nb = nin // 16
    bi, bw, bpart = alloc("f32", nin + 1), alloc("f32", (nin + 1) * (hid + 1)), alloc("f32", nb * hid)
    bd, bo = alloc("f32", hid + 1), alloc("f32", (nin + 1) * (hid + 1))
    tbi, tbw, tbp = _t(arena, bi, torch, device), _t(arena, bw, torch, device), _t(arena, bpart, torch, device)
    tbd, tbo = _t(arena, bd, torch, device), _t(arena, bo, torch, device)
    tbi.uniform_(0, 1, generator=g)
    tbw.uniform_(0, 1, generator=g)
    tbd.uniform_(-0.1, 0.1, generator=g)
    tbo.uniform_(-0.05, 0.05, generator=g)
    tbw0, tbo0 = tbw.clone(), tbo.clone()

    def bp_reset():
        tbw.copy_(tbw0)
        tbo.copy_(tbo0)

    def bp_fw_check():
        p = tbw0.view(nin + 1, hid + 1)[1:, 1:].reshape(nb, 16, hid) * tbi[1:].view(nb, 16, 1)
        while p.shape[1] > 1:  # Rodinia's tree: rows (0,1), (2,3), ... then pairs of pairs
            p = p[:, 0::2] + p[:, 1::2]
        return bool(torch.equal(tbp.view(nb, hid), p[:, 0, :]))

    def bp_adj_check():
        cx = 0.3 * tbd.double()
        a = cx[1:].view(1, hid) * tbi.double()[1:].view(nin, 1)
        b = 0.3 * tbo0.double().view(nin + 1, hid + 1)[1:, 1:]
        s_ = a + b
        w_ = (tbw0.double().view(nin + 1, hid + 1)[1:, 1:] + s_).float()
        return bool(torch.equal(tbw.view(nin + 1, hid + 1)[1:, 1:], w_)) and \
            bool(torch.equal(tbo.view(nin + 1, hid + 1)[1:, 1:], s_.float()))
    pk = PackedArgs([ArgSlot("handle", bi), ArgSlot("handle", bw), ArgSlot("handle", bpart),
                     ArgSlot("i32", hid)])
    cases.append(Case("bp_forward", "bp_forward", nin * (64 + 64 + 4 + 4), nin, "input unit",
                      [(routines.get("bpnn_layerforward"), Dim3(1, nb), Dim3(16, 16), 0, pk)],
                      check=bp_fw_check, reset=bp_reset,
                      note=f"Rodinia backprop bpnn_layerforward, {nin} inputs x 16 hidden, 16x16 blocks; "
                           "bytes/unit = 64 w read + 64 w written + 4 input + 4 partial"))
    pk = PackedArgs([ArgSlot("handle", bd), ArgSlot("i32", hid), ArgSlot("handle", bi), ArgSlot("i32", nin),
                     ArgSlot("handle", bw), ArgSlot("handle", bo)])
    cases.append(Case("bp_adjust", "bp_adjust", nin * (16 * 16 + 4), nin, "input unit",
                      [(routines.get("bpnn_adjust_weights"), Dim3(1, nb), Dim3(16, 16), 0, pk)],
                      check=bp_adj_check, reset=bp_reset,
                      note="bpnn_adjust_weights: w, oldw read + written (16 B x 16 per unit) + ly"))
    return cases


def bfs_case(arena, torch, device, log_v: int = 26, deg: int = 8) -> Case:
    """BFS over a random graph (2^log_v vertices x deg out-edges), full
    traversal from vertex 0: one `bfs` launch per level plus a 4-byte read of
    the changed flag (Rodinia's host loop)."""
    from paper_2206_07896_b200 import ArgSlot, Dim3, PackedArgs, routines

    nv = 1 << log_v
    ne = nv * deg
    row = arena.alloc("i32", nv + 1)
    col = arena.alloc("i32", ne)
    lvl = arena.alloc("i32", nv)
    chg = arena.alloc("i32", 1)
    g = torch.Generator(device=device)
    g.manual_seed(99)
    trow = _t(arena, row, torch, device)
    trow.copy_(torch.arange(0, nv + 1, dtype=torch.int64, device=device).mul_(deg).int())
    tcol = _t(arena, col, torch, device)
    tcol.random_(0, nv, generator=g)
    tl = _t(arena, lvl, torch, device)
    tch = _t(arena, chg, torch, device)
    routine = routines.get("bfs")
    levels = {"n": 0}

    def reset():
        tl.fill_(-1)
        tl[0] = 0

    def step(rt, stream):
        cur = 0
        while True:
            arena.fill_value(chg, 0)  # synchronous, ordered before the launch
            pk = PackedArgs([ArgSlot("handle", row), ArgSlot("handle", col), ArgSlot("handle", lvl),
                             ArgSlot("handle", chg), ArgSlot("i32", nv), ArgSlot("i32", cur)])
            rt.launch(routine, Dim3(nv // 256), Dim3(256), 0, pk)
            rt.device_synchronize()
            if int(tch.item()) == 0:
                break
            cur += 1
        levels["n"] = cur + 1
        return cur + 1


    def check():
        lv = tl.long()
        src = torch.repeat_interleave(torch.arange(nv, device=device), deg)
        dst = tcol.long()
        lu, lw = lv[src], lv[dst]
        ok = bool((lv[0] == 0).item())
        # every edge out of a reached vertex reaches its target within +1
        ok &= bool(((lu < 0) | ((lw >= 0) & (lw <= lu + 1))).all().item())
        # every reached vertex at level L > 0 has an in-edge from level L-1
        has_pred = torch.zeros(nv, dtype=torch.bool, device=device)
        m = (lu >= 0) & (lw == lu + 1)
        has_pred[dst[m]] = True
        ok &= bool(((lv <= 0) | has_pred).all().item())
        return ok

    saved = {}

    def check_and_save():
        ok = check()
        saved["lvl"] = tl.clone()
        return ok

    c = Case("bfs", "bfs_scan2+bfs_relax_v+bfs_apply", 4 * ne + 12 * nv, ne, "edge", [], host_loop=step, reset=reset,
             check=check_and_save,
             note=f"2^{log_v} vertices x {deg} random out-edges, full traversal by per-level "
                  "launches (Rodinia host loop); bytes = compulsory 4|E| + 12|V|, elem = edges (TEPS)")
    c.levels = levels

    from paper_2206_07896_b200 import graph

    def fused(rt, stream):
        levels["fused_depth"] = graph.bfs_levels(rt, row, col, lvl, nv, 0)
        return 1

    def fused_check():
        return bool(torch.equal(tl, saved["lvl"])) if "lvl" in saved else check()

    f = Case("bfs_fused", "bfs_expand_v+bfs_compact8s", 4 * ne + 12 * nv, ne, "edge", [], host_loop=fused,
             check=fused_check,
             note="same graph, whole traversal fused on the device, top-down only (bf_bfs_levels: frontier "
                  "queues + L2-resident visited bitmap); levels equal to the per-level launches")

    tg = {}

    def do_step(rt, stream):
        if "t" not in tg:  # the in-edge CSR is built once per graph, outside the timed steps
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            tg["t"] = graph.transpose(rt, row, col, nv)
            torch.cuda.synchronize()
            tg["build_ms"] = (time.perf_counter() - t0) * 1e3
        levels["do_depth"] = graph.bfs_levels(rt, row, col, lvl, nv, 0, transposed=tg["t"])
        return 1

    d = Case("bfs_do", "bfs_expand_v+bfs_bottom_up", 4 * ne + 12 * nv, ne, "edge", [], host_loop=do_step,
             check=fused_check,
             note="same graph, direction-optimizing fused traversal (bf_bfs_levels_do: top-down on small "
                  "frontiers, bottom-up over the in-edge CSR on large ones, chosen on the device per level); "
                  "levels equal to the per-level launches; bytes = the same compulsory 4|E| + 12|V|")
    d.levels = levels
    d.extra = tg
    return c, f, d


def time_case(case: Case, rt, torch, stream, reps: int, warmup: int) -> dict:
    """Device time per step (events on the worker stream) and per launch."""
    def issue():
        if case.host_loop is not None:
            return case.host_loop(rt, stream)
        for launch in case.launches:
            rt.launch(*launch)
        return len(case.launches)

    for _ in range(warmup):
        if case.reset:
            case.reset()
            torch.cuda.synchronize()
        issue()
    rt.device_synchronize()
    torch.cuda.synchronize()
    times = []
    nlaunch = 0
    for _ in range(reps):
        if case.reset:
            case.reset()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        a.record(stream)
        nlaunch = issue()
        b.record(stream)
        rt.device_synchronize()
        b.synchronize()
        wall = time.perf_counter() - t0
        times.append((a.elapsed_time(b) * 1e-3, wall))
    ok = None
    if case.check is not None:
        try:
            ok = bool(case.check())
        except Exception as e:  # a failed check is reported, never hidden
            ok = f"check error: {e!r}"
    dev = statistics.median(t for t, _ in times)
    wall = statistics.median(w for _, w in times)
    return {"dev_s": dev, "wall_s": wall, "launches": nlaunch, "checked": ok}


def sample_instance(name: str, log_n: int):
    """A seeded oracle.instances.Instance of one bench case at 2^log_n
    elements (points for kmeans, input units for backprop, cells for
    hotspot) -> (instance, elements).  bfs returns its graph instead
    (see bfs_sample)."""
    sys.path.insert(0, str(ROOT / "oracle"))
    import instances as I
    import numpy as np

    n = 1 << log_n
    if name in ("vecadd", "vecadd_pr1"):
        a = np.random.default_rng(1).uniform(-1, 1, n).astype(np.float32)
        b = np.random.default_rng(2).uniform(-1, 1, n).astype(np.float32)
        inst = I.Instance("vecadd", I.Geom(max(1, n // 256)), I.Geom(256), 0,
                          [I.Buf("a", "f32", n, a), I.Buf("b", "f32", n, b),
                           I.Buf("c", "f32", n, np.zeros(n, np.float32))],
                          [("buf", "a"), ("buf", "b"), ("buf", "c"), ("i32", n)], ["c"])
        return inst, n
    if name == "nn":
        return I.nn(n, 256), n
    if name == "hotspot":
        side = 1 << (log_n // 2)
        return I.hotspot(side, side, 16, 16, seed=0), side * side
    pix = np.random.default_rng(2).integers(0, 1 << 16, n).astype(np.int32)
    if name == "hist":
        return I.Instance("hist", I.Geom(max(1, n // 256)), I.Geom(256), 0,
                          [I.Buf("pix", "i32", n, pix), I.Buf("counts", "i32", 16, np.zeros(16, np.int32))],
                          [("buf", "pix"), ("buf", "counts"), ("i32", n), ("i32", 16)], ["counts"]), n
    if name == "hist_stride":
        return I.Instance("hist_stride", I.Geom(1), I.Geom(256), 0,
                          [I.Buf("pix", "i32", n, pix), I.Buf("counts", "i32", 16, np.zeros(16, np.int32))],
                          [("buf", "pix"), ("buf", "counts"), ("i32", max(1, n // 256)), ("i32", 16)],
                          ["counts"]), n
    if name == "reduce":
        return I.Instance("reduce", I.Geom(max(1, n // 256)), I.Geom(256), 0,
                          [I.Buf("x", "i32", n, pix),
                           I.Buf("out", "i32", max(1, n // 256), np.zeros(max(1, n // 256), np.int32))],
                          [("buf", "x"), ("buf", "out"), ("i32", n)], ["out"]), n
    if name == "wreduce":
        return I.Instance("wreduce", I.Geom(max(1, n // 256)), I.Geom(256), 0,
                          [I.Buf("x", "i32", n, pix), I.Buf("out", "i32", 1, np.zeros(1, np.int32))],
                          [("buf", "x"), ("buf", "out"), ("i32", n)], ["out"]), n
    if name == "fir":
        m = max(1, n // 256)
        x = np.random.default_rng(3).uniform(-1, 1, m * 256 + 8).astype(np.float32)
        w = np.random.default_rng(4).uniform(-1, 1, 8).astype(np.float32)
        return I.Instance("fir", I.Geom(1), I.Geom(256), 0,
                          [I.Buf("x", "f32", x.size, x),
                           I.Buf("y", "f32", m * 256, np.zeros(m * 256, np.float32)), I.Buf("w", "f32", 8, w)],
                          [("buf", "x"), ("buf", "y"), ("buf", "w"), ("i32", 8), ("i32", m)], ["y"]), m * 256
    if name in ("kmeans", "kmeans_loop"):
        return I.kmeans(n, 32, 16, 256), n
    if name == "nn_topk":
        return I.nn_topk(n, 5, seed=1, d=I.nn_inputs(n, 1)[0::2] + 90.0), n
    if name == "bp_forward":
        return I.backprop_forward(n, seed=1), n
    if name == "bp_adjust":
        return I.backprop_adjust(n, seed=1), n
    return None, 0


# bench-run sample sizes (log2): the C port, all host cores, ~0.5 s each
PORT_LOG = {"vecadd": 24, "vecadd_pr1": 20, "nn": 22, "hist": 24, "hist_stride": 22, "reduce": 24,
            "wreduce": 24, "fir": 20, "kmeans": 16, "kmeans_loop": 16, "bp_forward": 18,
            "bp_adjust": 18, "bfs": 22, "bfs_fused": 22, "bfs_do": 22, "hotspot": 22, "nn_topk": 22}
# the reference runtime (pure Python): SURVEY §8d sizes for the study
# (--workload cpu-runtime), and ~1 s samples for the default bench line
REF_LOG_SURVEY = {"vecadd_pr1": 20, "vecadd": 20, "hotspot": 16, "kmeans": 10, "bfs": 14, "nn": 20,
                  "hist": 16, "hist_stride": 16, "reduce": 16, "wreduce": 16, "fir": 16,
                  "bp_forward": 12, "bp_adjust": 12}
REF_LOG_BENCH = {"vecadd_pr1": 14, "vecadd": 14, "hotspot": 12, "kmeans": 7, "bfs": 11, "nn": 14,
                 "hist": 13, "hist_stride": 13, "reduce": 13, "wreduce": 13, "fir": 13,
                 "bp_forward": 9, "bp_adjust": 9, "nn_topk": 12}


def cpu_sample(name: str, threads: int, budget: float = 0.5) -> Optional[dict]:
    """Oracle port (oracle/oracle.c) throughput on a bounded sample of the
    same kernel, in elements/s, on all host threads: the launch's logical
    blocks split into one contiguous range per thread (oracle.run_par, the
    reference pool's average grain).  Single-block launches (fir and
    hist_stride are grid 1 in the corpus) run on one thread."""
    sys.path.insert(0, str(ROOT / "oracle"))
    import instances as I
    import oracle

    if name in ("bfs", "bfs_fused", "bfs_do"):
        nv = 1 << PORT_LOG["bfs"]
        row, col = I.random_graph(nv, 8, 1)
        t0 = time.perf_counter()
        oracle.bfs_full(row, col, nv, 0)
        dt = time.perf_counter() - t0
        return {"elem_per_s": col.size / dt, "cores": 1, "kind": "port",
                "sample": f"bfs 2^{PORT_LOG['bfs']} vertices x 8, frontier-queue restatement, {dt:.2f} s"}
    if name not in PORT_LOG:
        return None
    inst, elems = sample_instance(name, PORT_LOG[name])
    nt = threads if inst.grid.total > 1 else 1
    t0 = time.perf_counter()
    reps = 0
    while True:
        oracle.run_par(inst, nt)
        reps += 1
        if time.perf_counter() - t0 > budget:
            break
    dt = (time.perf_counter() - t0) / reps
    return {"elem_per_s": elems / dt, "cores": nt, "kind": "port",
            "sample": f"{name} {elems} elements, oracle/oracle.c over {nt} thread(s), {reps} run(s) of {dt:.3f} s"}


REF_NAME = {"kmeans_loop": "kmeans", "bfs_fused": "bfs", "bfs_do": "bfs"}
_REF_CACHE: dict = {}


def reference_runtime_pair(name: str, sizes: dict, threads: int) -> Optional[dict]:
    """reference_runtime_sample at pool = host cores and pool = 1 (the GIL
    makes them about equal), cached per kernel for one bench run."""
    key = REF_NAME.get(name, name)
    if key not in sizes:
        return None
    if (key, sizes[key]) not in _REF_CACHE:
        try:
            _REF_CACHE[(key, sizes[key])] = {
                "pool_cores": reference_runtime_sample(key, threads, sizes[key]),
                "pool_1": reference_runtime_sample(key, 1, sizes[key])}
        except Exception as e:  # reported, never hidden
            _REF_CACHE[(key, sizes[key])] = {"error": repr(e)}
    return _REF_CACHE[(key, sizes[key])]


def _reference_modules():
    for p in (ROOT / "baseline" / "_ref", Path("/root/reference/pkg/src")):
        if (p / "blockfuse" / "__init__.py").exists():
            if str(p) not in sys.path:
                sys.path.append(str(p))
            break
    import blockfuse.arena as A
    import blockfuse.bench as B
    import blockfuse.executor as E
    import blockfuse.hostprog as H
    import blockfuse.parser as P
    import blockfuse.runtime as R
    import blockfuse.syntax as S
    from blockfuse.transform import transform as T
    return A, B, E, H, P, R, S, T


_REF_KERNELS: dict = {}


def _reference_kernel(name: str, warp_size: int = 32):
    """The reference's compiled MpmdKernel of a corpus kernel, or of one of
    our north-star kernels (paper_2206_07896_b200/kernels/*.kn) parsed and
    transformed by the reference's own front end."""
    A, B, E, H, P, R, S, T = _reference_modules()
    if name not in _REF_KERNELS:
        if name in B.CORPUS:
            _REF_KERNELS[name] = B.CORPUS[name].compiled(warp_size)
        else:
            for f in (ROOT / "paper_2206_07896_b200" / "kernels").glob("*.kn"):
                for kname, prog in P.parse_unit(f.read_text()).items():
                    if kname == name:
                        _REF_KERNELS[name] = T(prog, warp_mode=False, warp_size=warp_size)
    return _REF_KERNELS[name]


def reference_runtime_sample(name: str, pool: int, log_n: int) -> Optional[dict]:
    """The unmodified reference runtime (blockfuse.Runtime: task queue +
    Python thread pool, runtime.py:216-350) running one launch of the case
    (bfs: Rodinia's per-level host loop to the end of the traversal) on a
    2^log_n sample; wall time of launch + device_synchronize.  The result is
    compared with the oracle (`matches_oracle`)."""
    sys.path.insert(0, str(ROOT / "oracle"))
    import instances as I
    import numpy as np
    import oracle
    A, B, E, H, P, R, S, T = _reference_modules()
    if name in ("bfs", "bfs_fused", "bfs_do"):
        nv = 1 << log_n
        row, col = I.random_graph(nv, 8, 1)
        want, depth = oracle.bfs_full(row, col, nv, 0)
        arena = A.DeviceArena()
        hr, hc, hl, hch = (arena.alloc("i32", nv + 1), arena.alloc("i32", col.size), arena.alloc("i32", nv),
                           arena.alloc("i32", 1))
        arena.fill(hr, row.tolist())
        arena.fill(hc, col.tolist())
        init = [-1] * nv
        init[0] = 0
        arena.fill(hl, init)
        mk = _reference_kernel("bfs")
        t0 = time.perf_counter()
        with R.Runtime(arena, pool_size=pool) as rt:
            cur = 0
            while True:
                arena.fill(hch, [0])
                pk = H.PackedArgs([E.ArgSlot("handle", hr), E.ArgSlot("handle", hc), E.ArgSlot("handle", hl),
                                   E.ArgSlot("handle", hch), E.ArgSlot("i32", nv), E.ArgSlot("i32", cur)])
                rt.launch(mk, S.Dim3(-(-nv // 256)), S.Dim3(256), 0, pk)
                rt.device_synchronize()
                if arena.to_list(hch)[0] == 0:
                    break
                cur += 1
        dt = time.perf_counter() - t0
        ok = bool(np.array_equal(np.array(arena.to_list(hl), np.int32), want))
        return {"elem_per_s": col.size / dt, "unit_elem": "edge", "seconds": round(dt, 3), "pool": pool,
                "kind": "reference", "matches_oracle": ok,
                "sample": f"blockfuse Runtime, bfs 2^{log_n} x 8 full traversal ({cur + 1} level launches), "
                          f"pool {pool}"}
    inst, elems = sample_instance(name, log_n)
    if inst is None:
        return None
    want, _ = oracle.run(inst)
    arena = A.DeviceArena()
    handles = {}
    for b in inst.buffers:
        h = arena.alloc(b.scalar, b.length)
        arena.fill(h, np.asarray(b.values).reshape(-1)[: b.length].tolist())
        handles[b.name] = h
    pk = H.PackedArgs([E.ArgSlot("handle", handles[a[1]]) if a[0] == "buf" else E.ArgSlot(a[0], a[1])
                       for a in inst.args])
    mk = _reference_kernel(inst.kernel)
    g = S.Dim3(inst.grid.x, inst.grid.y, inst.grid.z)
    bl = S.Dim3(inst.block.x, inst.block.y, inst.block.z)
    t0 = time.perf_counter()
    with R.Runtime(arena, pool_size=pool) as rt:
        rt.launch(mk, g, bl, inst.shmem, pk)
        rt.device_synchronize()
    dt = time.perf_counter() - t0
    ok = True
    for o in inst.outputs:
        got = np.array(arena.to_list(handles[o]), dtype=want[o].dtype)
        if inst.kernel == "kmeans" and o == "sums":
            ok &= bool(np.allclose(got, want[o], rtol=1e-4, atol=1e-4))
        else:
            ok &= bool(np.array_equal(got.view(np.uint8), want[o].view(np.uint8)))
    return {"elem_per_s": elems / dt, "seconds": round(dt, 3), "pool": pool, "kind": "reference",
            "matches_oracle": ok,
            "sample": f"blockfuse Runtime, {name} 2^{log_n} ({elems} elements), grid "
                      f"{inst.grid.x}x{inst.grid.y} x block {inst.block.x}x{inst.block.y}, pool {pool}"}
