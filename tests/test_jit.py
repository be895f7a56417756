"""JIT path: reference kernels compiled from their AST by
codegen.py + NVRTC run bit-exactly against the reference's own interpreter —
the corpus and north-star goldens forced through the JIT, the reference's
executor unit kernels (test_executor.py), and host scripts with ad-hoc
kernels (test_acceptance.py criterion 5)."""

import random

import numpy as np
import pytest

import golden
from conftest import has_gpu
from gpu_helpers import bit_equal, gpu_run

from paper_2206_07896_b200 import ArgSlot, DeviceArena, Dim3, PackedArgs, Runtime, RuntimeFault, codegen, routines


def test_codegen_compiles_every_kernel_kind(reference):
    """CPU: CUDA source is generated for every corpus and north-star kernel
    (nvcc compiles it in tests/test_abi-style builds; NVRTC on the box)."""
    from blockfuse.bench import CORPUS
    from blockfuse.parser import parse_unit
    from blockfuse.transform import transform
    for name, case in CORPUS.items():
        src, entry, spec = codegen.generate(case.compiled())
        assert entry in src and "__syncthreads" in src
    for nm in ("hotspot", "kmeans", "nn", "bfs"):
        kp = parse_unit(routines.kernel_source(nm))[nm]
        src, entry, spec = codegen.generate(transform(kp))
        assert len(spec) == len(kp.params)


gpu = pytest.mark.gpu


@pytest.fixture
def need_gpu():
    if not has_gpu():
        pytest.skip("no CUDA device")


@pytest.fixture
def force_jit(reference):
    routines.FORCE_JIT = True
    yield
    routines.FORCE_JIT = False


def _mk_for(reference, inst):
    from blockfuse.bench import CORPUS
    from blockfuse.parser import parse_unit
    from blockfuse.transform import transform
    if inst.kernel in CORPUS:
        return transform(CORPUS[inst.kernel].kernel(), warp_mode=inst.kernel == "wreduce",
                         warp_size=inst.warp_size)
    kp = parse_unit(routines.kernel_source(inst.kernel))[inst.kernel]
    return transform(kp)


@gpu
@pytest.mark.parametrize("name", golden.SETS)
def test_goldens_through_jit(need_gpu, reference, force_jit, name):
    cases = golden.load(name)
    for k, (inst, expected, trap) in enumerate(cases):
        if inst.kernel in ("reduce", "bpnn_layerforward") and inst.block.z > 1 or \
                inst.kernel == "reduce" and inst.block.y > 1:
            # duplicated threads update buf[t] in place without atomics: a
            # data race under CUDA semantics, ordered only by the reference's
            # sequential interpreter.  The hand-written reduce reproduces the
            # order (reduce_tree); generated code follows CUDA.
            # Same for backprop's in-place column tree with duplicated z threads.
            continue
        mk = _mk_for(reference, inst)
        got, got_trap, _, _ = gpu_run(inst, routine=mk)
        if trap is not None:
            assert got_trap is not None and got_trap[0] == trap, (name, k, trap, got_trap)
            continue
        assert got_trap is None, (name, k, inst.kernel, got_trap)
        for buf, want in expected.items():
            g = got[buf]
            if inst.kernel == "kmeans" and buf == "sums":
                scale = np.maximum(np.maximum(np.abs(g), np.abs(want)), 1.0)
                assert np.all(np.abs(g.astype(np.float64) - want) <= 1e-4 * scale), (name, k)
            else:
                assert bit_equal(g, want), (name, k, inst.kernel, buf)


def _run_ref_and_ours(reference, src, grid, block, buffers, scalars=(), warp_mode=False, warp_size=32,
                      dyn_bytes=0):
    """Run one ad-hoc kernel through the reference's run_mpmd and through our
    runtime (JIT); returns (ref buffers, ref trap kind, our buffers, our trap kind)."""
    from blockfuse.arena import DeviceArena as RefArena
    from blockfuse.executor import ArgSlot as RefSlot, run_mpmd
    from blockfuse.hostprog import PackedArgs as RefPacked
    from blockfuse.parser import parse
    from blockfuse.syntax import Dim3 as RefDim3
    from blockfuse.transform import transform
    mk = transform(parse(src), warp_mode=warp_mode, warp_size=warp_size)
    ra = RefArena()
    rh = []
    for scalar, vals in buffers:
        h = ra.alloc(scalar, len(vals))
        ra.fill(h, vals)
        rh.append(h)
    rslots = [RefSlot("handle", h) for h in rh] + [RefSlot(k, v) for k, v in scalars]
    rtrap = None
    try:
        run_mpmd(mk, RefDim3(*grid), RefDim3(*block), RefPacked(rslots), ra, dyn_bytes=dyn_bytes)
    except Exception as e:
        rtrap = getattr(e, "kind", repr(e))
    ref_out = [ra.to_list(h) for h in rh]
    arena = DeviceArena()
    oh = []
    for scalar, vals in buffers:
        h = arena.alloc(scalar, len(vals))
        arena.fill(h, vals)
        oh.append(h)
    slots = [ArgSlot("handle", h) for h in oh] + [ArgSlot(k, v) for k, v in scalars]
    otrap = None
    with Runtime(arena) as rt:
        rt.launch(mk, Dim3(*grid), Dim3(*block), dyn_bytes, PackedArgs(slots))
        try:
            rt.device_synchronize()
        except RuntimeFault as e:
            otrap = e.trap.kind
    our_out = [arena.to_list(h) for h in oh]
    return ref_out, rtrap, our_out, otrap


EXECUTOR_CASES = [
    # (name, source, grid, block, buffers, scalars, warp_mode, warp_size, dyn)   test_executor.py
    ("vecadd_small", "kernel vecadd(a: global f32[], b: global f32[], c: global f32[], n: i32) {\n"
     "  let id: i32 = blockIdx.x * blockDim.x + threadIdx.x;\n  if (id < n) { c[id] = a[id] + b[id]; }\n}\n",
     (2,), (2,), [("f32", [1, 2, 3, 4]), ("f32", [10, 20, 30, 40]), ("f32", [0] * 4)], [("i32", 4)], False, 32, 0),
    ("reverse_dyn", "kernel reverse(d: global i32[], n: i32) {\n  extern shared i32 s[];\n"
     "  let t: i32 = threadIdx.x;\n  let tr: i32 = n - t - 1;\n  s[t] = d[t];\n  barrier;\n  d[t] = s[tr];\n}\n",
     (1,), (8,), [("i32", list(range(8)))], [("i32", 8)], False, 32, 32),
    ("mark_3d", "kernel mark(o: global i32[]) {\n  let t: i32 = threadIdx.z * blockDim.y * blockDim.x"
     " + threadIdx.y * blockDim.x + threadIdx.x;\n  o[t] = t + 1;\n}\n",
     (1,), (2, 2, 2), [("i32", [0] * 8)], [], False, 32, 0),
    ("wrap", "kernel w(o: global i32[]) { o[0] = 2147483647 + 1; }", (1,), (1,), [("i32", [0])], [], False, 32, 0),
    ("cas_fail", "kernel c(x: global i32[]) { atomic_cas(x[0], 9, 5); }", (1,), (1,), [("i32", [3])], [], False, 32, 0),
    ("bump", "kernel bump(x: global i32[]) { atomic_add(x[0], 1); }", (50,), (7,), [("i32", [0])], [], False, 32, 0),
    ("oob_load", "kernel k(a: global i32[]) { let v: i32 = a[threadIdx.x + 100]; }", (1,), (4,),
     [("i32", [0] * 4)], [], False, 32, 0),
    ("oob_shared", "kernel k(a: global i32[]) { shared i32 s[2];\n  s[threadIdx.x] = 1; }", (1,), (4,),
     [("i32", [0] * 4)], [], False, 32, 0),
    ("div0", "kernel k(a: global i32[]) { a[0] = 1 / a[1]; }", (1,), (1,), [("i32", [0, 0, 0, 0])], [], False, 32, 0),
    ("dyn_missing", "kernel k(a: global i32[]) { extern shared i32 s[];\n  s[0] = 1; a[0] = s[0]; }", (1,), (1,),
     [("i32", [0])], [], False, 32, 0),
    ("shfl4", "kernel s(o: global i32[]) {\n  let v: i32 = threadIdx.x;\n  let w: i32 = shfl_down(v, 1);\n"
     "  o[threadIdx.x] = w;\n}\n", (1,), (8,), [("i32", [0] * 8)], [], True, 4, 0),
    ("shfl_partial", "kernel s(o: global i32[]) {\n  let v: i32 = threadIdx.x;\n  o[threadIdx.x] = shfl_down(v, 2);\n}\n",
     (1,), (6,), [("i32", [0] * 6)], [], True, 4, 0),
    ("votes", "kernel v(o: global i32[]) {\n  let a: i32 = vote_any(threadIdx.x == 3);\n"
     "  let b: i32 = vote_all(threadIdx.x < 8);\n  let c: i32 = vote_all(threadIdx.x < 3);\n"
     "  o[threadIdx.x] = a * 100 + b * 10 + c;\n}\n", (1,), (8,), [("i32", [0] * 8)], [], True, 8, 0),
    ("wsum", "kernel wsum(x: global i32[], out: global i32[]) {\n  let v: i32 = x[threadIdx.x];\n"
     "  let a: i32 = shfl_down(v, 2);\n  let b: i32 = v + a;\n  let c: i32 = shfl_down(b, 1);\n"
     "  let d: i32 = b + c;\n  if (threadIdx.x % 4 == 0) { atomic_add(out[0], d); }\n}\n",
     (1,), (8,), [("i32", [3, 1, 4, 1, 5, 9, 2, 6]), ("i32", [0])], [], True, 4, 0),
    ("floats", "kernel f(a: global f32[], o: global f64[], x: f32, y: f64) {\n"
     "  let t: i32 = threadIdx.x;\n  let u: f32 = a[t] * x + 0.1;\n  let q: f64 = y / (y + 1.0) - sqrt(y);\n"
     "  o[t] = q * q + y;\n  a[t] = min(u, 0.25) - max(-u, abs(u - 1.0)) + u / 3.0;\n}\n",
     (1,), (16,), [("f32", [i * 0.37 - 2 for i in range(16)]), ("f64", [0.0] * 16)], [("f32", 1.1), ("f64", 2.5)],
     False, 32, 0),
    ("ints64", "kernel g(a: global i64[], b: global i32[]) {\n  let t: i32 = threadIdx.x;\n"
     "  let v: i64 = a[t] * 3 - 7;\n  a[t] = v / 2 + v % 5;\n  b[t] = (t - 5) / 2 + (t - 5) % 3 - min(t, 3);\n}\n",
     (1,), (12,), [("i64", [2**40 + i * 123457 for i in range(12)]), ("i32", [0] * 12)], [], False, 32, 0),
    ("loops_barriers", "kernel l(x: global i32[], out: global i32[]) {\n  shared i32 buf[64];\n"
     "  let t: i32 = threadIdx.x;\n  buf[t] = x[blockIdx.x * blockDim.x + t];\n  barrier;\n"
     "  for (s = 1; s < blockDim.x; s += s) {\n    if (t % (s * 2) == 0 && t + s < blockDim.x) {\n"
     "      buf[t] = buf[t] + buf[t + s];\n    }\n    barrier;\n  }\n"
     "  for (j = 0; j < 3; j += 1) { if (t == j) { out[blockIdx.x * 3 + j] = buf[0] * (j + 1); } }\n}\n",
     (3,), (64,), [("i32", list(range(192))), ("i32", [0] * 9)], [], False, 32, 0),
    ("f32_atomics", "kernel fa(s: global f32[], x: global f32[]) {\n  atomic_add(s[threadIdx.x % 2], x[threadIdx.x]);\n}\n",
     (1,), (1,), [("f32", [0.0, 0.0]), ("f32", [0.1])], [], False, 32, 0),
    # a trapping loop step (0 after the trap) must end the loop, not hang:
    # the reference raises DivByZero at the first step
    ("trap_step_loop", "kernel k(a: global i32[], n: i32, d: i32) {\n"
     "  for (i = 0; i < n; i += n / d) { a[0] = a[0] + 1; }\n}\n",
     (1,), (4,), [("i32", [0])], [("i32", 10), ("i32", 0)], False, 32, 0),
    # the same inside a barrier loop (a LoopSection)
    ("trap_step_barrier_loop", "kernel k(a: global i32[], n: i32, d: i32) {\n  shared i32 s[4];\n"
     "  for (i = 0; i < n; i += n / d) { s[threadIdx.x] = i; barrier; a[threadIdx.x] = s[0]; barrier; }\n}\n",
     (2,), (4,), [("i32", [0] * 4)], [("i32", 10), ("i32", 0)], False, 32, 0),
]


@gpu
@pytest.mark.parametrize("case", EXECUTOR_CASES, ids=[c[0] for c in EXECUTOR_CASES])
def test_reference_executor_kernels_through_jit(need_gpu, reference, case):
    name, src, grid, block, buffers, scalars, wm, ws, dyn = case
    ref, rtrap, ours, otrap = _run_ref_and_ours(reference, src, grid, block, buffers, scalars, wm, ws, dyn)
    if rtrap is not None:
        assert otrap == rtrap, (name, rtrap, otrap)
        return
    assert otrap is None, (name, otrap)
    for r, o in zip(ref, ours):
        a, b = np.asarray(r), np.asarray(o)
        assert a.shape == b.shape and np.array_equal(a.view(np.uint8) if a.dtype.kind == "f" else a,
                                                     b.view(np.uint8) if b.dtype.kind == "f" else b), (name, r, o)


@gpu
def test_reference_implicit_sync_scripts_with_adhoc_kernels(need_gpu, reference):
    """test_acceptance.py:181-268 soundness half with its own writer/reader
    kernels, which now run through the JIT."""
    from blockfuse.hostprog import Alloc, BufferArg, Download, HostProgram, Launch, Upload
    from blockfuse.parser import parse
    from blockfuse.runtime import run_host_program
    from blockfuse.syntax import Dim3 as RDim3
    from test_dropin import our_runtime
    kernels = {"writer": parse("kernel writer(dst: global i32[], src: global i32[]) "
                               "{ dst[threadIdx.x] = src[threadIdx.x]; }"),
               "reader": parse("kernel reader(src: global i32[]) { let v: i32 = src[threadIdx.x]; }")}
    rng = random.Random(99)
    bufs = ["b0", "b1", "b2", "b3"]
    for trial in range(30):
        ops = [Alloc(b, "i32", 8) for b in bufs]
        for _ in range(rng.randint(2, 5)):
            kind = rng.randrange(3)
            if kind == 0:
                dst, src = rng.sample(bufs, 2)
                ops.append(Launch("writer", RDim3(2), RDim3(8), 0, [BufferArg(dst), BufferArg(src)]))
            elif kind == 1:
                ops.append(Upload(rng.choice(bufs), "fill:seq"))
            else:
                ops.append(Download(rng.choice(bufs), f"out{len(ops)}.bin"))
        program = HostProgram(ops)
        want = run_host_program(program, kernels, pool_size=2)
        with our_runtime(reference):
            got = run_host_program(program, kernels, pool_size=2, hold_blocks=True)
        assert got.conflicts == []
        assert got.downloads == want.downloads
