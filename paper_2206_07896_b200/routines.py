"""Routine handles: what `Runtime.launch` dispatches on.

The reference passes an `MpmdKernel` (transform.py:109-221) as the launch
routine; its `name` is the dispatch key, `warp_mode`/`warp_size` shape warp
intrinsics, `has_atomics()` and `static_instruction_estimate()` feed the
AutoAggressive grain (runtime.py:78-101) and `to_dict()` is a stable
fingerprint of the kernel body.

`Runtime.launch` accepts either a reference `MpmdKernel` (duck-typed) or a
`Routine` from this module, which carries the same fields for the kernels
implemented as hand-written sm_100a code.  A reference kernel whose name and
body fingerprint match a registered kernel runs the hand-written kernel (the
fingerprints were produced from the reference's own `transform()` by
oracle/gen_golden.py); any other reference kernel is compiled from its AST
by codegen.py + NVRTC (bf_jit_register) — never run on the CPU.
"""

from __future__ import annotations

import hashlib
import json
from dataclasses import dataclass
from pathlib import Path
from typing import Optional

KERNEL_DIR = Path(__file__).resolve().parent / "kernels"


class KernelNotImplemented(Exception):
    """No sm_100a implementation exists and none can be generated for this
    routine (there is no CPU fallback)."""


@dataclass(frozen=True)
class Routine:
    name: str
    params: tuple  # ((name, "global f32[]" | "i32" | ...), ...)
    atomics: bool
    estimate: int
    warp_mode: bool = False
    warp_size: int = 32
    source: Optional[str] = None  # .kn file for kernels this package defines

    def has_atomics(self) -> bool:
        return self.atomics

    def static_instruction_estimate(self) -> int:
        return self.estimate

    @property
    def param_signature(self):
        return self.params


def _p(*items):
    return tuple(items)


# name -> (params, has_atomics, static_instruction_estimate, warp_mode, source)
# values checked against the reference's transform() in tests/test_routines.py
_TABLE = {
    # the seven corpus kernels (blockfuse/corpus/*.kn)
    "vecadd": (_p(("a", "global f32[]"), ("b", "global f32[]"), ("c", "global f32[]"), ("n", "i32")),
               False, 3, False, None),
    "reverse": (_p(("d", "global i32[]"), ("n", "i32")), False, 4, False, None),
    "reduce": (_p(("x", "global i32[]"), ("out", "global i32[]"), ("n", "i32")), False, 11, False, None),
    "hist": (_p(("pix", "global i32[]"), ("counts", "global i32[]"), ("n", "i32"), ("nbins", "i32")),
             True, 3, False, None),
    "fir": (_p(("x", "global f32[]"), ("y", "global f32[]"), ("w", "global f32[]"), ("taps", "i32"),
               ("m", "i32")), False, 6, False, None),
    "hist_stride": (_p(("pix", "global i32[]"), ("counts", "global i32[]"), ("k", "i32"),
                       ("nbins", "i32")), True, 3, False, None),
    "wreduce": (_p(("x", "global i32[]"), ("out", "global i32[]"), ("n", "i32")), True, 11, True, None),
    # north-star kernels, written in the reference DSL (kernels/*.kn)
    "hotspot": (_p(("src", "global f32[]"), ("power", "global f32[]"), ("dst", "global f32[]"),
                   ("rows", "i32"), ("cols", "i32"), ("sdc", "f32"), ("rx1", "f32"), ("ry1", "f32"),
                   ("rz1", "f32"), ("amb", "f32")), False, 14, False, "hotspot.kn"),
    "nn": (_p(("ll", "global f32[]"), ("d", "global f32[]"), ("n", "i32"), ("x", "f32"), ("y", "f32")),
           False, 5, False, "nn.kn"),
    "nn_topk": (_p(("d", "global f32[]"), ("idx", "global i32[]"), ("dist", "global f32[]"), ("n", "i32"),
                   ("k", "i32")), False, 31, False, "nn_topk.kn"),
    "kmeans": (_p(("f", "global f32[]"), ("cent", "global f32[]"), ("member", "global i32[]"),
                  ("sums", "global f32[]"), ("counts", "global i32[]"), ("npts", "i32"), ("nf", "i32"),
                  ("k", "i32")), True, 16, False, "kmeans.kn"),
    "bfs": (_p(("row", "global i32[]"), ("col", "global i32[]"), ("lvl", "global i32[]"),
               ("changed", "global i32[]"), ("nv", "i32"), ("cur", "i32")), False, 8, False, "bfs.kn"),
    "bpnn_layerforward": (_p(("input", "global f32[]"), ("w", "global f32[]"), ("partial", "global f32[]"),
                             ("hid", "i32")), False, 14, False, "backprop.kn"),
    "bpnn_adjust_weights": (_p(("delta", "global f32[]"), ("hid", "i32"), ("ly", "global f32[]"),
                               ("inn", "i32"), ("w", "global f32[]"), ("oldw", "global f32[]")),
                            False, 11, False, "backprop.kn"),
}


def names() -> list[str]:
    return list(_TABLE)


def get(name: str, warp_mode: Optional[bool] = None, warp_size: int = 32) -> Routine:
    if name not in _TABLE:
        raise KernelNotImplemented(f"no sm_100a kernel for {name!r}")
    params, atomics, est, wm, src = _TABLE[name]
    return Routine(name, params, atomics, est, wm if warp_mode is None else warp_mode,
                   warp_size, src)


def kernel_source(name: str) -> str:
    src = _TABLE[name][4]
    if src is None:
        raise KeyError(f"{name} is a reference corpus kernel (blockfuse/corpus/{name}.kn)")
    return (KERNEL_DIR / src).read_text()


def fingerprint_of(d: dict) -> str:
    """Stable hash of an MpmdKernel.to_dict() with the warp shaping removed
    (warp_mode/warp_size/loop_shape change how, not what, a kernel computes)."""
    d = dict(d)
    d.pop("warp_mode", None)
    d.pop("warp_size", None)
    d["sections"] = [{k: v for k, v in s.items() if k != "loop_shape"} for s in d.get("sections", [])]
    return hashlib.sha256(json.dumps(d, sort_keys=True).encode()).hexdigest()


_FP_FILE = Path(__file__).resolve().parent / "fingerprints.json"
_fps: Optional[dict] = None


def expected_fingerprint(name: str) -> Optional[str]:
    global _fps
    if _fps is None:
        _fps = json.loads(_FP_FILE.read_text()) if _FP_FILE.exists() else {}
    return _fps.get(name)


# Tests set this to route even the registered kernels through the JIT path.
FORCE_JIT = False
_jit_keys: dict = {}


def _jit_key(routine) -> str:
    """Compile (once per process) a reference MpmdKernel through codegen.py +
    NVRTC and return its registry key."""
    import ctypes as C

    from . import _lib, codegen
    fp = codegen.fingerprint(routine)
    key = "jit:" + fp[:32]
    if key in _jit_keys:
        return key
    try:
        src, entry, spec = codegen.generate(routine)
    except codegen.CodegenError as e:
        raise KernelNotImplemented(f"kernel {routine.name!r}: cannot generate CUDA: {e}") from None
    n = len(spec)
    kinds = (C.c_int32 * max(n, 1))(*[_lib.SLOT_KINDS[k] for k, _ in spec])
    scal = (C.c_int32 * max(n, 1))(*[_lib.SCALARS[s] if s else 0 for _, s in spec])
    dyn = getattr(routine.shared_layout, "dynamic_scalar", None)
    rc = _lib.lib().bf_jit_register(key.encode(), src.encode(), entry.encode(), n, kinds, scal,
                                    _lib.SCALARS[dyn] if dyn else -1)
    if rc != _lib.OK:
        raise KernelNotImplemented(f"kernel {routine.name!r}: JIT compile failed: {_lib.last_error()}")
    _jit_keys[key] = src
    return key


def resolve(routine) -> tuple[str, bool, int]:
    """(registry key, warp_mode, warp_size) for a Routine or a reference
    MpmdKernel.

    A registered name with a matching body runs its hand-written sm_100a
    kernel.  Any other reference kernel (a different body under a known
    name, or an unregistered name) is compiled from its AST (codegen.py,
    NVRTC) and runs through the same runtime.  A `Routine` for an unknown
    name, or an object without an AST, raises KernelNotImplemented."""
    name = getattr(routine, "name", None)
    if not isinstance(name, str):
        raise TypeError(f"launch routine must have a .name, got {routine!r}")
    warp_mode = bool(getattr(routine, "warp_mode", False))
    warp_size = int(getattr(routine, "warp_size", 32)) if warp_mode else 0
    has_ast = hasattr(routine, "sections") and hasattr(routine, "to_dict")
    registered = name in _TABLE
    if registered and not FORCE_JIT:
        if isinstance(routine, Routine) or not hasattr(routine, "to_dict"):
            return name, warp_mode, warp_size
        want = expected_fingerprint(name)
        got = fingerprint_of(routine.to_dict())
        if want is None or got == want:
            return name, warp_mode, warp_size
    if has_ast:
        return _jit_key(routine), warp_mode, warp_size
    if registered:
        return name, warp_mode, warp_size
    raise KernelNotImplemented(
        f"kernel {name!r} has no sm_100a implementation and no AST to compile "
        f"(registered: {', '.join(_TABLE)})")
