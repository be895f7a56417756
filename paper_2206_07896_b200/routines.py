"""Routine handles: what `Runtime.launch` dispatches on.

The reference passes an `MpmdKernel` (transform.py:109-221) as the launch
routine; its `name` is the dispatch key, `warp_mode`/`warp_size` shape warp
intrinsics, `has_atomics()` and `static_instruction_estimate()` feed the
AutoAggressive grain (runtime.py:78-101) and `to_dict()` is a stable
fingerprint of the kernel body.

`Runtime.launch` accepts either a reference `MpmdKernel` (duck-typed; its
fingerprint must match the kernel this package implements — a different body
under a known name is rejected, never silently run) or a `Routine` from this
module, which carries the same fields for the kernels implemented as sm_100a
code.  The fingerprints were produced from the reference's own `transform()`
by oracle/gen_golden.py (see tests/golden/fingerprints.json).
"""

from __future__ import annotations

import hashlib
import json
from dataclasses import dataclass
from pathlib import Path
from typing import Optional

KERNEL_DIR = Path(__file__).resolve().parent / "kernels"


class KernelNotImplemented(Exception):
    """No sm_100a implementation exists for this routine (there is no CPU
    fallback)."""


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
    "kmeans": (_p(("f", "global f32[]"), ("cent", "global f32[]"), ("member", "global i32[]"),
                  ("sums", "global f32[]"), ("counts", "global i32[]"), ("npts", "i32"), ("nf", "i32"),
                  ("k", "i32")), True, 16, False, "kmeans.kn"),
    "bfs": (_p(("row", "global i32[]"), ("col", "global i32[]"), ("lvl", "global i32[]"),
               ("changed", "global i32[]"), ("nv", "i32"), ("cur", "i32")), False, 8, False, "bfs.kn"),
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


def resolve(routine) -> tuple[str, bool, int]:
    """(name, warp_mode, warp_size) for a Routine or a reference MpmdKernel.

    Raises KernelNotImplemented for names without an sm_100a kernel and for a
    reference kernel whose body differs from the implemented one."""
    name = getattr(routine, "name", None)
    if not isinstance(name, str):
        raise TypeError(f"launch routine must have a .name, got {routine!r}")
    if name not in _TABLE:
        raise KernelNotImplemented(
            f"kernel {name!r} has no sm_100a implementation (registered: {', '.join(_TABLE)})")
    if not isinstance(routine, Routine) and hasattr(routine, "to_dict"):
        want = expected_fingerprint(name)
        got = fingerprint_of(routine.to_dict())
        if want is not None and got != want:
            raise KernelNotImplemented(
                f"kernel {name!r}: body differs from the implemented one (fingerprint {got[:12]} "
                f"!= {want[:12]}); only the registered kernels run on the GPU")
    warp_mode = bool(getattr(routine, "warp_mode", False))
    warp_size = int(getattr(routine, "warp_size", 32)) if warp_mode else 0
    return name, warp_mode, warp_size
