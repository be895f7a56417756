"""The C-ABI library loads and exports every symbol include/bfgpu.h declares;
host-only entry points (task queue, grain law, registry) work without a GPU."""

import re
from pathlib import Path

import pytest

from paper_2206_07896_b200 import _lib

ROOT = Path(__file__).resolve().parents[1]


def declared_symbols() -> set:
    text = (ROOT / "include" / "bfgpu.h").read_text()
    return set(re.findall(r"^(?:int|const char \*)\s*(bf_\w+)\s*\(", text, re.M))


def test_exports_every_declared_symbol():
    L = _lib.lib()
    syms = declared_symbols()
    assert len(syms) >= 30
    missing = [s for s in syms if not hasattr(L, s)]
    assert not missing, missing
    assert set(_lib.EXPORTS) == syms


def test_abi_version_and_registry():
    L = _lib.lib()
    assert L.bf_abi_version() == 1
    ks = _lib.kernels()
    assert "vecadd" in ks and "hotspot" in ks
    assert ks["vecadd"] == [("handle", "f32"), ("handle", "f32"), ("handle", "f32"), ("i32", None)]


def test_registry_matches_routine_table():
    from paper_2206_07896_b200 import routines
    ks = _lib.kernels()
    for name, sig in ks.items():
        r = routines.get(name)
        assert len(r.params) == len(sig)
        for (pname, ptype), (kind, scalar) in zip(r.params, sig):
            if ptype.startswith("global"):
                assert kind == "handle" and ptype == f"global {scalar}[]", (name, pname)
            else:
                assert kind == ptype, (name, pname)


def test_fingerprints_registered_natively():
    """fingerprints.json reaches the C ABI at load (bf_kernel_set_fingerprint),
    so bf_launch_described rejects a different body under a registered name
    without the Python layer; unknown names are refused."""
    import json
    L = _lib.lib()
    fps = json.loads((ROOT / "paper_2206_07896_b200" / "fingerprints.json").read_text())
    assert {"vecadd", "hotspot", "kmeans", "bfs", "nn"} <= set(fps)
    assert L.bf_kernel_set_fingerprint(b"vecadd", bytes.fromhex(fps["vecadd"])) == _lib.OK
    assert L.bf_kernel_set_fingerprint(b"no_such_kernel", bytes(32)) == _lib.E_UNKNOWN_KERNEL
