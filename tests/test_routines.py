"""The routine table (paper_2206_07896_b200/routines.py) agrees with the
reference's own compiler: for every kernel, transform() of its .kn source
(/root/reference/pkg/src/blockfuse/transform.py:110-160) gives the same
parameter signature, has_atomics(), static_instruction_estimate() and warp
mode (the inputs of resolve_grain, runtime.py:83-101), and the fingerprint
the C ABI checks is the one of that MpmdKernel."""

import json
from pathlib import Path

from paper_2206_07896_b200 import routines

ROOT = Path(__file__).resolve().parents[1]


def _sig(mk):
    out = []
    for p in mk.param_signature:
        t = p.ptype
        out.append((p.name, f"global {t.scalar}[]" if t.is_global else t.scalar))
    return tuple(out)


def _compiled(name):
    from blockfuse.bench import CORPUS
    from blockfuse.parser import parse_unit
    from blockfuse.transform import transform
    if name in CORPUS:
        return CORPUS[name].compiled()
    r = routines.get(name)
    return transform(parse_unit(routines.kernel_source(name))[name], warp_mode=r.warp_mode)


def test_table_matches_reference_transform(reference):
    for name in routines.names():
        r = routines.get(name)
        mk = _compiled(name)
        assert tuple(r.params) == _sig(mk), name
        assert r.has_atomics() == mk.has_atomics(), name
        assert r.static_instruction_estimate() == mk.static_instruction_estimate(), name
        assert r.warp_mode == mk.warp_mode, name


def test_registered_fingerprints_are_the_reference_kernels(reference):
    fps = json.loads((ROOT / "paper_2206_07896_b200" / "fingerprints.json").read_text())
    for name, fp in fps.items():
        assert routines.fingerprint_of(_compiled(name).to_dict()) == fp, name
