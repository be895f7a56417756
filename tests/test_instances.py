"""The corpus instance generators of oracle/instances.py replay the
reference's (/root/reference/pkg/src/blockfuse/bench.py:78-180) draw for
draw: from the same seed they build the same geometry, buffers, arguments
and outputs, so the parity tests run exactly the reference's acceptance
instances."""

import random
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT / "oracle"))

import instances as I  # noqa: E402


@pytest.mark.parametrize("seed", [0, 1, 20260823, 99991])
def test_corpus_generators_replay_the_reference(reference, seed):
    from blockfuse.bench import CORPUS
    assert set(CORPUS) == set(I.CORPUS)
    for name, case in CORPUS.items():
        want = case.random_instance(random.Random(seed))
        got = I.CORPUS[name](random.Random(seed))
        assert (got.grid.x, got.grid.y, got.grid.z) == (want.grid.x, want.grid.y, want.grid.z), name
        assert (got.block.x, got.block.y, got.block.z) == (want.block.x, want.block.y, want.block.z), name
        assert got.shmem == want.shmem, name
        assert [(b.name, b.scalar, b.length) for b in got.buffers] == \
            [(b.name, b.scalar, b.length) for b in want.buffers], name
        for gb, wb in zip(got.buffers, want.buffers):
            assert list(gb.values) == list(wb.values), (name, gb.name)
        assert [tuple(a) for a in got.args] == [tuple(a) for a in want.args], name
        assert list(got.outputs) == list(want.outputs), name
