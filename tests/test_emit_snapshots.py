"""Emitter snapshots: generate() is deterministic and pinned (regenerate with
oracle/make_emit_snapshots.py after an intended change), and every snapshot
cross-compiles for sm_100a (covered by tests/test_codegen.py for the kinds)."""
import os
import sys

import pytest

from conftest import GOLDEN, ROOT

sys.path.insert(0, os.path.join(ROOT, "oracle"))
from make_emit_snapshots import CASES  # noqa: E402


@pytest.mark.parametrize("name", sorted(CASES))
def test_emitter_snapshot(fi, name):
    src = CASES[name]()
    got = fi.generate(src)
    assert got == fi.generate(src)  # deterministic
    with open(os.path.join(GOLDEN, "emit", f"{name}.cu")) as f:
        assert got == f.read()
