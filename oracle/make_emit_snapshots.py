#!/usr/bin/env python3
"""Regenerates tests/golden/emit/*.cu, the snapshots of the sm_100a emitter
(generate()). Run after an intended emitter change; the test
tests/test_emit_snapshots.py pins them (the reference pins its own emitted
text the same way, proj/tests/test_codegen.cpp:222-233)."""
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2003_06324_b200 as fi  # noqa: E402

G = ROOT / "tests" / "golden"
CASES = {
    "listing2": lambda: (G / "listings/listing2.fi").read_text(),
    "wmma_simple": lambda: (G / "listings/wmma_simple.fi").read_text(),
    "move_identity": lambda: (G / "listings/move_identity.fi").read_text(),
    "corpus_seed03": lambda: (G / "corpus/seed03.fi").read_text(),
    "reuse_buffer": lambda: (ROOT / "tests/fixtures/reuse_buffer.fi").read_text(),
    "paper_wmma": lambda: fi.strategies.wmma_decomp(256, 256, 256),
    "c2_tcgen05": fi.strategies.c2_strategy,
    "c3_splitk": fi.strategies.c3_strategy,
    "pair512_slabs": lambda: fi.strategies.tc_strategy(8192, 8192, 8192, tile_m=512),
    "pair_nhalves": lambda: fi.strategies.tc_strategy(8192, 8192, 8192, tile_n=512),
}

if __name__ == "__main__":
    for name, src in CASES.items():
        (G / "emit" / f"{name}.cu").write_text(fi.generate(src()))
    print("wrote", len(CASES), "snapshots")
