"""Edge cases of the tensor-core lowering, on the CPU (match_tc_strategy via
the protocol checker, which lowers exactly as Plan::create does): shapes that
are not multiples of the block tile, K blocks other than 64, tile shapes the
tcgen05 kernel family has no instance for, and refinement combinations it
cannot honour must be rejected with a reason -- never silently run on some
other path (the backend has no CPU fallback)."""
import pytest

import paper_2003_06324_b200 as fi
from paper_2003_06324_b200 import strategies


def _rejects(script, *fragments):
    with pytest.raises(fi.FiError) as e:
        fi.check_async(script)
    msg = str(e.value)
    assert any(f in msg for f in fragments), msg


@pytest.mark.parametrize("m,n,k,kw,frag", [
    (1000, 1024, 1024, dict(pair=True), ("multiple", "divid")),             # ragged M
    (1024, 1000, 1024, dict(pair=True), ("multiple", "divid")),             # ragged N
    (1024, 1024, 1000, dict(pair=True), ("multiple", "divid")),             # ragged K
    (1024, 1024, 1024, dict(pair=False, tile_n=96), ("N must be",)),        # no UMMA instance
    (1024, 1024, 1024, dict(pair=False, tile_n=512), ("N must be",)),       # N halves need a pair
    (1024, 1024, 1024, dict(pair=True, tile_n=128, tile_m=512), ("M 512 needs N 256",)),  # slabs need N 256
    (1024, 1024, 4096, dict(pair=True, tile_n=256, tile_m=512, split_k=2), ("no split-K",)),
    (1024, 1024, 1024, dict(pair=False, multicast=True), ("multicast", "pair")),
])
def test_unsupported_shapes_and_tiles_are_rejected(m, n, k, kw, frag):
    _rejects(strategies.tc_strategy(m, n, k, **kw), *frag)


def test_k_block_must_be_one_swizzle_span():
    s = strategies.tc_strategy(1024, 1024, 1024).replace("split 64\n", "split 32\n")
    _rejects(s, "K block must be 64")


def test_padded_operand_staging_is_rejected():
    s = strategies.tc_strategy(1024, 1024, 1024).replace("load a sh {", "load a sh .pad 8 {")
    _rejects(s, "pad")


def test_fp32_operands_have_no_tensor_core_lowering():
    s = strategies.tc_strategy(1024, 1024, 1024).replace("elems f16 f16 f32", "elems f32 f32 f32")
    with pytest.raises(fi.FiError):
        fi.check_async(s)


@pytest.mark.parametrize("m,n,k", [(256, 256, 64), (128, 64, 64), (512, 512, 64)])
def test_smallest_problems_lower(m, n, k):
    """One K block, one tile: the schedule degenerates cleanly."""
    for kw in (dict(pair=True, tile_n=64), dict(pair=False, tile_n=64)):
        if m % (256 if kw["pair"] else 128):
            continue
        r = fi.check_async(strategies.tc_strategy(m, n, k, **kw))
        assert r.ok and r.tiles >= 1, r.text
