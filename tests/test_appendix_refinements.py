"""The paper's pipelining refinements (Figure "HMMA
In-CTA-split-k"), first-class in the script language: `split .. .prefetchLoads`,
`split .. .doubleBufferLoop`, `load .. .doubleBuffer` and `load .. .postponed`.
They schedule, they do not change results: on the tcgen05 path they set the
TMA ring depth (deepest / 2 stages; a postponed load is what the
warp-specialised producer always does), on the generic path
`.doubleBufferLoop` is `.stages 2` and the others leave the program as is.
The reference parser rejects them, so there is no reference
output to match: the checks are round trips, lowering equivalences and
conflicts."""
import pytest

import paper_2003_06324_b200 as fi
from paper_2003_06324_b200 import strategies

PAIR = strategies.tc_strategy(4096, 4096, 4096, pair=True, tile_n=256)


def _with(script, old, new):
    assert old in script
    return script.replace(old, new, 1)


def test_round_trip_prints_the_paper_spelling():
    s = _with(PAIR, "split 64\n", "split 64 .prefetchLoads\n")
    s = _with(s, "load a sh {", "load a sh .postponed {")
    s = _with(s, "load b sh {", "load b sh .postponed {")
    out = fi.print_script(s)
    assert "split 64 .prefetchLoads" in out and out.count(".postponed") == 2
    assert fi.print_script(out) == out
    d = _with(PAIR, "split 64\n", "split 64 .doubleBufferLoop\n")
    assert "split 64 .doubleBufferLoop" in fi.print_script(d)


@pytest.mark.parametrize("edit,stages", [
    (("split 64\n", "split 64 .doubleBufferLoop\n"), 2),
    (("load a sh {", "load a sh .doubleBuffer {"), 2),
    (("split 64\n", "split 64 .prefetchLoads\n"), None),  # the deepest ring, as without refinements
    (("load b sh {", "load b sh .postponed {"), None),
])
def test_tcgen05_ring_depth(edit, stages):
    base = fi.check_async(PAIR).stages
    r = fi.check_async(_with(PAIR, *edit))
    assert r.ok
    assert r.stages == (stages if stages is not None else base)
    assert fi.check_async(_with(PAIR, "split 64\n", "split 64 .stages 2\n")).stages == 2


def test_double_buffer_loop_equals_two_stages_in_generated_code():
    a = fi.generate(_with(PAIR, "split 64\n", "split 64 .doubleBufferLoop\n"))
    b = fi.generate(_with(PAIR, "split 64\n", "split 64 .stages 2\n"))
    assert a == b


def test_generic_program_unchanged_by_postponed_and_prefetch():
    s = strategies.listing2(128, 128, 32)
    t = _with(s, "split 8 .sync", "split 8 .sync .prefetchLoads")
    t = _with(t, "load b sh {", "load b sh .postponed {")
    t = t.replace("load a rf {", "load a rf .doubleBuffer {", 1)
    assert fi.generate(t) == fi.generate(s)
    assert fi.elaborate(t) == fi.elaborate(s)


@pytest.mark.parametrize("edit", [
    ("split 64\n", "split 64 .doubleBufferLoop .stages 3\n"),
    ("split 64\n", "split 64 .prefetchLoads .stages 4\n"),
    ("split 64\n", "split 64 .prefetchLoads .doubleBufferLoop\n"),
])
def test_conflicting_pipeline_refinements_are_rejected(edit):
    with pytest.raises(fi.FiError):
        fi.validate(_with(PAIR, *edit))


def test_double_buffered_load_conflicts_with_deeper_stages():
    s = _with(PAIR, "split 64\n", "split 64 .stages 4\n")
    s = _with(s, "load a sh {", "load a sh .doubleBuffer {")
    with pytest.raises(fi.FiError):
        fi.check_async(s)
