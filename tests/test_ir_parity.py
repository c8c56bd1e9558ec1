"""The from-scratch strategy IR (include/fireiron/*.hpp) against the reference's
lowering, elaboration, validation and canonical printing, text-for-text, on
every reference listing and the reference's 50-tree random corpus
(fixtures: tests/golden/ir, made by oracle/make_golden.py)."""
import os

import pytest

from conftest import GOLDEN, golden_keys, golden_script


def _gold(key, ext):
    with open(os.path.join(GOLDEN, "ir", key.replace("/", "__") + f".{ext}.txt")) as f:
        return f.read()


@pytest.mark.parametrize("key", golden_keys())
def test_plan_text_matches_reference(fi, key):
    assert fi.plan_summary(golden_script(key)) == _gold(key, "plan")


@pytest.mark.parametrize("key", golden_keys())
def test_elaboration_matches_reference(fi, key):
    gold = _gold(key, "elab")
    if gold.startswith("ERROR"):
        with pytest.raises(fi.FiError):
            fi.elaborate(golden_script(key), True)
    else:
        assert fi.elaborate(golden_script(key), True) == gold


@pytest.mark.parametrize("key", golden_keys())
def test_print_and_validate_match_reference(fi, key):
    s = golden_script(key)
    assert fi.print_script(s) == _gold(key, "print")
    assert fi.print_script(fi.print_script(s)) == fi.print_script(s)  # fixpoint
    assert fi.validate(s) == _gold(key, "validate")


def test_listing1_trace_golden(fi):
    """Acceptance criterion 1 (proj/tests/test_acceptance.cpp:59-69): 12 entries."""
    t = fi.elaborate(golden_script("listings/listing1"))
    assert len(t.splitlines()) == 12
    assert t.splitlines()[-1].endswith("MatMul(1,1,512)(RF,RF,GL)(Thread)")


BAD = {
    "NonDivisible": "spec MatMul(100,128,32)(GL,GL,GL)(Kernel)\ntile 64 64 .to block\ndone\n",
    "HierarchyViolation": "spec MatMul(64,64,8)(GL,GL,GL)(Kernel)\ntile 32 32 .to warp\ndone\n",
    "UnitCountMismatch": ("spec MatMul(64,64,8)(GL,GL,GL)(Kernel)\ntile 64 64 .to block\ntile 32 32 .to warp\n"
                          "tile 4 4 .to thread\ndone\n"),
    "UpwardLoad": "spec MatMul(64,64,8)(SH,GL,GL)(Kernel)\nload a gl {\n  done\n}\ndone\n",
    "NoExecutableMatch": "spec MatMul(64,64,8)(GL,GL,GL)(Kernel)\ndone\n",
    "CNotInGL": ("spec MatMul(64,64,8)(GL,GL,RF)(Kernel)\nepilog rf {\n  init {\n    done\n  }\n"
                 "  store {\n    done\n  }\n}\ndone\n"),
    "InvalidRefinement": "spec MatMul(64,64,8)(GL,GL,GL)(Kernel)\ntile 8 8 .unroll .pair\ndone\n",
}


@pytest.mark.parametrize("kind", sorted(BAD))
def test_validation_collects_violation_kinds(fi, kind):
    try:
        report = fi.validate(BAD[kind])
    except fi.FiError as e:  # construction-time refinement errors surface as ParseError
        assert kind == "InvalidRefinement" and e.kind == "ParseError"
        return
    assert kind in report, report


def test_parse_errors_carry_line_and_column(fi):
    with pytest.raises(fi.FiError) as e:
        fi.validate("spec MatMul(64,64,8)(GL,GL,GL)(Kernel)\ntile 8 8 .bogus\ndone\n")
    assert e.value.kind == "ParseError" and "line 2" in str(e.value)


def test_swizzle_must_be_bijective(fi):
    s = ("spec MatMul(64,32,8)(RF,RF,RF)(Warp)\ntile 8 8 .to thread .swizzle 7\ntile 1 1\ndone\n")
    assert "SwizzleNotBijective" in fi.validate(s)


def test_reuse_buffer_aliasing(fi):
    """Acceptance criterion 10 (test_acceptance.cpp:303-351): barrier-separated
    reuse shares one max-extent allocation."""
    s = open(os.path.join(GOLDEN, "..", "fixtures", "reuse_buffer.fi")).read()
    plan = fi.plan_summary(s)
    assert "shared_bytes 16384" in plan
    assert any(" alias " in l and not l.endswith("alias -1") for l in plan.splitlines())


def test_tensor_core_strategies_validate(fi):
    for s in (fi.strategies.c2_strategy(), fi.strategies.c3_strategy(), fi.strategies.c5_strategy(),
              fi.strategies.tc_strategy(512, 512, 256, pair=False, tile_n=128, stages=4)):
        assert fi.validate(s).startswith("valid"), s
        assert fi.print_script(s) == s
        assert "tcgen05" in fi.generate(s)


def test_tc_trace_binds_sm100_leaves(fi):
    t = fi.elaborate(fi.strategies.c2_strategy(), True)
    assert "Move(256x64)(GL->SH)(Block)" in t       # TMA_LOAD
    assert "MatMul(256,256,64)(SH,SH,TM)(Block)" in t  # UMMA
    assert "Move(32x256)(TM->GL)(Warp)" in t          # TMEM_STORE


def test_splitk_must_feed_an_epilog(fi):
    s = ("spec MatMul(1024,1024,4096)(GL,GL,GL)(Kernel) elems f16 f16 f32\ntile 128 128 .to block\n"
         "split 1024 .splitk\nsplit 64\nload a sh {\n  done\n}\nload b sh {\n  done\n}\ndone\n")
    assert "InvalidRefinement" in fi.validate(s)
