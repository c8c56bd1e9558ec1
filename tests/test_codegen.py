"""sm_100a code generation: emitted kernels cross-compile for sm_100a (no GPU
needed), the FMA leaf is unfused (FMUL+FADD, no FFMA) so it is bit-exact with
the reference, and the tensor-core family really issues tcgen05/TMA."""
import os
import re
import shutil
import subprocess

import pytest

from conftest import ROOT, golden_script

NVCC = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
pytestmark = pytest.mark.skipif(not os.path.exists(NVCC), reason="nvcc absent")


def compile_sass(src: str, tmp_path, extra=()):
    cu = tmp_path / "k.cu"
    cu.write_text(src)
    cubin = tmp_path / "k.cubin"
    subprocess.run([NVCC, "-cubin", "-gencode", "arch=compute_100a,code=sm_100a", "--fmad=false", "-std=c++17",
                    *extra, "-o", str(cubin), str(cu)], check=True, capture_output=True, text=True)
    return subprocess.run(["cuobjdump", "-sass", str(cubin)], capture_output=True, text=True).stdout


def test_listing2_emits_unfused_fma(fi, tmp_path):
    src = fi.generate(golden_script("listings/listing2"))
    assert "fi_fma_unfused" in src and "__syncthreads();" in src
    sass = compile_sass(src, tmp_path)
    assert len(re.findall(r"\bFMUL\b", sass)) >= 64
    assert len(re.findall(r"\bFADD\b", sass)) >= 64
    assert not re.findall(r"\bFFMA\b", sass)


def test_wmma_listing_compiles_for_sm100a(fi, tmp_path):
    src = fi.generate(golden_script("listings/wmma_simple"))
    assert src.count("wmma::load_matrix_sync(") == 2 and "wmma::mma_sync(" in src
    sass = compile_sass(src, tmp_path)
    assert "HMMA" in sass


@pytest.mark.parametrize("key", ["corpus/seed03", "corpus/seed17", "corpus/seed42", "listings/move_identity"])
def test_corpus_kernels_compile(fi, key, tmp_path):
    compile_sass(fi.generate(golden_script(key)), tmp_path)


def test_listing1_micro_kernel_over_sm100_budget(fi):
    """Listing 1 stages 128x512 fp32 tiles: 512 KiB > 227 KiB (CapacityExceeded)."""
    with pytest.raises(fi.FiError) as e:
        fi.generate(golden_script("listings/listing1"))
    assert e.value.kind == "CapacityExceeded"


def test_tc_generated_source_compiles(fi, tmp_path):
    src = fi.generate(fi.strategies.c2_strategy())
    sass = compile_sass(src, tmp_path, extra=("-I", os.path.join(ROOT, "paper_2003_06324_b200", "csrc")))
    assert "UTCHMMA" in sass and "UTMALDG" in sass


def test_native_library_contains_tcgen05_family(fi):
    sass = subprocess.run(["cuobjdump", "-sass", fi.LIB_PATH], capture_output=True, text=True).stdout
    for mnemonic in ("UTCHMMA.2CTA", "UTCHMMA", "UTMALDG.2D", "LDTM", "UTCBAR"):
        assert mnemonic in sass, mnemonic
