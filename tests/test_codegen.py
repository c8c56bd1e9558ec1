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


def test_paper_wmma_strategy_compiles(fi, tmp_path):
    """the f32 epilog staging buffer reuses A's f16 shared
    storage (reuseBuffer) and is emitted as its own f32 view of it."""
    src = fi.generate(fi.strategies.wmma_decomp(1024, 1024, 1024))
    assert "float* const SRC_sh" in src
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


def _nvrtc_compile(src: str):
    """Compile as the runtime does (runtime/plan.cpp compile_cubin: NVRTC,
    sm_100a, --fmad=false); returns (ok, log). NVRTC needs no GPU."""
    import ctypes as C
    lib = None
    for name in ("libnvrtc.so.12", "/usr/local/cuda/lib64/libnvrtc.so.12"):
        try:
            lib = C.CDLL(name)
            break
        except OSError:
            pass
    if lib is None:
        pytest.skip("libnvrtc absent")
    prog = C.c_void_p()
    assert lib.nvrtcCreateProgram(C.byref(prog), src.encode(), b"k.cu", 0, None, None) == 0
    opts = [b"--gpu-architecture=sm_100a", b"--fmad=false", b"-std=c++17", b"-default-device", b"-lineinfo",
            b"--include-path=/usr/local/cuda/include"]
    rc = lib.nvrtcCompileProgram(prog, len(opts), (C.c_char_p * len(opts))(*opts))
    n = C.c_size_t()
    lib.nvrtcGetProgramLogSize(prog, C.byref(n))
    log = C.create_string_buffer(n.value)
    lib.nvrtcGetProgramLog(prog, log)
    lib.nvrtcDestroyProgram(C.byref(prog))
    return rc == 0, log.value.decode(errors="replace")


@pytest.mark.parametrize("key", ["listings/listing2", "listings/wmma_simple", "listings/move_identity",
                                 "corpus/seed03", "paper_wmma", "listing2_f16"])
def test_generic_sources_compile_with_nvrtc(fi, key):
    if key == "paper_wmma":
        script = fi.strategies.wmma_decomp(256, 256, 256)
    elif key == "listing2_f16":
        lines = golden_script("listings/listing2").splitlines()
        lines[0] += " elems f16 f16 f16"
        script = "\n".join(lines) + "\n"
    else:
        script = golden_script(key)
    ok, log = _nvrtc_compile(fi.generate(script))
    assert ok, log


def test_wait_profile_diagnostic_build_compiles(tmp_path):
    """The diagnostic build (-DFI_TC_WAITPROF=1) of one kernel
    instantiation still compiles for sm_100a and keeps the three producer warps'
    TMA issue and the single-asm K block (UTMALDG, UTCHMMA in the SASS)."""
    root = os.path.join(os.path.dirname(__file__), "..", "paper_2003_06324_b200", "csrc")
    src = tmp_path / "waitprof.cu"
    src.write_text('#include "sm100/gemm_kernel.cuh"\n'
                   "template __global__ void fireiron::sm100::fi_sm100_gemm<1, 64, 1, 1, 1>(\n"
                   "    const __grid_constant__ CUtensorMap, const __grid_constant__ CUtensorMap,\n"
                   "    const __grid_constant__ CUtensorMap, const __grid_constant__ CUtensorMap,\n"
                   "    const __grid_constant__ CUtensorMap, const __grid_constant__ fireiron::sm100::GemmArgs);\n")
    cubin = tmp_path / "waitprof.cubin"
    r = subprocess.run([NVCC, "-cubin", "-gencode", "arch=compute_100a,code=sm_100a", "-std=c++17", "-O2",
                        "-DFI_TC_WAITPROF=1", "-I", root, "-I", os.path.join(root, "..", "..", "include"),
                        "-o", str(cubin), str(src)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-2000:]
    sass = subprocess.run(["cuobjdump", "-sass", str(cubin)], capture_output=True, text=True).stdout
    assert "UTMALDG" in sass and "UTCHMMA" in sass and "CS2R" in sass  # clock reads of the wait profile
