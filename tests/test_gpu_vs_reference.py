"""GPU results against the compiled reference simulator (oracle/_ref, the
unmodified anvil headers) on identical inputs: FMA/HFMA/COPY strategies must
be bit-identical, including f16 variants (HFMA leaf, round_to_f16 on every
store) and row-major / padded layouts of the reference's random corpus.
Also: a user micro-kernel (verbatim CUDA, NVRTC) against the oracle."""
import os
import re

import numpy as np
import pytest

from conftest import golden_script

pytestmark = pytest.mark.gpu

REF = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref", "libanvil_ref.so")
needs_ref = pytest.mark.skipif(not os.path.exists(REF), reason="oracle/_ref not built")


def with_header(script, extra):
    lines = script.splitlines()
    lines[0] = lines[0] + " " + extra
    return "\n".join(lines) + "\n"


def dims(script):
    m, n, k = re.match(r"spec MatMul\((\d+),(\d+),(\d+)\)", script).groups()
    return int(m), int(n), int(k)


VARIANTS = {
    "f32": "",
    "f16": "elems f16 f16 f16",
    "rowmajor": "layouts rowmajor rowmajor rowmajor",
    "mixed_layouts": "layouts rowmajor colmajor rowmajor",
    "f16_rowmajor": "elems f16 f16 f16 layouts rowmajor rowmajor colmajor",
}


@needs_ref
@pytest.mark.parametrize("variant", sorted(VARIANTS))
@pytest.mark.parametrize("seed", [2, 9, 17, 33, 48])
def test_corpus_variant_bit_identical_to_reference(fi, oracle, variant, seed):
    s = with_header(golden_script(f"corpus/seed{seed:02d}"), VARIANTS[variant]).replace("  \n", "\n")
    s = fi.print_script(s)  # canonical
    m, n, k = dims(s)
    a = oracle.fill(m, k, 100 + seed, False)
    b = oracle.fill(k, n, 200 + seed, False)
    want, races = oracle.ref_run(s, a, b)
    assert races == 0
    got = fi.Plan(s).run_host(a, b)
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32)), variant


@needs_ref
@pytest.mark.parametrize("pad", [4, 8])
def test_padded_shared_tiles_bit_identical(fi, oracle, pad):
    s = golden_script("listings/listing2").replace("load a sh {", f"load a sh .pad {pad} {{")
    s = fi.print_script(s)
    a = oracle.fill(128, 32, 3, False)
    b = oracle.fill(32, 128, 4, False)
    want, _ = oracle.ref_run(s, a, b)
    got = fi.Plan(s).run_host(a, b)
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))


@needs_ref
def test_reuse_buffer_strategy_bit_identical(fi, oracle):
    path = os.path.join(os.path.dirname(__file__), "fixtures", "reuse_buffer.fi")
    s = open(path).read()
    a = oracle.fill(64, 32, 5, False)
    b = oracle.fill(32, 64, 6, False)
    want, races = oracle.ref_run(s, a, b)
    assert races == 0
    got = fi.Plan(s).run_host(a, b)
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))


MICRO = """spec MatMul(256,256,64)(GL,GL,GL)(Kernel)

microkernel dot.cu
pattern MatMul(1,1,K)(RF,RF,GL)(Thread)
vars K A.base A.off A.cs B.base B.off B.rs C
---
float acc = 0.0f;
for (int kk = 0; kk < {K}; ++kk) {
  acc = __fadd_rn(acc, __fmul_rn({A.base}[{A.off} + (kk * {A.cs})], {B.base}[{B.off} + (kk * {B.rs})]));
}
{C} = acc;
---

tile 128 128 .to block
load a sh {
  tile 16 64 .to warp
  tile 4 8 .to thread
  tile 1 1
  done
}
load b sh {
  tile 64 16 .to warp
  tile 8 4 .to thread
  tile 1 1
  done
}
tile 64 32 .to warp
tile 8 8 .to thread
load a rf {
  tile 1 1
  done
}
load b rf {
  tile 1 1
  done
}
tile 1 1
done dot.cu
"""


def test_micro_kernel_strategy_runs_verbatim(fi, oracle):
    """Listing 1's shape (micro-kernel leaf; the reference cannot simulate it,
    sim.hpp:436-437) on a size whose SH tiles fit: the per-thread dot product
    is sequential-k unfused fp32, i.e. seqk_f32."""
    plan = fi.Plan(MICRO)
    assert "dot.cu" not in plan.source() or "acc" in plan.source()
    a = oracle.fill(256, 64, 7, False)
    b = oracle.fill(64, 256, 8, False)
    got = plan.run_host(a, b)
    assert np.array_equal(got.view(np.uint32), oracle.seqk_f32(a, b).view(np.uint32))


@needs_ref
@pytest.mark.parametrize("integers", [True, False], ids=["int", "uniform"])
def test_paper_wmma_strategy_matches_reference(fi, oracle, integers):
    """The paper's staged WMMA strategy: its epilog stages
    the f32 accumulators through an SH buffer that reuses A's f16 storage
    (reuseBuffer); the alias is its own f32 view of that storage, as in the
    simulator (sim.hpp:314-339). Integer inputs: exact; uniform inputs: within
    the reference's WMMA bound 2^-8 (test_acceptance.cpp:132-154)."""
    m = n = k = 256
    s = fi.strategies.wmma_decomp(m, n, k)
    a = oracle.fill(m, k, 41, integers)
    b = oracle.fill(k, n, 42, integers)
    want, races = oracle.ref_run(s, a, b)
    assert races == 0
    got = fi.Plan(s).run_host(a, b)
    if integers:
        assert np.array_equal(got, want)
    else:
        assert oracle.max_abs_error(got, want) <= 2.0 ** -8


def test_paper_wmma_strategy_1024_vs_f64(fi, oracle):
    m = n = k = 1024
    plan = fi.Plan(fi.strategies.wmma_decomp(m, n, k))
    assert plan.kind == "generic"
    a = oracle.fill(m, k, 3, True)
    b = oracle.fill(k, n, 4, True)
    assert np.array_equal(plan.run_host(a, b), oracle.gemm_f64(a, b))
