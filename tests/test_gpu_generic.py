"""GPU parity of the generic sm_100a path (emitted CUDA, NVRTC, --fmad=false)
against the reference simulator's golden digests: FMA-leaf strategies are
bit-exact (listing2 incl. 512^3, all 50 corpus trees, integer and uniform
inputs); WMMA within the reference's 2^-8 (test_sim.cpp:248-263); Move is a
bitwise copy. Everything goes through the C ABI (fi_plan_create/run_host)."""
import re

import numpy as np
import pytest

from conftest import golden_digests, golden_script

pytestmark = pytest.mark.gpu


def dims(script, case):
    m = re.match(r"spec (MatMul|Move)\((\d+)[,x](\d+)(?:,(\d+))?\)", script)
    kind, a, b, c = m.groups()
    if kind == "Move":
        return "move", (case["m"] or int(a), case["n"] or int(b), 0)
    return "mm", (case["m"] or int(a), case["n"] or int(b), case["k"] or int(c))


FMA_CASES = [c for c in golden_digests() if c["script"].startswith(("listings/listing2", "corpus/"))]


@pytest.mark.parametrize("case", FMA_CASES,
                         ids=lambda c: f"{c['script']}-{c['m']}x{c['n']}x{c['k']}-s{c['seed']}-f{c['float']}")
def test_fma_strategies_bit_exact(fi, oracle, case):
    s = golden_script(case["script"])
    _, (m, n, k) = dims(s, case)
    plan = fi.Plan(s, case["m"], case["n"], case["k"])
    assert plan.kind == "generic"
    a = oracle.fill(m, k, case["seed"], not case["float"])
    b = oracle.fill(k, n, case["seed"] + 1, not case["float"])
    c = plan.run_host(a, b)
    assert oracle.digest(c) == case["digest"]


def test_listing2_large_uniform_bit_exact_vs_seqk(fi, oracle):
    s = golden_script("listings/listing2")
    plan = fi.Plan(s, 1024, 1024, 512)
    a = oracle.fill(1024, 512, 21, False)
    b = oracle.fill(512, 1024, 22, False)
    c = plan.run_host(a, b)
    want = oracle.seqk_f32(a, b)
    assert np.array_equal(c.view(np.uint32), want.view(np.uint32))


def test_wmma_within_reference_tolerance(fi, oracle):
    s = golden_script("listings/wmma_simple")
    plan = fi.Plan(s)
    for seed in (31, 41):
        a = oracle.fill(64, 16, seed, False)
        b = oracle.fill(16, 64, seed + 1, False)
        c = plan.run_host(a, b)
        want = oracle.gemm_f64(oracle.round_elem(a, "f16"), oracle.round_elem(b, "f16"))
        assert oracle.max_abs_error(c, want) <= 1.0 / 256.0
    # integer inputs are exact on every strategy
    a = oracle.fill(64, 16, 1, True)
    b = oracle.fill(16, 64, 2, True)
    assert oracle.digest(plan.run_host(a, b)) == "0x5b5f96ef67c52a00"


def test_move_copies_bitwise(fi, oracle):
    plan = fi.Plan(golden_script("listings/move_identity"))
    src = oracle.fill(8, 8, 11, False)
    out = plan.run_host(src)
    assert np.array_equal(out.view(np.uint32), src.view(np.uint32))


def test_launch_on_device_buffers_matches_run_host(fi, oracle):
    import torch
    s = golden_script("corpus/seed05")
    plan = fi.Plan(s)
    (m, k, ar), (_, n, br), (_, _, cr) = plan.shapes()
    a = oracle.fill(m, k, 5, False)
    b = oracle.fill(k, n, 6, False)
    host = plan.run_host(a, b)
    da = torch.from_numpy(a if ar else a.T.copy()).cuda().contiguous()
    db = torch.from_numpy(b if br else b.T.copy()).cuda().contiguous()
    dc = torch.full((m, n) if cr else (n, m), float("nan"), device="cuda")
    plan.launch(da.data_ptr(), db.data_ptr(), dc.data_ptr(), torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    got = dc.cpu().numpy()
    got = got if cr else got.T
    assert np.array_equal(got.view(np.uint32), host.view(np.uint32))


def test_hmma_leaf_is_rejected_on_sm100(fi):
    with pytest.raises(fi.FiError) as e:
        fi.Plan(golden_script("listings/hmma_ptx"))
    assert e.value.kind == "Unsupported"
