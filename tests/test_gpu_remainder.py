"""GPU parity of the K-slice tail with a remainder slice (sm100/gemm.cu
launch planner): main slices of W K-blocks on R*S clusters plus the remainder
kb - S*W of each leftover tile on the E idle clusters (q per cluster). Integer
inputs must equal the fp64 oracle exactly; uniform inputs must be
deterministic run to run and equal the plain even-slice schedule
(FI_REMAINDER=0) to fp32 reassociation (tolerance 1e-5 normwise, the summation
order of the partials differs)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

CASES = [
    # m, n, k, strategy kwargs, expected remainder
    (1024, 1024, 32768, dict(pair=True, tile_n=256, split_k=4), True),  # C3: S=4, E=10, q=2, W=114
    (512, 512, 16384, dict(pair=True, tile_n=256, split_k=4), True),    # q=1
    (2560, 2560, 10240, dict(pair=True, tile_n=256), True),             # 1 data-parallel wave + tail S=2, q=2
    (512, 512, 4096, dict(pair=True, tile_n=256, split_k=4), False),    # remainder too short: even slices
    (768, 1024, 9600, dict(pair=True, tile_n=256), False),              # 12 tiles -> 6 even K slices (peer staging fills the ring)
]


def _plan(fi, script, remainder, monkeypatch):
    monkeypatch.setenv("FI_REMAINDER", "1" if remainder else "0")  # read at plan creation
    return fi.Plan(script)


@pytest.mark.parametrize("m,n,k,kw,expect", CASES,
                         ids=lambda x: "_".join(f"{a}{b}" for a, b in x.items()) if isinstance(x, dict) else str(x))
def test_remainder_tail_exact_and_deterministic(fi, oracle, monkeypatch, m, n, k, kw, expect):
    monkeypatch.setenv("FI_HOST_PIPELINE", "0")  # one whole-matrix launch: the schedule under test
    script = fi.strategies.tc_strategy(m, n, k, **kw)
    plan = _plan(fi, script, True, monkeypatch)
    assert plan.kind == "tcgen05"
    assert (plan.info.remainder == 1) == expect
    even = _plan(fi, script, False, monkeypatch)
    assert even.info.remainder != 1
    # integer inputs: exact at 4096 sampled fp64 dot products, and bitwise equal
    # to the even-slice schedule over the whole matrix (both are exact)
    a = oracle.fill(m, k, 11, True)
    b = oracle.fill(k, n, 12, True)
    c = plan.run_host(a, b)
    rng = np.random.default_rng(1)
    rows, cols = rng.integers(0, m, 4096), rng.integers(0, n, 4096)
    want = oracle.sample_f64(oracle.round_elem(a, "f16"), oracle.round_elem(b, "f16"), rows, cols)
    assert np.array_equal(c[rows, cols].astype(np.float64), want)
    assert np.array_equal(c, even.run_host(a, b))

    a = oracle.fill(m, k, 13, False)
    b = oracle.fill(k, n, 14, False)
    c1, c2 = plan.run_host(a, b), plan.run_host(a, b)
    assert np.array_equal(c1.view(np.uint32), c2.view(np.uint32))
    c0 = even.run_host(a, b)
    assert np.max(np.abs(c1 - c0)) <= 1e-5 * np.max(np.abs(c0))
