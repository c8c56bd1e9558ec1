"""GPU parity of the tail schedules with every C element type and layout: the
2-slice pull fixup (run first), the symmetric K-slice fixup with remainder
slices, and N-split tails, with f16 / bf16 / f32 C in column- and row-major
storage (row-major C takes the per-thread store path instead of TMA stores).
Integer inputs; the fixups sum fp32 partials and round once, so C must equal
the fp64 oracle rounded to C's element type, exactly. K is kept small enough
for f16 C that no sum leaves the f16 range."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROW_C = ("colmajor", "colmajor", "rowmajor")
COL = ("colmajor", "colmajor", "colmajor")
CASES = [
    # m, n, k, strategy kwargs, FI_STREAMK, expected (plan.info.streamk, plan.info.remainder)
    (4096, 4096, 4096, dict(c="f16"), None, (1, 2)),              # 2-slice pull fixup, run first
    (4096, 4096, 4096, dict(c="bf16", layouts=ROW_C), None, (1, 2)),
    (1024, 1024, 8192, dict(c="bf16", split_k=4), None, (1, 0)),  # symmetric fixup, 4 even slices
    (1024, 1024, 4096, dict(c="f16", split_k=4, layouts=ROW_C), None, (1, 0)),
    (2560, 2560, 8192, dict(c="bf16"), None, (1, 1)),             # symmetric + remainder slices
    (2048, 2560, 2048, dict(c="f32", layouts=ROW_C), "1", (1, 0)),
    (4096, 4096, 1024, dict(c="bf16"), None, (2, 0)),             # N-split tail
]


@pytest.mark.parametrize("m,n,k,kw,streamk,expect", CASES)
def test_tail_schedule_all_output_types(fi, oracle, monkeypatch, m, n, k, kw, streamk, expect):
    monkeypatch.setenv("FI_HOST_PIPELINE", "0")  # one whole-matrix launch: the schedule under test
    if streamk is not None:
        monkeypatch.setenv("FI_STREAMK", streamk)
    plan = fi.Plan(fi.strategies.tc_strategy(m, n, k, pair=True, tile_n=256, **kw))
    mode, rem = expect
    assert plan.info.streamk == mode, (plan.info.streamk, plan.info.remainder)
    assert plan.info.remainder == rem
    a = oracle.fill(m, k, 21, True)
    b = oracle.fill(k, n, 22, True)
    c = plan.run_host(a, b)
    rng = np.random.default_rng(3)
    rows, cols = rng.integers(0, m, 4096), rng.integers(0, n, 4096)
    want = oracle.sample_f64(oracle.round_elem(a, "f16"), oracle.round_elem(b, "f16"), rows, cols).astype(np.float32)
    if kw["c"] != "f32":
        want = oracle.round_elem(want, kw["c"])
    assert np.array_equal(c[rows, cols], want)
