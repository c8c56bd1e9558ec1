"""GPU parity of the pipelined host paths of Plan.run_host on tcgen05 plans:
the blocked pipeline (A row panels and B column panels uploaded alternately,
one GEMM per landed panel over the C blocks it completes, pitched 2D copies for
any layout) and the column-panel pipeline (column-major B and C). The output
is computed while A/B are still crossing PCIe and earlier blocks are coming
back. The result must equal
the unpipelined path (FI_HOST_PIPELINE=0: whole H2D, one launch, whole D2H)
up to fp32 reassociation -- a panel launch may choose a
different tail schedule (K-sliced vs whole-K tiles) than the whole-matrix
launch -- and, on integer inputs, exactly the fp64 oracle."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

CASES = [
    # m, n, k, strategy kwargs
    (1024, 2048, 1024, dict(pair=True, tile_n=256)),
    (512, 4096, 1024, dict(pair=True, tile_n=256, c="f16")),     # f16 C widened per block
    (1024, 2048, 2048, dict(pair=True, tile_n=128, ab="bf16")),
    (512, 2048, 2048, dict(pair=False, tile_n=128)),             # 1-CTA MMA
    (1024, 1024, 32768, dict(pair=True, tile_n=256, split_k=4)), # C3: K slices per block
    (1024, 2048, 1024, dict(pair=True, tile_n=256, layouts=("rowmajor", "colmajor", "colmajor"))),
    (1024, 2048, 1024, dict(pair=True, tile_n=256, layouts=("colmajor", "rowmajor", "rowmajor"))),
    (2048, 2048, 1024, dict(pair=True, tile_n=256, tile_m=512, c="bf16")),  # slab tiles
    (1024, 2048, 1024, dict(pair=True, tile_n=128, multicast=True)),
]
MODES = ["blocked", "panels"]


def _unpipelined(plan, a, b):
    old = os.environ.get("FI_HOST_PIPELINE")
    os.environ["FI_HOST_PIPELINE"] = "0"
    try:
        return plan.run_host(a, b)
    finally:
        if old is None:
            del os.environ["FI_HOST_PIPELINE"]
        else:
            os.environ["FI_HOST_PIPELINE"] = old


@pytest.fixture
def pipeline_mode(request, monkeypatch):
    if request.param == "blocked":  # 1 MiB panels, short lines: the small cases split
        monkeypatch.setenv("FI_HOST_PANEL_MB", "1")
        monkeypatch.setenv("FI_HOST_MIN_LINE", "128")
        monkeypatch.setenv("FI_HOST_PIPELINE_TRACE", "1")
        monkeypatch.delenv("FI_HOST_PIPELINE", raising=False)
    else:
        monkeypatch.setenv("FI_HOST_PIPELINE", "panels")
    return request.param


@pytest.mark.parametrize("pipeline_mode", MODES, indirect=True)
@pytest.mark.parametrize("m,n,k,kw", CASES, ids=lambda x: str(x) if not isinstance(x, dict) else
                         "_".join(f"{a}{b}" for a, b in x.items()))
def test_pipelined_run_host_matches_plain_and_oracle(fi, oracle, m, n, k, kw, pipeline_mode, capfd):
    plan = fi.Plan(fi.strategies.tc_strategy(m, n, k, **kw))
    assert plan.kind == "tcgen05"
    ab = kw.get("ab", "f16")
    # integer mode: exact against fp64 (f16 C holds every value |x| <= 2048 here
    # only for small k; compare the f16-output case against the rounded oracle)
    a = oracle.fill(m, k, 3, True)
    b = oracle.fill(k, n, 4, True)
    c = plan.run_host(a, b)
    if pipeline_mode == "blocked":
        assert "blocked" in capfd.readouterr().err  # the blocked pipeline ran
    want = oracle.gemm_f64(oracle.round_elem(a, ab), oracle.round_elem(b, ab))
    if kw.get("c", "f32") == "f32":
        assert np.array_equal(c, want)
    else:
        assert np.array_equal(c, oracle.round_elem(want, kw["c"]))
    # uniform mode: the pipelined path and the whole-matrix path agree to fp32
    # reassociation (tolerance 1e-5 normwise; f16/bf16 C: one unit of rounding),
    # and each path is deterministic
    a = oracle.fill(m, k, 5, False)
    b = oracle.fill(k, n, 6, False)
    c1 = plan.run_host(a, b)
    c0 = _unpipelined(plan, a, b)
    tol = 1e-5 if kw.get("c", "f32") == "f32" else 1e-2
    assert np.max(np.abs(c1 - c0)) <= tol * np.max(np.abs(c0))
    assert np.array_equal(plan.run_host(a, b).view(np.uint32), c1.view(np.uint32))
