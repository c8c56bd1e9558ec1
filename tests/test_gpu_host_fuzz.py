"""Randomised GPU parity of the host side of run_host (fi_plan_run_host): the
blocked and column-panel pipelines with random panel and piece sizes, host
snapping ratios, pinned or pageable input and output buffers, operand layouts
and element types, over random tcgen05 strategies (drawn as in
test_gpu_fuzz). Integer inputs: every case is exact against the fp64 oracle,
and the bytes the runtime reports moving match the pieces it snapped."""
import re

import numpy as np
import pytest

from test_gpu_fuzz import draw

pytestmark = pytest.mark.gpu


def draw_host(rng):
    while True:
        m, n, k, kw = draw(rng)
        bm = kw.get("tile_m") or (256 if kw["pair"] else 128)
        bn = kw["tile_n"] * (2 if kw.get("multicast") else 1)
        # at least 2 row and 2 column panels of >= 1 MiB: the pipelines engage
        if kw.get("split_k", 1) == 1 and m >= 2 * bm and n >= 2 * bn and 4 * m * k >= 2 << 20 and 4 * k * n >= 2 << 20:
            break
    env = {
        "FI_HOST_PIPELINE": str(rng.choice(["1", "panels"])),
        "FI_HOST_PANEL_MB": str(rng.choice(["1", "2"])),
        "FI_HOST_MIN_LINE": "128",
        "FI_HOST_PIECE_MB": str(rng.choice(["0.5", "1", "2"])),
        "FI_HOST_SNAP_RATIO": str(rng.choice(["0", "0.5", "0.8", "1"])),
        "FI_HOST_SNAP_SKIP": str(rng.choice(["0", "1", "3"])),
    }
    pins = (bool(rng.random() < 0.6), bool(rng.random() < 0.6))  # inputs, output
    return m, n, k, kw, env, pins


CASES = []
_rng = np.random.default_rng(20261020)
while len(CASES) < 24:
    CASES.append(draw_host(_rng))


PIPELINED = {}


@pytest.mark.parametrize("case", range(len(CASES)))
def test_random_host_pipeline(fi, oracle, monkeypatch, capfd, case):
    import torch
    m, n, k, kw, env, (pin_in, pin_out) = CASES[case]
    for key, v in env.items():
        monkeypatch.setenv(key, v)
    monkeypatch.setenv("FI_HOST_PIPELINE_TRACE", "1")
    ab = "bf16" if case % 4 == 3 else "f16"
    kw = dict(kw, ab=ab)
    plan = fi.Plan(fi.strategies.tc_strategy(m, n, k, **kw))
    a = oracle.fill(m, k, 700 + case, True)
    b = oracle.fill(k, n, 800 + case, True)
    # physical storage of the roots in the strategy's layouts
    lay = kw["layouts"]
    pa = (np.ascontiguousarray(a) if lay[0] == "rowmajor" else np.asfortranarray(a)).ravel(order="K")
    pb = (np.ascontiguousarray(b) if lay[1] == "rowmajor" else np.asfortranarray(b)).ravel(order="K")

    def buf(x, pinned):
        t = torch.from_numpy(np.ascontiguousarray(x))
        return t.pin_memory() if pinned else t

    hA, hB = buf(pa, pin_in), buf(pb, pin_in)
    hC = buf(np.zeros(m * n, np.float32), pin_out)
    plan.run_host_ptr(hA.data_ptr(), hB.data_ptr(), hC.data_ptr())
    err = capfd.readouterr().err
    PIPELINED[case] = ("blocked" in err or "pipeline" in err, bool(re.search(r" [AB]\d+h", err)))
    flat = hC.numpy()
    c = flat.reshape(m, n) if lay[2] == "rowmajor" else flat.reshape(n, m).T
    want = oracle.gemm_f64(oracle.round_elem(a, ab), oracle.round_elem(b, ab))
    if kw["c"] != "f32":
        want = oracle.round_elem(want, kw["c"])
    assert np.array_equal(c, want), (m, n, k, kw, env, pin_in, pin_out)
    up, down = plan.host_bytes()
    assert down == 4 * m * n
    assert 2 * (m * k + k * n) <= up <= 4 * (m * k + k * n)


def test_fuzz_cases_exercised_the_pipelines():
    """Most drawn cases ran a pipelined host path, and some snapped on the host."""
    assert len(PIPELINED) == len(CASES), PIPELINED
    assert sum(p for p, _ in PIPELINED.values()) >= len(CASES) // 2, PIPELINED
    assert sum(h for _, h in PIPELINED.values()) >= len(CASES) // 4, PIPELINED
