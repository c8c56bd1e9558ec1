"""Randomised GPU parity over the tcgen05 strategy space: tile variant (1-CTA,
pair, 512x256 slabs, 256x512 N halves, multicast pairs), tile N, split-K,
pipeline depth, operand layouts, C element type and problem shape, drawn with
a fixed seed. Every case must be integer-exact against the fp64 oracle at
sampled points (C in f16/bf16: exact after rounding the oracle) and must pass
the CPU protocol checker first. 80 f16 cases, 16 with bf16 operands, and 16
gated launches (the fused all-gather's GEMM: random chunk widths and first
chunks)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

LAYOUTS = [("colmajor", "colmajor", "colmajor"), ("rowmajor", "colmajor", "colmajor"),
           ("colmajor", "rowmajor", "rowmajor"), ("rowmajor", "rowmajor", "colmajor")]


def draw(rng):
    kind = rng.choice(["cta", "pair", "slab", "nhalf", "mcast"], p=[0.25, 0.35, 0.1, 0.1, 0.2])
    kw = {}
    if kind == "cta":
        kw.update(pair=False, tile_n=int(rng.choice([64, 128, 256])))
        bm, bn = 128, kw["tile_n"]
    elif kind == "pair":
        kw.update(pair=True, tile_n=int(rng.choice([64, 128, 256])))
        bm, bn = 256, kw["tile_n"]
    elif kind == "slab":
        kw.update(pair=True, tile_n=256, tile_m=512)
        bm, bn = 512, 256
    elif kind == "nhalf":
        kw.update(pair=True, tile_n=512)
        bm, bn = 256, 512
    else:
        kw.update(pair=True, tile_n=int(rng.choice([64, 128, 256])), multicast=True)
        bm, bn = 256, 2 * kw["tile_n"]
    lay = LAYOUTS[int(rng.integers(0, 4))]
    if kw["tile_n"] == 64 and kw["pair"] and lay[1] == "rowmajor":
        lay = LAYOUTS[int(rng.integers(0, 2))]  # N = 64 pair tiles need K-major B
    kw["layouts"] = lay
    m = bm * int(rng.integers(1, max(2, 2048 // bm) + 1))
    n = bn * int(rng.integers(1, max(2, 2048 // bn) + 1))
    k = 64 * int(rng.integers(1, 33))
    if kind in ("cta", "pair") and rng.random() < 0.3:
        s = int(rng.choice([2, 4]))
        if k % (64 * s) == 0 and (kw["tile_n"] // s) >= 32 and not (kind == "pair" and kw["tile_n"] == 64):
            kw["split_k"] = s
    if rng.random() < 0.3:
        kw["stages"] = int(rng.integers(2, 5))
    kw["c"] = str(rng.choice(["f32", "f32", "f16", "bf16"]))
    return m, n, k, kw


# FI_FUZZ_CASES / FI_FUZZ_SEED widen a one-off stress run (defaults: the fixed 80)
import os  # noqa: E402

CASES = []
_rng = np.random.default_rng(int(os.environ.get("FI_FUZZ_SEED", "20261017")))
while len(CASES) < int(os.environ.get("FI_FUZZ_CASES", "80")):
    CASES.append(draw(_rng))


@pytest.mark.parametrize("case", range(len(CASES)))
def test_random_tcgen05_strategy(fi, oracle, case):
    m, n, k, kw = CASES[case]
    script = fi.strategies.tc_strategy(m, n, k, **kw)
    chk = fi.check_async(script)
    assert chk.ok, (kw, chk.text)
    plan = fi.Plan(script)
    assert plan.kind == "tcgen05"
    a = oracle.fill(m, k, 100 + case, True)
    b = oracle.fill(k, n, 200 + case, True)
    c = plan.run_host(a, b)
    rng = np.random.default_rng(case)
    rows, cols = rng.integers(0, m, 2048), rng.integers(0, n, 2048)
    want = oracle.sample_f64(oracle.round_elem(a, "f16"), oracle.round_elem(b, "f16"), rows, cols).astype(np.float32)
    if kw["c"] != "f32":
        want = oracle.round_elem(want, kw["c"])
    assert np.array_equal(c[rows, cols], want), (m, n, k, kw)


GATED = []
_rg = np.random.default_rng(20261018)
while len(GATED) < 16:
    m, n, k, kw = draw(_rg)
    if kw.get("split_k", 1) > 1:
        continue
    unit = kw["tile_n"] * (2 if kw.get("multicast") else 1)  # N columns of one scheduled unit
    chunks = [c for c in range(1, n // unit + 1) if (n // unit) % c == 0]
    nch = int(_rg.choice(chunks))
    GATED.append((m, n, k, kw, n // nch, int(_rg.integers(0, nch))))


@pytest.mark.parametrize("case", range(len(GATED)))
def test_random_gated_launch(fi, oracle, case):
    """Gated launches (the fused all-gather's GEMM) over random strategies,
    chunk widths and first chunks, every flag already at the epoch: exact."""
    import torch
    m, n, k, kw, chunk_cols, first = GATED[case]
    kw = dict(kw, c="f32", layouts=("colmajor", "colmajor", "colmajor"))
    plan = fi.Plan(fi.strategies.tc_strategy(m, n, k, **kw))
    a = oracle.fill(m, k, 300 + case, True)
    b = oracle.fill(k, n, 400 + case, True)
    dt = torch.bfloat16 if kw.get("ab") == "bf16" else torch.float16
    dA = torch.from_numpy(np.ascontiguousarray(a.T).ravel()).cuda().to(dt)
    dB = torch.from_numpy(np.asfortranarray(b).ravel(order="F").copy()).cuda().to(dt)
    dC = torch.full((m * n,), float("nan"), device="cuda")
    ready = torch.full((n // chunk_cols,), 3, device="cuda", dtype=torch.int32)
    plan.launch_gated(dA.data_ptr(), dB.data_ptr(), dC.data_ptr(), torch.cuda.current_stream().cuda_stream,
                      ready.data_ptr(), 3, chunk_cols, first)
    torch.cuda.synchronize()
    c = dC.cpu().numpy().reshape(n, m).T
    assert np.array_equal(c, oracle.gemm_f64(a, b)), (m, n, k, kw, chunk_cols, first)


BF16 = []
_rb = np.random.default_rng(20261019)
while len(BF16) < 16:
    BF16.append(draw(_rb))


@pytest.mark.parametrize("case", range(len(BF16)))
def test_random_bf16_strategy(fi, oracle, case):
    """The same random strategy space with bf16 operands (the C5 element type)."""
    m, n, k, kw = BF16[case]
    kw = dict(kw, ab="bf16")
    script = fi.strategies.tc_strategy(m, n, k, **kw)
    chk = fi.check_async(script)
    assert chk.ok, (kw, chk.text)
    plan = fi.Plan(script)
    a = oracle.fill(m, k, 500 + case, True)
    b = oracle.fill(k, n, 600 + case, True)
    c = plan.run_host(a, b)
    rng = np.random.default_rng(case)
    rows, cols = rng.integers(0, m, 2048), rng.integers(0, n, 2048)
    want = oracle.sample_f64(oracle.round_elem(a, "bf16"), oracle.round_elem(b, "bf16"), rows, cols).astype(np.float32)
    if kw["c"] != "f32":
        want = oracle.round_elem(want, kw["c"])
    assert np.array_equal(c[rows, cols], want), (m, n, k, kw)
