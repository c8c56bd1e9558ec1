"""GPU parity of the tensor-core (tcgen05/TMA/TMEM) strategies. Integer-mode
inputs ({-3..3}, exact in f16/bf16, partial sums < 2^24) must equal the fp64
oracle exactly for every strategy, split-K included; uniform inputs must meet
the north-star bound max|C - C64| / max|C64| <= 1e-2 with C64 the fp64 GEMM
on grid-rounded inputs (tolerance stated here: 1e-2)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL_NORMWISE = 1e-2


def run(fi, oracle, script, m, n, k, integers, seed=1, elem="f16"):
    plan = fi.Plan(script)
    assert plan.kind == "tcgen05", plan.source()[:200]
    a = oracle.fill(m, k, seed, integers)
    b = oracle.fill(k, n, seed + 1, integers)
    c = plan.run_host(a, b)
    ar, br = oracle.round_elem(a, elem), oracle.round_elem(b, elem)
    return c, ar, br


CFGS = [dict(pair=True, tile_n=256), dict(pair=True, tile_n=128), dict(pair=False, tile_n=256),
        dict(pair=False, tile_n=128), dict(pair=False, tile_n=64)]
LAYOUTS = [("colmajor", "colmajor", "colmajor"), ("rowmajor", "colmajor", "colmajor"),
           ("colmajor", "rowmajor", "rowmajor"), ("rowmajor", "rowmajor", "colmajor")]


@pytest.mark.parametrize("cfg", CFGS, ids=lambda c: f"pair{int(c['pair'])}_n{c['tile_n']}")
@pytest.mark.parametrize("layouts", LAYOUTS, ids=lambda l: "".join(x[0] for x in l))
def test_integer_exact_all_tiles_and_layouts(fi, oracle, cfg, layouts):
    m, n, k = 512, 768 if cfg["tile_n"] != 256 else 512, 320
    s = fi.strategies.tc_strategy(m, n, k, layouts=layouts, **cfg)
    c, ar, br = run(fi, oracle, s, m, n, k, True)
    assert np.array_equal(c, oracle.gemm_f64(ar, br))


@pytest.mark.parametrize("ab", ["f16", "bf16"])
@pytest.mark.parametrize("cout", ["f32", "f16", "bf16"])
def test_element_types(fi, oracle, ab, cout):
    m, n, k = 512, 512, 256
    s = fi.strategies.tc_strategy(m, n, k, ab=ab, c=cout)
    c, ar, br = run(fi, oracle, s, m, n, k, False, elem=ab)
    want = oracle.gemm_f64(ar, br)
    err = np.max(np.abs(c - want)) / np.max(np.abs(want))
    bound = TOL_NORMWISE if cout == "f32" else 2.0 ** -7
    assert err <= bound
    if cout == "f32":
        assert err <= 1e-5  # fp32 accumulation on exact products


@pytest.mark.parametrize("pair,tile_n,split", [(False, 128, 2), (False, 128, 4), (False, 256, 4),
                                               (True, 256, 2), (True, 256, 4), (True, 128, 2)])
def test_splitk_integer_exact_and_deterministic(fi, oracle, pair, tile_n, split):
    m, n, k = 512, 512, 4096
    s = fi.strategies.tc_strategy(m, n, k, pair=pair, tile_n=tile_n, split_k=split)
    c, ar, br = run(fi, oracle, s, m, n, k, True)
    assert np.array_equal(c, oracle.gemm_f64(ar, br))
    plan = fi.Plan(s)
    a = oracle.fill(m, k, 9, False)
    b = oracle.fill(k, n, 10, False)
    c1, c2 = plan.run_host(a, b), plan.run_host(a, b)
    assert np.array_equal(c1.view(np.uint32), c2.view(np.uint32))  # fixed reduction order


def test_c2_strategy_4096_uniform_within_tolerance(fi, oracle):
    s = fi.strategies.c2_strategy()
    c, ar, br = run(fi, oracle, s, 4096, 4096, 4096, False, seed=1)
    rng = np.random.default_rng(0)
    rows = rng.integers(0, 4096, 4096)
    cols = rng.integers(0, 4096, 4096)
    want = oracle.sample_f64(ar, br, rows, cols)
    got = c[rows, cols].astype(np.float64)
    assert np.max(np.abs(got - want)) / np.max(np.abs(want)) <= TOL_NORMWISE
    assert np.max(np.abs(got - want)) <= 1e-3


def test_c2_strategy_4096_integer_exact_sampled(fi, oracle):
    s = fi.strategies.c2_strategy()
    c, ar, br = run(fi, oracle, s, 4096, 4096, 4096, True, seed=3)
    assert np.array_equal(c, np.round(c))
    rng = np.random.default_rng(1)
    rows, cols = rng.integers(0, 4096, 8192), rng.integers(0, 4096, 8192)
    assert np.array_equal(c[rows, cols].astype(np.float64), oracle.sample_f64(ar, br, rows, cols))


def test_c3_splitk_strategy_integer_exact_sampled(fi, oracle):
    s = fi.strategies.c3_strategy()
    c, ar, br = run(fi, oracle, s, 1024, 1024, 32768, True, seed=5)
    rng = np.random.default_rng(2)
    rows, cols = rng.integers(0, 1024, 4096), rng.integers(0, 1024, 4096)
    assert np.array_equal(c[rows, cols].astype(np.float64), oracle.sample_f64(ar, br, rows, cols))


def test_block_swizzle_schedule_is_honoured(fi, oracle):
    # tiles visited in reverse order: results must not depend on the schedule
    m, n, k = 1024, 1024, 256
    units = (m // 256) * (n // 256)
    s = fi.strategies.tc_strategy(m, n, k, swizzle=f"(id*5)%{units}")  # 5 is coprime with 16
    c, ar, br = run(fi, oracle, s, m, n, k, True)
    assert np.array_equal(c, oracle.gemm_f64(ar, br))


def test_device_launch_equals_host_run(fi, oracle):
    import torch
    m, n, k = 512, 512, 512
    plan = fi.Plan(fi.strategies.tc_strategy(m, n, k))
    a = oracle.fill(m, k, 7, False)
    b = oracle.fill(k, n, 8, False)
    host = plan.run_host(a, b)
    da = torch.from_numpy(a.T.copy()).cuda().half()  # col-major A
    db = torch.from_numpy(b.T.copy()).cuda().half()  # col-major B
    dc = torch.empty((n, m), device="cuda")
    plan.launch(da.data_ptr(), db.data_ptr(), dc.data_ptr(), torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    assert np.array_equal(dc.cpu().numpy().T.view(np.uint32), host.view(np.uint32))


def test_unsupported_tile_reports_cleanly(fi):
    s = fi.strategies.tc_strategy(512, 480, 256, pair=False, tile_n=96)
    with pytest.raises(fi.FiError) as e:
        fi.Plan(s)
    assert e.value.kind in ("Unsupported", "NonDivisible")


@pytest.mark.parametrize("pair,tile_n,shape", [(True, 256, (1280, 1024, 2048)), (False, 128, (2048, 2560, 2048)),
                                               (True, 256, (1024, 1024, 32768)), (True, 128, (4096, 4096, 4096)),
                                               (False, 256, (4096, 4096, 4096)), (True, 256, (4096, 4096, 4096))])
def test_tail_split_exact_and_deterministic(fi, oracle, monkeypatch, pair, tile_n, shape):
    """The partial last wave's tiles are split into K-slices across idle
    clusters (fixups of up to 6 slices): integer inputs stay exact, uniform
    inputs are bitwise reproducible and within tolerance."""
    m, n, k = shape
    s = fi.strategies.tc_strategy(m, n, k, pair=pair, tile_n=tile_n)
    plan = fi.Plan(s)
    a = oracle.fill(m, k, 11, True)
    b = oracle.fill(k, n, 12, True)
    c = plan.run_host(a, b)
    rng = np.random.default_rng(3)
    rows, cols = rng.integers(0, m, 4096), rng.integers(0, n, 4096)
    ar, br = oracle.round_elem(a, "f16"), oracle.round_elem(b, "f16")
    assert np.array_equal(c[rows, cols].astype(np.float64), oracle.sample_f64(ar, br, rows, cols))
    assert np.array_equal(c, np.round(c))
    a = oracle.fill(m, k, 13, False)
    b = oracle.fill(k, n, 14, False)
    c1, c2 = plan.run_host(a, b), plan.run_host(a, b)
    assert np.array_equal(c1.view(np.uint32), c2.view(np.uint32))
    want = oracle.sample_f64(oracle.round_elem(a, "f16"), oracle.round_elem(b, "f16"), rows, cols)
    assert np.max(np.abs(c1[rows, cols] - want)) / np.max(np.abs(want)) <= TOL_NORMWISE


def test_c2_plan_uses_tail_split(fi):
    plan = fi.Plan(fi.strategies.c2_strategy())
    assert plan.info.streamk == 1 and plan.info.launch_ctas == 148  # K-sliced partial wave


@pytest.mark.parametrize("mode", ["1", "2"])
@pytest.mark.parametrize("layouts", [("colmajor", "colmajor", "colmajor"), ("rowmajor", "rowmajor", "rowmajor")])
def test_forced_tail_modes(fi, oracle, monkeypatch, mode, layouts):
    """Both tail modes on a 3.46-wave problem, both B majors: integer exact."""
    monkeypatch.setenv("FI_STREAMK", mode)
    m, n, k = 4096, 4096, 1024
    plan = fi.Plan(fi.strategies.tc_strategy(m, n, k, layouts=layouts))
    assert plan.info.streamk == int(mode)
    a = oracle.fill(m, k, 21, True)
    b = oracle.fill(k, n, 22, True)
    c = plan.run_host(a, b)
    rng = np.random.default_rng(4)
    rows, cols = rng.integers(0, m, 8192), rng.integers(0, n, 8192)
    ar, br = oracle.round_elem(a, "f16"), oracle.round_elem(b, "f16")
    assert np.array_equal(c[rows, cols].astype(np.float64), oracle.sample_f64(ar, br, rows, cols))
    # the last tiles (the tail) explicitly: a full 256-column strip at the end
    assert np.array_equal(c[-256:, -256:].astype(np.float64),
                          oracle.gemm_f64(ar[-256:], br[:, -256:]).astype(np.float64))


WIDE = {"slab512x256": dict(tile_m=512), "nhalf256x512": dict(tile_n=512)}


@pytest.mark.parametrize("wide", sorted(WIDE))
@pytest.mark.parametrize("layouts", LAYOUTS, ids=lambda l: "".join(x[0] for x in l))
@pytest.mark.parametrize("cout", ["f32", "f16"])
def test_wide_pair_tiles_integer_exact(fi, oracle, wide, layouts, cout):
    """tile 512 256 .pair (two A slabs per CTA, two M=256 MMAs sharing B) and
    tile 256 512 .pair (two N=256 MMAs sharing A through the A collector): the
    whole TMEM per accumulator, whole-tile schedule."""
    m, n, k = 1024, 512, 320
    s = fi.strategies.tc_strategy(m, n, k, layouts=layouts, c=cout, **WIDE[wide])
    plan = fi.Plan(s)
    assert plan.kind == "tcgen05" and plan.info.tile_m * plan.info.tile_n == 512 * 256 and plan.info.streamk == 0
    a = oracle.fill(m, k, 21, True)
    b = oracle.fill(k, n, 22, True)
    want = oracle.gemm_f64(oracle.round_elem(a, "f16"), oracle.round_elem(b, "f16"))
    got = plan.run_host(a, b)
    assert np.array_equal(got, want if cout == "f32" else oracle.round_elem(want, "f16"))


@pytest.mark.parametrize("wide", sorted(WIDE))
def test_wide_pair_tiles_multi_wave_uniform(fi, oracle, monkeypatch, wide):
    # 4096 x 4096: 128 wide tiles over 74 clusters (two waves, the last one partial)
    monkeypatch.setenv("FI_HOST_PIPELINE", "0")
    m = n = 4096
    k = 1024
    s = fi.strategies.tc_strategy(m, n, k, **WIDE[wide])
    c, ar, br = run(fi, oracle, s, m, n, k, False, seed=31)
    rng = np.random.default_rng(3)
    rows, cols = rng.integers(0, m, 4096), rng.integers(0, n, 4096)
    want = oracle.sample_f64(ar, br, rows, cols)
    got = c[rows, cols].astype(np.float64)
    assert np.max(np.abs(got - want)) / np.max(np.abs(want)) <= TOL_NORMWISE
    assert np.max(np.abs(got - want)) <= 1e-3
    plain = fi.Plan(fi.strategies.tc_strategy(m, n, k))  # same products, 256x256 tiles
    assert np.max(np.abs(plain.run_host(oracle.fill(m, k, 31, False), oracle.fill(k, n, 32, False)) - c)) <= 1e-4


@pytest.mark.parametrize("layouts", LAYOUTS[:2], ids=lambda l: "".join(x[0] for x in l))
@pytest.mark.parametrize("m,n,k", [(512, 256, 320), (4096, 256, 1024)])
def test_pair_256x64_tile_integer_exact(fi, oracle, layouts, m, n, k):
    """Narrow pair tile (cta_group::2, N = 64, 9-stage ring; K-major B only)."""
    s = fi.strategies.tc_strategy(m, n, k, layouts=layouts, tile_n=64)
    plan = fi.Plan(s)
    assert plan.kind == "tcgen05" and plan.info.cta_group == 2 and plan.info.tile_n == 64
    a = oracle.fill(m, k, 41, True)
    b = oracle.fill(k, n, 42, True)
    want = oracle.gemm_f64(oracle.round_elem(a, "f16"), oracle.round_elem(b, "f16"))
    assert np.array_equal(plan.run_host(a, b), want)


@pytest.mark.parametrize("tn", [64, 128, 256])
@pytest.mark.parametrize("layouts", LAYOUTS, ids=lambda l: "".join(x[0] for x in l))
def test_multicast_pair_tiles_integer_exact(fi, oracle, tn, layouts):
    """.multicast: two pair tiles (neighbours along N) form a 4-CTA cluster and
    share each A stage -- each CTA loads one 64-row half and multicasts it."""
    if tn == 64 and layouts[1] == "rowmajor":
        pytest.skip("N = 64 pair tiles need K-major B")
    m, n, k = 512, 4 * tn, 320
    s = fi.strategies.tc_strategy(m, n, k, layouts=layouts, tile_n=tn, multicast=True)
    plan = fi.Plan(s)
    assert plan.kind == "tcgen05" and plan.info.cluster == 4
    a = oracle.fill(m, k, 51, True)
    b = oracle.fill(k, n, 52, True)
    want = oracle.gemm_f64(oracle.round_elem(a, "f16"), oracle.round_elem(b, "f16"))
    assert np.array_equal(plan.run_host(a, b), want)


def test_multicast_multi_wave_uniform(fi, oracle, monkeypatch):
    monkeypatch.setenv("FI_HOST_PIPELINE", "0")
    m = n = 4096
    k = 1024
    s = fi.strategies.tc_strategy(m, n, k, multicast=True)
    c, ar, br = run(fi, oracle, s, m, n, k, False, seed=61)
    plain = fi.Plan(fi.strategies.tc_strategy(m, n, k))
    assert np.max(np.abs(plain.run_host(oracle.fill(m, k, 61, False), oracle.fill(k, n, 62, False)) - c)) <= 1e-4


def _sampled_exact(torch, np, A_km, B_nk, C_nm, m, n, samples=1024, seed=5):
    """C (column-major M x N, stored as [n][m]) against fp64 dot products of sampled
    (row, col) pairs of the integer operands (A stored [k][m], B stored [n][k])."""
    rng = np.random.default_rng(seed)
    rows, cols = rng.integers(0, m, samples), rng.integers(0, n, samples)
    ri, ci = torch.from_numpy(rows).cuda(), torch.from_numpy(cols).cuda()
    a = A_km[:, ri].T.float().cpu().numpy().astype(np.float64)   # samples x k
    b = B_nk[ci, :].float().cpu().numpy().astype(np.float64)      # samples x k
    want = np.einsum("sk,sk->s", a, b)
    got = C_nm.view(n, m)[ci, ri].cpu().numpy().astype(np.float64)
    return np.array_equal(got, want)


def test_c5_full_size_sampled_exact(fi):
    """configs[4] at full size on one GPU (16384^3 bf16, 512x256 slab tiles):
    integer operands generated on the device, 1024 sampled outputs exact."""
    import torch
    m = n = k = 16384
    plan = fi.Plan(fi.strategies.c5_strategy())
    g = torch.Generator(device="cuda").manual_seed(7)
    A = torch.randint(-3, 4, (k, m), device="cuda", generator=g).to(torch.bfloat16)
    B = torch.randint(-3, 4, (n, k), device="cuda", generator=g).to(torch.bfloat16)
    C = torch.empty(n * m, device="cuda")
    plan.launch(A.data_ptr(), B.data_ptr(), C.data_ptr(), torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    assert _sampled_exact(torch, np, A, B, C, m, n)


def test_c5_band_gated_full_size_sampled_exact(fi):
    """The 8-GPU shard of configs[4] as the fused all-gather runs it: one gated
    launch over a 2048 x 16384 x 16384 band, B in 8 chunks, starting at chunk 3."""
    import torch
    m, n, k = 2048, 16384, 16384
    plan = fi.Plan(fi.strategies.c5_strategy(m, n, k))
    g = torch.Generator(device="cuda").manual_seed(8)
    A = torch.randint(-3, 4, (k, m), device="cuda", generator=g).to(torch.bfloat16)
    B = torch.randint(-3, 4, (n, k), device="cuda", generator=g).to(torch.bfloat16)
    C = torch.full((n * m,), float("nan"), device="cuda")
    ready = torch.ones(8, device="cuda", dtype=torch.int32)
    plan.launch_gated(A.data_ptr(), B.data_ptr(), C.data_ptr(), torch.cuda.current_stream().cuda_stream,
                      ready.data_ptr(), 1, n // 8, 3)
    torch.cuda.synchronize()
    assert not torch.isnan(C).any().item()
    assert _sampled_exact(torch, np, A, B, C, m, n)


def test_f16_ingestion_saturates_like_round_to_f16(fi, oracle):
    """run_host snaps fp32 host data to f16 on the device with the reference's
    saturation (matrix.hpp:76): finite |x| >= 2^16 becomes +-65504 where IEEE
    RNE gives inf. C = A * I reproduces the snapped A exactly."""
    m = n = k = 256
    plan = fi.Plan(fi.strategies.tc_strategy(m, n, k, pair=True, tile_n=256))
    rng = np.random.default_rng(5)
    a = rng.uniform(-2.0, 2.0, (m, k)).astype(np.float32)
    special = np.array([70000.0, -70000.0, 1e6, -3e38, 65504.0, 65519.0, -65519.0, 65536.0, 1e-8, -2.0 ** -24],
                       dtype=np.float32)
    a.flat[rng.choice(m * k, special.size * 20, replace=False)] = np.tile(special, 20)
    c = plan.run_host(a, np.eye(k, n, dtype=np.float32))
    want = oracle.round_elem(a, "f16")
    assert np.isfinite(c).all()
    assert np.array_equal(c, want)


# Three producer warps fill the ring stages s % 3 = 0, 1, 2 (gemm_kernel.cuh); ring
# depths that are and are not multiples of three, and shallower than three, must
# all give the exact result -- over units that wrap the ring several times.
@pytest.mark.parametrize("stages", [2, 3, 4, 5, 6, 7])
@pytest.mark.parametrize("cfg", [dict(pair=False, tile_n=64), dict(pair=True, tile_n=128),
                                 dict(pair=True, tile_n=64, multicast=True), dict(pair=True, tile_n=256, tile_m=512)],
                         ids=["cta64", "pair128", "pair64_mcast", "slab512"])
def test_ring_depths_with_three_producers(fi, oracle, stages, cfg):
    m, n, k = 1024, 512, 1472  # 23 K blocks per tile: not a multiple of any ring depth
    s = fi.strategies.tc_strategy(m, n, k, stages=stages, **cfg)
    c, ar, br = run(fi, oracle, s, m, n, k, True, seed=11 + stages)
    assert np.array_equal(c, oracle.gemm_f64(ar, br))
