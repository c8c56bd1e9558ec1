"""CPU checker of the tcgen05 launch protocol (include/fireiron/async_check.hpp,
SURVEY.md 8(f) rank 4): every strategy the GPU tests and the bench run must
replay race-free, within its shared-memory / TMEM / workspace allocations,
storing each output chunk exactly once; every injected protocol fault must
be reported -- the B200 counterpart of the reference's race and ownership
checks (proj/include/anvil/sim.hpp:63-104, 546-561; tests/test_sim.cpp)."""
import pytest


@pytest.fixture(scope="module")
def tc(fi):
    return fi.strategies.tc_strategy


CFGS = [dict(pair=True, tile_n=256), dict(pair=True, tile_n=128), dict(pair=False, tile_n=256),
        dict(pair=False, tile_n=128), dict(pair=False, tile_n=64)]
LAYOUTS = [("colmajor", "colmajor", "colmajor"), ("rowmajor", "colmajor", "colmajor"),
           ("colmajor", "rowmajor", "rowmajor"), ("rowmajor", "rowmajor", "colmajor")]


@pytest.mark.parametrize("cfg", CFGS, ids=lambda c: f"pair{int(c['pair'])}_n{c['tile_n']}")
@pytest.mark.parametrize("layouts", LAYOUTS, ids=lambda l: "".join(x[0] for x in l))
@pytest.mark.parametrize("cout", ["f32", "f16"])
def test_gpu_test_strategies_are_race_free(fi, tc, cfg, layouts, cout):
    m, n, k = 512, 768 if cfg["tile_n"] != 256 else 512, 320
    r = fi.check_async(tc(m, n, k, layouts=layouts, c=cout, **cfg))
    assert r.ok, r.text


@pytest.mark.parametrize("pair,tile_n,split", [(False, 128, 2), (False, 128, 4), (False, 256, 4),
                                               (True, 256, 2), (True, 256, 4), (True, 128, 2)])
@pytest.mark.parametrize("k", [4096, 16384])
def test_splitk_lowerings_are_race_free(fi, tc, pair, tile_n, split, k):
    # pairs: cross-cluster K slices (+ remainder at k=16384); 1-CTA: cluster DSMEM reduction
    r = fi.check_async(tc(512, 512, k, pair=pair, tile_n=tile_n, split_k=split))
    assert r.ok, r.text
    assert r.split_k == split


@pytest.mark.parametrize("mode", [-1, 0, 1, 2])
@pytest.mark.parametrize("shape", [(4096, 4096, 4096), (4096, 4096, 1024), (2560, 2560, 10240), (768, 1024, 9600),
                                   (4096, 4096, 32768), (8192, 8192, 2048)])
def test_tail_schedules_are_race_free(fi, tc, mode, shape):
    r = fi.check_async(tc(*shape), streamk=mode)
    assert r.ok, r.text


def test_bench_workload_schedules(fi, tc):
    """The schedules the bench lines measure."""
    c2 = fi.check_async(fi.strategies.c2_strategy())
    assert c2.ok and c2.mode == 1 and c2.slices == 2 and not c2.remainder and c2.units == 222 + 68
    c3 = fi.check_async(fi.strategies.c3_strategy())
    assert c3.ok and c3.mode == 1 and c3.slices == 4 and c3.remainder and c3.clusters == 74
    assert c3.units == 16 * 4 + 16  # 64 main slices + 16 remainders on 10 extra clusters
    c5 = fi.check_async(fi.strategies.c5_strategy(2048, 2048, 16384))  # an 8-way shard chunk
    assert c5.ok


@pytest.mark.parametrize("m,n,k", [(1024, 1024, 1024), (2048, 2048, 2048), (4096, 256, 4096), (512, 8192, 8192)])
def test_sweep_strategies_are_race_free(fi, m, n, k):
    for name, script in fi.strategies.sweep_strategies(m, n, k).items():
        r = fi.check_async(script)
        assert r.ok, (name, r.text)


@pytest.mark.parametrize("kw", [dict(tile_m=512), dict(tile_n=512)], ids=["slab512x256", "nhalf256x512"])
@pytest.mark.parametrize("shape", [(1024, 512, 320), (4096, 4096, 1024), (8192, 8192, 2048)])
def test_wide_pair_tiles_are_race_free(fi, tc, kw, shape):
    r = fi.check_async(tc(*shape, **kw))
    assert r.ok and r.mode == 0, r.text


@pytest.mark.parametrize("stages", [2, 3, 4])
def test_shallow_rings_are_race_free(fi, tc, stages):
    r = fi.check_async(tc(1024, 1024, 2048, stages=stages))
    assert r.ok and r.stages == stages, r.text


def test_without_ring_drain_or_tma_store(fi, tc):
    assert fi.check_async(tc(4096, 4096, 1024), ring_drain=0).ok
    assert fi.check_async(tc(4096, 4096, 1024), c_tma=0).ok


# ---------------------------------------------------------------- fault injection
MUTANTS = [
    ("ring_drain_every_unit", (4096, 4096, 1024), {}, "races"),           # C staged over in-flight TMA loads
    ("flag_before_bulk_wait", (1024, 1024, 32768), dict(split_k=4), "races"),  # peers read unwritten partials
    ("skip_tmem_empty_wait", (4096, 4096, 1024), {}, "races"),            # MMA overwrites an undrained accumulator
    ("remainder_slot_collision", (1024, 1024, 32768), dict(split_k=4), "races"),
    ("unpacked_peer_staging", (768, 1024, 9600), {}, "capacity_errors"),  # 6 slices: staging past the ring
    ("skip_empty_wait", (1024, 1024, 4096), {}, "deadlocks"),             # parity runs ahead of the consumer
    ("tx_undercount", (1024, 1024, 1024), dict(tile_n=512), "deadlocks"),  # N-half tile: B half 2 not expected
    ("mcast_single_release", (2048, 2048, 2048), dict(multicast=True), "races"),  # twin pair still reading
]


@pytest.mark.parametrize("mutation,shape,kw,field", MUTANTS, ids=[m[0] for m in MUTANTS])
def test_injected_faults_are_reported(fi, tc, mutation, shape, kw, field):
    clean = fi.check_async(tc(*shape, **kw))
    assert clean.ok, clean.text
    bad = fi.check_async(tc(*shape, **kw), mutation=mutation)
    assert not bad.ok
    assert getattr(bad, field) > 0, bad.text


# ---------------------------------------------------------------- gated launches
GATED = [  # (shape, strategy kwargs, chunks, first chunk): the fused all-gather's GEMM
    ((2048, 16384, 1024), dict(ab="bf16", tile_m=512), 8, 3),  # C5 band at 8 GPUs, slab tiles
    ((2048, 4096, 2048), {}, 4, 0),
    ((1024, 2048, 512), dict(tile_n=128, multicast=True), 4, 1),
    ((512, 1024, 4096), dict(pair=False, tile_n=128), 2, 1),   # K-slice tail units gated too
]


@pytest.mark.parametrize("shape,kw,chunks,first", GATED)
def test_gated_launch_protocol(fi, tc, shape, kw, chunks, first):
    """B chunks landed by a copy engine and released by ready flags: every TMA
    read of a chunk must happen after the producer acquired its flag; a
    producer that skips the acquire races the copy engine."""
    s = tc(*shape, **kw)
    r = fi.check_async(s, gated_chunks=chunks, gated_first=first)
    assert r.ok, r.text
    bad = fi.check_async(s, gated_chunks=chunks, gated_first=first, mutation="gate_skip_acquire")
    assert bad.races > 0 and "B chunk" in bad.text


def test_gated_chunks_must_split_the_tile_columns(fi, tc):
    r = fi.check_async(tc(2048, 4096, 1024), gated_chunks=3)
    assert not r.ok and r.capacity_errors > 0


def test_non_tensor_core_tree_is_rejected(fi):
    from paper_2003_06324_b200 import FiError
    with pytest.raises(FiError):
        fi.check_async(fi.strategies.listing2(128, 128, 32))


@pytest.mark.parametrize("shape", [(4096, 256, 4096), (1024, 1024, 1024), (2048, 2048, 2048), (4096, 4096, 1024)])
@pytest.mark.parametrize("mode", [-1, 1])
def test_pair_256x64_schedules_are_race_free(fi, tc, shape, mode):
    r = fi.check_async(tc(*shape, tile_n=64), streamk=mode)
    assert r.ok, r.text


@pytest.mark.parametrize("tn", [64, 128, 256])
@pytest.mark.parametrize("shape", [(4096, 256, 4096), (2048, 2048, 2048), (1024, 1024, 1024), (4096, 4096, 1024)])
@pytest.mark.parametrize("layouts", [("colmajor", "colmajor", "colmajor"), ("rowmajor", "colmajor", "colmajor")],
                         ids=["ccc", "rcc"])
def test_multicast_pairs_are_race_free(fi, tc, tn, shape, layouts):
    if shape[1] % (2 * tn):
        pytest.skip("N must hold two tiles")
    r = fi.check_async(tc(*shape, tile_n=tn, multicast=True, layouts=layouts))
    assert r.ok and r.cluster_size == 4 and r.mode == 0, r.text


# three producer warps over ring depths that are and are not multiples of three
# (the GPU side: tests/test_gpu_tc.py::test_ring_depths_with_three_producers)
@pytest.mark.parametrize("stages", [2, 3, 4, 5, 7])
@pytest.mark.parametrize("kw", [dict(pair=False, tile_n=64), dict(pair=True, tile_n=128),
                                dict(pair=True, tile_n=64, multicast=True)], ids=["cta64", "pair128", "pair64_mcast"])
def test_three_producers_any_ring_depth(fi, tc, stages, kw):
    r = fi.check_async(tc(1024, 512, 1472, stages=stages, **kw))
    assert r.ok and r.stages == stages, r.text
