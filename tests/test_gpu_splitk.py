"""Both lowerings of the `.splitk` refinement on CTA pairs:
  * cross-cluster K slices (every (tile, slice) fits one wave): partials
    exchanged through L2 and summed in shared memory in slice order;
  * in-cluster DSMEM reduction (too many tiles for one wave).
Integer inputs are exact; uniform inputs bitwise reproducible."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("shape,split,expect_global", [((1024, 1024, 32768), 4, 1), ((512, 1024, 8192), 2, 1),
                                                       ((4096, 2048, 1024), 2, 0)])
def test_pair_splitk_lowerings(fi, oracle, shape, split, expect_global):
    m, n, k = shape
    plan = fi.Plan(fi.strategies.tc_strategy(m, n, k, pair=True, tile_n=256, split_k=split))
    a = oracle.fill(m, k, 31, True)
    b = oracle.fill(k, n, 32, True)
    c = plan.run_host(a, b)
    rng = np.random.default_rng(5)
    rows, cols = rng.integers(0, m, 4096), rng.integers(0, n, 4096)
    ar, br = oracle.round_elem(a, "f16"), oracle.round_elem(b, "f16")
    assert np.array_equal(c[rows, cols].astype(np.float64), oracle.sample_f64(ar, br, rows, cols))
    assert np.array_equal(c, np.round(c))
    u = oracle.fill(m, k, 33, False), oracle.fill(k, n, 34, False)
    c1, c2 = plan.run_host(*u), plan.run_host(*u)
    assert np.array_equal(c1.view(np.uint32), c2.view(np.uint32))
    # which lowering ran: cross-cluster slices use a plain pair cluster
    assert (plan.info.cluster == 2) == bool(expect_global)
