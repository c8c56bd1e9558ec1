"""Host snapping on the GPU box: fi_host_snap_f32 (host cores) against
fi_convert_f32 (the device conversion, runtime/convert.cu) bit for bit, and
fi_plan_run_host with host-snapped panels against the same call with every
panel snapped on the device (FI_HOST_SNAP_SKIP past the panel count): the
output must be bit-identical, including inputs beyond the f16 range that the
reference saturates (anvil::round_to_f16, matrix.hpp:67-80)."""
import re

import numpy as np
import pytest

from test_host_snap import SPECIALS, payload_nans

pytestmark = pytest.mark.gpu


def device_convert(fi, x, code):
    import torch
    src = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).cuda()
    dst = torch.empty(src.numel(), dtype=torch.int16, device="cuda")
    fi._native.check(fi.lib.fi_convert_f32(src.data_ptr(), dst.data_ptr(), src.numel(), code,
                                           torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    return dst.cpu().numpy().view(np.uint16)


@pytest.mark.parametrize("elem,code", [("f16", 1), ("bf16", 2)])
def test_host_snap_equals_device_conversion(fi, elem, code):
    rng = np.random.default_rng(7)
    bits = rng.integers(0, 2**32, size=1 << 20, dtype=np.uint64).astype(np.uint32).view(np.float32)
    x = np.concatenate([SPECIALS, -SPECIALS, payload_nans(), bits,
                        rng.uniform(-70000, 70000, 4096).astype(np.float32)])
    np.testing.assert_array_equal(fi.host_snap(x, elem), device_convert(fi, x, code))


CASES = [
    (1024, 2048, 1024, dict(pair=True, tile_n=256)),
    (1024, 2048, 2048, dict(pair=True, tile_n=128, ab="bf16")),
    (1024, 2048, 1024, dict(pair=True, tile_n=256, layouts=("rowmajor", "colmajor", "colmajor"))),
    (1024, 2048, 1024, dict(pair=True, tile_n=256, layouts=("colmajor", "rowmajor", "rowmajor"))),
]


@pytest.mark.parametrize("m,n,k,kw", CASES, ids=lambda x: str(x) if not isinstance(x, dict) else
                         "_".join(f"{a}{b}" for a, b in x.items()))
def test_run_host_host_snapped_panels_bit_identical(fi, oracle, monkeypatch, capfd, m, n, k, kw):
    monkeypatch.setenv("FI_HOST_PANEL_MB", "1")
    monkeypatch.setenv("FI_HOST_MIN_LINE", "128")
    monkeypatch.setenv("FI_HOST_PIPELINE_TRACE", "1")
    monkeypatch.delenv("FI_HOST_PIPELINE", raising=False)
    plan = fi.Plan(fi.strategies.tc_strategy(m, n, k, **kw))
    a = oracle.fill(m, k, 11, False) * np.float32(3.0)
    b = oracle.fill(k, n, 12, False)
    a[::97, ::89] = np.float32(70000.0)   # beyond f16: saturates to 65504 (f16 roots)
    b[::61, ::53] = np.float32(-1e-7)     # f16 subnormal range
    monkeypatch.setenv("FI_HOST_SNAP_SKIP", "1")
    c_host = plan.run_host(a, b)
    trace = capfd.readouterr().err
    assert "blocked" in trace and re.search(r" [AB]\d+h", trace), trace  # pieces were host-snapped
    up, down = plan.host_bytes()  # host-snapped pieces cross PCIe in 2-byte elements
    assert down == 4 * m * n and 2 * (m * k + k * n) <= up < 4 * (m * k + k * n), (up, down)
    monkeypatch.setenv("FI_HOST_SNAP_SKIP", "100000")
    c_dev = plan.run_host(a, b)
    trace = capfd.readouterr().err
    assert "blocked" in trace and not re.search(r" [AB]\d+h", trace), trace
    assert plan.host_bytes() == (4 * (m * k + k * n), 4 * m * n)
    np.testing.assert_array_equal(c_host.view(np.uint32), c_dev.view(np.uint32))
    # and exact against fp64 on integer inputs with host-snapped panels
    monkeypatch.setenv("FI_HOST_SNAP_SKIP", "0")
    ab = kw.get("ab", "f16")
    a = oracle.fill(m, k, 3, True)
    b = oracle.fill(k, n, 4, True)
    want = oracle.gemm_f64(oracle.round_elem(a, ab), oracle.round_elem(b, ab))
    assert np.array_equal(plan.run_host(a, b), want)


@pytest.mark.parametrize("pin_in,pin_out", [(True, False), (False, True), (False, False), (True, True)])
def test_run_host_pinned_and_pageable_buffers(fi, oracle, monkeypatch, capfd, pin_in, pin_out):
    """anvil::Matrix holds std::vector storage (pageable); the benchmark uses
    pinned buffers. Pageable inputs are snapped on the host entirely, a
    pageable C is staged in pinned memory and copied out by the host pool;
    every combination is exact against fp64 on integer inputs, in both
    pipelines (blocked and column panels)."""
    import torch
    monkeypatch.setenv("FI_HOST_PIPELINE_TRACE", "1")
    m, n, k = 1024, 2048, 1024
    plan = fi.Plan(fi.strategies.tc_strategy(m, n, k, pair=True, tile_n=256))
    a = oracle.fill(m, k, 3, True)
    b = oracle.fill(k, n, 4, True)
    want = oracle.gemm_f64(oracle.round_elem(a, "f16"), oracle.round_elem(b, "f16"))
    # physical col-major storage of the roots
    pa, pb = np.asfortranarray(a).ravel(order="K"), np.asfortranarray(b).ravel(order="K")
    def buf(x, pinned):
        t = torch.from_numpy(np.ascontiguousarray(x))
        return t.pin_memory() if pinned else t
    hA, hB = buf(pa, pin_in), buf(pb, pin_in)
    hC = buf(np.zeros(m * n, np.float32), pin_out)
    for mode in ["blocked", "panels"]:
        monkeypatch.setenv("FI_HOST_PIPELINE", "1" if mode == "blocked" else "panels")
        monkeypatch.setenv("FI_HOST_PANEL_MB", "1")
        monkeypatch.setenv("FI_HOST_MIN_LINE", "128")
        monkeypatch.setenv("FI_HOST_PIECE_MB", "1")
        hC.zero_()
        plan.run_host_ptr(hA.data_ptr(), hB.data_ptr(), hC.data_ptr())
        trace = capfd.readouterr().err
        assert ("pageable input" in trace) == (not pin_in), trace
        assert ("pageable C" in trace) == (not pin_out), trace
        c = hC.numpy().reshape(n, m).T  # col-major C
        assert np.array_equal(c, want), mode


def test_run_host_rejects_device_pointers(fi, monkeypatch):
    """The host pipelines read and write host memory: a device pointer is an
    argument error (FI_ERR_ARGUMENT), not a crash."""
    import torch
    monkeypatch.setenv("FI_HOST_PANEL_MB", "1")
    monkeypatch.setenv("FI_HOST_MIN_LINE", "128")
    m, n, k = 1024, 2048, 1024
    plan = fi.Plan(fi.strategies.tc_strategy(m, n, k, pair=True, tile_n=256))
    hA = torch.zeros(m * k, dtype=torch.float32, pin_memory=True)
    hB = torch.zeros(k * n, dtype=torch.float32, pin_memory=True)
    dC = torch.zeros(m * n, dtype=torch.float32, device="cuda")
    with pytest.raises(fi.FiError) as e:
        plan.run_host_ptr(hA.data_ptr(), hB.data_ptr(), dC.data_ptr())
    assert e.value.code == 104
