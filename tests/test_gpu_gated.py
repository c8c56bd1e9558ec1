"""Gated launches (fi_plan_launch_gated): ONE persistent tcgen05 GEMM whose B
column chunks become readable only when their ready flags reach the launch's
epoch -- the multi-GPU driver's fused all-gather -> GEMM. Integer inputs,
compared exactly with the fp64 oracle: with every flag already set; with a
chunk that lands (copy + stream-ordered flag write on another stream) only
after the kernel is running, so an early read would see garbage; and with a
chunk that never lands, which must fail the launch (trap) instead of hanging."""
import os
import subprocess
import sys
import time

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
M, N, K, CHUNK = 512, 1024, 512, 256


def _setup(fi, oracle, torch, **kw):
    plan = fi.Plan(fi.strategies.tc_strategy(M, N, K, **kw))
    a = oracle.fill(M, K, 11, True)
    b = oracle.fill(K, N, 12, True)
    dev = torch.device("cuda", 0)
    dA = torch.from_numpy(np.ascontiguousarray(a.T).ravel()).to(dev).half()   # col-major
    b_cm = torch.from_numpy(np.asfortranarray(b).ravel(order="F").copy()).to(dev).half()
    dC = torch.full((M * N,), float("nan"), device=dev)
    want = oracle.gemm_f64(a, b)
    return plan, dA, b_cm, dC, want


def _band(dC):
    return dC.cpu().numpy().reshape(N, M).T


@pytest.mark.parametrize("kw", [dict(pair=True, tile_n=256), dict(pair=False, tile_n=128),
                                dict(pair=True, tile_n=128, multicast=True)],
                         ids=["pair256", "cta128", "mcast128"])
@pytest.mark.parametrize("first", [0, 3])
def test_gated_all_ready(fi, oracle, kw, first):
    import torch
    plan, dA, dB, dC, want = _setup(fi, oracle, torch, **kw)
    ready = torch.full((N // CHUNK,), 7, device="cuda", dtype=torch.int32)
    s = torch.cuda.current_stream().cuda_stream
    plan.launch_gated(dA.data_ptr(), dB.data_ptr(), dC.data_ptr(), s, ready.data_ptr(), 7, CHUNK, first)
    torch.cuda.synchronize()
    assert np.array_equal(_band(dC), want)


def test_gated_waits_for_a_late_chunk(fi, oracle):
    import torch
    from paper_2003_06324_b200 import _native as N_
    import ctypes as C
    plan, dA, dB, dC, want = _setup(fi, oracle, torch)
    late = 2
    o = late * CHUNK * K
    good = dB[o:o + CHUNK * K].clone()
    dB[o:o + CHUNK * K].fill_(float("nan"))       # what an early read would see
    ready = torch.tensor([1, 1, 0, 1], device="cuda", dtype=torch.int32)
    torch.cuda.synchronize()
    main, side = torch.cuda.current_stream(), torch.cuda.Stream()
    plan.launch_gated(dA.data_ptr(), dB.data_ptr(), dC.data_ptr(), main.cuda_stream, ready.data_ptr(), 1, CHUNK, 0)
    time.sleep(0.2)                                # the kernel is now spinning on chunk 2
    N_.check(N_.lib.fi_copy_async(C.c_void_p(dB.data_ptr() + 2 * o), C.c_void_p(good.data_ptr()),
                                  good.numel() * 2, C.c_void_p(side.cuda_stream)))
    N_.check(N_.lib.fi_stream_write_u32(C.c_void_p(ready.data_ptr() + 4 * late), C.c_uint32(1),
                                        C.c_void_p(side.cuda_stream)))
    torch.cuda.synchronize()
    assert np.array_equal(_band(dC), want)


def test_gated_missing_chunk_fails_instead_of_hanging():
    code = f"""
import sys; sys.path.insert(0, {ROOT!r})
import torch, paper_2003_06324_b200 as fi
plan = fi.Plan(fi.strategies.tc_strategy({M}, {N}, {K}))
a = torch.zeros({M * K}, device="cuda", dtype=torch.float16); b = torch.zeros({K * N}, device="cuda", dtype=torch.float16)
c = torch.empty({M * N}, device="cuda"); ready = torch.zeros({N // CHUNK}, device="cuda", dtype=torch.int32)
plan.launch_gated(a.data_ptr(), b.data_ptr(), c.data_ptr(), 0, ready.data_ptr(), 1, {CHUNK}, 0)
try:
    torch.cuda.synchronize()
    print("NO-ERROR")
except Exception as e:
    print("ERROR", type(e).__name__)
"""
    t0 = time.time()
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=120)
    assert "NO-ERROR" not in r.stdout, r.stdout + r.stderr
    assert time.time() - t0 < 100


def test_gated_rejects_chunks_that_split_a_tile(fi):
    import torch
    plan = fi.Plan(fi.strategies.tc_strategy(M, N, K))
    z = torch.zeros(16, device="cuda")
    with pytest.raises(fi.FiError):
        plan.launch_gated(z.data_ptr(), z.data_ptr(), z.data_ptr(), 0, z.data_ptr(), 1, 384, 0)
