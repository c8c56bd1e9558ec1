"""The M/N-sharded multi-GPU driver with the real tcgen05 kernels: two ranks
share the one GPU of this environment (gloo for the process group), each
computes its C row band with the B chunks gathered either by per-owner
broadcasts, by copy-engine pulls from the peers' IPC-mapped buffers
(PeerGather), or not at all (the chunk GEMM's TMA reads the owner's buffer
through its IPC mapping), overlapped with chunk GEMMs -- or, fused (the GPU
driver's default), by sequential copy-engine pulls that release per-chunk
ready flags to ONE gated persistent GEMM over the whole band. Integer
inputs: every rank's band must equal the fp64 oracle exactly, two steps in a
row (the second re-gathers into buffers the first step read)."""
import os
import socket
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q, transport="broadcast"):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import torch
    import torch.distributed as dist
    import oracle
    import paper_2003_06324_b200 as fi
    from paper_2003_06324_b200.dist import (PeerGather, make_shard, sharded_step, sharded_step_direct,
                                            sharded_step_fused, sharded_step_peer)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    m, n, k = 1024, 1024, 512
    sh = make_shard(m, n, k, world, rank)
    a = oracle.fill(m, k, 5, True)
    b = oracle.fill(k, n, 6, True)
    dev = torch.device("cuda", 0)
    # col-major storage: A_r band (m_local x k), B chunk (k x n/g), C band (m_local x n)
    a_r = torch.from_numpy(np.ascontiguousarray(a[rank * sh.m_local:(rank + 1) * sh.m_local].T).ravel()).to(dev).half()
    b_cm = np.asfortranarray(b).ravel(order="F")
    off = sh.b_chunk_offset(rank)
    b_l = torch.from_numpy(b_cm[off:off + sh.b_chunk_elems].copy()).to(dev).half()
    b_f = torch.empty(k * n, device=dev, dtype=torch.float16)
    c_r = torch.full((sh.c_elems,), float("nan"), device=dev)
    plan = fi.Plan(fi.strategies.tc_strategy(sh.m_local, sh.n_chunk, k))
    stream = torch.cuda.current_stream()

    def gemm(j, aa, bb, cc):
        plan.launch(aa.data_ptr(), bb.data_ptr(), cc.data_ptr(), stream.cuda_stream)

    want = oracle.gemm_f64(a[rank * sh.m_local:(rank + 1) * sh.m_local], b)
    ok = True
    pg = PeerGather(sh, b_f, dist) if transport in ("peer", "direct", "fused") else None
    band_plan = fi.Plan(fi.strategies.tc_strategy(sh.m_local, n, k)) if transport == "fused" else None
    ready = torch.zeros(2, device=dev, dtype=torch.int32)

    def gemm_ptr(j, aa, bptr, cc):
        plan.launch(aa.data_ptr(), bptr, cc.data_ptr(), stream.cuda_stream)

    for step in range(2):
        c_r.fill_(float("nan"))
        if transport == "fused":
            sharded_step_fused(sh, a_r, b_l, b_f, c_r, band_plan, dist, pg, ready, step + 1)
        elif transport == "direct":
            sharded_step_direct(sh, a_r, b_l, b_f, c_r, gemm_ptr, dist, pg)
        elif pg is not None:
            sharded_step_peer(sh, a_r, b_l, b_f, c_r, gemm, dist, pg)
        else:
            sharded_step(sh, a_r, b_l, b_f, c_r, gemm, dist)
        torch.cuda.synchronize()
        band = c_r.cpu().numpy().reshape(n, sh.m_local).T
        ok = ok and bool(np.array_equal(band, want))
    dist.barrier()
    if pg is not None:
        pg.close()
    q.put((rank, ok))
    dist.destroy_process_group()


@pytest.mark.parametrize("transport", ["broadcast", "peer", "direct", "fused"])
def test_sharded_gemm_two_ranks_one_gpu(transport):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q, transport)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {0: True, 1: True}
