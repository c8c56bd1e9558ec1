"""Host logic of the M/N-sharded multi-GPU driver (paper_2003_06324_b200/dist.py),
exercised with world_size 2 over gloo on CPU: every rank must end with its C
row band equal to A_r @ B, with B assembled from per-owner broadcast chunks."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2003_06324_b200.dist import make_shard, sharded_step


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, m, n, k, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(0)
    A = rng.integers(-3, 4, (m, k)).astype(np.float32)
    B = rng.integers(-3, 4, (k, n)).astype(np.float32)
    sh = make_shard(m, n, k, world, rank, tile_m=4, tile_n=4)
    a_local = torch.from_numpy(np.ascontiguousarray(A[rank * sh.m_local:(rank + 1) * sh.m_local].T).ravel())
    b_col = np.asfortranarray(B)  # col-major storage: column chunks are contiguous
    flat_b = torch.from_numpy(b_col.ravel(order="F").copy())
    b_local = flat_b[sh.b_chunk_offset(rank):sh.b_chunk_offset(rank) + sh.b_chunk_elems].clone()
    b_full = torch.zeros(k * n)
    c_local = torch.zeros(sh.c_elems)
    order = []

    def gemm(j, a, b, c):
        order.append(j)
        am = a.numpy().reshape(k, sh.m_local).T                    # col-major A_r
        bm = b.numpy().reshape(sh.n_chunk, k).T                    # col-major chunk
        c.copy_(torch.from_numpy(np.ascontiguousarray((am @ bm).T).ravel()))

    sharded_step(sh, a_local, b_local, b_full, c_local, gemm, dist)
    band = c_local.numpy().reshape(n, sh.m_local).T
    want = A[rank * sh.m_local:(rank + 1) * sh.m_local] @ B
    q.put((rank, bool(np.array_equal(band, want)), order, bool(torch.equal(b_full, flat_b))))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_sharded_allgather_gemm_gloo(world):
    m, n, k = 16, 24, 12
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, m, n, k, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, ok, order, gathered in res:
        assert ok and gathered
        assert order[0] == rank and sorted(order) == list(range(world))


def test_shard_geometry():
    sh = make_shard(16384, 16384, 16384, 8, 3)
    assert sh.m_local == 2048 and sh.n_chunk == 2048
    assert sh.b_chunk_offset(2) == 2 * 16384 * 2048
    assert sh.c_chunk_offset(1) == 2048 * 2048
    assert sh.order()[0] == 3
    with pytest.raises(ValueError):
        make_shard(1000, 1000, 64, 8, 0)


def _ipc_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2003_06324_b200.dist import PeerGather
    sh = make_shard(16, 24, 12, world, rank, tile_m=4, tile_n=4)
    try:
        PeerGather(sh, torch.zeros(12 * 24), dist)  # host memory: the export fails on every rank
        q.put((rank, "no error"))
    except RuntimeError as e:
        q.put((rank, str(e)))
    dist.destroy_process_group()


def test_peer_gather_failure_is_collective():
    """A rank whose CUDA IPC export fails must not strand its peers inside the
    handle exchange: every rank raises, so bench.py can agree on the NCCL
    fallback."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ipc_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert sorted(res) == [0, 1]
    assert all("fi_ipc_export failed" in v for v in res.values()), res


def _handshake_worker(rank, world, port, path, steps, q):
    import time
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2003_06324_b200.dist import _publish_own_chunk
    sh = make_shard(8, 8, 4, world, rank, tile_m=4, tile_n=4)
    # one shared gathered-B buffer stands in for the IPC-mapped peer buffers:
    # each rank writes only its own slot, peers read it in place
    b_full = torch.from_file(path, shared=True, size=sh.k * sh.n)
    seen = []
    for step in range(1, steps + 1):
        _publish_own_chunk(sh, torch.full((sh.b_chunk_elems,), float(10 * step + rank)), b_full, dist)
        peer = (rank + 1) % world
        if rank == 1:
            time.sleep(0.3)  # a slow reader of rank 0's slot
        o = sh.b_chunk_offset(peer)
        seen.append(float(b_full[o:o + sh.b_chunk_elems].max()))
    q.put((rank, seen))
    dist.destroy_process_group()


def test_own_chunk_publish_waits_for_slow_readers(tmp_path):
    """A peer still reading my slot for step t must see step t's chunk, not
    step t+1's (the own-slot write waits for every rank's previous reads)."""
    world, steps = 2, 3
    path = str(tmp_path / "b_full.bin")
    torch.zeros(8 * 4).numpy().tofile(path)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_handshake_worker, args=(r, world, port, path, steps, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    for rank in range(world):
        peer = (rank + 1) % world
        assert res[rank] == [float(10 * s + peer) for s in range(1, steps + 1)], res
