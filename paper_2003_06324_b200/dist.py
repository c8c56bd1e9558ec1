"""Multi-GPU execution of a Fireiron GEMM strategy, sharded by M/N output
blocks across the GPUs of one node (BASELINE.json configs[4]).

Partitioning (1-D over N): with g ranks, rank r owns
  A_r  = A[r*M/g:(r+1)*M/g, :]     (row shard, never communicated)
  B_r  = B[:, r*N/g:(r+1)*N/g]     (column shard, contiguous in col-major B)
and computes the row band C_r = A_r * B (M/g x N). B is all-gathered over
NVLink, by default with copy-engine pulls from every peer's buffer mapped
through CUDA IPC (PeerGather, no SM time), or with NCCL as g per-owner
broadcasts (sharded_step); the GEMM of column chunk j starts as soon as chunk
j has arrived, so the transfer overlaps the tensor-core work chunk by chunk
(the own chunk needs no communication and runs first).

Each chunk GEMM is the same tcgen05 strategy on the (M/g) x (N/g) x K shard
shape; column chunks of col-major B and C are contiguous, so chunk j is a
plain pointer offset.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, List


@dataclass(frozen=True)
class Shard:
    rank: int
    world: int
    m: int           # global
    n: int
    k: int
    m_local: int     # rows of A / C owned by this rank
    n_chunk: int     # columns per B chunk (one per owner rank)

    @property
    def a_elems(self) -> int:
        return self.m_local * self.k

    @property
    def b_chunk_elems(self) -> int:
        return self.k * self.n_chunk

    @property
    def c_elems(self) -> int:
        return self.m_local * self.n

    def b_chunk_offset(self, j: int) -> int:
        """Element offset of owner j's chunk in the gathered col-major B (K x N)."""
        return j * self.b_chunk_elems

    def c_chunk_offset(self, j: int) -> int:
        """Element offset of column chunk j in the col-major C band (M/g x N)."""
        return j * self.m_local * self.n_chunk

    def order(self) -> List[int]:
        """Chunk compute order: own chunk first, then the others rotated (rank
        r pulls from r+1 first, so no owner is every rank's first source; the
        fused GEMM's tile raster starts at chunk r and wraps the same way)."""
        return [(self.rank + i) % self.world for i in range(self.world)]


def make_shard(m: int, n: int, k: int, world: int, rank: int, tile_m: int = 256, tile_n: int = 256) -> Shard:
    if m % world or n % world:
        raise ValueError(f"{m}x{n} does not split over {world} ranks")
    ml, nc = m // world, n // world
    if ml % tile_m or nc % tile_n:
        raise ValueError(f"shard {ml}x{nc} is not a multiple of the {tile_m}x{tile_n} block tile")
    return Shard(rank, world, m, n, k, ml, nc)


def sharded_step(shard: Shard, a_local, b_local, b_full, c_local, gemm: Callable, dist, stream_wait=None):
    """One step: broadcast every owner's B chunk into b_full (async, NCCL
    queues them in order) and run the chunk GEMMs as chunks arrive.

    gemm(j, a_local, b_chunk_view, c_chunk_view) launches chunk j.
    b_full is a flat buffer of K*N elements; b_local is this rank's chunk.
    Works for any torch.distributed backend (nccl on GPUs, gloo in tests)."""
    me = shard.rank
    off = shard.b_chunk_offset(me)
    b_full[off:off + shard.b_chunk_elems].copy_(b_local)
    works = {}
    for j in range(shard.world):
        o = shard.b_chunk_offset(j)
        works[j] = dist.broadcast(b_full[o:o + shard.b_chunk_elems], src=j, async_op=True)
    for j in shard.order():
        if j != me:
            works[j].wait()  # stream-ordered on NCCL: the GEMM waits only for chunk j
        bo, co = shard.b_chunk_offset(j), shard.c_chunk_offset(j)
        gemm(j, a_local, b_full[bo:bo + shard.b_chunk_elems],
             c_local[co:co + shard.m_local * shard.n_chunk])
    works[me].wait()


class PeerGather:
    """B all-gather over CUDA IPC and copy engines (the default transport of the
    GPU driver): every rank exports its gathered-B buffer once, maps every
    peer's buffer, and each step pulls the peers' chunks with DMA on one stream
    per peer. The transfers use NVLink/NVSwitch copy engines and no SM time, so
    they overlap the persistent tcgen05 GEMM, which keeps all SMs (NCCL's
    broadcast kernels would take SMs from it). Chunk GEMM j waits only for the
    event of chunk j."""

    def __init__(self, shard: Shard, b_full, dist):
        import ctypes as C
        import torch
        from . import _native as N
        self.shard, self.N, self.C = shard, N, C
        h = (C.c_char * 64)()
        off = C.c_int64()
        mine = None
        if N.lib.fi_ipc_export(C.c_void_p(b_full.data_ptr()), h, C.byref(off)) == 0:
            mine = (bytes(h), off.value)
        # the exchange is reached by every rank even when an export failed, so a
        # failure raises on every rank instead of leaving peers in the collective
        objs = [None] * shard.world
        dist.all_gather_object(objs, mine)
        self.peer = {}
        if any(o is None for o in objs):
            raise RuntimeError("fi_ipc_export failed on rank(s) %s" % [j for j, o in enumerate(objs) if o is None])
        for j, (hb, o) in enumerate(objs):
            if j == shard.rank:
                continue
            p = C.c_void_p()
            N.check(N.lib.fi_ipc_open(hb, o, C.byref(p)))
            self.peer[j] = (p.value, o)
        dev = b_full.device
        self.streams = {j: torch.cuda.Stream(device=dev) for j in self.peer}
        # sharded_step_fused: pulls in rotated order, dealt round-robin over a few
        # streams (FI_DIST_PULL_STREAMS, default 2) so more than one copy engine
        # can run while the chunks still land roughly in compute order
        import os
        n = max(1, int(os.environ.get("FI_DIST_PULL_STREAMS", "2")))
        self.seq_streams = [torch.cuda.Stream(device=dev) for _ in range(n)]
        self.events = {j: torch.cuda.Event() for j in self.peer}
        self.esize = b_full.element_size()

    def pull(self, j: int, b_full):
        """Issue the copy of owner j's chunk into b_full on j's stream; returns its event."""
        import torch
        p, _ = self.peer[j]
        o = self.shard.b_chunk_offset(j) * self.esize
        s = self.streams[j]
        self.N.check(self.N.lib.fi_copy_async(self.C.c_void_p(b_full.data_ptr() + o), self.C.c_void_p(p + o),
                                              self.shard.b_chunk_elems * self.esize, self.C.c_void_p(s.cuda_stream)))
        self.events[j].record(s)
        return self.events[j]

    def close(self):
        for p, o in self.peer.values():
            self.N.lib.fi_ipc_close(self.C.c_void_p(p), o)
        self.peer = {}


def _publish_own_chunk(shard: Shard, b_local, b_full, dist):
    """Write this rank's chunk into its slot of b_full, which peers read
    directly (copy-engine pulls or TMA loads through their IPC mappings).

    Two handshakes: (1) before the write, every rank synchronises its stream --
    which holds all of its previous-step reads of peers' slots (pulls and GEMMs)
    -- and meets at a barrier, so no peer can still be reading the old contents
    of my slot; (2) after the write, synchronise and meet again, so every
    owner's chunk is in place before anyone reads it. A host barrier alone does
    not order a peer's in-flight device reads, hence the syncs."""
    import torch
    sync = torch.cuda.current_stream().synchronize if b_full.is_cuda else (lambda: None)
    sync()
    dist.barrier()
    off = shard.b_chunk_offset(shard.rank)
    b_full[off:off + shard.b_chunk_elems].copy_(b_local)
    sync()
    dist.barrier()


def sharded_step_peer(shard: Shard, a_local, b_local, b_full, c_local, gemm: Callable, dist, pg: PeerGather):
    """One step with copy-engine pulls: write my chunk into my gathered buffer
    (_publish_own_chunk: after every peer finished reading the previous step's,
    and in place on every rank before any pull), pull the peers' chunks in
    rotated order and run each chunk GEMM as soon as its chunk has landed."""
    import torch
    me = shard.rank
    _publish_own_chunk(shard, b_local, b_full, dist)
    cur = torch.cuda.current_stream()
    events = {j: pg.pull(j, b_full) for j in shard.order() if j != me}
    for j in shard.order():
        if j != me:
            cur.wait_event(events[j])
        bo, co = shard.b_chunk_offset(j), shard.c_chunk_offset(j)
        gemm(j, a_local, b_full[bo:bo + shard.b_chunk_elems],
             c_local[co:co + shard.m_local * shard.n_chunk])


def sharded_step_fused(shard: Shard, a_local, b_local, b_full, c_local, plan, dist, pg: PeerGather, ready,
                       epoch: int):
    """One step as ONE persistent GEMM over this rank's whole C band with the
    B all-gather fused in: copy engines pull the peers' chunks in rotated
    order, dealt over FI_DIST_PULL_STREAMS streams (default 2) that each copy
    sequentially -- so chunks land roughly in compute order instead of all at
    the end -- each copy followed by a stream-ordered write of its ready flag
    (fi_stream_write_u32: no SM needed, the GEMM holds them all); the GEMM starts on my own chunk and each tile's producer waits
    for its chunk's flag before its first TMA load (fi_plan_launch_gated).
    `plan` covers (m_local x N x K); `ready` is a device int32[world] buffer
    whose entries only ever increase (epoch = 1, 2, ... per step).
    b_local goes into this rank's slot of b_full through _publish_own_chunk,
    after every peer's pulls of the previous step completed (their streams
    wait for the pull streams at the end of each step).
    The epoch is a host value written by stream memops and passed to the
    launch, so a captured step would replay with a frozen epoch: run it
    eagerly (the GEMM's own stream-K epoch is device-side and graph-safe)."""
    import torch
    me = shard.rank
    cur = torch.cuda.current_stream()
    _publish_own_chunk(shard, b_local, b_full, dist)
    N, C = pg.N, pg.C
    rp = ready.data_ptr()
    N.check(N.lib.fi_stream_write_u32(C.c_void_p(rp + 4 * me), C.c_uint32(epoch), C.c_void_p(cur.cuda_stream)))
    for s in pg.seq_streams:
        s.wait_stream(cur)
    for i, j in enumerate(x for x in shard.order() if x != me):
        s = pg.seq_streams[i % len(pg.seq_streams)]
        p, _ = pg.peer[j]
        o = shard.b_chunk_offset(j) * pg.esize
        N.check(N.lib.fi_copy_async(C.c_void_p(b_full.data_ptr() + o), C.c_void_p(p + o),
                                    shard.b_chunk_elems * pg.esize, C.c_void_p(s.cuda_stream)))
        N.check(N.lib.fi_stream_write_u32(C.c_void_p(rp + 4 * j), C.c_uint32(epoch), C.c_void_p(s.cuda_stream)))
    plan.launch_gated(a_local.data_ptr(), b_full.data_ptr(), c_local.data_ptr(), cur.cuda_stream, rp, epoch,
                      shard.n_chunk, me)
    for s in pg.seq_streams:
        cur.wait_stream(s)  # the next step's barrier then also covers these pulls


def sharded_step_direct(shard: Shard, a_local, b_local, b_full, c_local, gemm_ptr: Callable, dist, pg: PeerGather):
    """One step with no gather at all: chunk GEMM j's TMA descriptors point at
    owner j's buffer through its IPC mapping, so B streams over NVLink tile by
    tile inside the GEMM (the transfer fused into the kernel's loads).
    gemm_ptr(j, a_local, b_ptr, c_chunk) launches chunk j on a raw B pointer.
    The peers' GEMMs of the previous step read my slot until their streams
    drain: _publish_own_chunk waits for that before overwriting it."""
    me = shard.rank
    _publish_own_chunk(shard, b_local, b_full, dist)
    for j in shard.order():
        bo, co = shard.b_chunk_offset(j), shard.c_chunk_offset(j)
        ptr = b_full.data_ptr() + bo * pg.esize if j == me else pg.peer[j][0] + bo * pg.esize
        gemm_ptr(j, a_local, ptr, c_local[co:co + shard.m_local * shard.n_chunk])
