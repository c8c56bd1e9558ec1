#!/usr/bin/env python3
"""Benchmark: GEMM TFLOP/s of the Fireiron tensor-core strategy on B200.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workloads (BASELINE.json configs):
  N = 1  -> configs[1]: 4096^3, f16 in / f32 acc, the paper's staged strategy
            with MMA leaves lowered to tcgen05/TMEM (strategies.c2_strategy).
  N > 1  -> configs[4]: 16384^3 bf16 sharded by M/N output blocks across the N
            GPUs, B all-gathered over NVLink (NCCL broadcasts overlapped with
            the chunk GEMMs), strong scaling (total work fixed).
  --workload c3|c5|c2 overrides (c3: 1024x1024x32768 split-K).

A step = one execution of the strategy over the whole problem. `value` is
device-timed (CUDA events on the launch stream, inputs resident in HBM, L2
flushed by a 512 MiB write before every timed step, max over ranks). `e2e` is
the same metric through the reference-facing C ABI fi_plan_run_host with
pinned fp32 host matrices: H2D copies, grid snapping, the GEMM and the D2H of C
are all inside the timed region. The reference arm (--impl reference) times
the reference CPU simulator (oracle/_ref: the unmodified anvil headers built
in place) on the paper's tensor-core (WMMA) strategy for the same problem, on
a bounded sample of CTA blocks over all host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "GEMM TFLOP/s (fp16 in/fp32 acc) and % of B200 tensor peak at 1/2/4/8 GPUs"
UNIT = "TFLOP/s"
L2_FLUSH_BYTES = 512 << 20
DATA = "synthetic (uniform [-1,1) matrices; no dataset)"


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return {"tflops": p["bf16_tflops"], "tflops_sustained": p.get("bf16_tflops_sustained"),
                "hbm": p["hbm_gbs"], "src": "measured"}
    except Exception:
        return {"tflops": 1590.0, "tflops_sustained": 1400.0, "hbm": 6650.0, "src": "fallback"}


def workload_of(args, world):
    w = args.workload
    if w == "auto":
        w = "c2" if world == 1 else "c5"
    if w == "c2":
        return dict(name="c2_4096^3_f16_f32acc_tcgen05_pair256x256", m=4096, n=4096, k=4096, ab="f16")
    if w == "c3":
        return dict(name="c3_1024x1024x32768_f16_splitk4_pair256x256", m=1024, n=1024, k=32768, ab="f16")
    if w == "c5":
        return dict(name="c5_16384^3_bf16_sharded_MN_allgatherB", m=16384, n=16384, k=16384, ab="bf16")
    raise SystemExit(f"unknown workload {w}")


def problem_config(wl, world):
    """The `config` both arms print (identical, so the driver can pair them):
    the problem only. Each arm's implementation details go under `impl_config`."""
    cfg = {"workload": wl["name"], "m": wl["m"], "n": wl["n"], "k": wl["k"],
           "ab_type": wl["ab"], "c_type": "f32", "layout": "col-major A, B, C (Fireiron default)",
           "inputs": "synthetic uniform [-1,1), snapped to the A/B type",
           "l2": "GPU arm: flushed (512 MiB write) before every timed step"}
    if world > 1:
        cfg["parallelism"] = f"mn-shard{world}"
    return cfg


def strategy_for(fi, wl, m, n, k):
    if wl["name"].startswith("c3"):
        return fi.strategies.c3_strategy()
    if wl["name"].startswith("c5"):
        return fi.strategies.c5_strategy(m, n, k)  # per-shard shape under torchrun
    return fi.strategies.tc_strategy(m, n, k, ab=wl["ab"], pair=True, tile_n=256)


# ------------------------------------------------------------------ clocks
def gpu_local_affinity(device_index):
    """Restrict this process to the CPUs NVML reports as local to the GPU (its
    NUMA node), so pinned host buffers allocated next are first-touched there
    and the copy engines do not cross the socket link. Returns the previous
    affinity to restore, or None when NVML / affinity is unavailable."""
    try:
        import pynvml
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
        ncpu = os.cpu_count() or 1
        words = pynvml.nvmlDeviceGetCpuAffinity(h, (ncpu + 63) // 64)
        cpus = {w * 64 + b for w, word in enumerate(words) for b in range(64) if (word >> b) & 1 and w * 64 + b < ncpu}
        prev = os.sched_getaffinity(0)
        if cpus and cpus != prev:
            os.sched_setaffinity(0, cpus & prev or cpus)
            return prev
    except Exception:
        pass
    return None


class ClockSampler:
    """Samples SM clock + throttle reasons (NVML) while the timed region runs."""
    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x2: "applications_clocks_setting"}

    def __init__(self, device_index=0, period=0.001):
        self.samples, self.reasons, self.period = [], set(), period
        self.power_w = []
        self.max_mhz = None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.power_w.append(self.nv.nvmlDeviceGetPowerUsage(self.h) / 1000.0)
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.nv:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        out = {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
               "reasons": sorted(self.reasons), "samples": len(self.samples)}
        if self.power_w:
            out["power_w_median"] = statistics.median(self.power_w)
            out["power_w_max"] = max(self.power_w)
        return out


# ------------------------------------------------------------------ CPU baseline (reference)
def cpu_reference_sample(fi, wl, blocks_per_thread=2, threads=None):
    """The reference simulator (oracle/_ref) on the paper's WMMA strategy for
    the same problem: `threads` host threads, each running blocks of the grid
    through anvil::detail::Machine; the rate is extrapolated per block."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle
    if not oracle.have_reference():
        return None
    threads = threads or os.cpu_count() or 1
    m, n, k = wl["m"], wl["n"], wl["k"]
    # past K = 4096 a block runs a 4096-deep slice of its K loop so that a step
    # stays a few seconds at 16384^3; the simulator is faster per FLOP on the
    # shallower slice (1.85x here: its working set fits the caches), so the
    # reported reference rate is an upper bound -- conservative for the ratio
    ks = min(k, 4096)
    script = fi.strategies.wmma_decomp(m, n, ks)
    blocks = blocks_per_thread * threads
    secs, grid = oracle.ref_time_blocks(script, 0, 0, 0, blocks, threads)
    flops_per_block = 2.0 * m * n * ks / grid
    rate = flops_per_block * blocks / secs / 1e12
    kdesc = f"full K={k}" if ks == k else f"a K={ks} slice of K={k}: an upper bound on the full-K rate"
    return {"value": rate, "unit": UNIT, "cores": threads, "kind": "reference",
            "sample": f"{blocks} of {grid} CTA blocks (128x128 tiles, {kdesc}) of the paper's WMMA strategy "
                      f"(PAPER.md:927-974) through anvil::detail::Machine on {threads} threads, {secs:.1f} s; "
                      f"extrapolated full-problem time {2.0*m*n*k/(rate*1e12):.0f} s",
            "seconds": secs}


def reference_arm(args, fi, rank, world):
    import torch.distributed as dist
    wl = workload_of(args, world)
    if rank != 0:
        if dist.is_initialized():
            dist.barrier()
        return
    threads = os.cpu_count() or 1
    vals = []
    for i in range(args.warmup + args.steps):
        r = cpu_reference_sample(fi, wl, blocks_per_thread=1, threads=threads)
        if r is None:
            print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref (reference build) missing"}))
            return
        if i >= args.warmup:
            vals.append(r)
    v = statistics.median([x["value"] for x in vals])
    secs = sum(x["seconds"] for x in vals)
    flops = 2.0 * wl["m"] * wl["n"] * wl["k"]
    line = {"metric": METRIC, "value": v, "unit": UNIT, "impl": "reference", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": secs / len(vals) * 1e3, "higher_is_better": True,
            "scaling": "strong" if world > 1 else "weak", "vs_baseline": None, "dtype": wl["ab"] + " in / f32 acc",
            "data": DATA,
            "config": problem_config(wl, world),
            "impl_config": {"engine": "reference CPU simulator (oracle/_ref: anvil::detail::Machine, unmodified "
                                      "headers built in place)",
                            "strategy": "paper WMMA decomposition (GL->SH->FR, WMMA leaves; f16 inputs, fp32 "
                                        "accumulate) on the anvil CPU model",
                            "inputs": "splitmix64 uniform fills (the reference's own generator)",
                            "extrapolated_full_problem_s": flops / (v * 1e12)},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": "reference",
                             "sample": vals[-1]["sample"]},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    if dist.is_initialized():
        dist.barrier()


# ------------------------------------------------------------------ our arm
def profile_traffic(workload_name):
    """Per-launch DRAM bytes of the dominant kernel from the committed ncu summary."""
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return d.get(workload_name, {}).get("dram_bytes_per_launch")
    except Exception:
        return None


def ours_single(args, fi, torch):
    wl = workload_of(args, 1)
    m, n, k = wl["m"], wl["n"], wl["k"]
    plan = fi.Plan(strategy_for(fi, wl, m, n, k))
    assert plan.kind == "tcgen05"
    dt = torch.float16 if wl["ab"] == "f16" else torch.bfloat16
    dev = torch.device("cuda", 0)
    gen = torch.Generator(device=dev).manual_seed(1)
    # col-major A (M x K) and B (K x N): stored as (K, M) / (N, K) row-major tensors
    A = (torch.rand((k, m), device=dev, generator=gen) * 2 - 1).to(dt)
    B = (torch.rand((n, k), device=dev, generator=gen) * 2 - 1).to(dt)
    C = torch.empty((n, m), device=dev, dtype=torch.float32)
    flush = torch.empty(L2_FLUSH_BYTES // 4, device=dev, dtype=torch.float32)
    stream = torch.cuda.current_stream()
    sp = stream.cuda_stream
    flops = plan.flops

    for _ in range(args.warmup):
        plan.launch(A.data_ptr(), B.data_ptr(), C.data_ptr(), sp)
    torch.cuda.synchronize()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    with ClockSampler(0) as clocks:
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for i in range(args.steps):
            flush.zero_()                      # L2 flush (untimed by the events)
            starts[i].record(stream)
            plan.launch(A.data_ptr(), B.data_ptr(), C.data_ptr(), sp)
            ends[i].record(stream)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
    ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    ms_mean = statistics.mean(ms)
    value = flops / (ms_mean * 1e-3) / 1e12
    # sanity: result finite
    assert torch.isfinite(C[:, :64]).all().item()

    # ---- e2e through the C ABI with pinned fp32 host buffers
    import numpy as np
    saved_affinity = gpu_local_affinity(0)  # host buffers on the GPU's NUMA node
    hA = torch.empty((k, m), dtype=torch.float32, pin_memory=True)
    hB = torch.empty((n, k), dtype=torch.float32, pin_memory=True)
    hC = torch.empty((n, m), dtype=torch.float32, pin_memory=True)
    hA.copy_(A.float().cpu())
    hB.copy_(B.float().cpu())
    e2e_steps = max(3, min(args.steps, 10))
    for _ in range(2):
        plan.run_host_ptr(hA.data_ptr(), hB.data_ptr(), hC.data_ptr())
    e2e_t = []
    for _ in range(e2e_steps):  # each call is synchronous: H2D, snap, GEMM panels, D2H
        t0 = time.perf_counter()
        plan.run_host_ptr(hA.data_ptr(), hB.data_ptr(), hC.data_ptr())
        e2e_t.append(time.perf_counter() - t0)
    e2e_s = statistics.median(e2e_t)  # a host hiccup in one call does not set the number
    h2d_bytes, d2h_bytes = plan.host_bytes()  # counted by the runtime from the copies it issued
    assert np.isfinite(hC[:4, :4].numpy()).all()
    if saved_affinity is not None:
        os.sched_setaffinity(0, saved_affinity)

    peaks = load_peaks()
    roof = {"bound": "tensor", "achieved": value, "peak": peaks["tflops"], "unit": UNIT,
            "frac": value / peaks["tflops"], "traffic": profile_traffic(wl["name"]),
            "peak_source": f"{peaks['src']} bf16_tflops (burst; kernel timed alone)",
            "frac_of_sustained": value / peaks["tflops_sustained"] if peaks["tflops_sustained"] else None,
            "algorithmic_flops_per_launch": flops}
    cpu = None if args.no_cpu_baseline else cpu_reference_sample(fi, wl, blocks_per_thread=2)
    info = plan.info
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_mean, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": wl["ab"] + " in / f32 acc", "data": DATA,
            "config": problem_config(wl, 1),
            "impl_config": {"engine": "tcgen05 persistent GEMM (TMA -> SW128 smem ring -> tcgen05.mma -> TMEM)",
                            "tile": f"{info.tile_m}x{info.tile_n}",
                            "cta_group": info.cta_group, "split_k": info.split_k, "stages": info.stages,
                            "ctas": info.launch_ctas, "inputs": "torch uniform [-1,1) generated on the device",
                            "percent_of_peak": 100.0 * value / peaks["tflops"],
                            "ms_min": min(ms), "ms_median": statistics.median(ms), "wall_s": wall},
            "roofline": roof,
            "cpu_baseline": cpu,
            "e2e": {"value": flops / e2e_s / 1e12, "unit": UNIT,
                    "h2d_bytes_per_step": h2d_bytes, "d2h_bytes_per_step": d2h_bytes,
                    "host_input_bytes_per_step": 4 * (m * k + k * n),
                    "ms_per_step": e2e_s * 1e3, "ms_mean": statistics.mean(e2e_t) * 1e3,
                    "steps": e2e_steps, "timing": "median of per-call wall times",
                    "api": "fi_plan_run_host (pinned fp32 host buffers; input pieces snapped to f16 by host "
                           "threads and uploaded as 2-byte elements, the first piece uploaded fp32 and snapped "
                           "on the device)"},
            "gpu_launches": args.steps,
            "clocks": clocks.summary()}
    print(json.dumps(line), flush=True)


def ours_multi(args, fi, torch, rank, world):
    import torch.distributed as dist
    from paper_2003_06324_b200.dist import (PeerGather, make_shard, sharded_step, sharded_step_direct,
                                            sharded_step_fused, sharded_step_peer)
    wl = workload_of(args, world)
    m, n, k = wl["m"], wl["n"], wl["k"]
    shard = make_shard(m, n, k, world, rank)
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", rank)) % torch.cuda.device_count())
    torch.cuda.set_device(dev)
    dt = torch.float16 if wl["ab"] == "f16" else torch.bfloat16
    plan = fi.Plan(strategy_for(fi, wl, shard.m_local, shard.n_chunk, k), device=dev.index)
    gen = torch.Generator(device=dev).manual_seed(1 + rank)
    A = (torch.rand(shard.a_elems, device=dev, generator=gen) * 2 - 1).to(dt)
    Bl = (torch.rand(shard.b_chunk_elems, device=dev, generator=gen) * 2 - 1).to(dt)
    Bf = torch.empty(k * n, device=dev, dtype=dt)
    C = torch.empty(shard.c_elems, device=dev, dtype=torch.float32)
    flush = torch.empty(L2_FLUSH_BYTES // 4, device=dev, dtype=torch.float32)
    stream = torch.cuda.current_stream()

    def gemm(j, a, b, c):
        plan.launch(a.data_ptr(), b.data_ptr(), c.data_ptr(), stream.cuda_stream)

    # B transport: copy-engine pulls releasing per-chunk flags to ONE gated
    # persistent GEMM over the whole band (default, "fused"), copy-engine pulls
    # with one GEMM per chunk ("peer"), NCCL per-owner broadcasts ("nccl"), or
    # direct TMA reads of the owners' buffers inside the chunk GEMMs ("direct")
    transport = os.environ.get("FI_DIST_TRANSPORT", "fused")
    pg = None
    if transport in ("peer", "direct", "fused"):
        # every rank must map every peer's buffer; if any rank cannot (no IPC /
        # P2P between these GPUs), all ranks fall back to NCCL broadcasts
        err = None
        try:
            pg = PeerGather(shard, Bf, dist)
        except Exception as e:  # noqa: BLE001 - reported below, decided collectively
            err = e
        ok = torch.tensor([0 if err else 1], device=dev, dtype=torch.int32)
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        if ok.item() == 0:
            if pg is not None:
                pg.close()
                pg = None
            if rank == 0:
                print(f"bench: CUDA IPC transport unavailable ({err or 'on a peer rank'}); using NCCL broadcasts",
                      file=sys.stderr)
            transport = "nccl"

    def gemm_ptr(j, a, bptr, c):
        plan.launch(a.data_ptr(), bptr, c.data_ptr(), stream.cuda_stream)

    band_plan = fi.Plan(strategy_for(fi, wl, shard.m_local, n, k), device=dev.index) if transport == "fused" else None
    ready = torch.zeros(world, device=dev, dtype=torch.int32)
    epoch = [0]

    def step():
        if transport == "fused":
            epoch[0] += 1
            sharded_step_fused(shard, A, Bl, Bf, C, band_plan, dist, pg, ready, epoch[0])
        elif transport == "direct":
            sharded_step_direct(shard, A, Bl, Bf, C, gemm_ptr, dist, pg)
        elif pg is not None:
            sharded_step_peer(shard, A, Bl, Bf, C, gemm, dist, pg)
        else:
            sharded_step(shard, A, Bl, Bf, C, gemm, dist)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ms_steps = []
    with ClockSampler(dev.index) as clocks:
        for i in range(args.steps):
            flush.zero_()
            torch.cuda.synchronize()
            dist.barrier()
            e0.record(stream)
            step()
            e1.record(stream)
            torch.cuda.synchronize()
            ms_steps.append(e0.elapsed_time(e1))
    t = torch.tensor([statistics.mean(ms_steps)], device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = t.item()
    flops = 2.0 * m * n * k
    value = flops / (ms * 1e-3) / 1e12
    # e2e: every step also moves this rank's operand shards up from pinned host
    # memory (A row band, own B chunk, in the compute type) and its C band down
    hA = torch.empty(shard.a_elems, dtype=dt, pin_memory=True)
    hB = torch.empty(shard.b_chunk_elems, dtype=dt, pin_memory=True)
    hC = torch.empty(shard.c_elems, dtype=torch.float32, pin_memory=True)
    hA.copy_(A)
    hB.copy_(Bl)
    e2e_steps = max(2, min(args.steps, 5))
    e2e_ms = []
    for i in range(e2e_steps + 1):
        torch.cuda.synchronize()
        dist.barrier()
        t0 = time.perf_counter()
        A.copy_(hA, non_blocking=True)
        Bl.copy_(hB, non_blocking=True)
        step()
        hC.copy_(C, non_blocking=True)
        torch.cuda.synchronize()
        if i:  # the first pass warms the pinned-copy path
            e2e_ms.append((time.perf_counter() - t0) * 1e3)
    te = torch.tensor([statistics.mean(e2e_ms)], device=dev)
    dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_ms_step = te.item()
    if rank == 0:
        peaks = load_peaks()
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": wl["ab"] + " in / f32 acc", "data": DATA,
                "config": problem_config(wl, world),
                "impl_config": {"shard": f"{shard.m_local}x{n} rows of C per GPU, B chunks of {shard.n_chunk} columns",
                           "comm": {"fused": "copy-engine pulls of B chunks from IPC-mapped peer buffers in "
                                             "rotated order, each releasing a ready flag to ONE gated persistent "
                                             "GEMM over the whole C band (tiles wait per chunk)",
                                    "peer": "copy-engine pulls of B chunks from IPC-mapped peer buffers, "
                                            "overlapped with chunk GEMMs",
                                    "direct": "chunk GEMMs read B over NVLink from the owners' IPC-mapped buffers",
                                    }.get(transport, "NCCL per-owner broadcasts of B chunks, overlapped with chunk GEMMs"),
                           "percent_of_peak": 100.0 * value / (world * peaks["tflops"])},
                "roofline": {"bound": "tensor", "achieved": value / world, "peak": peaks["tflops"], "unit": UNIT,
                             "frac": value / world / peaks["tflops"], "traffic": None,
                             "peak_source": f"{peaks['src']} bf16_tflops per GPU"},
                "cpu_baseline": None,
                "e2e": {"value": flops / (e2e_ms_step * 1e-3) / 1e12, "unit": UNIT,
                        "h2d_bytes_per_step": world * (hA.numel() + hB.numel()) * hA.element_size(),
                        "d2h_bytes_per_step": world * hC.numel() * 4, "ms_per_step": e2e_ms_step,
                        "steps": e2e_steps,
                        "api": "dist.sharded_step* per rank with pinned host shards (A band, own B chunk "
                               "up; C band down), wall clock, max over ranks"},
                # fused: one GEMM per rank per step; else one chunk GEMM per B chunk per rank per step
                "gpu_launches": args.steps * world * (1 if transport == "fused" else world),
                "clocks": clocks.summary()}
        print(json.dumps(line), flush=True)
    if pg is not None:
        dist.barrier()
        pg.close()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="auto", choices=["auto", "c2", "c3", "c5"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    import torch
    import torch.distributed as dist
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if args.impl == "ours":
            torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)) % torch.cuda.device_count())
            # FI_DIST_BACKEND=gloo runs the sharded driver with several ranks on one
            # GPU (logic check only; the measured configuration is NCCL, 1 rank/GPU)
            dist.init_process_group(os.environ.get("FI_DIST_BACKEND", "nccl"))
        else:
            dist.init_process_group("gloo")
    import paper_2003_06324_b200 as fi

    if args.impl == "reference":
        reference_arm(args, fi, rank, world)
    elif world == 1:
        ours_single(args, fi, torch)
    else:
        ours_multi(args, fi, torch, rank, world)
    if dist.is_initialized():
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
