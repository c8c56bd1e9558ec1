"""run_host e2e (pinned fp32 host buffers, host snapping on) for the C2/C3 plans
under several host-pipeline shapes, interleaved in one process: blocked with
4 KiB / 8 KiB / whole-column C lines (FI_HOST_MIN_LINE), and column panels x2/x4/x8.
Median wall time per call over 3 interleaved rounds of 9 calls, then one traced
call per setting."""
import os, statistics, sys, time
sys.path.insert(0, ".")
import torch
import paper_2003_06324_b200 as fi

SETTINGS = {
    "blocked(default)": {},
    "blocked min_line 2048": {"FI_HOST_MIN_LINE": "2048"},
    "blocked min_line 4096": {"FI_HOST_MIN_LINE": "4096"},
    "blocked 8MiB panels": {"FI_HOST_PANEL_MB": "8"},
    "panels x2": {"FI_HOST_PIPELINE": "panels", "FI_HOST_PANELS": "2"},
    "panels x4": {"FI_HOST_PIPELINE": "panels", "FI_HOST_PANELS": "4"},
    "panels x8": {"FI_HOST_PIPELINE": "panels", "FI_HOST_PANELS": "8"},
    "blocked piece16": {"FI_HOST_PIECE_MB": "16"},
    "blocked piece32": {"FI_HOST_PIECE_MB": "32"},
    "blocked piece16 skip0": {"FI_HOST_PIECE_MB": "16", "FI_HOST_SNAP_SKIP": "0"},
    "blocked 8MiB panels piece16": {"FI_HOST_PANEL_MB": "8", "FI_HOST_PIECE_MB": "16"},
    "blocked 32MiB panels piece16": {"FI_HOST_PANEL_MB": "32", "FI_HOST_PIECE_MB": "16"},
    "panels x4 piece16": {"FI_HOST_PIPELINE": "panels", "FI_HOST_PANELS": "4", "FI_HOST_PIECE_MB": "16"},
    "panels x8 piece16": {"FI_HOST_PIPELINE": "panels", "FI_HOST_PANELS": "8", "FI_HOST_PIECE_MB": "16"},
}
if len(sys.argv) > 1:
    SETTINGS = {k: v for k, v in SETTINGS.items() if any(a == k for a in sys.argv[1:])}
KEYS = sorted({k for v in SETTINGS.values() for k in v} | {"FI_HOST_PIPELINE_TRACE"})


def apply(env):
    for k in KEYS:
        os.environ.pop(k, None)
    os.environ.update(env)


for name, strat, (m, n, k) in [("c2", fi.strategies.c2_strategy(), (4096, 4096, 4096)),
                               ("c3", fi.strategies.c3_strategy(), (1024, 1024, 32768))]:
    plan = fi.Plan(strat)
    hA = torch.empty((k, m), dtype=torch.float32, pin_memory=True)
    hB = torch.empty((n, k), dtype=torch.float32, pin_memory=True)
    hC = torch.empty((n, m), dtype=torch.float32, pin_memory=True)
    hA.copy_(torch.rand((k, m)) * 2 - 1)
    hB.copy_(torch.rand((n, k)) * 2 - 1)
    times = {s: [] for s in SETTINGS}
    ref = None
    for rnd in range(3):
        for s, env in SETTINGS.items():
            apply(env)
            for _ in range(2):
                plan.run_host_ptr(hA.data_ptr(), hB.data_ptr(), hC.data_ptr())
            if ref is None:
                ref = hC.clone()
            # sub-GEMM schedules (stream-K slices) differ per blocking: same up to rounding
            assert (hC - ref).abs().max().item() < 1e-3, s
            for _ in range(9):
                t = time.perf_counter()
                plan.run_host_ptr(hA.data_ptr(), hB.data_ptr(), hC.data_ptr())
                times[s].append((time.perf_counter() - t) * 1e3)
    for s in SETTINGS:
        ts = times[s]
        print(f"{name} {s:24s} median {statistics.median(ts):.3f} ms  min {min(ts):.3f}", flush=True)
    for s, env in SETTINGS.items():
        apply(dict(env, FI_HOST_PIPELINE_TRACE="1"))
        print(f"trace {name} {s}:", file=sys.stderr, flush=True)
        plan.run_host_ptr(hA.data_ptr(), hB.data_ptr(), hC.data_ptr())
        sys.stderr.flush()
    apply({})
