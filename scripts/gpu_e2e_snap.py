"""run_host e2e with host snapping: median wall time per call for the C2/C3
plans under the environment this process was started with (FI_HOST_SNAP*,
FI_HOST_PANEL_MB), plus one traced call. Run once per configuration:
  FI_HOST_SNAP=0 python scripts/gpu_e2e_snap.py ; python scripts/gpu_e2e_snap.py"""
import os, statistics, sys, time
sys.path.insert(0, ".")
import torch
import paper_2003_06324_b200 as fi

tag = " ".join(f"{k}={v}" for k, v in sorted(os.environ.items()) if k.startswith("FI_HOST")) or "defaults"
for name, strat, (m, n, k) in [("c2", fi.strategies.c2_strategy(), (4096, 4096, 4096)),
                               ("c3", fi.strategies.c3_strategy(), (1024, 1024, 32768))]:
    plan = fi.Plan(strat)
    hA = torch.empty((k, m), dtype=torch.float32, pin_memory=True)
    hB = torch.empty((n, k), dtype=torch.float32, pin_memory=True)
    hC = torch.empty((n, m), dtype=torch.float32, pin_memory=True)
    hA.copy_(torch.rand((k, m)) * 2 - 1)
    hB.copy_(torch.rand((n, k)) * 2 - 1)
    for _ in range(3):
        plan.run_host_ptr(hA.data_ptr(), hB.data_ptr(), hC.data_ptr())
    ts = []
    for _ in range(15):
        t = time.perf_counter()
        plan.run_host_ptr(hA.data_ptr(), hB.data_ptr(), hC.data_ptr())
        ts.append((time.perf_counter() - t) * 1e3)
    print(f"{name} [{tag}]: median {statistics.median(ts):.3f} ms  min {min(ts):.3f}  max {max(ts):.3f}", flush=True)
    os.environ["FI_HOST_PIPELINE_TRACE"] = "1"
    plan.run_host_ptr(hA.data_ptr(), hB.data_ptr(), hC.data_ptr())
    del os.environ["FI_HOST_PIPELINE_TRACE"]
    sys.stderr.flush()
