"""Pipelined run_host timeline (FI_HOST_PIPELINE_TRACE) for the C2 plan, and wall time per call."""
import os, sys, time
sys.path.insert(0, ".")
import torch
import paper_2003_06324_b200 as fi
m = n = k = 4096
plan = fi.Plan(fi.strategies.c2_strategy())
hA = torch.rand((k, m), dtype=torch.float32).pin_memory()
hB = torch.rand((n, k), dtype=torch.float32).pin_memory()
hC = torch.empty((n, m), dtype=torch.float32).pin_memory()
for mode in ["1", "panels", "0"]:
    os.environ["FI_HOST_PIPELINE"] = mode
    for _ in range(2): plan.run_host_ptr(hA.data_ptr(), hB.data_ptr(), hC.data_ptr())
    t = time.perf_counter()
    for _ in range(5): plan.run_host_ptr(hA.data_ptr(), hB.data_ptr(), hC.data_ptr())
    print(f"pipeline={mode}: {(time.perf_counter() - t) / 5 * 1e3:.3f} ms per run_host", flush=True)
os.environ["FI_HOST_PIPELINE_TRACE"] = "1"
for mode in ["1", "panels"]:
    os.environ["FI_HOST_PIPELINE"] = mode
    for _ in range(2): plan.run_host_ptr(hA.data_ptr(), hB.data_ptr(), hC.data_ptr())
del os.environ["FI_HOST_PIPELINE_TRACE"]
os.environ["FI_HOST_PIPELINE"] = "1"
for mb in ["4", "16"]:
    os.environ["FI_HOST_PANEL_MB"] = mb
    for _ in range(2): plan.run_host_ptr(hA.data_ptr(), hB.data_ptr(), hC.data_ptr())
    t = time.perf_counter()
    for _ in range(5): plan.run_host_ptr(hA.data_ptr(), hB.data_ptr(), hC.data_ptr())
    print(f"blocked panel {mb} MiB: {(time.perf_counter() - t) / 5 * 1e3:.3f} ms per run_host", flush=True)
