"""run_host per call for the C5 plan (16384^3 bf16) across host-pipeline variants."""
import os, sys, time
sys.path.insert(0, ".")
import torch
import paper_2003_06324_b200 as fi
n = 16384
plan = fi.Plan(fi.strategies.c5_strategy())
hA = torch.rand((n, n), dtype=torch.float32).pin_memory()
hB = torch.rand((n, n), dtype=torch.float32).pin_memory()
hC = torch.empty((n, n), dtype=torch.float32).pin_memory()
KEYS = ("FI_HOST_PIPELINE", "FI_HOST_PANELS", "FI_HOST_PANEL_MB", "FI_HOST_MIN_LINE", "FI_HOST_BLOCKED_MAX_MB")
VARS = [{"FI_HOST_PIPELINE": "panels"},
        {"FI_HOST_BLOCKED_MAX_MB": "100000", "FI_HOST_PANEL_MB": "128", "FI_HOST_MIN_LINE": "4096"},
        {"FI_HOST_BLOCKED_MAX_MB": "100000", "FI_HOST_PANEL_MB": "128", "FI_HOST_MIN_LINE": "8192"},
        {"FI_HOST_BLOCKED_MAX_MB": "100000", "FI_HOST_PANEL_MB": "64", "FI_HOST_MIN_LINE": "4096"},
        {"FI_HOST_BLOCKED_MAX_MB": "100000", "FI_HOST_PANEL_MB": "256", "FI_HOST_MIN_LINE": "4096"}]
for rnd in range(2):
    for env in VARS:
        for k in KEYS: os.environ.pop(k, None)
        os.environ.update(env)
        plan.run_host_ptr(hA.data_ptr(), hB.data_ptr(), hC.data_ptr())
        t = time.perf_counter()
        for _ in range(3): plan.run_host_ptr(hA.data_ptr(), hB.data_ptr(), hC.data_ptr())
        print(f"{env}: {(time.perf_counter() - t) / 3 * 1e3:.2f} ms", flush=True)
for k in KEYS: os.environ.pop(k, None)
os.environ.update(VARS[1]); os.environ["FI_HOST_PIPELINE_TRACE"] = "1"
plan.run_host_ptr(hA.data_ptr(), hB.data_ptr(), hC.data_ptr())
