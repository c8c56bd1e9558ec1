"""run_host timeline for the C5 plan (16384^3 bf16) with the column-panel pipeline."""
import os, sys, time
sys.path.insert(0, ".")
import torch
import paper_2003_06324_b200 as fi
n = 16384
plan = fi.Plan(fi.strategies.c5_strategy())
hA = torch.rand((n, n), dtype=torch.float32).pin_memory()
hB = torch.rand((n, n), dtype=torch.float32).pin_memory()
hC = torch.empty((n, n), dtype=torch.float32).pin_memory()
for panels in ("8", "16", "4"):
    os.environ["FI_HOST_PANELS"] = panels
    plan.run_host_ptr(hA.data_ptr(), hB.data_ptr(), hC.data_ptr())
    t = time.perf_counter()
    for _ in range(3): plan.run_host_ptr(hA.data_ptr(), hB.data_ptr(), hC.data_ptr())
    print(f"panels<={panels}: {(time.perf_counter() - t) / 3 * 1e3:.2f} ms", flush=True)
os.environ["FI_HOST_PANELS"] = "8"
os.environ["FI_HOST_PIPELINE_TRACE"] = "1"
plan.run_host_ptr(hA.data_ptr(), hB.data_ptr(), hC.data_ptr())
