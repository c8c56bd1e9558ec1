"""run_host per call for the C2 plan: median of 7, for the current FI_TC_COOP setting."""
import os, sys, time
sys.path.insert(0, ".")
import torch
import paper_2003_06324_b200 as fi
plan = fi.Plan(fi.strategies.c2_strategy())
hA = torch.rand((4096, 4096), dtype=torch.float32).pin_memory()
hB = torch.rand((4096, 4096), dtype=torch.float32).pin_memory()
hC = torch.empty((4096, 4096), dtype=torch.float32).pin_memory()
for _ in range(2): plan.run_host_ptr(hA.data_ptr(), hB.data_ptr(), hC.data_ptr())
ts = []
for _ in range(7):
    t = time.perf_counter(); plan.run_host_ptr(hA.data_ptr(), hB.data_ptr(), hC.data_ptr()); ts.append(time.perf_counter() - t)
ts.sort()
print(f"FI_TC_COOP={os.environ.get('FI_TC_COOP', '1')}: median {ts[3]*1e3:.3f} ms", flush=True)
if os.environ.get("TRACE"):
    os.environ["FI_HOST_PIPELINE_TRACE"] = "1"
    plan.run_host_ptr(hA.data_ptr(), hB.data_ptr(), hC.data_ptr())
