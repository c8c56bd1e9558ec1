"""run_host wall time per call for the C2 plan across host-pipeline variants."""
import os, sys, time
sys.path.insert(0, ".")
import torch
import paper_2003_06324_b200 as fi
plan = fi.Plan(fi.strategies.c2_strategy())
hA = torch.rand((4096, 4096), dtype=torch.float32).pin_memory()
hB = torch.rand((4096, 4096), dtype=torch.float32).pin_memory()
hC = torch.empty((4096, 4096), dtype=torch.float32).pin_memory()
VARS = [("blocked", {"FI_HOST_PANEL_MB": mb, "FI_HOST_MIN_LINE": ml}) for mb, ml in
        (("16", "1024"), ("8", "2048"), ("16", "2048"), ("4", "2048"), ("8", "4096"), ("32", "1024"))] + \
       [("panels", {"FI_HOST_PIPELINE": "panels", "FI_HOST_PANELS": p}) for p in ("2", "4", "8")] + \
       [("plain", {"FI_HOST_PIPELINE": "0"})]
for rnd in range(2):
    for name, env in VARS:
        for key in ("FI_HOST_PANEL_MB", "FI_HOST_PIPELINE", "FI_HOST_PANELS", "FI_HOST_MIN_LINE"):
            os.environ.pop(key, None)
        os.environ.update(env)
        for _ in range(2): plan.run_host_ptr(hA.data_ptr(), hB.data_ptr(), hC.data_ptr())
        ts = []
        for _ in range(7):
            t = time.perf_counter(); plan.run_host_ptr(hA.data_ptr(), hB.data_ptr(), hC.data_ptr())
            ts.append(time.perf_counter() - t)
        ts.sort()
        print(f"{name:8s} {env}: median {ts[3] * 1e3:.3f} ms  min {ts[0] * 1e3:.3f} ms", flush=True)
