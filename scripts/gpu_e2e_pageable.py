"""run_host e2e from PAGEABLE host memory (what anvil::run's std::vector-backed
Matrix gives the C++ drop-in), C2 plan, under this process's FI_HOST_* env."""
import os, statistics, sys, time
sys.path.insert(0, ".")
import numpy as np
import paper_2003_06324_b200 as fi

tag = " ".join(f"{k}={v}" for k, v in sorted(os.environ.items()) if k.startswith("FI_HOST")) or "defaults"
m = n = k = 4096
plan = fi.Plan(fi.strategies.c2_strategy())
rng = np.random.default_rng(1)
hA = (rng.random((k, m), dtype=np.float32) * 2 - 1)
hB = (rng.random((n, k), dtype=np.float32) * 2 - 1)
hC = np.empty((n, m), dtype=np.float32)
for _ in range(3):
    plan.run_host_ptr(hA.ctypes.data, hB.ctypes.data, hC.ctypes.data)
ts = []
for _ in range(10):
    t = time.perf_counter()
    plan.run_host_ptr(hA.ctypes.data, hB.ctypes.data, hC.ctypes.data)
    ts.append((time.perf_counter() - t) * 1e3)
print(f"pageable c2 [{tag}]: median {statistics.median(ts):.3f} ms  min {min(ts):.3f}  bytes {plan.host_bytes()}", flush=True)
