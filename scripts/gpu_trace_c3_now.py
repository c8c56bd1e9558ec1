"""Timeline of the current C3 launch (bench strategy, default schedule), and of C2."""
import os, sys
sys.path.insert(0, ".")
import torch
import paper_2003_06324_b200 as fi
s = torch.cuda.current_stream().cuda_stream
flush = torch.empty(128 << 20, device="cuda")
for name, strat, (m, n, k) in [("c3", fi.strategies.c3_strategy(), (1024, 1024, 32768)),
                               ("c2", fi.strategies.c2_strategy(), (4096, 4096, 4096))]:
    A = torch.randn(m * k, device="cuda").half(); B = torch.randn(k * n, device="cuda").half()
    C = torch.empty(m * n, device="cuda")
    plan = fi.Plan(strat)
    for _ in range(5): plan.launch(A.data_ptr(), B.data_ptr(), C.data_ptr(), s)
    flush.zero_(); torch.cuda.synchronize()
    os.environ["FI_TC_TRACE"] = f"gpurun_out/trace_{name}_now.txt"
    plan.launch(A.data_ptr(), B.data_ptr(), C.data_ptr(), s); torch.cuda.synchronize()
    del os.environ["FI_TC_TRACE"]
print("ok")
