"""Timelines of C3 with/without the remainder slice."""
import os, sys
sys.path.insert(0, ".")
import torch
import paper_2003_06324_b200 as fi
A = torch.randn(1024 * 32768, device="cuda").half(); B = torch.randn(1024 * 32768, device="cuda").half()
C = torch.empty(1024 * 1024, device="cuda")
flush = torch.empty(128 << 20, device="cuda")
s = torch.cuda.current_stream().cuda_stream
for name, rem in [("rem0", "0"), ("rem1", "1")]:
    os.environ["FI_REMAINDER"] = rem
    plan = fi.Plan(fi.strategies.c3_strategy())
    for _ in range(3): plan.launch(A.data_ptr(), B.data_ptr(), C.data_ptr(), s)
    flush.zero_(); torch.cuda.synchronize()
    os.environ["FI_TC_TRACE"] = f"gpurun_out/trace_c3b_{name}.txt"
    plan.launch(A.data_ptr(), B.data_ptr(), C.data_ptr(), s); torch.cuda.synchronize()
    del os.environ["FI_TC_TRACE"]
print("ok")
