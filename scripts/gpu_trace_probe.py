"""Timeline + effective SM clock of the 4096^3 pair kernel, cold (after an L2
flush, idle GPU) and warm (after ~1.5 s of back-to-back GEMMs at the power cap)."""
import os, sys, time
sys.path.insert(0, ".")
import torch
import paper_2003_06324_b200 as fi
os.environ["FI_STREAMK"] = sys.argv[1] if len(sys.argv) > 1 else "-1"
plan = fi.Plan(fi.strategies.tc_strategy(4096, 4096, 4096))
A = torch.randn(4096 * 4096, device="cuda").half(); B = torch.randn(4096 * 4096, device="cuda").half()
C = torch.empty(4096 * 4096, device="cuda")
flush = torch.empty(128 << 20, device="cuda")
s = torch.cuda.current_stream().cuda_stream
go = lambda: plan.launch(A.data_ptr(), B.data_ptr(), C.data_ptr(), s)
for _ in range(3): go()
torch.cuda.synchronize(); time.sleep(0.5)
flush.zero_(); torch.cuda.synchronize()
os.environ["FI_TC_TRACE"] = f"gpurun_out/trace_cold_m{os.environ['FI_STREAMK']}.txt"; go(); torch.cuda.synchronize()
del os.environ["FI_TC_TRACE"]
t0 = time.time()
while time.time() - t0 < 1.5:
    for _ in range(50): go()
    torch.cuda.synchronize()
flush.zero_()
os.environ["FI_TC_TRACE"] = f"gpurun_out/trace_warm_m{os.environ['FI_STREAMK']}.txt"; go(); torch.cuda.synchronize()
print("done")
