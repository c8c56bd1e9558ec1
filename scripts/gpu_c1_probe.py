"""configs[0] on the GPU: the paper's Listing 2 (FMA leaf, fp32) at 512^3 through
the generic NVRTC path -- device time of the launch (inputs resident, L2 flushed)
and run_host end to end, against the reference simulator's 42 s."""
import statistics, sys, time
sys.path.insert(0, ".")
sys.path.insert(0, "oracle")
import numpy as np
import torch
import paper_2003_06324_b200 as fi
import oracle

m = n = k = 512
plan = fi.Plan(fi.strategies.listing2(m, n, k))
print("kind", plan.kind)
A = torch.rand(m * k, device="cuda"); B = torch.rand(k * n, device="cuda"); C = torch.empty(m * n, device="cuda")
flush = torch.empty(128 << 20, device="cuda")
s = torch.cuda.current_stream()
for _ in range(3): plan.launch(A.data_ptr(), B.data_ptr(), C.data_ptr(), s.cuda_stream)
ts = []
for _ in range(30):
    flush.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s); plan.launch(A.data_ptr(), B.data_ptr(), C.data_ptr(), s.cuda_stream); e1.record(s)
    torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
t = statistics.median(ts)
print(f"listing2 512^3 fp32 FMA leaf: device {t*1e3:.1f} us = {2*m*n*k/t/1e9:.2f} TFLOP/s")
a = oracle.fill(m, k, 1, False); b = oracle.fill(k, n, 2, False)
plan.run_host(a, b)
tw = []
for _ in range(10):
    t0 = time.perf_counter(); c = plan.run_host(a, b); tw.append(time.perf_counter() - t0)
print(f"run_host e2e (pageable numpy): {statistics.median(tw)*1e3:.2f} ms; digest {oracle.digest(c)}")
