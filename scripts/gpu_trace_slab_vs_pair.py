"""Per-unit main-loop time of the 512x256 slab tile vs the 256x256 pair tile at
4096^3 (FI_TC_TRACE), same box: does a slab unit beat two pair units?"""
import os, sys
sys.path.insert(0, ".")
import torch
import paper_2003_06324_b200 as fi
m = n = k = 4096
s = torch.cuda.current_stream().cuda_stream
A = torch.randn(m * k, device="cuda").half(); B = torch.randn(k * n, device="cuda").half()
C = torch.empty(m * n, device="cuda")
flush = torch.empty(128 << 20, device="cuda")
for name, kw in [("pair", dict(pair=True, tile_n=256)), ("slab", dict(pair=True, tile_n=256, tile_m=512))]:
    plan = fi.Plan(fi.strategies.tc_strategy(m, n, k, **kw))
    for _ in range(5): plan.launch(A.data_ptr(), B.data_ptr(), C.data_ptr(), s)
    for rep in range(3):
        flush.zero_(); torch.cuda.synchronize()
        os.environ["FI_TC_TRACE"] = f"gpurun_out/trace_{name}.txt"
        plan.launch(A.data_ptr(), B.data_ptr(), C.data_ptr(), s); torch.cuda.synchronize()
        del os.environ["FI_TC_TRACE"]
    print("==", name, flush=True)
    os.system(f"python scripts/trace_report.py gpurun_out/trace_{name}.txt")
