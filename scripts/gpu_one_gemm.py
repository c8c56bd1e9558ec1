"""Run one tcgen05 strategy a few times (for ncu): args m n k pair tn [streamk]."""
import os, sys
sys.path.insert(0, ".")
import torch
import paper_2003_06324_b200 as fi
m, n, k, pair, tn = (int(x) for x in sys.argv[1:6])
if len(sys.argv) > 6:
    os.environ["FI_STREAMK"] = sys.argv[6]
plan = fi.Plan(fi.strategies.tc_strategy(m, n, k, pair=bool(pair), tile_n=tn))
A = torch.randn(k, m, device="cuda").half(); B = torch.randn(n, k, device="cuda").half()
C = torch.empty(n, m, device="cuda")
for _ in range(4):
    plan.launch(A.data_ptr(), B.data_ptr(), C.data_ptr(), torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
print("ok", plan.info.streamk, plan.info.launch_ctas)
