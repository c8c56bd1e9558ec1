"""One of our tensor-core launches (for ncu): m n k pair tile_n [multicast] [stages]."""
import sys
sys.path.insert(0, ".")
import torch
import paper_2003_06324_b200 as fi
m, n, k, pair, tn = (int(x) for x in sys.argv[1:6])
mc = int(sys.argv[6]) if len(sys.argv) > 6 else 0
st = int(sys.argv[7]) if len(sys.argv) > 7 else 0
plan = fi.Plan(fi.strategies.tc_strategy(m, n, k, pair=bool(pair), tile_n=tn, multicast=bool(mc), stages=st))
A = (torch.rand(m * k, device="cuda") - 0.5).half(); B = (torch.rand(k * n, device="cuda") - 0.5).half()
C = torch.empty(m * n, device="cuda")
s = torch.cuda.current_stream().cuda_stream
for _ in range(4):
    plan.launch(A.data_ptr(), B.data_ptr(), C.data_ptr(), s)
torch.cuda.synchronize()
print("ok")
