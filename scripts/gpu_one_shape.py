"""A few launches of one tcgen05 strategy on one shape (for ncu):
  python scripts/gpu_one_shape.py M N K [pair 0|1] [tile_n] [multicast 0|1]"""
import sys
sys.path.insert(0, ".")
import torch
import paper_2003_06324_b200 as fi
m, n, k = (int(x) for x in sys.argv[1:4])
pair = bool(int(sys.argv[4])) if len(sys.argv) > 4 else True
tile_n = int(sys.argv[5]) if len(sys.argv) > 5 else 256
mc = bool(int(sys.argv[6])) if len(sys.argv) > 6 else False
plan = fi.Plan(fi.strategies.tc_strategy(m, n, k, pair=pair, tile_n=tile_n, multicast=mc))
A = (torch.rand(m * k, device="cuda") - 0.5).half(); B = (torch.rand(k * n, device="cuda") - 0.5).half()
C = torch.empty(m * n, device="cuda")
flush = torch.empty(128 << 20, device="cuda")
for _ in range(4):
    flush.zero_()
    plan.launch(A.data_ptr(), B.data_ptr(), C.data_ptr(), torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
print("ok")
