"""One traced C2 launch (FI_TC_TRACE) after warm-up and an L2 flush: argv[1] = output file."""
import os, sys, torch
sys.path.insert(0, ".")
import paper_2003_06324_b200 as fi
A = torch.randn(4096 * 4096, device="cuda").half(); B = torch.randn(4096 * 4096, device="cuda").half()
C = torch.empty(4096 * 4096, device="cuda")
flush = torch.empty(128 << 20, device="cuda"); s = torch.cuda.current_stream().cuda_stream
plan = fi.Plan(fi.strategies.c2_strategy())
for _ in range(3): plan.launch(A.data_ptr(), B.data_ptr(), C.data_ptr(), s)
flush.zero_(); torch.cuda.synchronize()
os.environ["FI_TC_TRACE"] = sys.argv[1]
plan.launch(A.data_ptr(), B.data_ptr(), C.data_ptr(), s); torch.cuda.synchronize()
