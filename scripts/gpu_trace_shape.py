"""Traced launches (FI_TC_TRACE) of tensor-core strategies after warm-up and an
L2 flush. argv: out_prefix then one or more m,n,k,pair,tile_n,split[,multicast[,stages]] specs."""
import os, sys, torch
sys.path.insert(0, ".")
import paper_2003_06324_b200 as fi
flush = torch.empty(128 << 20, device="cuda"); s = torch.cuda.current_stream().cuda_stream
prefix = sys.argv[1]
for spec in sys.argv[2:]:
    m, n, k, pair, tn, sk, *mc = (int(x) for x in spec.split(","))
    plan = fi.Plan(fi.strategies.tc_strategy(m, n, k, pair=bool(pair), tile_n=tn, split_k=sk,
                                             multicast=bool(mc and mc[0]), stages=mc[1] if len(mc) > 1 else 0))
    A = torch.randn(m * k, device="cuda").half(); B = torch.randn(k * n, device="cuda").half()
    C = torch.empty(m * n, device="cuda")
    for _ in range(3): plan.launch(A.data_ptr(), B.data_ptr(), C.data_ptr(), s)
    flush.zero_(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); plan.launch(A.data_ptr(), B.data_ptr(), C.data_ptr(), s); e1.record(); torch.cuda.synchronize()
    print(spec, "event ms", round(e0.elapsed_time(e1), 4), "TF", round(2*m*n*k/e0.elapsed_time(e1)/1e9, 1), flush=True)
    flush.zero_(); torch.cuda.synchronize()
    os.environ["FI_TC_TRACE"] = f"{prefix}_{spec.replace(',', '_')}.txt"
    plan.launch(A.data_ptr(), B.data_ptr(), C.data_ptr(), s); torch.cuda.synchronize()
    del os.environ["FI_TC_TRACE"]
