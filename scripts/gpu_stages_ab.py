"""Pipeline depth (.stages) of the pair 256x256 tile on C2 and C3: median of 30 launches,
L2 flushed before each, interleaved over two rounds."""
import statistics, sys
sys.path.insert(0, ".")
import torch
import paper_2003_06324_b200 as fi
flush = torch.empty(128 << 20, device="cuda")
s = torch.cuda.current_stream()
for (m, n, k, sk) in [(4096, 4096, 4096, 1), (1024, 1024, 32768, 4)]:
    A = torch.randn(m * k, device="cuda").half(); B = torch.randn(k * n, device="cuda").half()
    C = torch.empty(m * n, device="cuda")
    plans = {st: fi.Plan(fi.strategies.tc_strategy(m, n, k, pair=True, tile_n=256, split_k=sk, stages=st))
             for st in (3, 4, 5, 6)}
    for rnd in range(2):
        for st, plan in plans.items():
            for _ in range(3): plan.launch(A.data_ptr(), B.data_ptr(), C.data_ptr(), s.cuda_stream)
            ts = []
            for _ in range(30):
                flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(s); plan.launch(A.data_ptr(), B.data_ptr(), C.data_ptr(), s.cuda_stream); e1.record(s)
                torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
            t = statistics.median(ts)
            print(f"{m}x{n}x{k} stages {st}: {2*m*n*k/t/1e9:7.1f} TF  {t*1e3:6.1f} us", flush=True)
