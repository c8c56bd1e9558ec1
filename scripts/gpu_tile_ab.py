"""Interleaved A/B of block-tile strategies on large GEMMs (device time, L2
flushed before every launch): 256x256 pair tile vs the 512x256 slab tile vs the 256x512 N-half tile.
argv: m n k ab [rounds]"""
import statistics, sys, time
sys.path.insert(0, ".")
from bench import ClockSampler
import torch
import paper_2003_06324_b200 as fi
m, n, k = (int(x) for x in sys.argv[1:4])
ab = sys.argv[4] if len(sys.argv) > 4 else "f16"
rounds = int(sys.argv[5]) if len(sys.argv) > 5 else 3
dt = torch.float16 if ab == "f16" else torch.bfloat16
A = (torch.rand(k * m, device="cuda") - 0.5).to(dt); B = (torch.rand(n * k, device="cuda") - 0.5).to(dt)
C = torch.empty(m * n, device="cuda")
flush = torch.empty(128 << 20, device="cuda"); s = torch.cuda.current_stream()
plans = {"pair256x256": fi.Plan(fi.strategies.tc_strategy(m, n, k, ab=ab)),
         "pair512x256": fi.Plan(fi.strategies.tc_strategy(m, n, k, ab=ab, tile_m=512)),
         "pair256x512": fi.Plan(fi.strategies.tc_strategy(m, n, k, ab=ab, tile_n=512))}
for p in plans.values():
    for _ in range(3): p.launch(A.data_ptr(), B.data_ptr(), C.data_ptr(), s.cuda_stream)
torch.cuda.synchronize()
for r in range(rounds):
    for name, p in plans.items():
        time.sleep(3)  # let clocks and temperature recover between arms
        ts = []
        cs = ClockSampler(0)
        cs.__enter__()
        for _ in range(10):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s); p.launch(A.data_ptr(), B.data_ptr(), C.data_ptr(), s.cuda_stream); e1.record(s)
            torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
        cs.__exit__()
        ms = statistics.median(ts)
        print(f"{m}x{n}x{k} {ab} {name}: {2*m*n*k/ms/1e9:7.1f} TF  median {ms:.3f} ms  min {min(ts):.3f}  "
              f"clocks {cs.summary()}", flush=True)
