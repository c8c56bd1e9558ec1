"""Per-K-block time vs pipeline depth (.stages) for the pair 256x256 tile, and
the 1-CTA tiles, interleaved; distinguishes latency- from bandwidth-bound."""
import os, statistics, sys
sys.path.insert(0, ".")
import torch
import paper_2003_06324_b200 as fi
os.environ["FI_STREAMK"] = "0"
flush = torch.empty(128 << 20, device="cuda")
m = n = k = 4096
variants = {}
for st in (2, 3, 4, 5, 6):
    variants[f"pair256 st{st}"] = fi.Plan(fi.strategies.tc_strategy(m, n, k, stages=st))
for st in (2, 3, 4):
    variants[f"cta128x256 st{st}"] = fi.Plan(fi.strategies.tc_strategy(m, n, k, pair=False, stages=st))
for st in (3, 6, 8):
    variants[f"pair128 st{st}"] = fi.Plan(fi.strategies.tc_strategy(m, n, k, tile_n=128, stages=st))
A = torch.randn(k * m, device="cuda").half(); B = torch.randn(k * n, device="cuda").half()
C = torch.empty(m * n, device="cuda")
s = torch.cuda.current_stream()
times = {v: [] for v in variants}
names = list(variants)
for step in range(25):
    for name in names[step % len(names):] + names[:step % len(names)]:
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s); variants[name].launch(A.data_ptr(), B.data_ptr(), C.data_ptr(), s.cuda_stream); e1.record(s)
        torch.cuda.synchronize()
        if step >= 3: times[name].append(e0.elapsed_time(e1))
for name in names:
    ms = statistics.median(times[name])
    print(f"{name:18s} stages={variants[name].info.stages}  {2*m*n*k/ms/1e9:7.1f} TF  {ms*1e3:6.1f} us", flush=True)
