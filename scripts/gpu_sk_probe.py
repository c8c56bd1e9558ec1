"""Stream-K vs data-parallel on the shapes that matter (L2 flushed between steps)."""
import os, sys, statistics
sys.path.insert(0, ".")
import torch
import paper_2003_06324_b200 as fi

flush = torch.empty(128 << 20, device="cuda")

def bench(script, ab=torch.float16, steps=30):
    plan = fi.Plan(script)
    m, n, k = plan.m, plan.n, plan.k
    A = torch.randn(k, m, device="cuda").to(ab); B = torch.randn(n, k, device="cuda").to(ab)
    C = torch.empty(n, m, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    for _ in range(5): plan.launch(A.data_ptr(), B.data_ptr(), C.data_ptr(), s)
    ts = []
    for _ in range(steps):
        flush.zero_()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); plan.launch(A.data_ptr(), B.data_ptr(), C.data_ptr(), s); e1.record()
        torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    ms = statistics.mean(ts)
    return f"{plan.flops/ms/1e9:7.1f} TF  ({ms*1e3:.1f} us, ctas {plan.info.launch_ctas}, sk {plan.info.streamk})"

for mode in ["0", "1"]:
    os.environ["FI_STREAMK"] = mode
    for (m, n, k, pair, tn) in [(4096, 4096, 4096, True, 256), (8192, 8192, 8192, True, 256),
                                (2048, 2048, 16384, True, 256), (1024, 1024, 32768, True, 256),
                                (4096, 4096, 4096, False, 256), (2048, 2048, 2048, True, 256)]:
        print(f"streamk={mode} {m}x{n}x{k} pair={pair} tn={tn}:", bench(fi.strategies.tc_strategy(m, n, k, pair=pair, tile_n=tn)), flush=True)
