"""C3 shape (1024x1024x32768 f16 -> f32) under several split-K trees: median of 30
launches, L2 flushed before each (events on the launch stream)."""
import statistics, sys
sys.path.insert(0, ".")
import torch
import paper_2003_06324_b200 as fi
m, n, k = 1024, 1024, 32768
A = torch.randn(m * k, device="cuda").half(); B = torch.randn(k * n, device="cuda").half()
C = torch.empty(m * n, device="cuda"); flush = torch.empty(128 << 20, device="cuda")
s = torch.cuda.current_stream()
VARS = {"pair256 split4": dict(pair=True, tile_n=256, split_k=4), "pair256 split2": dict(pair=True, tile_n=256, split_k=2),
        "pair256 no split (auto tail)": dict(pair=True, tile_n=256), "pair128 split2": dict(pair=True, tile_n=128, split_k=2),
        "cta128x256 split4": dict(pair=False, tile_n=256, split_k=4), "pair128 no split": dict(pair=True, tile_n=128),
        "pair256x128 mcast": dict(pair=True, tile_n=128, multicast=True)}
for rnd in range(2):
    for name, kw in VARS.items():
        try:
            plan = fi.Plan(fi.strategies.tc_strategy(m, n, k, **kw))
        except Exception as e:  # noqa: BLE001
            print(name, "rejected:", str(e)[:80]); continue
        for _ in range(3): plan.launch(A.data_ptr(), B.data_ptr(), C.data_ptr(), s.cuda_stream)
        ts = []
        for _ in range(30):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s); plan.launch(A.data_ptr(), B.data_ptr(), C.data_ptr(), s.cuda_stream); e1.record(s)
            torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
        t = statistics.median(ts)
        i = plan.info
        print(f"{name:30s} {2*m*n*k/t/1e9:7.1f} TF  {t*1e3:6.1f} us  ctas {i.launch_ctas} streamk {i.streamk}", flush=True)
