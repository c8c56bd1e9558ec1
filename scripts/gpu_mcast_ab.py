"""Interleaved device-time A/B of pair tiles with and without .multicast (L2 flushed)."""
import statistics, sys, time
sys.path.insert(0, ".")
import torch
import paper_2003_06324_b200 as fi
flush = torch.empty(128 << 20, device="cuda"); s = torch.cuda.current_stream()
shapes = [(4096, 256, 4096, 64), (4096, 256, 4096, 128), (256, 4096, 4096, 64), (4096, 512, 4096, 128), (1024, 1024, 1024, 64),
          (2048, 2048, 2048, 256), (2048, 2048, 2048, 128), (4096, 4096, 4096, 256), (8192, 8192, 8192, 256)]
for m, n, k, tn in shapes:
    A = (torch.rand(k * m, device="cuda") - 0.5).half(); B = (torch.rand(n * k, device="cuda") - 0.5).half()
    C = torch.empty(m * n, device="cuda")
    res = {}
    for mc in (False, True):
        p = fi.Plan(fi.strategies.tc_strategy(m, n, k, tile_n=tn, multicast=mc))
        for _ in range(3): p.launch(A.data_ptr(), B.data_ptr(), C.data_ptr(), s.cuda_stream)
        ts = []
        for _ in range(15):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s); p.launch(A.data_ptr(), B.data_ptr(), C.data_ptr(), s.cuda_stream); e1.record(s)
            torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
        res[mc] = 2 * m * n * k / statistics.median(ts) / 1e9
    print(f"{m}x{n}x{k} pair 256x{tn}: plain {res[False]:7.1f} TF  multicast {res[True]:7.1f} TF  ({res[True] / res[False]:.2f}x)", flush=True)
