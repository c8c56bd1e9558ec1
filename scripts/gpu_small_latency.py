"""Small shapes: is the main loop latency- or bandwidth-bound? Event-timed median
of single launches with and without an L2 flush before each, for ring depths
(strategy .stages) and tile variants, beside cuBLAS (torch.mm, f32 out) under the
same conditions."""
import statistics, sys
sys.path.insert(0, ".")
import torch
import paper_2003_06324_b200 as fi

flush = torch.empty(128 << 20, device="cuda")
s = torch.cuda.current_stream().cuda_stream


def timed(fn, do_flush, reps=30):
    ts = []
    for _ in range(3):
        fn()
    for _ in range(reps):
        if do_flush:
            flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    return statistics.median(ts)


def empty():
    pass


for m, n, k in [(1024, 1024, 1024), (512, 512, 512), (2048, 2048, 2048), (4096, 256, 4096)]:
    A = (torch.rand(m * k, device="cuda") - 0.5).half()
    B = (torch.rand(k * n, device="cuda") - 0.5).half()
    C = torch.empty(m * n, device="cuda")
    At, Bt = A.view(k, m).t(), B.view(n, k).t()  # column-major views
    cub = lambda: torch.mm(At, Bt, out_dtype=torch.float32)
    print(f"{m}x{n}x{k}: cuBLAS flush {timed(cub, True):.1f} us, warm {timed(cub, False):.1f} us", flush=True)
    for name, kw in [("cta128x64", dict(pair=False, tile_n=64)), ("cta128x128", dict(pair=False, tile_n=128)),
                     ("pair256x64", dict(pair=True, tile_n=64)), ("pair256x64_mcast", dict(pair=True, tile_n=64, multicast=True)),
                     ("pair256x128", dict(pair=True, tile_n=128)), ("pair256x256", dict(pair=True, tile_n=256))]:
        for st in (0, 4):
            try:
                plan = fi.Plan(fi.strategies.tc_strategy(m, n, k, stages=st, **kw))
            except Exception as e:  # shape not divisible
                continue
            fn = lambda: plan.launch(A.data_ptr(), B.data_ptr(), C.data_ptr(), s)
            print(f"  {name:18s} stages {st or 'max':>3}: flush {timed(fn, True):6.1f} us, warm {timed(fn, False):6.1f} us",
                  flush=True)
