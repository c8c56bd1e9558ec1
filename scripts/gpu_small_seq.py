"""Small-shape device time without event quantisation: one event pair around
R x (L2 flush + launch) minus one around R x (L2 flush) alone, divided by R,
for our best trees and cuBLAS (torch.mm, f32 out). Interleaved rounds, median."""
import statistics, sys
sys.path.insert(0, ".")
import torch
import paper_2003_06324_b200 as fi

flush = torch.empty(128 << 20, device="cuda")
s = torch.cuda.current_stream().cuda_stream
R = 40


def seq(fn):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(R):
        flush.zero_()
        if fn:
            fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3


shapes = [(256, 256, 256), (512, 512, 512), (1024, 1024, 1024), (2048, 2048, 2048), (4096, 256, 4096),
          (256, 4096, 4096), (4096, 512, 4096)]
trees = [("cta128x64", dict(pair=False, tile_n=64)), ("cta128x128", dict(pair=False, tile_n=128)),
         ("pair256x64", dict(pair=True, tile_n=64)), ("pair256x128", dict(pair=True, tile_n=128)),
         ("pair256x256", dict(pair=True, tile_n=256))]
for m, n, k in shapes:
    A = (torch.rand(m * k, device="cuda") - 0.5).half()
    B = (torch.rand(k * n, device="cuda") - 0.5).half()
    C = torch.empty(m * n, device="cuda")
    At, Bt = A.view(k, m).t(), B.view(n, k).t()
    fns = {"cuBLAS": lambda: torch.mm(At, Bt, out_dtype=torch.float32)}
    for name, kw in trees:
        try:
            plan = fi.Plan(fi.strategies.tc_strategy(m, n, k, **kw))
        except Exception:
            continue
        fns[name] = (lambda p: lambda: p.launch(A.data_ptr(), B.data_ptr(), C.data_ptr(), s))(plan)
    res = {name: [] for name in fns}
    for fn in fns.values():
        seq(fn)
    for _ in range(5):
        base = seq(None)
        for name, fn in fns.items():
            res[name].append((seq(fn) - base) / R)
    line = "  ".join(f"{name} {statistics.median(v):5.2f}" for name, v in res.items())
    print(f"{m}x{n}x{k} (us per launch): {line}", flush=True)
