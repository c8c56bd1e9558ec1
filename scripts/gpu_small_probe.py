"""Small-shape overheads: host cost per plan.launch, back-to-back device time
(events around 200 launches), CUDA-graph replay time (no host in the loop),
single flushed launch; the same for cuBLAS (torch.mm, f32 out)."""
import statistics, sys, time
sys.path.insert(0, ".")
import torch
import paper_2003_06324_b200 as fi

flush = torch.empty(64 << 20, device="cuda")
s = torch.cuda.current_stream()


def measure(f, label):
    for _ in range(5):
        f()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(2000):
        f()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    host = (t1 - t0) / 2000 * 1e6
    wall = (t2 - t0) / 2000 * 1e6
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(200):
        f()
    e1.record(s)
    torch.cuda.synchronize()
    b2b = e0.elapsed_time(e1) / 200 * 1e3
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(20):
            f()
    g.replay(); torch.cuda.synchronize()
    e0.record(s)
    for _ in range(10):
        g.replay()
    e1.record(s)
    torch.cuda.synchronize()
    graph = e0.elapsed_time(e1) / 200 * 1e3
    ts = []
    for _ in range(30):
        flush.zero_()
        e0.record(s); f(); e1.record(s)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    print(f"{label:40s} host {host:6.1f}us wall {wall:6.1f}us b2b {b2b:6.1f}us graph {graph:6.1f}us flushed {statistics.median(ts):6.1f}us",
          flush=True)


SHAPES = [(512, 512, 512), (1024, 1024, 1024), (2048, 2048, 2048), (4096, 512, 4096)]
if len(sys.argv) > 1:
    SHAPES = [tuple(int(x) for x in a.split("x")) for a in sys.argv[1:]]
for (m, n, k) in SHAPES:
    for name, scr in fi.strategies.sweep_strategies(m, n, k).items():
        if "splitk" in name or "mcast" in name and m * n > 2048 * 2048:
            continue
        plan = fi.Plan(scr)
        A = torch.rand(m * k, device="cuda").half(); B = torch.rand(k * n, device="cuda").half()
        C = torch.empty(m * n, device="cuda")
        try:
            measure(lambda: plan.launch(A.data_ptr(), B.data_ptr(), C.data_ptr(), torch.cuda.current_stream().cuda_stream),
                    f"{m}x{n}x{k} {name}")
        except Exception as e:  # noqa: BLE001
            print(m, n, k, name, "failed", e, flush=True)
    a = torch.rand((k, m), device="cuda").half(); b = torch.rand((n, k), device="cuda").half()
    measure(lambda: torch.mm(b, a, out_dtype=torch.float32), f"{m}x{n}x{k} cublas_f32out")
