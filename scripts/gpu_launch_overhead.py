"""Host cost of one Plan.launch (tensor-map encode + schedule + cudaLaunchKernelEx)
and the device time of small GEMMs: eager event-timed (the sweep's method),
back-to-back eager, and CUDA-graph replay, beside cuBLAS."""
import statistics, sys, time
sys.path.insert(0, ".")
import torch
import paper_2003_06324_b200 as fi

s = torch.cuda.current_stream()
for (m, n, k), kw in [((256, 256, 256), dict(pair=False, tile_n=64)), ((512, 512, 512), dict(pair=False, tile_n=128)),
                      ((1024, 1024, 1024), dict(pair=False, tile_n=128)), ((2048, 2048, 2048), dict(pair=False, tile_n=256)),
                      ((4096, 4096, 4096), dict(pair=True, tile_n=256))]:
    plan = fi.Plan(fi.strategies.tc_strategy(m, n, k, **kw))
    A = (torch.rand(m * k, device="cuda") - 0.5).half()
    B = (torch.rand(k * n, device="cuda") - 0.5).half()
    C = torch.empty(m * n, device="cuda")
    for _ in range(5):
        plan.launch(A.data_ptr(), B.data_ptr(), C.data_ptr(), s.cuda_stream)
    torch.cuda.synchronize()
    # host submission cost
    t = time.perf_counter()
    for _ in range(200):
        plan.launch(A.data_ptr(), B.data_ptr(), C.data_ptr(), s.cuda_stream)
    host_us = (time.perf_counter() - t) / 200 * 1e6
    torch.cuda.synchronize()
    # eager, event-timed single launches (sweep method, no flush)
    ts = []
    for _ in range(50):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s); plan.launch(A.data_ptr(), B.data_ptr(), C.data_ptr(), s.cuda_stream); e1.record(s)
        torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1) * 1e3)
    # back-to-back eager: 100 launches between two events
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record(s)
    for _ in range(100):
        plan.launch(A.data_ptr(), B.data_ptr(), C.data_ptr(), s.cuda_stream)
    e1.record(s); torch.cuda.synchronize()
    b2b = e0.elapsed_time(e1) * 1e3 / 100
    # graph replay of 20 launches
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(20):
            plan.launch(A.data_ptr(), B.data_ptr(), C.data_ptr(), torch.cuda.current_stream().cuda_stream)
    g.replay(); torch.cuda.synchronize()
    e0.record(s); g.replay(); e1.record(s); torch.cuda.synchronize()
    gr = e0.elapsed_time(e1) * 1e3 / 20
    # cuBLAS
    a = (torch.rand((k, m), device="cuda") - 0.5).half(); b = (torch.rand((n, k), device="cuda") - 0.5).half()
    for _ in range(5): torch.mm(b, a, out_dtype=torch.float32)
    tc = []
    for _ in range(50):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s); torch.mm(b, a, out_dtype=torch.float32); e1.record(s)
        torch.cuda.synchronize(); tc.append(e0.elapsed_time(e1) * 1e3)
    t = time.perf_counter()
    for _ in range(200): torch.mm(b, a, out_dtype=torch.float32)
    cub_host = (time.perf_counter() - t) / 200 * 1e6
    torch.cuda.synchronize()
    print(f"{m}x{n}x{k} {kw}: host {host_us:.1f} us/launch | eager event {statistics.median(ts):.1f} us | "
          f"back-to-back {b2b:.1f} us | graph {gr:.1f} us || cuBLAS eager {statistics.median(tc):.1f} us host {cub_host:.1f} us",
          flush=True)
