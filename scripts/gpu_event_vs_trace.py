"""Event-timed duration vs device timeline span for the same launches."""
import os, sys, statistics, time
sys.path.insert(0, ".")
import torch
import paper_2003_06324_b200 as fi
flush = torch.empty(128 << 20, device="cuda")
s = torch.cuda.current_stream()
def run(name, script, mode, m, n, k):
    os.environ["FI_STREAMK"] = mode
    plan = fi.Plan(script)
    A = torch.randn(k * m, device="cuda").half(); B = torch.randn(k * n, device="cuda").half(); C = torch.empty(m * n, device="cuda")
    go = lambda: plan.launch(A.data_ptr(), B.data_ptr(), C.data_ptr(), s.cuda_stream)
    for _ in range(3): go()
    ev = []
    for i in range(8):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s); go(); e1.record(s); torch.cuda.synchronize(); ev.append(e0.elapsed_time(e1) * 1e3)
    # host launch overhead alone
    torch.cuda.synchronize(); t0 = time.perf_counter(); go(); t1 = time.perf_counter(); torch.cuda.synchronize()
    flush.zero_(); torch.cuda.synchronize()
    path = f"gpurun_out/evt_{name}.txt"
    if os.path.exists(path): os.remove(path)
    os.environ["FI_TC_TRACE"] = path
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s); go(); e1.record(s); torch.cuda.synchronize()
    del os.environ["FI_TC_TRACE"]
    rows = [list(map(int, l.split())) for l in open(path) if not l.startswith("launch")]
    t_first = min(r[2] for r in rows if r[2]); t_last = max(max(r[3], r[5]) for r in rows)
    print(f"{name:14s} mode {plan.info.streamk}: events median {statistics.median(ev):7.1f} us (min {min(ev):.1f}); "
          f"traced launch events {e0.elapsed_time(e1)*1e3:7.1f} us, device span {(t_last - t_first)/1e3:6.1f} us; "
          f"host launch call {1e6*(t1-t0):6.1f} us  -> {plan.flops/statistics.median(ev)/1e6:7.1f} TF", flush=True)
run("c2_dp", fi.strategies.c2_strategy(), "0", 4096, 4096, 4096)
run("c2_kslice", fi.strategies.c2_strategy(), "1", 4096, 4096, 4096)
run("c3pair_kslice", fi.strategies.tc_strategy(1024, 1024, 32768), "1", 1024, 1024, 32768)
run("c3_dsmem", fi.strategies.c3_strategy(), "0", 1024, 1024, 32768)
