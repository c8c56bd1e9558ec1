"""Interleaved A/B of a per-launch environment knob on tensor-core launches:
event-timed median over rounds (L2 flushed before every timed launch), and the
outputs of every setting compared bit for bit.
  python scripts/gpu_env_ab.py FI_SK_EARLY 0,1 c3 4096,256,4096,1,256,4 ...
Shapes: c2 / c3 (the bench strategies) or m,n,k,pair,tile_n,split_k."""
import os, statistics, sys
sys.path.insert(0, ".")
import torch
import paper_2003_06324_b200 as fi

var, values, shapes = sys.argv[1], sys.argv[2].split(","), sys.argv[3:]
flush = torch.empty(128 << 20, device="cuda")
s = torch.cuda.current_stream().cuda_stream
for spec in shapes:
    if spec == "c2":
        strat, (m, n, k) = fi.strategies.c2_strategy(), (4096, 4096, 4096)
    elif spec == "c3":
        strat, (m, n, k) = fi.strategies.c3_strategy(), (1024, 1024, 32768)
    else:
        m, n, k, pair, tn, sk = (int(x) for x in spec.split(","))
        strat = fi.strategies.tc_strategy(m, n, k, pair=bool(pair), tile_n=tn, split_k=sk)
    plan = fi.Plan(strat)
    g = torch.Generator(device="cuda").manual_seed(7)
    A = (torch.rand(m * k, device="cuda", generator=g) * 2 - 1).half()
    B = (torch.rand(k * n, device="cuda", generator=g) * 2 - 1).half()
    C = torch.empty(m * n, device="cuda")
    outs, times = {}, {v: [] for v in values}
    for rnd in range(25):
        for v in values:
            os.environ[var] = v
            if rnd == 0:
                for _ in range(3):
                    plan.launch(A.data_ptr(), B.data_ptr(), C.data_ptr(), s)
                torch.cuda.synchronize()
                outs[v] = C.clone()
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            plan.launch(A.data_ptr(), B.data_ptr(), C.data_ptr(), s)
            e1.record()
            torch.cuda.synchronize()
            times[v].append(e0.elapsed_time(e1) * 1e3)
    same = all(torch.equal(outs[v], outs[values[0]]) for v in values)
    line = " | ".join(f"{var}={v}: {statistics.median(times[v]):.1f} us ({2 * m * n * k / statistics.median(times[v]) / 1e6:.0f} TF)"
                      for v in values)
    print(f"{spec}: {line} | outputs identical: {same}", flush=True)
os.environ.pop(var, None)
