"""Timelines (FI_TC_TRACE) of small GEMMs after an L2 flush: where a 6-10 us launch goes."""
import os, sys
sys.path.insert(0, ".")
import torch
import paper_2003_06324_b200 as fi
s = torch.cuda.current_stream().cuda_stream
flush = torch.empty(128 << 20, device="cuda")
for (m, n, k), kw in [((512, 512, 512), dict(pair=False, tile_n=128)), ((1024, 1024, 1024), dict(pair=False, tile_n=128)),
                      ((1024, 1024, 1024), dict(pair=True, tile_n=128))]:
    A = (torch.rand(m * k, device="cuda") - 0.5).half(); B = (torch.rand(k * n, device="cuda") - 0.5).half()
    C = torch.empty(m * n, device="cuda")
    plan = fi.Plan(fi.strategies.tc_strategy(m, n, k, **kw))
    for _ in range(5): plan.launch(A.data_ptr(), B.data_ptr(), C.data_ptr(), s)
    name = f"{m}_{'pair' if kw['pair'] else 'cta'}{kw['tile_n']}"
    for rep in range(3):
        (flush.zero_() if os.environ.get("NOFLUSH") != "1" else None); torch.cuda.synchronize()
        os.environ["FI_TC_TRACE"] = f"gpurun_out/trace_small_{name}.txt"
        plan.launch(A.data_ptr(), B.data_ptr(), C.data_ptr(), s); torch.cuda.synchronize()
        del os.environ["FI_TC_TRACE"]
    print(name, flush=True)
    os.system(f"python scripts/trace_report.py gpurun_out/trace_small_{name}.txt")
