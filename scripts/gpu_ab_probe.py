"""Interleaved A/B timing of tcgen05 plan variants (each step: L2 flush, one
launch per variant in rotating order) so clock/power drift hits all variants
alike. Usage: python scripts/gpu_ab_probe.py [steps]"""
import os
import statistics
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_2003_06324_b200 as fi  # noqa: E402

STEPS = int(sys.argv[1]) if len(sys.argv) > 1 else 40
flush = torch.empty(128 << 20, device="cuda")


def make(m, n, k, streamk, **kw):
    os.environ["FI_STREAMK"] = str(streamk)
    plan = fi.Plan(fi.strategies.tc_strategy(m, n, k, **kw))
    ab = torch.bfloat16 if kw.get("ab") == "bf16" else torch.float16
    A = torch.randn(k * m, device="cuda").to(ab)
    B = torch.randn(k * n, device="cuda").to(ab)
    C = torch.empty(m * n, device="cuda")
    return plan, A, B, C


def ab(label, variants):
    s = torch.cuda.current_stream()
    times = {name: [] for name in variants}
    names = list(variants)
    for step in range(STEPS):
        order = names[step % len(names):] + names[:step % len(names)]
        for name in order:
            plan, A, B, C = variants[name]
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            plan.launch(A.data_ptr(), B.data_ptr(), C.data_ptr(), s.cuda_stream)
            e1.record(s)
            torch.cuda.synchronize()
            if step >= 3:
                times[name].append(e0.elapsed_time(e1))
    for name in names:
        plan = variants[name][0]
        ms = statistics.median(times[name])
        print(f"{label:28s} {name:12s} {plan.flops / ms / 1e9:8.1f} TF  {ms * 1e3:7.1f} us  "
              f"(mode {plan.info.streamk}, ctas {plan.info.launch_ctas})", flush=True)


for (m, n, k) in [(4096, 4096, 4096), (8192, 8192, 8192), (1024, 1024, 32768), (2048, 2048, 16384), (4096, 4096, 1024)]:
    ab(f"{m}x{n}x{k} pair256", {"dp": make(m, n, k, 0), "auto": make(m, n, k, -1),
                                "kslice": make(m, n, k, 1), "nsplit": make(m, n, k, 2)})
ab("4096^3 cta128x256", {"dp": make(4096, 4096, 4096, 0, pair=False), "auto": make(4096, 4096, 4096, -1, pair=False)})
ab("c3 splitk (dsmem)", {"c3": (fi.Plan(fi.strategies.c3_strategy()), torch.randn(1024 * 32768, device="cuda").half(),
                                torch.randn(1024 * 32768, device="cuda").half(), torch.empty(1024 * 1024, device="cuda"))})
