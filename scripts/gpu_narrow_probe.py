"""Narrow shapes: which tail schedule the planner picks, and its time vs
pure data-parallel (FI_STREAMK=0) and forced K-slices, event-timed after a flush."""
import os, statistics, sys
sys.path.insert(0, ".")
sys.path.insert(0, "scripts")
import torch
import paper_2003_06324_b200 as fi
from sweep import time_plan

flush = torch.empty(128 << 20, device="cuda")
for (m, n, k) in [(4096, 256, 4096), (8192, 256, 8192), (4096, 512, 4096), (2048, 2048, 2048)]:
    for name, kw in [("pair256x64", dict(pair=True, tile_n=64)), ("pair256x128", dict(pair=True, tile_n=128)),
                     ("pair256x256", dict(pair=True, tile_n=256)), ("cta128x64", dict(pair=False, tile_n=64)),
                     ("cta128x128", dict(pair=False, tile_n=128))]:
        if n % kw["tile_n"]:
            continue
        row = []
        for sk in ["-1", "0", "1", "2"]:
            os.environ["FI_STREAMK"] = sk
            plan = fi.Plan(fi.strategies.tc_strategy(m, n, k, **kw))
            t = time_plan(plan, 15, flush) * 1e3
            row.append(f"sk{sk}={t:.1f}us(mode{plan.info.streamk},ctas{plan.info.launch_ctas})")
        print(f"{m}x{n}x{k} {name}: " + "  ".join(row), flush=True)
os.environ.pop("FI_STREAMK")
