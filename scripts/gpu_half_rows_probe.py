"""Half-row pair tiles (128 x N, 64 rows per CTA) vs the existing trees and cuBLAS
on the small / narrow C4 shapes (event-timed after an L2 flush, median of 30)."""
import sys
sys.path.insert(0, ".")
sys.path.insert(0, "scripts")
import torch
import paper_2003_06324_b200 as fi
from sweep import time_plan, time_cublas

flush = torch.empty(128 << 20, device="cuda")
for (m, n, k) in [(256, 256, 256), (512, 512, 512), (1024, 1024, 1024), (2048, 2048, 2048), (4096, 256, 4096),
                  (4096, 512, 4096), (256, 4096, 4096), (8192, 256, 8192)]:
    res = {}
    for name, kw in [("cta128x64", dict(pair=False, tile_n=64)), ("cta128x128", dict(pair=False, tile_n=128)),
                     ("pair256x128", dict(pair=True, tile_n=128)), ("pair256x256", dict(pair=True, tile_n=256)),
                     ("half128x64", dict(pair=True, tile_m=128, tile_n=64)),
                     ("half128x128", dict(pair=True, tile_m=128, tile_n=128)),
                     ("half128x256", dict(pair=True, tile_m=128, tile_n=256))]:
        if m % (kw.get("tile_m") or (256 if kw["pair"] else 128)) or n % kw["tile_n"]:
            continue
        try:
            plan = fi.Plan(fi.strategies.tc_strategy(m, n, k, **kw))
            res[name] = time_plan(plan, 30, flush) * 1e3
        except Exception as e:  # noqa: BLE001
            res[name] = float("nan")
            print(name, "failed:", e)
    cub = time_cublas(m, n, k, 30, flush) * 1e3
    best = min(res, key=lambda x: res[x])
    print(f"{m}x{n}x{k}: " + "  ".join(f"{a}={b:.1f}" for a, b in res.items()) +
          f"  | cuBLAS {cub:.1f} us | best {best} {2*m*n*k/res[best]/1e6:.0f} TF vs cuBLAS {2*m*n*k/cub/1e6:.0f} TF",
          flush=True)
