"""Per-launch device time of several trees on one shape (sequence method of
scripts/sweep.py: 20 x (L2 flush + launch) minus 20 x flush), interleaved rounds.
  python scripts/gpu_shape_trees.py 4096 4096 4096 pair256 pair256_mcast slab512 nhalf512"""
import statistics, sys
sys.path.insert(0, ".")
import torch
import paper_2003_06324_b200 as fi
from scripts.sweep import per_launch_ms

TREES = {
    "pair256": dict(pair=True, tile_n=256), "pair256_mcast": dict(pair=True, tile_n=256, multicast=True),
    "pair128": dict(pair=True, tile_n=128), "pair128_mcast": dict(pair=True, tile_n=128, multicast=True),
    "pair64": dict(pair=True, tile_n=64), "pair64_mcast": dict(pair=True, tile_n=64, multicast=True),
    "cta64": dict(pair=False, tile_n=64),
    "pair256_s5": dict(pair=True, tile_n=256, stages=5), "pair256_s4": dict(pair=True, tile_n=256, stages=4),
    "pair256_sk2": dict(pair=True, tile_n=256, split_k=2), "pair256_sk4": dict(pair=True, tile_n=256, split_k=4),
    "pair256_sk8": dict(pair=True, tile_n=256, split_k=8), "pair128_sk4": dict(pair=True, tile_n=128, split_k=4),
    "slab512": dict(pair=True, tile_n=256, tile_m=512), "nhalf512": dict(pair=True, tile_n=512),
    "cta256": dict(pair=False, tile_n=256), "cta128": dict(pair=False, tile_n=128),
}
m, n, k = (int(x) for x in sys.argv[1:4])
names = sys.argv[4:]
flush = torch.empty(128 << 20, device="cuda")
A = (torch.rand(m * k, device="cuda") - 0.5).half()
B = (torch.rand(k * n, device="cuda") - 0.5).half()
C = torch.empty(m * n, device="cuda")
s = torch.cuda.current_stream().cuda_stream
plans = {nm: fi.Plan(fi.strategies.tc_strategy(m, n, k, **TREES[nm])) for nm in names}
res = {nm: [] for nm in names}
for _ in range(3):
    for nm, p in plans.items():
        res[nm].append(per_launch_ms(lambda: p.launch(A.data_ptr(), B.data_ptr(), C.data_ptr(), s), 3, flush))
for nm in names:
    ms = statistics.median(res[nm])
    print(f"{m}x{n}x{k} {nm:14s} {ms * 1e3:7.2f} us  {2 * m * n * k / ms / 1e9:7.1f} TF", flush=True)
