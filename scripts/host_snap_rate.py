"""Host conversion throughput of fi_host_snap_f32 (the product's snap) on T
threads over 128 MiB of fp32 (pinned or pageable), f16 and bf16."""
import ctypes as C, sys, time
from concurrent.futures import ThreadPoolExecutor
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_2003_06324_b200 as fi

n = 32 << 20
pin = torch.cuda.is_available()
src = torch.empty(n, dtype=torch.float32, pin_memory=pin)
src.copy_(torch.rand(n) * 2 - 1)
dst = torch.empty(n, dtype=torch.int16, pin_memory=pin)
piece = 256 * 1024
for elem, code in (("f16", 1), ("bf16", 2)):
    for T in (1, 4, 8, 16):
        def work(i):
            fi.lib.fi_host_snap_f32(src.data_ptr() + i * piece * 4, dst.data_ptr() + i * piece * 2, piece, code)
        with ThreadPoolExecutor(T) as ex:
            list(ex.map(work, range(n // piece)))
            best = 1e9
            for _ in range(5):
                t = time.perf_counter()
                list(ex.map(work, range(n // piece)))
                best = min(best, time.perf_counter() - t)
        print(f"{elem} T={T:2d}: {n * 4 / best / 1e9:6.1f} GB/s of fp32 in", flush=True)
