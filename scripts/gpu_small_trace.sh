#!/bin/bash
# Device-side view of small launches: ncu durations of ours vs cuBLAS, plus a unit timeline.
python scripts/gpu_small_probe.py 512x512x512 1024x1024x1024 2>&1 | grep -v Warn
ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__cluster_dim_x --clock-control none --csv \
  --log-file gpurun_out/small_ncu.csv python scripts/gpu_one_gemm.py 512 512 512 1 256 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/small_ncu_1k.csv \
  python scripts/gpu_one_gemm.py 1024 1024 1024 0 128 > /dev/null 2>&1
FI_TC_TRACE=gpurun_out/small_trace.txt python scripts/gpu_one_gemm.py 512 512 512 1 256
python - <<'PY'
import torch, time
a = torch.rand((512, 512), device="cuda").half(); b = torch.rand((512, 512), device="cuda").half()
for _ in range(3): torch.mm(b, a, out_dtype=torch.float32)
torch.cuda.synchronize()
PY
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/small_ncu_cublas.csv \
  python -c "
import torch
for s in (512, 1024):
    a = torch.rand((s, s), device='cuda').half(); b = torch.rand((s, s), device='cuda').half()
    for _ in range(3): torch.mm(b, a, out_dtype=torch.float32)
torch.cuda.synchronize()" > /dev/null 2>&1
