#!/bin/bash
# cuBLAS kernel choice and time for the C4 shapes where it leads (f32 out)
for s in "4096 256 4096" "256 4096 4096" "4096 512 4096" "1024 1024 1024" "2048 2048 2048" "512 512 512"; do
  timeout 120 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__cluster_dim_x,launch__shared_mem_per_block_dynamic --clock-control none -k regex:"nvjet|gemm|xmma|cutlass|splitK|reduce" -s 1 -c 3 python scripts/gpu_cublas_one.py $s 2>/dev/null | grep -E "nvjet|gemm|xmma|cutlass|Kernel|splitK|reduce|duration|grid_size|cluster_dim" | sed "s/^/[$s] /" | head -12
done
