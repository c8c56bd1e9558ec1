#!/bin/bash
# ncu full captures: ours vs cuBLAS (f32 out) at 8192^3, plus ours at 2048^3
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fi_sm100_gemm -s 3 -c 1 \
    -o gpurun_out/prof_8192_ours python scripts/gpu_one_gemm.py 8192 8192 8192 1 256 > gpurun_out/ncu_8192_ours.log 2>&1
timeout 900 ncu --set full --clock-control none -s 3 -c 1 \
    -o gpurun_out/prof_8192_cublas python scripts/gpu_cublas_one.py 8192 8192 8192 > gpurun_out/ncu_8192_cublas.log 2>&1
timeout 900 ncu --set full --clock-control none -s 3 -c 1 \
    -o gpurun_out/prof_2048_cublas python scripts/gpu_cublas_one.py 2048 2048 2048 > gpurun_out/ncu_2048_cublas.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fi_sm100_gemm -s 3 -c 1 \
    -o gpurun_out/prof_2048_ours python scripts/gpu_one_gemm.py 2048 2048 2048 1 256 > gpurun_out/ncu_2048_ours.log 2>&1
timeout 900 python scripts/sweep.py --tag round1 > gpurun_out/sweep.log 2>&1; echo "sweep rc=$?"
cp profiles/round1_sweep.json gpurun_out/round1_sweep.json
cut -c1-150 gpurun_out/sweep.log
ls gpurun_out/*.ncu-rep
