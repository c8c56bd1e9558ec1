#!/bin/bash
# Full ncu capture (with source) of the C3 split-K kernel and the 2048^3 kernel.
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fi_sm100_gemm -s 3 -c 1 \
    -o gpurun_out/prof_c3r python bench.py --workload c3 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_c3r.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/ncu_c3r.log
ls -la gpurun_out/*.ncu-rep
