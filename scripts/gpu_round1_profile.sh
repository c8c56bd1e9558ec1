#!/bin/bash
# ncu evidence for the current kernels + config-4 sweep + CLI/GPU tests
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv \
    python bench.py --steps 5 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fi_sm100_gemm -s 3 -c 1 \
    -o gpurun_out/prof_c2b python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_c2b.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fi_sm100_gemm -s 3 -c 1 \
    -o gpurun_out/prof_c3b python bench.py --workload c3 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_c3b.log 2>&1
timeout 900 python scripts/sweep.py --tag round1 > gpurun_out/sweep.log 2>&1
cp profiles/round1_sweep.json gpurun_out/round1_sweep.json 2>/dev/null
timeout 300 python -m pytest tests/test_cli.py -q 2>&1 | tail -2
