#!/bin/bash
# TMA L2 eviction hints (FI_TC_L2HINT) vs DRAM traffic and throughput on C5
for h in 0 1 2; do
  FI_TC_L2HINT=$h timeout 180 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum --clock-control none -k regex:fi_sm100_gemm -s 1 -c 1 python bench.py --workload c5 --steps 1 --warmup 3 --no-cpu-baseline 2>/dev/null | grep -E "dram__bytes_read|gpu__time" | sed "s/^/hint=$h /"
done
for r in 1 2 3; do for h in 0 1 2; do FI_TC_L2HINT=$h timeout 120 python bench.py --workload c5 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('c5 l2hint=$h', round(d['value'],1), 'med', round(d['impl_config']['ms_median'],3))"; done; done
