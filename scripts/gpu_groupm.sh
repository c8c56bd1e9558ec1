#!/bin/bash
# Raster band height (FI_TC_GROUP_M) vs DRAM traffic and throughput on C5 (16384^3 bf16, 512x256 slab tiles)
for g in 8 4 2 16 32; do
  FI_TC_GROUP_M=$g timeout 180 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum --clock-control none -k regex:fi_sm100_gemm -s 1 -c 1 python bench.py --workload c5 --steps 1 --warmup 3 --no-cpu-baseline 2>/dev/null | grep -E "dram__bytes_read|gpu__time" | sed "s/^/g=$g /"
done
for r in 1 2; do for g in 8 4 2 16 32; do FI_TC_GROUP_M=$g timeout 120 python bench.py --workload c5 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('c5 group_m=$g', round(d['value'],1), 'med', round(d['impl_config']['ms_median'],3))"; done; done
