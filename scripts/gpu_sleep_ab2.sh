#!/bin/bash
mkdir -p gpurun_out
for v in 0 2000 20000; do
FI_TC_EPI_SLEEP=$v timeout 600 ncu --metrics smsp__inst_executed.sum,gpc__cycles_elapsed.avg.per_second,gpu__time_duration.sum,gpc__cycles_elapsed.max --clock-control none -k regex:fi_sm100_gemm -s 3 -c 1 \
    python scripts/gpu_one_gemm.py 8192 8192 8192 1 256 > gpurun_out/ncu_8192_sleep$v.log 2>&1
grep -E "inst_executed|per_second|gpu__time|elapsed.max" gpurun_out/ncu_8192_sleep$v.log | sed "s/^/sleep$v /"
done
for v in 0 2000 0 2000; do FI_TC_EPI_SLEEP=$v timeout 300 python bench.py --workload c5 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('c5 sleep=$v', round(d['value'],1), 'min', round(d['impl_config']['ms_min'],3), 'med', round(d['impl_config']['ms_median'],3), d['clocks'])"; done
VAR=FI_TC_EPI_SLEEP A=0 B=2000 WL=c2 bash scripts/gpu_ab.sh
