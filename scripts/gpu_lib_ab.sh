#!/bin/bash
# Interleaved A/B of two builds of the native library on one workload:
# OLD=path/to/old.so WL=c3 bash scripts/gpu_lib_ab.sh
for i in 1 2 3; do
  for lib in "$OLD" ""; do
    FI_LIB_PATH=$lib timeout 300 python bench.py --workload ${WL:-c2} --steps 40 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('${lib:-new}', round(d['value'],1), 'TF min_ms', round(d['impl_config']['ms_min']*1e3,1), 'med_ms', round(d['impl_config']['ms_median']*1e3,1))"
  done
done
