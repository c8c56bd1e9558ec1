#!/bin/bash
# Interleaved A/B of an environment toggle on one workload: VAR=name A=val B=val WL=c2
for i in 1 2 3; do
  for v in $A $B; do
    env $VAR=$v timeout 300 python bench.py --workload ${WL:-c2} --steps 40 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$VAR=$v', round(d['value'],1), 'TF min_ms', round(d['impl_config']['ms_min']*1e3,1), 'med_ms', round(d['impl_config']['ms_median']*1e3,1))"
  done
done
