#!/bin/bash
# Interleaved A/B over several values of one environment knob: VAR=name VALS="a b c" WL=c3
for i in 1 2 3; do
  for v in $VALS; do
    env $VAR=$v timeout 300 python bench.py --workload ${WL:-c2} --steps 40 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$VAR=$v', round(d['value'],1), 'TF min_us', round(d['impl_config']['ms_min']*1e3,1), 'med_us', round(d['impl_config']['ms_median']*1e3,1))"
  done
done
