#!/bin/bash
# Interleaved A/B/C of library builds on one workload: LIBS="a.so b.so" WL=c2 (""=in-tree build)
for i in 1 2 3; do
  for lib in $LIBS in-tree; do
    l=$lib; [ "$l" = in-tree ] && l=""
    FI_LIB_PATH=$l timeout 300 python bench.py --workload ${WL:-c2} --steps 40 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$lib', round(d['value'],1), 'TF min_us', round(d['impl_config']['ms_min']*1e3,1), 'med_us', round(d['impl_config']['ms_median']*1e3,1))"
  done
done
