#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest -x -q -m gpu tests/test_gpu_remainder.py tests/test_gpu_tc.py tests/test_gpu_host_pipeline.py > gpurun_out/pytest_iter.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_iter.log
for i in 1 2; do for v in "FI_TC_HEAD=0 FI_TC_PULL_D=-1" "FI_TC_HEAD=0" "FI_TC_HEAD=1"; do
  env $v timeout 300 python bench.py --workload c2 --steps 40 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$v', round(d['value'],1), 'TF min_ms', round(d['impl_config']['ms_min']*1e3,1), 'med_ms', round(d['impl_config']['ms_median']*1e3,1))"
done; done
for v in 0 1; do FI_TC_HEAD=$v python scripts/gpu_trace_c2.py gpurun_out/trace_c2_head$v.txt; echo "== head $v"; python scripts/trace_report.py gpurun_out/trace_c2_head$v.txt; done
