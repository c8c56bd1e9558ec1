#!/bin/bash
# Iteration call: targeted GPU tests, bench lines, C3 timeline.
mkdir -p gpurun_out
timeout 900 python -m pytest -x -q -m gpu ${TESTS:-tests/test_gpu_remainder.py tests/test_gpu_host_pipeline.py tests/test_gpu_tc.py tests/test_gpu_splitk.py} > gpurun_out/pytest_iter.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_iter.log
for wl in ${WLS:-c2 c3}; do
    timeout 300 python bench.py --workload $wl --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/b_${wl}.json 2>/dev/null
    python -c "import json;d=json.load(open('gpurun_out/b_${wl}.json'));print('$wl', round(d['value'],1), 'TF', 'e2e', round(d['e2e']['value'],1), round(d['e2e']['ms_per_step'],3), 'ms', d['clocks'])"
done
python scripts/gpu_trace_c3b.py > /dev/null 2>&1; for f in gpurun_out/trace_c3b_*.txt; do echo == $f; python scripts/trace_report.py $f; done
if [ -n "$SWEEP" ]; then timeout 900 python scripts/sweep.py --tag iter --quick > gpurun_out/sweep_iter.log 2>&1; cut -c1-120 gpurun_out/sweep_iter.log; fi
