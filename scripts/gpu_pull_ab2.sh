#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest -x -q -m gpu tests/test_gpu_remainder.py tests/test_gpu_tc.py > gpurun_out/pytest_iter.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_iter.log
for i in 1 2; do for d in -1 12 16 20; do
  FI_TC_PULL_D=$d timeout 300 python bench.py --workload c2 --steps 40 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('pull_d=$d', round(d['value'],1), 'TF min_ms', round(d['impl_config']['ms_min']*1e3,1), 'med_ms', round(d['impl_config']['ms_median']*1e3,1))"
done; done
cat > /tmp/tr.py <<'PY'
import os, sys, torch
sys.path.insert(0, ".")
import paper_2003_06324_b200 as fi
A = torch.randn(4096*4096, device="cuda").half(); B = torch.randn(4096*4096, device="cuda").half(); C = torch.empty(4096*4096, device="cuda")
flush = torch.empty(128 << 20, device="cuda"); s = torch.cuda.current_stream().cuda_stream
plan = fi.Plan(fi.strategies.c2_strategy())
for _ in range(3): plan.launch(A.data_ptr(), B.data_ptr(), C.data_ptr(), s)
flush.zero_(); torch.cuda.synchronize()
os.environ["FI_TC_TRACE"] = sys.argv[1]
plan.launch(A.data_ptr(), B.data_ptr(), C.data_ptr(), s); torch.cuda.synchronize()
PY
for d in -1 16; do FI_TC_PULL_D=$d python /tmp/tr.py gpurun_out/trace_c2_pull$d.txt; echo "== pull $d"; python scripts/trace_report.py gpurun_out/trace_c2_pull$d.txt; done
