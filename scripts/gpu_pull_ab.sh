#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest -x -q -m gpu tests/test_gpu_tc.py tests/test_gpu_remainder.py tests/test_gpu_host_pipeline.py tests/test_gpu_splitk.py > gpurun_out/pytest_iter.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_iter.log
VAR=FI_TC_PULL_D A=-1 B=8 WL=c2 bash scripts/gpu_ab.sh
VAR=FI_TC_PULL_D A=4 B=12 WL=c2 bash scripts/gpu_ab.sh
FI_TC_PULL_D=8 python scripts/gpu_trace_probe.py > /dev/null 2>&1
python - <<'PY'
import os, sys, torch
sys.path.insert(0, ".")
import paper_2003_06324_b200 as fi
A = torch.randn(4096*4096, device="cuda").half(); B = torch.randn(4096*4096, device="cuda").half(); C = torch.empty(4096*4096, device="cuda")
flush = torch.empty(128 << 20, device="cuda"); s = torch.cuda.current_stream().cuda_stream
for d in ["-1", "8"]:
    os.environ["FI_TC_PULL_D"] = d
    plan = fi.Plan(fi.strategies.c2_strategy())
    for _ in range(3): plan.launch(A.data_ptr(), B.data_ptr(), C.data_ptr(), s)
    flush.zero_(); torch.cuda.synchronize()
    os.environ["FI_TC_TRACE"] = f"gpurun_out/trace_c2_pull{d}.txt"
    plan.launch(A.data_ptr(), B.data_ptr(), C.data_ptr(), s); torch.cuda.synchronize()
    del os.environ["FI_TC_TRACE"]
PY
for f in gpurun_out/trace_c2_pull*.txt; do echo "== $f"; python scripts/trace_report.py $f; done
