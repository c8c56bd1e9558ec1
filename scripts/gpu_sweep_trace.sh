#!/bin/bash
# C4 sweep (+cuBLAS reference column), C5 at 1 GPU, C3 timelines.
mkdir -p gpurun_out
timeout 1200 python scripts/sweep.py --tag round1 > gpurun_out/sweep.log 2>&1; echo "sweep rc=$?"
cp profiles/round1_sweep.json gpurun_out/round1_sweep.json 2>/dev/null
timeout 600 python bench.py --workload c5 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5_n1.json 2> gpurun_out/bench_c5_n1.err; echo "c5 rc=$?"
timeout 300 python scripts/gpu_trace_c3.py > gpurun_out/trace_c3.log 2>&1; echo "trace rc=$?"
for f in gpurun_out/trace_c3_*.txt; do echo "== $f"; python scripts/trace_report.py $f; done
cat gpurun_out/bench_c5_n1.json
tail -30 gpurun_out/sweep.log
