#!/bin/bash
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none -k regex:"nvjet|gemm|xmma|cutlass" -s 1 -c 1 \
    -o gpurun_out/prof_8192_cublas python scripts/gpu_cublas_one.py 8192 8192 8192 > gpurun_out/ncu_8192_cublas.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:"nvjet|gemm|xmma|cutlass" -s 1 -c 1 \
    -o gpurun_out/prof_2048_cublas python scripts/gpu_cublas_one.py 2048 2048 2048 > gpurun_out/ncu_2048_cublas.log 2>&1
for h in 1 2; do
FI_TC_L2HINT=$h timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:fi_sm100_gemm -s 3 -c 1 \
    python scripts/gpu_one_gemm.py 8192 8192 8192 1 256 > gpurun_out/ncu_8192_hint$h.log 2>&1
grep -E "dram__bytes|gpu__time|hit_rate" gpurun_out/ncu_8192_hint$h.log | sed "s/^/hint$h /"
done
cat > /tmp/b8192.py <<'PY'
import sys; sys.argv=['bench.py']
PY
for wl in c2 c5; do VAR=FI_TC_L2HINT A=0 B=1 WL=$wl bash scripts/gpu_ab.sh; done
