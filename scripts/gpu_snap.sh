#!/bin/bash
# host snapping: GPU parity, then e2e A/B of device vs host snapping
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_host_snap.py tests/test_gpu_host_pipeline.py -x -q 2>&1 | tail -5
for cfg in "FI_HOST_SNAP=0" "FI_HOST_SNAP=1" "FI_HOST_SNAP_RATIO=0.75" "FI_HOST_SNAP_RATIO=0.85" "FI_HOST_SNAP_RATIO=0.9" \
           "FI_HOST_PIECE_MB=12" "FI_HOST_SNAP_SKIP=2" "FI_HOST_SNAP=0" "FI_HOST_SNAP=1"; do
  env $cfg timeout 300 python scripts/gpu_e2e_snap.py 2>&1 | grep -v "^$"
done
