#!/bin/bash
# host snapping: GPU parity, then e2e A/B of device vs host snapping
mkdir -p gpurun_out
# (parity: tests/test_gpu_host_snap.py, tests/test_gpu_host_pipeline.py)
for cfg in "FI_HOST_SNAP=1" "FI_HOST_PANEL_MB=8" "FI_HOST_PANEL_MB=4" "FI_HOST_PANEL_MB=8 FI_HOST_PIECE_MB=4" \
           "FI_HOST_PANEL_MB=32" "FI_HOST_SNAP=1"; do
  env $cfg timeout 300 python scripts/gpu_e2e_snap.py 2>&1 | grep -v "^$"
done
