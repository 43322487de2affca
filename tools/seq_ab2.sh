#!/bin/bash
# Same-box A/B of the r02 persistent-GEMM options on the slice-sequential cfg 3 schedule (N_t = 6):
# 3-D tensor maps (one TMA per k-major operand, SQOC_TMA3D) and Hermitian mirror-tile skipping (SQOC_HERM).
mkdir -p gpurun_out
for cfg in "0 0" "1 0" "0 1" "1 1"; do
  set -- $cfg
  echo "tma3d=$1 herm=$2 $(SQOC_DEBUG=1 SQOC_TMA3D=$1 SQOC_HERM=$2 python tools/gemm_stats.py 3 6 sequential 2 2>&1 | tail -2 | tr '\n' ' ')"
done
