#!/bin/bash
# Same-box A/B of the slice-sequential cfg 3 schedule options (N_t = 6): U_j history and the all-sparse
# derivative chain (env SQOC_UHIST / SQOC_SPCHAIN), each printed as one gemm_stats line.
mkdir -p gpurun_out
for cfg in "0 0" "1 0" "0 1" "1 1"; do
  set -- $cfg
  echo "uhist=$1 spchain=$2 $(SQOC_UHIST=$1 SQOC_SPCHAIN=$2 python tools/gemm_stats.py 3 6 sequential 2)"
done
