#!/bin/bash
# Dense-path (SQOC_SPARSE=0) determinism check: tools/sparse_dense_vs_oracle.py (dense vs sparse only) N times
# under the environment given as arguments, e.g.  bash tools/race_ab.sh 6 SQOC_PT_TRACE=0
n=$1; shift
export SKIP_ORACLE=1
for r in $(seq 1 $n); do echo "$* $(env "$@" python tools/sparse_dense_vs_oracle.py 4 2>&1 | tail -1 | cut -c1-260)"; done
