#!/bin/bash
# Same-box A/B of library variants built into tools/bin/variants/*.so (large.cu compiled with different
# -D flags, linked with the same other objects): each is copied over the in-tree library and timed on the
# slice-sequential cfg 3 schedule (N_t = 6) and cfg 4 (N_t = 4); the original library is restored.
set -u
LIB=paper_2309_05884_b200/libsymqoc_b200.so
cp $LIB /tmp/lib_orig.so
for v in "$@"; do
  cp tools/bin/variants/$v.so $LIB
  echo "$v cfg3 $(python tools/gemm_stats.py 3 6 sequential 2 2>&1 | tail -1 | python -c 'import sys,json; d=json.loads(sys.stdin.read()); print(round(d["step_ms"],1), round(d["gemm_ms"],1), round(d["dmma_pipe_frac_gemm"],4))')"
  echo "$v cfg4 $(python tools/gemm_stats.py 4 4 auto 2 2>&1 | tail -1 | python -c 'import sys,json; d=json.loads(sys.stdin.read()); print(round(d["step_ms"],1), round(d["gemm_ms"],1), round(d["dmma_pipe_frac_gemm"],4))')"
done
cp /tmp/lib_orig.so $LIB
