#!/bin/bash
# cfg 3 slice-sequential schedule (the N_t = 500 bench path) at a few slices: event timing, ncu launch list,
# one full capture each of the persistent GEMM and the two sparse-generator kernels.
set -u
mkdir -p gpurun_out
T="python tools/gemm_stats.py 3 4 sequential"
$T 2 > gpurun_out/gs_cfg3_n4.json 2>&1; echo "gs rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg3_n4.csv $T 1 > /dev/null 2>&1; echo "ll rc=$?"
ncu --set full --clock-control none --import-source on -k regex:zgemm3m_pt -s 20 -c 1 -o gpurun_out/zgemm_pt_cfg3 $T 1 > gpurun_out/ncu_zgemm.log 2>&1; echo "z rc=$?"
ncu --set full --clock-control none --import-source on -k regex:spmm_cols -s 2 -c 1 -o gpurun_out/spmm_cols_cfg3 $T 1 > gpurun_out/ncu_sp.log 2>&1; echo "s rc=$?"
ncu --set full --clock-control none --import-source on -k regex:spmm_rows -s 2 -c 1 -o gpurun_out/spmm_rows_cfg3 $T 1 > gpurun_out/ncu_sp2.log 2>&1; echo "s2 rc=$?"
ncu --set full --clock-control none --import-source on -k regex:sp_trace -s 1 -c 1 -o gpurun_out/sp_trace_cfg3 $T 1 > gpurun_out/ncu_sp3.log 2>&1; echo "s3 rc=$?"
ls -la gpurun_out
