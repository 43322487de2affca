#!/bin/bash
# Round profiling recipe (run on the GPU box from the repo root):
#   plain bench line, launch list of the same command, one full capture of the dominant kernel.
set -u
mkdir -p gpurun_out
python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
rc=$?
echo "bench rc=$rc"; cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err
if [ $rc -eq 0 ]; then
  python bench.py --steps 2 --warmup 3 --skip-cpu > gpurun_out/bench_plain2.json 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv \
      python bench.py --steps 2 --warmup 3 --skip-cpu > /dev/null 2>&1
  echo "launch list rc=$?"
fi
