#!/bin/bash
# GPU box: the whole GPU suite, bench lines of configs 2 / 4, and the projection
# GEMM's per-launch times under ncu (launch list only).
t=${1:-g}
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/${t}_gputest.txt 2>&1
tail -2 gpurun_out/${t}_gputest.txt
for c in fc-rnnt stateless-b512; do
  timeout 300 python bench.py --config $c --no-cpu-baseline > gpurun_out/${t}_bench_$c.json 2> gpurun_out/${t}_bench_$c.err
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${t}_gemm.csv \
  python bench.py --config stateless-b512 --steps 2 --warmup 1 --no-cpu-baseline --clock-window 0 > /dev/null 2>&1
