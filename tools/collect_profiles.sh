#!/bin/bash
# Round evidence for profiles/ (GPU box): bench lines, ncu launch list, one
# ncu --set full capture of the decode kernel, per-warp timeline.
#   tools/collect_profiles.sh <tag>      -> gpurun_out/<tag>_*
t=${1:-r02}
o=gpurun_out
for c in fc-rnnt fc-tdt stateless-b512; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 > $o/${t}_bench_$c.json 2> $o/${t}_bench_$c.err
done
timeout 600 python bench.py --config fc-rnnt-4x --steps 10 --warmup 3 > $o/${t}_bench_fc-rnnt-4x.json 2> $o/${t}_bench_fc-rnnt-4x.err
for c in fc-rnnt stateless-b512 fc-rnnt-4x; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --frame-looping --no-cpu-baseline \
    > $o/${t}_bench_${c}_frame-looping.json 2> $o/${t}_bench_${c}_frame-looping.err
done
for c in fc-rnnt fc-tdt; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --schedule batched \
    > $o/${t}_bench_${c}_alg3-batched.json 2> $o/${t}_bench_${c}_alg3-batched.err
done
for c in sweep-rnnt sweep-tdt; do
  timeout 900 python bench.py --config $c --steps 3 --warmup 3 > $o/${t}_bench_$c.json 2> $o/${t}_bench_$c.err
done
# the sweep as B=32 launches (the metric's batch) on 4 concurrent streams
timeout 900 python bench.py --config sweep-rnnt --chunk 32 --streams 4 --steps 3 --warmup 3 --no-cpu-baseline \
  > $o/${t}_bench_sweep-rnnt_b32x4.json 2> $o/${t}_bench_sweep-rnnt_b32x4.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $o/${t}_launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline > $o/${t}_launches.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:decode_kernel -s 2 -c 1 \
  -o $o/${t}_decode python tools/one_decode.py fc-rnnt 3 > $o/${t}_ncu.log 2>&1
timeout 300 python tools/timeline.py fc-rnnt --tj > $o/${t}_timeline.txt 2>&1; timeout 300 python tools/timeline.py fc-tdt --tj >> $o/${t}_timeline.txt 2>&1
