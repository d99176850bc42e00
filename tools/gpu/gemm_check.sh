#!/bin/bash
# GPU box: suite + bench lines + the projection GEMM's launch times (config 4, config 2).
t=${1:-g}
cd "$GRAFT_REPO_ROOT"
touch paper_2406_06220_b200/libll.so
bash tools/gpu/tjrun.sh $t > /dev/null 2>&1
tail -2 gpurun_out/${t}_gputest.log
for c in fc-rnnt fc-tdt stateless-b512; do python -c "
import json; d=json.loads(open(\"gpurun_out/${t}_bench_$c.json\").read().strip().splitlines()[-1]); s=d[\"decode_stats\"]; print(\"$c\", round(d[\"ms_per_step\"],4), int(d[\"value\"]), 'kernel', round(d['roofline']['kernel_ms'],4), s[\"group_rows\"], s[\"window\"])"; done
for c in stateless-b512 fc-rnnt; do
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${t}_gemm_$c.csv \
  python bench.py --config $c --steps 1 --warmup 1 --no-cpu-baseline --clock-window 0 > /dev/null 2>&1
python - gpurun_out/${t}_gemm_$c.csv <<'PY'
import csv, sys, collections
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]; ki = h.index("Kernel Name"); vi = h.index("Metric Value")
d = collections.defaultdict(list)
for r in rows[1:]:
    d[r[ki][:60]].append(float(r[vi]))
for k, v in d.items(): print(f"  {k:60s} n={len(v):3d} median {sorted(v)[len(v)//2]/1000:.3f} us-> ms")
PY
done
