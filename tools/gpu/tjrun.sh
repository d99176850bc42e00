#!/bin/bash
# GPU box: GPU suite, TJ timelines, config sweeps, bench lines.   tools/gpu/tjrun.sh <tag>
t=${1:-tj}
cd "$GRAFT_REPO_ROOT"
touch paper_2406_06220_b200/libll.so
timeout 900 python -m pytest tests -x -q -m gpu -s > gpurun_out/${t}_gputest.log 2>&1; echo "gpu tests rc=$?"; tail -3 gpurun_out/${t}_gputest.log
python tools/timeline.py fc-rnnt --tj > gpurun_out/${t}_tl.txt 2>&1; python tools/timeline.py fc-tdt --tj >> gpurun_out/${t}_tl.txt 2>&1
for c in fc-rnnt fc-tdt stateless-b512; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/${t}_bench_$c.json 2> gpurun_out/${t}_bench_$c.err
  python - gpurun_out/${t}_bench_$c.json <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); s=d['decode_stats']
    print(d['config']['workload'], round(d['ms_per_step'],4),'ms', int(d['value']), 'audio-s/s kernel', round(d['roofline'].get('kernel_ms',0),4), 'labels', s.get('labels'), 'R', s.get('group_rows'), 'W', s.get('window'))
except Exception as e: print('parse fail', e)
PY
done
