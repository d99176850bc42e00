#!/bin/bash
# GPU box: whole GPU suite (stop at first failure) + bench lines of the main configs.
#   tools/gpu/quick.sh <tag> [pytest -k expr]
t=${1:-q}; k=${2:-}
cd "$GRAFT_REPO_ROOT"
o=gpurun_out; mkdir -p $o
python -m paper_2406_06220_b200.build > $o/${t}_build.log 2>&1 || { echo BUILD FAILED; tail -20 $o/${t}_build.log; exit 1; }
if [ -n "$k" ]; then
  timeout 1500 python -m pytest tests -x -q -m gpu -s -k "$k" > $o/${t}_gputest.log 2>&1; echo "gpu tests rc=$?"
else
  timeout 1500 python -m pytest tests -x -q -m gpu -s > $o/${t}_gputest.log 2>&1; echo "gpu tests rc=$?"
fi
tail -15 $o/${t}_gputest.log
for c in fc-rnnt fc-tdt stateless-b512; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > $o/${t}_bench_$c.json 2> $o/${t}_bench_$c.err
  echo "$c rc=$?"; python - $o/${t}_bench_$c.json <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(d['config']['workload'], round(d['ms_per_step'],4),'ms', int(d['value']), 'audio-s/s', 'kernel', round(d['roofline'].get('kernel_ms',0),4), d.get('decode_stats',{}).get('labels'))
except Exception as e: print('parse fail', e)
PY
done
