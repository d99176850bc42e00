#!/bin/bash
# A/B timing over environment settings: tools/ab_env.sh <config> "ENV=..;" ...   (GPU box)
cfg=$1; shift
for e in "$@"; do
  env $e timeout 300 python bench.py --config $cfg --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); s=d['decode_stats']; print('$e', '$cfg', round(d['ms_per_step'],4), 'ms kernel', round(d['roofline']['kernel_ms'],4), 'rounds', s['joint_rounds'], 'outer', s['outer_steps'])"
done
