#!/bin/bash
# A/B of two prebuilt libraries on the bench configs (GPU box):
#   tools/gpu/ab.sh <libA> <libB> [configs...]   -> one line per (lib, config, repeat)
cd "$GRAFT_REPO_ROOT"
A=$1; B=$2; shift 2
cfgs=${@:-fc-rnnt fc-tdt stateless-b512}
for rep in 1 2; do
  for lib in $A $B; do
    for c in $cfgs; do
      LL_LIB_PATH=$lib timeout 300 python bench.py --config $c --steps 30 --warmup 3 --no-cpu-baseline --clock-window 0 2>/dev/null \
        | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib'.split('/')[-1], '$c', round(d['ms_per_step'],4), 'ms  kernel', round(d['roofline']['kernel_ms'],4), 'labels', d['decode_stats']['labels'])"
    done
  done
done
