#!/bin/bash
# A/B timing of library variants: tools/ab.sh <config> <lib1> [lib2 ...]  (GPU box)
cfg=$1; shift
for lib in "$@"; do
  for rep in 1 2; do
    LL_LIB_PATH=$lib timeout 300 python bench.py --config $cfg --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', '$cfg', round(d['ms_per_step'],4), 'ms', d['roofline']['kernel_ms'])"
  done
done
