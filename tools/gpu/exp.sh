#!/bin/bash
# GPU box: timeline of fc-rnnt for the base build and experiment variants.  tools/gpu/exp.sh <tag> exp1 exp2 ...
t=$1; shift
cd "$GRAFT_REPO_ROOT"
python tools/timeline.py fc-rnnt --tj > gpurun_out/${t}_base.txt 2>&1
for e in "$@"; do python tools/timeline.py fc-rnnt --tj --$e > gpurun_out/${t}_$e.txt 2>&1; done
for f in gpurun_out/${t}_*.txt; do echo "== $f"; sed -n 3,20p $f; done
