#!/bin/bash
# GPU box: rebuild, the whole GPU suite, smoke, bench lines (default + sweep).
#   tools/gpu/full_check.sh <tag>      -> gpurun_out/<tag>_*
t=${1:-chk}
cd "$GRAFT_REPO_ROOT"
o=gpurun_out
mkdir -p $o
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $o/${t}_smi.txt
python -m paper_2406_06220_b200.build > $o/${t}_build.log 2>&1 || { echo BUILD FAILED; tail -20 $o/${t}_build.log; exit 1; }
timeout 2400 python -m pytest tests -q -m gpu -s --durations=15 > $o/${t}_gputest.log 2>&1; echo "gpu tests rc=$?"
tail -25 $o/${t}_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $o/${t}_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 $o/${t}_smoke.log
timeout 600 python bench.py --steps 20 --warmup 3 > $o/${t}_bench_fc-rnnt.json 2> $o/${t}_bench_fc-rnnt.err; echo "bench rc=$?"
head -c 1500 $o/${t}_bench_fc-rnnt.json; echo
timeout 900 python bench.py --config sweep-rnnt --steps 3 --warmup 1 --no-cpu-baseline > $o/${t}_bench_sweep-rnnt.json 2> $o/${t}_bench_sweep-rnnt.err; echo "sweep rc=$?"
head -c 1500 $o/${t}_bench_sweep-rnnt.json; echo; tail -3 $o/${t}_bench_sweep-rnnt.err
