# unequal groups: GPU suite + A/B (group plan on / off), RNN-T and TDT
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gp_gputest.txt 2>&1
tail -2 gpurun_out/gp_gputest.txt
for c in fc-rnnt fc-tdt; do
  for f in "" "--no-group-plan"; do
    timeout 300 python bench.py --config $c --no-cpu-baseline --steps 20 $f 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); s=d['decode_stats']; print('$c $f', round(d['ms_per_step'],4), 'kernel', round(d['roofline']['kernel_ms'],4), 'chain', d['chain_floor']['critical_cluster'], s['window'])"
  done
done
