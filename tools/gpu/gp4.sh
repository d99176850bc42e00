# length-ranked groups for multi-group decodes: GPU suite + A/B on config 4 and the sweep
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gp4_gputest.txt 2>&1
tail -2 gpurun_out/gp4_gputest.txt
for c in stateless-b512 sweep-rnnt; do
  for f in "" "--no-group-plan"; do
    timeout 600 python bench.py --config $c --no-cpu-baseline --steps 5 --warmup 3 $f 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c $f', round(d['ms_per_step'],4), round(d['value']))"
  done
done
