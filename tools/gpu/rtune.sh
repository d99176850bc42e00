# rows-per-group tuning under length-ranked groups (config 4 stateless, sweep LSTM)
for R in 8 12 16 20 24; do
  timeout 600 python bench.py --config stateless-b512 --no-cpu-baseline --steps 5 --warmup 3 --group-rows $R 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('stateless R=$R', round(d['ms_per_step'],3), round(d['value']), d['decode_stats']['window'])"
done
for R in 4 6 8 10 12; do
  timeout 600 python bench.py --config sweep-rnnt --no-cpu-baseline --steps 3 --warmup 3 --group-rows $R 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('sweep-rnnt R=$R', round(d['ms_per_step'],3), round(d['value']))"
done
