# OTF (on-the-fly projections, Table 3 ablation): parity tests + A/B bench lines
tag=${1:-o2}
timeout 600 python -m pytest tests/test_gpu_otf.py -x -q > gpurun_out/${tag}_test.txt 2>&1
for b in 32 4 1; do
 for pj in precompute on-the-fly; do
  timeout 300 python bench.py --batch $b --projections $pj --no-cpu-baseline --steps 20 > gpurun_out/${tag}_b${b}_${pj}.json 2> gpurun_out/${tag}_b${b}_${pj}.err
 done
done
for pj in precompute on-the-fly; do
  timeout 300 python bench.py --config fc-tdt --projections $pj --no-cpu-baseline --steps 20 > gpurun_out/${tag}_tdt_${pj}.json 2> gpurun_out/${tag}_tdt_${pj}.err
done
