set -x
cd "$GRAFT_REPO_ROOT"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m paper_2406_06220_b200.build > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests -x -q -m gpu -s -k "production_kernel or config4_random or cat_dog or schedules or guard or frame_looping_cat" > gpurun_out/gputest_new.log 2>&1; echo "new tests rc=$?"
tail -30 gpurun_out/gputest_new.log
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/bench_r02a.json 2> gpurun_out/bench_r02a.err; echo "bench rc=$?"
cat gpurun_out/bench_r02a.json | head -c 3000
