timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/x8_gputest.txt 2>&1
for r in 1 2 3; do timeout 300 python -m pytest tests/test_gpu_parity.py -q -k "production_kernel" -s 2>&1 | grep -E "g err|passed|failed"; done
timeout 300 python tools/gpu/gerr_debug.py 2>&1 | head -3
for c in fc-rnnt fc-tdt; do bash tools/ab.sh $c paper_2406_06220_b200/libll_base.so paper_2406_06220_b200/libll.so; done
