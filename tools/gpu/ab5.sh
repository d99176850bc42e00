timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/ab5_gputest.txt 2>&1
tail -2 gpurun_out/ab5_gputest.txt
for c in fc-tdt fc-rnnt; do bash tools/ab.sh $c paper_2406_06220_b200/libll_base.so paper_2406_06220_b200/libll.so; done
