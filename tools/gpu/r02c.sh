#!/bin/bash
cd "$GRAFT_REPO_ROOT"
o=gpurun_out
touch paper_2406_06220_b200/libll.so   # prebuilt here: do not rebuild on the box
bash tools/gpu/ab.sh paper_2406_06220_b200/libll_base.so paper_2406_06220_b200/libll.so > $o/r02c_ab.txt 2>&1
cat $o/r02c_ab.txt
timeout 1200 python -m pytest tests -q -m gpu -x -s -k "scores or production_kernel or fc_random or fc_rnnt_planted or fc_tdt_planted or schedules or determinism" > $o/r02c_tests.log 2>&1; echo "tests rc=$?"; tail -15 $o/r02c_tests.log
