#!/bin/bash
# Round evidence on one GPU box: the GPU suite, smoke, every bench line + ncu
# launch list + one ncu --set full decode capture + timeline (collect_profiles.sh),
# and the on-the-fly projection A/B lines (otf_run.sh).
t=${1:-r02}
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/${t}_gputest.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${t}_smoke.txt 2>&1
bash tools/collect_profiles.sh $t
bash tools/gpu/otf_run.sh ${t}otf
