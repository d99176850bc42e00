#!/bin/bash
# compute-sanitizer memcheck / synccheck / racecheck / initcheck over tools/sanitize_run.py
# (every kernel family, small shapes); summaries to gpurun_out/sanitizer.txt.
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
out=gpurun_out/sanitizer.txt
: > "$out"
for t in memcheck synccheck racecheck initcheck; do
  timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool $t --print-limit 20 python tools/sanitize_run.py \
    > gpurun_out/san_$t.txt 2>&1
  rc=$?
  {
    echo "== compute-sanitizer --tool $t python tools/sanitize_run.py  (exit $rc)"
    grep -v "^=========     \|Host Frame" gpurun_out/san_$t.txt
    echo
  } >> "$out"
done
cat "$out"
