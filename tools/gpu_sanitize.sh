#!/bin/bash
# NOTE: compute-sanitizer is closed on the GPU pool since round 2 session 3 (runs exit 86).
# compute-sanitizer on config 1 (outputs under gpurun_out/r2s3/)
mkdir -p gpurun_out/r2s3
python -c "import __graft_entry__ as g; g.build()" || exit 1
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize.py > gpurun_out/r2s3/sanitizer_$tool.txt 2>&1
  echo "$tool rc=$?"; tail -3 gpurun_out/r2s3/sanitizer_$tool.txt
done
