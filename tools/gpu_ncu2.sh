#!/bin/bash
# ncu --set full (with source) of the first kernel whose DEMANGLED name matches $1 on c4: bash tools/gpu_ncu2.sh REGEX NAME k=v ...
python -c "import __graft_entry__ as g; g.build()" || exit 1
K="$1"; N="$2"; shift 2
timeout 1500 ncu --set full --clock-control none --import-source on --profile-from-start off --kernel-name-base demangled -k regex:"$K" -c 1 -o gpurun_out/prof_$N python tools/profile_step.py --config c4 --set "$@" > gpurun_out/ncu_$N.log 2>&1; tail -2 gpurun_out/ncu_$N.log
python tools/ncu_summary.py gpurun_out/prof_$N.ncu-rep > gpurun_out/ncu_${N}_summary.txt 2>&1
