#!/bin/bash
# launch list (per-kernel device times, ncu, cold-cache serialised) of one c4 substep: bash tools/gpu_launches.sh NAME [k=v ...]
python -c "import __graft_entry__ as g; g.build()" || exit 1
N="$1"; shift
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches_$N.csv python tools/profile_step.py --config c4 --set "$@" > /dev/null 2>&1
python tools/launches.py gpurun_out/launches_$N.csv > gpurun_out/launches_${N}_summary.txt; cat gpurun_out/launches_${N}_summary.txt
