#!/bin/bash
# ncu --set full (with source) of the pair kernels of one c4 substep: $1 = kernel regex, $2 = report name
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1500 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"$1" -o gpurun_out/$2 python tools/profile_step.py --config ${3:-c4} > gpurun_out/$2.log 2>&1; tail -2 gpurun_out/$2.log
