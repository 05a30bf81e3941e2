#!/bin/bash
# session baseline: build, per-pass sweep on c4, ncu --set full (with source) of the hot pass kernels
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python tools/pass_sweep.py --config c4 --steps 5 "grav_kernel=0"
timeout 1500 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"grav_pipe|list_kernel|pair_kernel" -c 7 -o gpurun_out/prof_base python tools/profile_step.py --config c4 > gpurun_out/ncu_base.log 2>&1; tail -2 gpurun_out/ncu_base.log
python tools/ncu_summary.py gpurun_out/prof_base.ncu-rep > gpurun_out/ncu_base_summary.txt 2>&1
