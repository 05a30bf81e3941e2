#!/bin/bash
# executed-FP32/DRAM counters and ncu --set full of the dominant kernels with the final kernels (gpurun_out/final/)
mkdir -p gpurun_out/final
python -c "import __graft_entry__ as g; g.build()" || exit 1
M=$(python tools/ncu_fp32.py --metrics)
timeout 900 ncu --metrics $M --clock-control none --profile-from-start off -k regex:"grav_pipe|pair_kernel|list_kernel" -o gpurun_out/final/fp32 python tools/profile_step.py --config c4 > gpurun_out/final/fp32.log 2>&1
python tools/ncu_fp32.py gpurun_out/final/fp32.ncu-rep gpurun_out/final/ncu_fp32.json
timeout 1500 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"grav_pipe|list_kernel|GeoPass|k_entry_masks|k_lists" -c 6 -o gpurun_out/final/prof_full python tools/profile_step.py --config c4 > gpurun_out/final/ncu_full.log 2>&1; tail -1 gpurun_out/final/ncu_full.log
python tools/ncu_summary.py gpurun_out/final/prof_full.ncu-rep > gpurun_out/final/ncu_full_summary.txt 2>&1
