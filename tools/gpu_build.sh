#!/bin/bash
# build pass iteration: build, bit-exact build/list parity + counts + decomposition tests, sweep, launch list of the build
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_counts.py tests/test_domain.py tests/test_subcycle.py -q -x -m "gpu and not slow" 2>&1 | tail -3
timeout 900 python tools/pass_sweep.py --config c4 --steps 5 "grav_kernel=0"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches_build.csv python tools/profile_step.py --config c4 > /dev/null 2>&1
python tools/launches.py gpurun_out/launches_build.csv > gpurun_out/launches_build.txt; head -24 gpurun_out/launches_build.txt
