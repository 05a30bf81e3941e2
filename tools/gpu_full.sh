#!/bin/bash
# build + smoke, full GPU tests, bench (with cpu baseline), reference arm, launch list, ncu full of the
# pair kernels (+ per-pass traffic JSON).  Outputs under gpurun_out/.
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -2
timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -3
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -c 4000 gpurun_out/bench.json; tail -3 gpurun_out/bench.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; tail -c 1500 gpurun_out/bench_ref.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches.csv python tools/profile_step.py --config c4 > /dev/null 2>&1
python tools/launches.py gpurun_out/launches.csv | tee gpurun_out/launches_summary.txt
timeout 1500 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"grav_pipe|pair_kernel|list_kernel" -o gpurun_out/prof_full python tools/profile_step.py --config c4 > gpurun_out/ncu_full.log 2>&1; tail -1 gpurun_out/ncu_full.log
python tools/make_traffic.py gpurun_out/prof_full.ncu-rep gpurun_out/ncu_traffic.json > /dev/null
python tools/ncu_summary.py gpurun_out/prof_full.ncu-rep > gpurun_out/ncu_full_summary.txt
