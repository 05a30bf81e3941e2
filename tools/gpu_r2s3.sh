#!/bin/bash
# round-2 session-3 measurement set (outputs under gpurun_out/r2s3/): full GPU test suite, smoke, bench
# (c4) + reference arm, launch list, executed-FP32/DRAM counters, ncu --set full of the dominant kernels
mkdir -p gpurun_out/r2s3
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -2
if [ "$1" != "nobench" ]; then
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r2s3/bench_c4.json 2> gpurun_out/r2s3/bench_c4.err; tail -c 4000 gpurun_out/r2s3/bench_c4.json
fi
if [ "$1" == "full" ]; then
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2s3/bench_ref_c4.json 2> gpurun_out/r2s3/bench_ref.err; tail -c 1500 gpurun_out/r2s3/bench_ref_c4.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/r2s3/launches_c4.csv python tools/profile_step.py --config c4 > /dev/null 2>&1
python tools/launches.py gpurun_out/r2s3/launches_c4.csv > gpurun_out/r2s3/launches_c4_summary.txt; cat gpurun_out/r2s3/launches_c4_summary.txt
M=$(python tools/ncu_fp32.py --metrics)
timeout 900 ncu --metrics $M --clock-control none --profile-from-start off -k regex:"grav_pipe|pair_kernel|list_kernel" -o gpurun_out/r2s3/fp32 python tools/profile_step.py --config c4 > gpurun_out/r2s3/fp32.log 2>&1
python tools/ncu_fp32.py gpurun_out/r2s3/fp32.ncu-rep gpurun_out/r2s3/ncu_fp32.json
timeout 1500 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"grav_pipe|list_kernel|GeoPass|k_entry_masks|k_lists" -c 6 -o gpurun_out/r2s3/prof_full python tools/profile_step.py --config c4 > gpurun_out/r2s3/ncu_full.log 2>&1; tail -1 gpurun_out/r2s3/ncu_full.log
python tools/ncu_summary.py gpurun_out/r2s3/prof_full.ncu-rep > gpurun_out/r2s3/ncu_full_summary.txt 2>&1
timeout 3000 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
fi
