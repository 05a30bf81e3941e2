#!/bin/bash
# round-2 measurement set (outputs under gpurun_out/r2/): bench (c4) + reference arm, the launch
# list, executed-FP32/DRAM counters of the pass kernels, an ncu --set full capture of the dominant
# kernels, the slow parity tests, per-rank decomposed times
mkdir -p gpurun_out/r2
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -2
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r2/bench_c4.json 2> gpurun_out/r2/bench_c4.err; tail -c 3000 gpurun_out/r2/bench_c4.json
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2/bench_ref_c4.json 2> gpurun_out/r2/bench_ref.err; tail -c 1500 gpurun_out/r2/bench_ref_c4.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/r2/launches_c4.csv python tools/profile_step.py --config c4 > /dev/null 2>&1
python tools/launches.py gpurun_out/r2/launches_c4.csv > gpurun_out/r2/launches_c4_summary.txt; cat gpurun_out/r2/launches_c4_summary.txt
M=$(python tools/ncu_fp32.py --metrics)
timeout 900 ncu --metrics $M --clock-control none --profile-from-start off -k regex:"grav_pipe|pair_kernel|list_kernel" -o gpurun_out/r2/fp32 python tools/profile_step.py --config c4 > gpurun_out/r2/fp32.log 2>&1
python tools/ncu_fp32.py gpurun_out/r2/fp32.ncu-rep gpurun_out/r2/ncu_fp32.json
timeout 1500 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"grav_pipe|list_kernel" -c 3 -o gpurun_out/r2/prof_full python tools/profile_step.py --config c4 > gpurun_out/r2/ncu_full.log 2>&1; tail -1 gpurun_out/r2/ncu_full.log
python tools/ncu_summary.py gpurun_out/r2/prof_full.ncu-rep > gpurun_out/r2/ncu_full_summary.txt 2>&1
if [ "$1" != "quick" ]; then
timeout 2400 python -m pytest tests/test_gpu_parity.py tests/test_domain.py -m "gpu and slow" -q -x 2>&1 | tail -3
for P in 2 4; do timeout 1200 python tools/decomp_bench.py --P $P --reps 3 > gpurun_out/r2/decomp_P$P.json 2>&1; tail -1 gpurun_out/r2/decomp_P$P.json; done
timeout 1200 python tools/decomp_bench.py --P 8 --reps 3 --config lat:128,128,128:0.1:16522 > gpurun_out/r2/decomp_P8_128.json 2>&1; tail -1 gpurun_out/r2/decomp_P8_128.json
fi
