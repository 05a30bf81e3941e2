#!/bin/bash
# build, selected tests, sweep, and an ncu --set full capture of kernels matching $1 (regex) on c4
python -c "import __graft_entry__ as g; g.build()" || exit 1
K="$1"; T="$2"; shift 2
if [ -n "$T" ]; then timeout 1200 python -m pytest $T -q -x 2>&1 | tail -5; fi
if [ "$#" -gt 0 ]; then timeout 900 python tools/pass_sweep.py --config c4 --steps 5 "$@"; fi
if [ -n "$K" ]; then
timeout 1200 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"$K" -c 4 -o gpurun_out/prof_k python tools/profile_step.py --config c4 > gpurun_out/ncu_k.log 2>&1; tail -2 gpurun_out/ncu_k.log
python tools/ncu_summary.py gpurun_out/prof_k.ncu-rep > gpurun_out/ncu_k_summary.txt 2>&1
fi
ncu --query-metrics 2>/dev/null | grep -E "sass_thread_inst_executed_op_f|inst_executed_op_f" | head -20 > gpurun_out/ncu_fp_metrics.txt
