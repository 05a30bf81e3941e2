#!/bin/bash
# end-of-session validation: smoke, the whole -m gpu suite, c4 bench, launch list, variant portfolio
mkdir -p gpurun_out/final
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/final/bench_c4.json 2> gpurun_out/final/bench_c4.err; tail -c 600 gpurun_out/final/bench_c4.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/final/launches_c4.csv python tools/profile_step.py --config c4 > /dev/null 2>&1
python tools/launches.py gpurun_out/final/launches_c4.csv > gpurun_out/final/launches_c4_summary.txt; head -3 gpurun_out/final/launches_c4_summary.txt
timeout 1200 python tools/variant_portfolio.py --config c4 --out gpurun_out/final/variant_portfolio.json > gpurun_out/final/variant_portfolio.log 2>&1; tail -3 gpurun_out/final/variant_portfolio.log
timeout 3000 python -m pytest tests -m gpu -q 2>&1 | tail -3
