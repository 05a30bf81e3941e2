#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_counts.py -m "gpu and not slow" -q -x 2>&1 | tail -3
timeout 600 python tools/pass_sweep.py --config c4 --steps 5 "hydro_kernel=0"
mkdir -p gpurun_out/r2
timeout 900 python bench.py --steps 10 --warmup 3 --symmetric 0 --no-cpu-baseline > gpurun_out/r2/bench_c4_icentric.json 2>&1; tail -c 600 gpurun_out/r2/bench_c4_icentric.json
bash tools/gpu_sanitize.sh
