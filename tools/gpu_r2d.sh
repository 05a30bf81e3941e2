#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_counts.py -m "gpu and not slow" -q -x 2>&1 | tail -5
timeout 1500 python -m pytest tests/test_domain.py -m gpu -q -x 2>&1 | tail -5
timeout 600 python tools/pass_sweep.py --config c4 --steps 5 "hydro_kernel=0" "hydro_kernel=1"
timeout 1200 python tools/decomp_bench.py --P 8 --reps 3 --config lat:128,128,128:0.1:16522 2>&1 | tail -1
timeout 600 python tools/pass_sweep.py --config lat:128,128,128:0.1:16522 --steps 5 "hydro_kernel=0"
