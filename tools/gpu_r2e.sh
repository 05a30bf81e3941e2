#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "one_walk or full_chain" 2>&1 | tail -3
timeout 1200 python tools/decomp_bench.py --P 8 --reps 3 --config lat:128,128,128:0.1:16522 2>&1 | tail -1
timeout 1200 python tools/decomp_bench.py --P 4 --reps 3 2>&1 | tail -1
timeout 1200 python tools/variant_portfolio.py --config c4 --out gpurun_out/r2/variant_portfolio.json 2>&1 | tail -12
timeout 3000 python -m pytest tests/test_domain.py -m "gpu and slow" -q -x 2>&1 | tail -3
