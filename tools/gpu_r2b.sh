#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" || exit 1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/pipes tools/micro/pipes.cu && /tmp/pipes
timeout 1800 python -m pytest tests/test_domain.py -m gpu -q -x 2>&1 | tail -5
timeout 600 python tools/pass_sweep.py --config lat:128,128,128:0.1:16522 --steps 5 "grav_kernel=0"
timeout 1200 python tools/decomp_bench.py --P 8 --reps 2 --config lat:128,128,128:0.1:16522 2>&1 | tail -2
timeout 1200 python tools/decomp_bench.py --P 4 --reps 3 2>&1 | tail -2
timeout 2400 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "sampled" 2>&1 | tail -5
