#!/bin/bash
# per-rank emulated decomposed-substep times with the current kernels (profiles/r02/decomposed_*.json)
python -c "import __graft_entry__ as g; g.build()" || exit 1
mkdir -p gpurun_out/r2s3
timeout 600 python tools/pass_sweep.py --config c4 --steps 5 "grav_kernel=0" | tee gpurun_out/r2s3/single_domain.json
timeout 1200 python tools/decomp_bench.py --P 2 --reps 3 2>&1 | tail -1 > gpurun_out/r2s3/decomposed_P2_c4.json; cat gpurun_out/r2s3/decomposed_P2_c4.json | cut -c1-300
timeout 1200 python tools/decomp_bench.py --P 4 --reps 3 2>&1 | tail -1 > gpurun_out/r2s3/decomposed_P4_c4.json; cat gpurun_out/r2s3/decomposed_P4_c4.json | cut -c1-300
timeout 1200 python tools/decomp_bench.py --P 8 --reps 3 --config lat:128,128,128:0.1:16522 2>&1 | tail -1 > gpurun_out/r2s3/decomposed_P8_2x128cubed.json; cat gpurun_out/r2s3/decomposed_P8_2x128cubed.json | cut -c1-300
timeout 600 python tools/pass_sweep.py --config lat:128,128,128:0.1:16522 --steps 5 "grav_kernel=0" | tee gpurun_out/r2s3/single_domain_128.json
