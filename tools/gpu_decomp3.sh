#!/bin/bash
# decomposition changes: domain GPU tests (incl. the slow weak-scaled ones), then per-rank emulated times
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 2400 python -m pytest tests/test_domain.py tests/test_bench.py -q -x -m gpu 2>&1 | tail -3
mkdir -p gpurun_out/r2s3b
timeout 1200 python tools/decomp_bench.py --P 2 --reps 3 2>&1 | tail -1 > gpurun_out/r2s3b/decomposed_P2_c4.json; cut -c1-200 gpurun_out/r2s3b/decomposed_P2_c4.json
timeout 1200 python tools/decomp_bench.py --P 4 --reps 3 2>&1 | tail -1 > gpurun_out/r2s3b/decomposed_P4_c4.json; cut -c1-200 gpurun_out/r2s3b/decomposed_P4_c4.json
timeout 1200 python tools/decomp_bench.py --P 8 --reps 3 --config lat:128,128,128:0.1:16522 2>&1 | tail -1 > gpurun_out/r2s3b/decomposed_P8_2x128cubed.json; cut -c1-200 gpurun_out/r2s3b/decomposed_P8_2x128cubed.json
