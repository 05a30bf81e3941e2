#!/bin/bash
# sanitizers on config 1 (current kernels) + the variant portfolio on c4
bash tools/gpu_sanitize.sh
timeout 1500 python tools/variant_portfolio.py --config c4 --out gpurun_out/r2s2/variant_portfolio.json | tail -15
