#!/bin/bash
# decomposed-substep checks: GPU domain tests, per-rank emulated times at P = 1 (single domain), 2, 4, 8
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1200 python -m pytest tests/test_domain.py -m gpu -q -x 2>&1 | tail -5
timeout 600 python tools/pass_sweep.py --config c4 --steps 5 "grav_kernel=0"
for P in 2 4 8; do timeout 1200 python tools/decomp_bench.py --P $P --reps 2 2>&1 | tail -2; done
