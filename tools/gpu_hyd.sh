#!/bin/bash
# hydro kernel iteration: build, hydro parity/count tests, sweep on c4
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_counts.py tests/test_domain.py tests/test_subcycle.py -q -x -m "gpu and not slow" 2>&1 | tail -4
timeout 900 python tools/pass_sweep.py --config c4 --steps 5 "$@"
