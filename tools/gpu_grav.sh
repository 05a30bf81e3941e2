#!/bin/bash
# gravity kernel iteration: build, gravity parity/count tests of the variants, sweep on c4
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_counts.py tests/test_domain.py tests/test_subcycle.py -q -x -k "symmetric_variants or pipe_configurations or decomposed_substep or skin or kdk or counts_and_full_chain or gravity" 2>&1 | tail -4
timeout 900 python tools/pass_sweep.py --config c4 --steps 5 "$@"
