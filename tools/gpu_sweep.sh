#!/bin/bash
# build + per-pass sweep of crk_params variants on a config: bash tools/gpu_sweep.sh CONFIG "k=v ..." ...
python -c "import __graft_entry__ as g; g.build()" || exit 1
C="$1"; shift
timeout 1500 python tools/pass_sweep.py --config $C --steps 5 "$@"
