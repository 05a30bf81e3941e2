#!/bin/bash
# iteration check on the GPU box: build, selected GPU tests, per-pass sweep of solver options on c4
#   bash tools/gpu_iter.sh "<pytest -k expr or test files>" "opt=v ..." "opt=v ..." ...
python -c "import __graft_entry__ as g; g.build()" || exit 1
T="$1"; shift
if [ -n "$T" ]; then eval "timeout 1200 python -m pytest $T -q -x" 2>&1 | tail -15; fi
if [ "$#" -gt 0 ]; then timeout 900 python tools/pass_sweep.py --config c4 --steps 5 "$@"; fi
