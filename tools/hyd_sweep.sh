#!/bin/bash
# CRK_HYD_VARIANT sweep on c4 (digits: geo cor ext acc); usage: hyd_sweep.sh v1 v2 ...
python -c "import __graft_entry__ as g; g.build()"
for v in "$@"; do CRK_HYD_VARIANT=$v timeout 600 python bench.py --steps 6 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('var $v', round(d['ms_per_step'],2), d['pass_ms'])"; done
