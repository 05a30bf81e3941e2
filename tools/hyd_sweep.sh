#!/bin/bash
python -c "import __graft_entry__ as g; g.build()"
for v in 0000 1111; do CRK_HYD_VARIANT=$v timeout 600 python bench.py --steps 6 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('var $v', round(d['ms_per_step'],2), d['pass_ms'])"; done
