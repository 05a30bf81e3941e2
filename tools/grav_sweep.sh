#!/bin/bash
python -c "import __graft_entry__ as g; g.build()"
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "c2z" 2>&1 | tail -1
for v in 0 1 2 3; do CRK_GRAV_VARIANT=$v timeout 600 python bench.py --steps 6 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('grav var $v', round(d['ms_per_step'],2), d['pass_ms']['gravity'])"; done
