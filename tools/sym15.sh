#!/bin/bash
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "full_chain or kicks" 2>&1 | tail -2
for s in 1 5; do timeout 600 python bench.py --steps 6 --warmup 3 --no-cpu-baseline --symmetric $s 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('sym $s', round(d['ms_per_step'],2), d['pass_ms'])"; done
