#!/bin/bash
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "full_chain or kicks or coincident" 2>&1 | tail -2
for e in "" "CRK_ACC_SCALAR=1"; do env $e timeout 600 python bench.py --steps 6 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('acc [$e]', round(d['ms_per_step'],2), d['pass_ms'])"; done
