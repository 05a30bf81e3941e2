#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_counts.py tests/test_subcycle.py -q -x -m "gpu and not slow" 2>&1 | tail -2
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x -m "gpu and slow" -k "c3" 2>&1 | tail -2
python -c "
import sys; sys.path.insert(0,'.')
from gen import make_config; import numpy as np
parts, params = make_config('c3')
import oracle
order, keys, cellm = oracle.sort_order(parts, params)
c = np.bincount(cellm[order] if cellm.shape[0]==parts['x'].shape[0] else cellm)
print('c3 max particles per cell', c.max(), 'cells > 256:', (c > 256).sum())
" 2>&1 | tail -2
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_sortfix.json 2> gpurun_out/bench_sortfix.err
python -c "
import json; d=json.loads(open('gpurun_out/bench_sortfix.json').read().strip().splitlines()[-1])
print(d['ms_per_step'], d['pass_ms'], d['e2e'])"
