#!/bin/bash
python -c "import __graft_entry__ as g; g.build()"
for c in c2z c3; do timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null > gpurun_out/bench_$c.json; python -c "
import json; d=json.loads(open('gpurun_out/bench_$c.json').read().strip().splitlines()[-1]); print('$c', round(d['ms_per_step'],2), 'pairs/s %.3e' % d['value'], d['pass_ms'], d['pairs'])"; done
