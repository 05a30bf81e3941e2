#!/bin/bash
# build, fast GPU parity tests, bench on c4, launch list (used with gpurun)
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests -m "gpu and not slow" -q -x 2>&1 | tail -3
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
python -c "
import json; d=json.loads(open('gpurun_out/bench_c4.json').read().strip().splitlines()[-1]); print('ms/step', round(d['ms_per_step'],2), d['pass_ms'], 'frac', round(d['roofline']['frac'],3), 'value %.3e' % d['value'], d['clocks'])"
tail -3 gpurun_out/bench_c4.err
if [ "$1" == "launches" ]; then
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches_c4.csv python tools/profile_step.py --config c4 > /dev/null 2>&1
python tools/launches.py gpurun_out/launches_c4.csv
fi
