#!/bin/bash
python -c "import __graft_entry__ as g; g.build()"
cat > /tmp/p.py <<'PY'
import sys, torch
sys.path.insert(0, '.')
from gen import make_config
from paper_2310_16122_b200 import Particles, Solver
parts, params = make_config('c2z')
for sym in (1, 5):
    params['symmetric'] = sym
    p = Particles.from_host(parts, 'cuda'); s = Solver(params, 0)
    s.substep(p); torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStart(); s.substep(p); torch.cuda.synchronize(); torch.cuda.cudart().cudaProfilerStop()
    s.close()
PY
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"acc_cmp|AccPass" -o gpurun_out/prof_acc python /tmp/p.py > gpurun_out/ncu_acc.log 2>&1; tail -1 gpurun_out/ncu_acc.log
