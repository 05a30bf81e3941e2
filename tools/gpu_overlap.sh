#!/bin/bash
# the overlapped ghost exchange: domain tests, then 2 ranks sharing the GPU over gloo with the overlap forced
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1500 python -m pytest tests/test_domain.py -q -x -m gpu -k "overlap or decomposed_substep or kicks or migration" 2>&1 | tail -3
CRK_DIST_BACKEND=gloo CRK_SHARE_GPU=1 CRK_OVERLAP=1 timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 2 --warmup 3 > gpurun_out/bench_2ranks_gloo_overlap.json 2> gpurun_out/bench_2ranks_gloo_overlap.err
tail -c 1500 gpurun_out/bench_2ranks_gloo_overlap.json; tail -3 gpurun_out/bench_2ranks_gloo_overlap.err
