python -c "import __graft_entry__ as g; g.build()" > /dev/null
CRK_DIST_BACKEND=gloo CRK_SHARE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 --steps 3 --warmup 3 > gpurun_out/multi2.json 2> gpurun_out/multi2.err; tail -c 1500 gpurun_out/multi2.json; tail -3 gpurun_out/multi2.err
timeout 600 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c3.json 2>/dev/null; tail -c 600 gpurun_out/bench_c3.json
timeout 600 python bench.py --config c2z --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2z.json 2>/dev/null; tail -c 600 gpurun_out/bench_c2z.json
