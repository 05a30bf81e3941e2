#!/bin/bash
# FP32 pipe microbenchmark (scalar FFMA vs packed FFMA2), then the quick GPU check (used with gpurun)
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ffma2 tools/micro/ffma2.cu && /tmp/ffma2
bash tools/gpu_hyd.sh "$@"
