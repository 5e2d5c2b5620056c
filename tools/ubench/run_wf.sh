#!/bin/bash
cd "$(dirname "$0")"; mkdir -p ../../gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/wf warp_fold.cu && /tmp/wf 2>&1 | tee ../../gpurun_out/warp_fold.log
