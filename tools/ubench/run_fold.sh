#!/bin/bash
cd "$(dirname "$0")"
mkdir -p ../../gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -DELM_QR_TRACE -I ../../include -I ../../paper_1911_13252_b200/csrc -o /tmp/fb fold_bench.cu -lcuda
for n in 21 65 129; do /tmp/fb $n; done 2>&1 | tee ../../gpurun_out/fold_bench.log
