#!/bin/bash
# microbenchmarks: reflector-chain latencies and the WY panel alone (one warp)
cd "$(dirname "$0")"
mkdir -p ../../gpurun_out
for b in refl_lat panel_bench; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -I ../../include -I ../../paper_1911_13252_b200/csrc -o /tmp/$b $b.cu -lcuda && /tmp/$b
done 2>&1 | tee ../../gpurun_out/ubench.log
