#!/bin/bash
cd "$(dirname "$0")"; mkdir -p ../../gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/fv fold_var.cu && /tmp/fv 2>&1 | tee ../../gpurun_out/fold_var.log
cd ../..; python -m paper_1911_13252_b200.build > /dev/null
timeout 900 python -m pytest tests -m gpu -q -x -k "solve or ridge or nonfinite or virtual or full_config or tsqr or train or smoke" 2>&1 | tail -2
for c in C1 C2j; do timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch3_$c.csv python bench.py --config $c --profile --steps 1 --warmup 1 > /dev/null 2>&1; done
