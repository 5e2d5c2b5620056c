#!/bin/bash
# Every bench configuration on one GPU (dev tool): one JSON line each in gpurun_out/bench_all.jsonl
mkdir -p gpurun_out; : > gpurun_out/bench_all.jsonl
for c in C4 C1 C2j C2n C2n_ef C3gru C3fc C3lstm_diag C3gru_diag C3fc_eq8 C5lstm1024 C5gru1024; do
  timeout 900 python bench.py --config $c 2>> gpurun_out/bench_all.err | tail -1 >> gpurun_out/bench_all.jsonl
done
timeout 900 python bench.py --config C4 --weight-grid 1 2>> gpurun_out/bench_all.err | tail -1 >> gpurun_out/bench_all.jsonl
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 2>> gpurun_out/bench_all.err | tail -1 >> gpurun_out/bench_all.jsonl
wc -l gpurun_out/bench_all.jsonl
