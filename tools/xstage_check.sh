#!/bin/bash
# a1 / f3 check: the GPU suite, then build timings at M = 256: default (X staged,
# last K-slice bypassing the staging area) vs nohold (unstaged, round-2 layout)
mkdir -p gpurun_out
python -m paper_1911_13252_b200.build > /dev/null
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > gpurun_out/xs_tests.log
for rep in 1 2 3; do
for v in "" tools/dbg/libelmrnn_nohold.so; do
  for args in "lstm 256 50 4000000 1" "lstm 128 50 2000000 1"; do
    echo -n "$v "; ELMRNN_LIB=$v timeout 300 python tools/prof.py build $args 3
  done
done
done > gpurun_out/xs_times.jsonl 2>&1
cat gpurun_out/xs_tests.log gpurun_out/xs_times.jsonl
