#!/bin/bash
# wide builders: N = 256 chunk-pair MMA units vs N = 128 (ELMRNN_WIDE_PAIR=0), parity + timing
mkdir -p gpurun_out
python -m paper_1911_13252_b200.build > /dev/null
timeout 900 python -m pytest tests -m gpu -q -x -k "wide or c5 or well_cond or readout or x_staging" 2>&1 | tail -3
for rep in 1 2; do
for v in 1 0; do
  for a in "gru 1024 10 2000000 1" "gru 512 10 2000000 1" "gru 384 10 1000000 1"; do
    echo -n "pair=$v "; ELMRNN_TESTING=1 ELMRNN_WIDE_PAIR=$v timeout 300 python tools/prof.py build $a 3
  done
done
done 2>&1 | tee gpurun_out/wide_ab.jsonl
