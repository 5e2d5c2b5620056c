#!/bin/bash
# LSTM M = 128: x(t) W + b inside the MMA (XM, default) vs in the epilogue (tools/dbg/libelmrnn_noxm.so)
mkdir -p gpurun_out
python -m paper_1911_13252_b200.build > /dev/null
timeout 1200 python -m pytest tests -m gpu -q -x -k "lstm or tc or readout or staging or c5 or well_cond" 2>&1 | tail -3
for rep in 1 2; do for v in "" tools/dbg/libelmrnn_noxm.so; do
  for a in "lstm 128 50 2000000 1" "lstm 128 10 2000000 1" "lstm 128 30 1000000 4" "lstm 256 50 4000000 1"; do echo -n "$v "; ELMRNN_LIB=$v timeout 300 python tools/prof.py build $a 3; done
done; done 2>&1 | tee gpurun_out/lstm128_ab.jsonl
