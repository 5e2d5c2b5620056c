#!/bin/bash
# TSQR A/B: default lib vs tools/dbg variants at the C4/C3/C5 shapes, plus the trace.
mkdir -p gpurun_out
python -m paper_1911_13252_b200.build > /dev/null
for rep in 1 2; do
for v in "" $(ls tools/dbg/libelmrnn_*.so | grep -v trace); do
  for s in "256 4000000" "128 1000000" "512 2000000" "1024 2000000" "64 100000"; do
    echo -n "$v "; ELMRNN_LIB=$v timeout 300 python tools/prof.py qr $s 3
  done
done
done 2>&1 | tee gpurun_out/qr_ab.jsonl
bash tools/qr_trace.sh 256 4000000 > gpurun_out/qtrace_256.txt 2>&1; tail -18 gpurun_out/qtrace_256.txt
timeout 900 python -m pytest tests -m gpu -q -x -k "tsqr or solve or wy or virtual or multi or train" 2>&1 | tail -3
