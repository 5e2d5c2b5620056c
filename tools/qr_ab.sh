#!/bin/bash
# TSQR A/B: default lib vs tools/dbg variants (interleaved, 2 rounds) + the TSQR GPU tests.
mkdir -p gpurun_out
python -m paper_1911_13252_b200.build > /dev/null
for rep in 1 2; do
for s in "256 4000000" "128 1000000" "512 2000000" "1024 2000000" "64 100000"; do
for v in "" $(ls tools/dbg/libelmrnn_*.so 2>/dev/null | grep -v trace); do
    echo -n "$v "; ELMRNN_LIB=$v timeout 300 python tools/prof.py qr $s 3
done
done
done 2>&1 | tee gpurun_out/qr_ab.jsonl
timeout 900 python -m pytest tests -m gpu -q -x -k "tsqr or solve or wy or virtual or multi or train" 2>&1 | tail -3
