#!/bin/bash
mkdir -p gpurun_out
python -m paper_1911_13252_b200.build > /dev/null
for s in "256 4000000" "128 1000000" "512 2000000" "1024 2000000"; do python tools/qr_time.py $s '{}' '{"ELMRNN_PW_MODE": "0"}'; done 2>&1 | tee gpurun_out/qr_ab2.jsonl
timeout 900 python -m pytest tests -m gpu -q -x -k "tsqr or solve or wy or virtual or multi or train" 2>&1 | tail -3
