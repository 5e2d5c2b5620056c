#!/bin/bash
mkdir -p gpurun_out
python -m paper_1911_13252_b200.build > /dev/null
for s in "256 4000000" "256 500000" "128 1000000" "512 2000000" "1024 2000000"; do python tools/qr_time.py $s '{}' '{"ELMRNN_MERGE_SMALL": "0"}'; done 2>&1 | tee gpurun_out/qr_ab3.jsonl
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/n500k_launches2.csv python bench.py --config C4 --n 500000 --profile --steps 1 --warmup 1 > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -k "tsqr or solve or wy or virtual or multi or train" 2>&1 | tail -3
