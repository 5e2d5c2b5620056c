#!/bin/bash
mkdir -p gpurun_out
python -m paper_1911_13252_b200.build > /dev/null
for rep in 1 2; do
python tools/qr_time.py 256 4000000 '{}' '{"ELMRNN_TSQR_WY_ROWS": "48"}' '{"ELMRNN_TSQR_WY_ROWS": "48", "ELMRNN_PW_MODE": "0"}'
python tools/qr_time.py 256 500000 '{}' '{"ELMRNN_TSQR_WY_ROWS": "48"}'
python tools/qr_time.py 128 1000000 '{}' '{"ELMRNN_TSQR_WY_ROWS": "48"}'
done 2>&1 | tee gpurun_out/qr_ab4.jsonl
