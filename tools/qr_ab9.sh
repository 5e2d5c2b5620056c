#!/bin/bash
mkdir -p gpurun_out
python -m paper_1911_13252_b200.build > /dev/null
python tools/qr_time.py 1024 2000000 '{"ELMRNN_WY_2PHASE": "0", "ELMRNN_TSQR_WY_ROWS": "24", "ELMRNN_WY_NW": "16"}' '{"ELMRNN_WY_2PHASE": "0", "ELMRNN_TSQR_WY_ROWS": "24", "ELMRNN_WY_NW": "12"}' 2>&1 | tee gpurun_out/qr_ab9.jsonl
python tools/qr_time.py 512 2000000 '{"ELMRNN_WY_2PHASE": "0", "ELMRNN_TSQR_WY_ROWS": "48", "ELMRNN_WY_NW": "16"}' '{"ELMRNN_WY_2PHASE": "0", "ELMRNN_TSQR_WY_ROWS": "48", "ELMRNN_WY_NW": "12"}' '{}' 2>&1 | tee -a gpurun_out/qr_ab9.jsonl
python tools/qr_time.py 400 2000000 '{"ELMRNN_WY_2PHASE": "0", "ELMRNN_TSQR_WY_ROWS": "48", "ELMRNN_WY_NW": "12"}' '{}' 2>&1 | tee -a gpurun_out/qr_ab9.jsonl
