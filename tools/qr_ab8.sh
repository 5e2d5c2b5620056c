#!/bin/bash
mkdir -p gpurun_out
python -m paper_1911_13252_b200.build > /dev/null
python tools/qr_time.py 1024 2000000 '{}' '{"ELMRNN_WY_2PHASE": "0", "ELMRNN_TSQR_WY_ROWS": "24", "ELMRNN_WY_NW": "8"}' '{"ELMRNN_WY_2PHASE": "0", "ELMRNN_TSQR_WY_ROWS": "24", "ELMRNN_WY_NW": "12"}' '{"ELMRNN_WY_2PHASE": "0", "ELMRNN_TSQR_WY_ROWS": "16", "ELMRNN_WY_NW": "8"}' 2>&1 | tee gpurun_out/qr_ab8.jsonl
python tools/qr_time.py 512 2000000 '{"ELMRNN_WY_2PHASE": "0", "ELMRNN_TSQR_WY_ROWS": "24", "ELMRNN_WY_NW": "12"}' 2>&1 | tee -a gpurun_out/qr_ab8.jsonl
