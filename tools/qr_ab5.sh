#!/bin/bash
mkdir -p gpurun_out
python -m paper_1911_13252_b200.build > /dev/null
for s in "256 4000000" "256 500000" "192 2000000"; do
python tools/qr_time.py $s '{}' '{"ELMRNN_TSQR_WY_ROWS": "48", "ELMRNN_WY_NW": "6", "ELMRNN_PW_MODE": "0"}' '{"ELMRNN_TSQR_WY_ROWS": "48", "ELMRNN_WY_NW": "5", "ELMRNN_PW_MODE": "0"}' '{"ELMRNN_TSQR_WY_ROWS": "40", "ELMRNN_WY_NW": "6", "ELMRNN_PW_MODE": "0"}' '{"ELMRNN_TSQR_WY_ROWS": "40", "ELMRNN_WY_NW": "5", "ELMRNN_PW_MODE": "0"}' '{"ELMRNN_TSQR_WY_ROWS": "48", "ELMRNN_WY_NW": "6", "ELMRNN_PW_MODE": "0", "ELMRNN_LIB": "tools/dbg/libelmrnn_noilp48.so"}'
done 2>&1 | tee gpurun_out/qr_ab5.jsonl
