#!/bin/bash
# WY TSQR leaf variants (tile rows x warps per CTA) at the C3/C4/C5 shapes (dev tool, GPU box).
python tools/qr_time.py 128 2000000 '{}' '{"ELMRNN_TSQR_WY_ROWS":"96","ELMRNN_WY_NW":"4"}' '{"ELMRNN_TSQR_WY_ROWS":"64","ELMRNN_WY_NW":"8"}' '{"ELMRNN_TSQR_WY_ROWS":"32","ELMRNN_WY_NW":"4"}'
python tools/qr_time.py 64 100000 '{}' '{"ELMRNN_TSQR_WY":"1"}' '{"ELMRNN_TSQR_WY":"1","ELMRNN_TSQR_WY_ROWS":"96"}'
python tools/qr_time.py 20 1000 '{}' '{"ELMRNN_TSQR_WY":"1"}'
