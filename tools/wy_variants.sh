#!/bin/bash
# WY TSQR leaf wavefront sharing (CTAs per R slab) at the C3/C4/C5 shapes (dev tool, GPU box).
python tools/qr_time.py 256 4000000 '{"ELMRNN_LEAF_SHARE":"1"}' '{}' '{"ELMRNN_LEAF_SHARE":"2"}' '{"ELMRNN_LEAF_SHARE":"3"}' '{"ELMRNN_LEAF_SHARE":"12"}'
python tools/qr_time.py 256 500000 '{"ELMRNN_LEAF_SHARE":"1"}' '{}' '{"ELMRNN_LEAF_SHARE":"12"}'
python tools/qr_time.py 128 2000000 '{"ELMRNN_LEAF_SHARE":"1"}' '{}'
python tools/qr_time.py 512 2000000 '{"ELMRNN_LEAF_SHARE":"1"}' '{}'
python tools/qr_time.py 1024 2000000 '{"ELMRNN_LEAF_SHARE":"1"}' '{}'
