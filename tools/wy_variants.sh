#!/bin/bash
# WY TSQR leaf: two-phase pipelined vs single-chain at the C3/C4/C5 shapes (dev tool, GPU box).
for MN in "256 4000000" "256 500000" "512 2000000" "1024 2000000" "300 1000000" "400 1000000" "192 1000000"; do
  python tools/qr_time.py $MN '{"ELMRNN_WY_2PHASE":"0"}' '{}'
done
