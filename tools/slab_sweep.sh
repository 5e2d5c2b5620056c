#!/bin/bash
# TSQR leaf-count sweep at the small configs (dev tool, GPU box): C1 (M=20, 1k rows), C2 (M=64, 100k rows)
for M_N in "20 1000" "64 100000" "128 1000000"; do
  set -- $M_N
  args=""
  for s in 0 2 4 8 16 32 64 148 296 444; do args="$args {\"ELMRNN_TSQR_MAXSLABS\":\"$s\"}"; done
  python tools/qr_time.py $1 $2 $args
done
