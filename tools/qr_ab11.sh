#!/bin/bash
mkdir -p gpurun_out
python -m paper_1911_13252_b200.build > /dev/null
for rep in 1 2; do for v in "" tools/dbg/libelmrnn_oldmerge.so; do
for s in "1024 2000000" "512 2000000" "768 1000000"; do echo -n "$v "; ELMRNN_LIB=$v python tools/prof.py qr $s 3; done; done; done 2>&1 | tee gpurun_out/qr_ab11.jsonl
timeout 1500 python -m pytest tests -m gpu -q -x -k "tsqr or solve or wy or virtual or multi or train or c5 or wide or well_cond or ridge" 2>&1 | tail -3
