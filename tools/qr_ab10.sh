#!/bin/bash
mkdir -p gpurun_out
python -m paper_1911_13252_b200.build > /dev/null
python tools/qr_time.py 768 1000000 '{}' '{"ELMRNN_WY_2PHASE": "3"}' 2>&1 | tee gpurun_out/qr_ab10.jsonl
for s in "512 2000000" "1024 2000000" "400 2000000"; do python tools/prof.py qr $s 3; done 2>&1 | tee -a gpurun_out/qr_ab10.jsonl
timeout 1500 python -m pytest tests -m gpu -q -x -k "tsqr or solve or wy or virtual or multi or train or c5 or wide or well_cond" 2>&1 | tail -3
for c in C5lstm1024 C5gru1024; do timeout 900 python bench.py --config $c --no-cpu-baseline | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'][:20], d['value'], d['ms_per_step'], d['config']['phases_ms'])"; done
