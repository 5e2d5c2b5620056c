#!/bin/bash
mkdir -p gpurun_out
python -m paper_1911_13252_b200.build > /dev/null
for s in "256 4000000" "256 500000" "192 2000000" "128 1000000" "512 2000000"; do python tools/prof.py qr $s 3; done 2>&1 | tee gpurun_out/qr_ab6.jsonl
timeout 1500 python -m pytest tests -m gpu -q -x -k "tsqr or solve or wy or virtual or multi or train or full_config or well_cond or smoke" 2>&1 | tail -3
timeout 600 python bench.py --no-cpu-baseline | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['config']['phases_ms'], d['clocks'])"
