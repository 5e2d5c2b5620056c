#!/bin/bash
# Multi-GPU projection inputs: one rank's share of C4 at 8 GPUs (N = 500k) on one B200,
# plus the TSQR at that size under leaf-count caps (testing knob).
mkdir -p gpurun_out
python -m paper_1911_13252_b200.build > /dev/null
timeout 600 python bench.py --config C4 --n 500000 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/n500k_bench.json
python tools/qr_time.py 256 500000 '{}' '{"ELMRNN_TSQR_MAXSLABS": "296"}' '{"ELMRNN_TSQR_MAXSLABS": "222"}' '{"ELMRNN_TSQR_MAXSLABS": "148"}' | tee gpurun_out/n500k_qr.txt
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/n500k_launches.csv python bench.py --config C4 --n 500000 --profile --steps 1 --warmup 1 > /dev/null 2>&1
python -c "
import json; d=json.load(open('gpurun_out/n500k_bench.json')); print(d['value'], d['ms_per_step'], d['config']['phases_ms'], d['clocks'])"
