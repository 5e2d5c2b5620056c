#!/bin/bash
set -o pipefail
python -m paper_1911_13252_b200.build >/dev/null
timeout 1800 python -m pytest tests -q -m gpu -x 2>&1 | tail -3
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -6
timeout 900 python bench.py > gpurun_out/bench_C4.json 2> gpurun_out/bench_C4.err; cat gpurun_out/bench_C4.json
rm -f gpurun_out/bench_all.jsonl
for c in C1 C2j C2n C3gru C3fc C3lstm_diag C3gru_diag C3fc_eq8; do timeout 600 python bench.py --config $c 2>>gpurun_out/bench_other.err >> gpurun_out/bench_all.jsonl; done
timeout 600 python bench.py --weight-grid 1 --no-cpu-baseline >> gpurun_out/bench_all.jsonl 2>>gpurun_out/bench_other.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_C4.json 2>&1; cat gpurun_out/bench_ref_C4.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench_C4.csv python bench.py --profile --steps 1 --warmup 1 > /dev/null 2>&1
python - <<'PY'
import json
for l in open('gpurun_out/bench_all.jsonl'):
    d = json.loads(l)
    print(d['config']['workload'][:34], '| value', round(d['value']), '| ms', round(d['ms_per_step'], 3), '| phases', {k: round(v, 2) for k, v in d['config']['phases_ms'].items()}, '| roof', d['roofline']['bound'], round(d['roofline']['frac'], 3), '| cpu', d['cpu_baseline'] and round(d['cpu_baseline']['value']), '| e2e', round(d['e2e']['value']), '| clk', d['clocks']['sm_mhz'])
PY
