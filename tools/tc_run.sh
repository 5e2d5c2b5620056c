#!/bin/bash
set -o pipefail
python -m paper_1911_13252_b200.build >/dev/null
for wg in 0 1; do
timeout 600 python bench.py --steps 3 --no-cpu-baseline --weight-grid $wg 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('wg', $wg, 'value', round(d['value']), 'e2e', round(d['e2e']['value']), 'phases', {k: round(v,1) for k,v in d['config']['phases_ms'].items()}, 'roof', round(d['roofline']['achieved']), round(d['roofline']['frac'],3), 'clk', d['clocks'])"
done
timeout 300 python -m pytest tests/test_gpu_parity.py -q -k "two_pass" 2>&1 | tail -1
