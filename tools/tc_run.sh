#!/bin/bash
# per-call GPU script (edited per experiment)
set -o pipefail
python -m paper_1911_13252_b200.build >/dev/null
timeout 300 python tools/fc_check.py 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "fc" 2>&1 | tail -3
