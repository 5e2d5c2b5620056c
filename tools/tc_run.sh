#!/bin/bash
set -o pipefail
python -m paper_1911_13252_b200.build >/dev/null
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "gru" 2>&1 | tail -2
timeout 300 python tools/tc_check.py 2>&1 | grep -E "gru|GRU|C4"
