#!/bin/bash
set -o pipefail
timeout 900 python tools/qr3.py 32 4 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "wy_and_fold or solve_parity or virtual" 2>&1 | tail -2
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -6
