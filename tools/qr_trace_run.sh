#!/bin/bash
# Per-panel phase trace of the WY leaf at the C4 shape (block 0's last tile).
set -e
tools/build_variant.sh trace -DELM_QR_TRACE >/dev/null
cat > /tmp/qtr.py <<'PY'
import sys, torch
sys.path.insert(0, '.')
from paper_1911_13252_b200 import ELMRNN
M, N = 256, 4_000_000
e = ELMRNN('lstm', 1, M, 4, 1, force_path=1)
H = torch.rand(N, M, device='cuda') - 0.5; Y = torch.rand(N, device='cuda') - 0.5
e.solve_beta(H, Y); torch.cuda.synchronize()
PY
ELMRNN_LIB=tools/dbg/libelmrnn_trace.so ELMRNN_TSQR_LEVELS=0 ELMRNN_TRACE_QR=gpurun_out/qtrace.csv python /tmp/qtr.py
python tools/qt_wy2.py gpurun_out/qtrace.csv
