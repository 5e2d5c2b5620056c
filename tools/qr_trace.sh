#!/bin/bash
# Per-panel-step clock trace of the WY leaf (CTA 0's last tile) at a given shape:
#   tools/qr_trace.sh M N   (tracing build tools/dbg/libelmrnn_trace.so, -DELM_QR_TRACE)
M=${1:-256}; N=${2:-4000000}
mkdir -p gpurun_out
cat > /tmp/qtr.py <<PY
import sys, torch
sys.path.insert(0, '.')
from paper_1911_13252_b200 import ELMRNN
M, N = $M, $N
e = ELMRNN('lstm', 1, M, 4, 1, force_path=1)
H = torch.rand(N, M, device='cuda') - 0.5; Y = torch.rand(N, device='cuda') - 0.5
b = torch.empty(M, dtype=torch.float64, device='cuda')
e.solve_beta(H, Y, b, info=False); torch.cuda.synchronize()
PY
ELMRNN_LIB=tools/dbg/libelmrnn_trace.so ELMRNN_TRACE_QR=gpurun_out/qtrace_${M}.csv python /tmp/qtr.py
python tools/qt_parse.py gpurun_out/qtrace_${M}.csv
