#!/bin/bash
# Panel-step phase trace of the WY leaf under env variants (C4 shape).
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
for v in "" "ELMRNN_TSQR_WY_CTAS=1" "ELMRNN_TSQR_WY_CTAS=1 ELMRNN_TSQR_WY_WARPS=2" "ELMRNN_TSQR_WY_WARPS=8"; do
  echo "== $v"
  env $v ELMRNN_LIB=tools/dbg/libelmrnn_trace.so ELMRNN_TSQR_LEVELS=0 ELMRNN_TRACE_QR=/tmp/q.csv python /tmp/qtr.py
  python tools/qt_wy2.py /tmp/q.csv | sed -n '1p;5p;9p;13p;$p'
done
