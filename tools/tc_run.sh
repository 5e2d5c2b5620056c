TAG=rev timeout 300 python tools/qr_debug2.py
ELMRNN_TSQR_VAR=3 ELMRNN_TRACE_QR=gpurun_out/qrtrace2.csv timeout 120 python tools/prof_qr.py 256 100000
timeout 300 python tools/qt.py
timeout 300 python tools/qr_check.py 2>&1 | tail -6
