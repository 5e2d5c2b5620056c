TAG=lag timeout 300 python tools/qr_debug2.py 2>&1 | grep -E "var=4|nonfinite=[1-9]"
timeout 300 python tools/qt.py
ELMRNN_TSQR_VAR=4 ELMRNN_TRACE_QR=gpurun_out/qrtrace3.csv timeout 120 python tools/prof_qr.py 256 100000
timeout 300 python tools/tc_check.py 2>&1 | grep -E "gru|GRU"
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "gru" 2>&1 | tail -2
