ELMRNN_TRACE=gpurun_out/trace.csv timeout 120 python tools/prof_build.py lstm 256 50 37888
timeout 300 python tools/tc_check.py 2>&1 | tail -3
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_tsqr_leaf -s 1 -c 1 -o gpurun_out/prof_qr1 python tools/prof_qr.py 256 500000 > gpurun_out/prof_qr1.log 2>&1
tail -1 gpurun_out/prof_qr1.log
