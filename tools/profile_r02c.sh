#!/bin/bash
# Round-2 profiling pass (one GPU): launch list of the default bench command and one
# `ncu --set full` capture per hot kernel at full benchmark size.
mkdir -p gpurun_out
python -m paper_1911_13252_b200.build > /dev/null
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_lstm_tc -c 1 -o gpurun_out/r02c_full_lstm_tc_C4 python tools/prof.py build lstm 256 50 4000000 1 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_tsqr_leaf_wy -c 1 -o gpurun_out/r02c_full_tsqr_wy_C4 python tools/prof.py qr 256 4000000 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gru_tc -c 1 -o gpurun_out/r02c_full_gru_C3 python tools/prof.py build gru 128 30 1000000 4 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_tsqr_leaf_wy -c 1 -o gpurun_out/r02c_full_tsqr_wy_C3 python tools/prof.py qr 128 1000000 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_teacher_forced -c 1 -o gpurun_out/r02c_full_tf_C2 python tools/prof.py build jordan 64 20 100000 1 1 > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/r02c_ncu_summary.json gpurun_out/r02c_full_*.ncu-rep > /dev/null; rm -f gpurun_out/r02c_full_*.ncu-rep; ls -la gpurun_out
