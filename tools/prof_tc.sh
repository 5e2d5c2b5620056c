set -x
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_lstm_tc -s 1 -c 1 -o gpurun_out/prof_tc python tools/prof_build.py lstm 256 50 37888 > gpurun_out/prof_tc.log 2>&1
tail -5 gpurun_out/prof_tc.log
