# Round profiling pass (one GPU): launch list of the bench command + one
# `ncu --set full` capture per hot kernel at full benchmark size.
set -x
mkdir -p gpurun_out
python -m paper_1911_13252_b200.build > /dev/null
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench_C4.csv python bench.py --profile --steps 1 --warmup 1 > gpurun_out/launches_bench_C4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_tsqr_leaf_wy -s 1 -c 1 -o gpurun_out/full_tsqr_wy_C4 python tools/prof_qr.py 256 4000000 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fc_tc -s 1 -c 1 -o gpurun_out/full_fc_C3 python tools/prof_build.py fc 128 30 1000000 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gru_tc -s 1 -c 1 -o gpurun_out/full_gru_C3 python tools/prof_build.py gru 128 30 1000000 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_tsqr_leaf -s 1 -c 1 -o gpurun_out/full_tsqr_1d_C3 python tools/prof_qr.py 128 1000000 > /dev/null 2>&1
ls -la gpurun_out
