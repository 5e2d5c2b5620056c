# Round profiling pass (one GPU): launch list of the bench command + one
# `ncu --set full` capture per hot kernel at full benchmark size.
set -x
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench_C4.csv python bench.py --profile --steps 1 --warmup 1 > gpurun_out/launches_bench_C4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_lstm_tc -s 1 -c 1 -o gpurun_out/full_lstm_C4 python tools/prof_build.py lstm 256 50 4000000 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_tsqr_leaf -s 1 -c 1 -o gpurun_out/full_tsqr_leaf_C4 python tools/prof_qr.py 256 4000000 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gru_tc -s 1 -c 1 -o gpurun_out/full_gru_C3 python tools/prof_build.py gru 128 30 1000000 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_teacher_forced -s 1 -c 1 -o gpurun_out/full_jordan_C2 python tools/prof_build.py jordan 64 20 100000 > /dev/null 2>&1
ls -la gpurun_out
timeout 900 python bench.py > gpurun_out/bench_C4.json 2> gpurun_out/bench_C4.err
for c in C1 C2j C2n C3gru C3fc; do timeout 600 python bench.py --config $c --no-cpu-baseline >> gpurun_out/bench_other.jsonl 2>> gpurun_out/bench_other.err; done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_C4.json 2>&1
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm --format=csv > gpurun_out/gpu_info.csv
lscpu | head -20 > gpurun_out/host_cpu.txt; nproc >> gpurun_out/host_cpu.txt
