set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python __graft_entry__.py smoke 2>&1 | tail -5
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -rA 2>&1 | grep -E "PASS|FAIL|rel dbeta|passed|failed|Error" | tail -80
timeout 600 python bench.py 2>&1 | tail -3
for c in C1 C2j C3gru C3fc; do timeout 300 python bench.py --config $c --no-cpu-baseline 2>&1 | tail -1; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv python bench.py --profile --steps 1 --warmup 1 > gpurun_out/ncu_c4.log 2>&1
tail -3 gpurun_out/ncu_c4.log
