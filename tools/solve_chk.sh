python -m paper_1911_13252_b200.build >/dev/null
timeout 900 python -m pytest tests -m gpu -q -x -k "solve or ridge or nonfinite or virtual or full_config or tsqr or train or smoke" 2>&1 | tail -3
for c in C1 C2j; do timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch2_$c.csv python bench.py --config $c --profile --steps 1 --warmup 1 > /dev/null 2>&1; done
for c in C1 C2j C3gru; do timeout 300 python bench.py --config $c --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['config']['workload'][:30], d['value'], d['ms_per_step'], d['config']['phases_ms'])"; done
