#!/bin/bash
# GRU M = 128: x(t) W + b inside the MMA (XMMA, default) vs in the epilogue (tools/dbg/libelmrnn_noxmma.so)
mkdir -p gpurun_out
python -m paper_1911_13252_b200.build > /dev/null
timeout 900 python -m pytest tests -m gpu -q -x -k "gru" 2>&1 | tail -3
for rep in 1 2; do for v in "" tools/dbg/libelmrnn_noxmma.so; do
  for a in "gru 128 30 1000000 4" "gru 128 10 2000000 1" "gru 128 50 2000000 1"; do echo -n "$v "; ELMRNN_LIB=$v timeout 300 python tools/prof.py build $a 3; done
done; done 2>&1 | tee gpurun_out/gru_ab.jsonl
for v in "" tools/dbg/libelmrnn_noxmma.so; do ELMRNN_LIB=$v timeout 300 python bench.py --config C3gru --no-cpu-baseline | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['config']['phases_ms'])"; done
