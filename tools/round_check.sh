#!/bin/bash
# Full round check on one GPU: build, gpu tests, smoke, default bench (+ reference arm),
# the bench launch list and one ncu capture of the TSQR leaf.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/rc_build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -8 > gpurun_out/rc_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/rc_smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/rc_bench.json 2> gpurun_out/rc_bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/rc_ref.json 2> gpurun_out/rc_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/rc_launches_C4.csv python bench.py --profile --steps 1 --warmup 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_tsqr_leaf_wy -s 1 -c 1 -o gpurun_out/rc_full_tsqr_wy_C4 python tools/prof_qr.py 256 4000000 > /dev/null 2>&1
cat gpurun_out/rc_tests.log gpurun_out/rc_smoke.log; tail -c 2500 gpurun_out/rc_bench.json; tail -c 800 gpurun_out/rc_ref.json
