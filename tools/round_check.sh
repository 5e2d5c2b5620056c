#!/bin/bash
# Full round check on one GPU: build, gpu tests, smoke, default bench (+ reference arm).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/rc_build.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -8 > gpurun_out/rc_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/rc_smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/rc_bench.json 2> gpurun_out/rc_bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/rc_ref.json 2> gpurun_out/rc_ref.err
cat gpurun_out/rc_tests.log gpurun_out/rc_smoke.log; tail -c 2500 gpurun_out/rc_bench.json; tail -c 800 gpurun_out/rc_ref.json
