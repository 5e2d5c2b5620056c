#!/bin/bash
timeout 300 ncu --set full --clock-control none -k regex:k_elman -s 1 -c 1 -o gpurun_out/full_eq8 python tools/prof_build.py fc_eq8 128 30 1000000 > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/full_eq8.ncu-rep
