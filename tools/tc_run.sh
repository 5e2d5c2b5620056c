#!/bin/bash
timeout 300 ncu --set full --import-source on --clock-control none -k regex:kp -c 1 -o gpurun_out/panel32 -f tools/ubench/panel_bench > gpurun_out/ncu_panel.log 2>&1
tail -3 gpurun_out/ncu_panel.log
