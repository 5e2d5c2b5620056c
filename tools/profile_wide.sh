#!/bin/bash
# ncu capture of the wide-layer builders at the C5 shape (2M x Q=10, M=1024)
mkdir -p gpurun_out
python -m paper_1911_13252_b200.build > /dev/null
timeout 900 ncu --set full --clock-control none -k regex:k_lstm_wide -c 1 -o gpurun_out/r02e_full_lstm_wide python tools/prof.py build lstm 1024 10 2000000 1 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none -k regex:k_gru_wide -c 1 -o gpurun_out/r02e_full_gru_wide python tools/prof.py build gru 1024 10 2000000 1 1 > /dev/null 2>&1
for r in lstm_wide gru_wide; do
  ncu -i gpurun_out/r02e_full_$r.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,lts__throughput.avg.pct_of_peak_sustained_elapsed,l1tex__throughput.avg.pct_of_peak_sustained_active,smsp__average_warp_latency_issue_stalled_barrier,sm__warps_active.avg.pct_of_peak_sustained_active > gpurun_out/r02e_$r.csv
  ncu -i gpurun_out/r02e_full_$r.ncu-rep --page details --csv > gpurun_out/r02e_${r}_details.csv
done
rm -f gpurun_out/r02e_full_*.ncu-rep
cat gpurun_out/r02e_lstm_wide.csv gpurun_out/r02e_gru_wide.csv
