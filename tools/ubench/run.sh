#!/bin/bash
# Microbenchmarks (one GPU): reflector-chain latencies, the WY panel alone, the
# per-column fold with parts switched off, and the per-warp fold prototype.
#   bash tools/ubench/run.sh            -> gpurun_out/ubench.log
cd "$(dirname "$0")"
mkdir -p ../../gpurun_out
F="-gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -I ../../include -I ../../paper_1911_13252_b200/csrc"
{
  nvcc $F -o /tmp/refl_lat refl_lat.cu && /tmp/refl_lat
  nvcc $F -o /tmp/panel_bench panel_bench.cu -lcuda && /tmp/panel_bench
  nvcc $F -DELM_QR_TRACE -o /tmp/fold_bench fold_bench.cu -lcuda && for n in 21 65 129; do /tmp/fold_bench $n; done
  nvcc $F -o /tmp/fold_var fold_var.cu && /tmp/fold_var
  nvcc $F -o /tmp/warp_fold warp_fold.cu && /tmp/warp_fold
} 2>&1 | tee ../../gpurun_out/ubench.log
