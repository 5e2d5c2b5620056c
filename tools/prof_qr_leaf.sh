#!/bin/bash
# ncu capture of one WY leaf launch at the C4 shape (source-level stall sampling).
python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_tsqr_leaf_wy -s 1 -c 1 \
    -o gpurun_out/leaf_wy python tools/prof_qr.py 256 4000000 > gpurun_out/ncu_leaf.log 2>&1
ncu -i gpurun_out/leaf_wy.ncu-rep --page source --csv --print-source sass > gpurun_out/leaf_wy_sass.csv 2>&1
ncu -i gpurun_out/leaf_wy.ncu-rep --page raw --csv > gpurun_out/leaf_wy_raw.csv 2>&1
ls -la gpurun_out/leaf_wy*
