#!/bin/bash
# Build a debug variant of libelmrnn.so with extra defines into tools/dbg/ (testing aid).
#   tools/build_variant.sh trace -DELM_QR_TRACE
set -e
name=$1; shift
out=tools/dbg/obj_$name; mkdir -p $out
for f in paper_1911_13252_b200/csrc/*.cu; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -Xcompiler -fvisibility=hidden \
    --expt-relaxed-constexpr -I include -I paper_1911_13252_b200/csrc "$@" -c $f -o $out/$(basename $f).o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o tools/dbg/libelmrnn_$name.so $out/*.o -lcuda
rm -rf $out
echo tools/dbg/libelmrnn_$name.so
