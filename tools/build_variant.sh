#!/bin/bash
# Build an experiment variant of libelmrnn.so with extra -D defines into tools/dbg/
# (git-ignored; travels to the GPU box).  Load it with ELMRNN_LIB=<path>.
#   tools/build_variant.sh epi -DELM_TC_EPI_ACCURATE
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
