#!/bin/bash
# Panel-loop unroll variants of the WY leaf, timed at the C4 and C5 shapes.
python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
for u in 4 8 16; do tools/build_variant.sh u$u -DELM_PANEL_UNROLL=$u > /dev/null 2>&1; done
for lib in paper_1911_13252_b200/libelmrnn.so tools/dbg/libelmrnn_u4.so tools/dbg/libelmrnn_u8.so tools/dbg/libelmrnn_u16.so; do
  echo "== $lib"; ELMRNN_LIB=$lib QR_VARIANTS="{}" python tools/qr_time.py 256 4000000; ELMRNN_LIB=$lib QR_VARIANTS="{}" python tools/qr_time.py 1024 2000000
done
