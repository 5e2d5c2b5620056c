TAG=fast timeout 300 python tools/qr_debug2.py
cp paper_1911_13252_b200/libelmrnn.so /tmp/keep.so; cp tools/dbg/libelmrnn_ieee.so paper_1911_13252_b200/libelmrnn.so
TAG=ieee timeout 300 python tools/qr_debug2.py
cp /tmp/keep.so paper_1911_13252_b200/libelmrnn.so
