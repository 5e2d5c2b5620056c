python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
QR_VARIANTS='{};{"ELMRNN_TSQR_MAXSLABS":"592"};{"ELMRNN_TSQR_MAXSLABS":"296"};{"ELMRNN_TSQR_MAXSLABS":"148"};{"ELMRNN_TSQR_MAXSLABS":"74"};{"ELMRNN_TSQR_WY":"1"};{"ELMRNN_TSQR_WY":"1","ELMRNN_TSQR_MAXSLABS":"148"}' python tools/qr_time.py 64 100000
QR_VARIANTS='{};{"ELMRNN_TSQR_MAXSLABS":"8"};{"ELMRNN_TSQR_MAXSLABS":"4"};{"ELMRNN_TSQR_MAXSLABS":"1"}' python tools/qr_time.py 20 1000
