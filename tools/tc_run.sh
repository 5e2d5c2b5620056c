timeout 300 python tools/qr_check.py 2>&1 | tail -6
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "solve or virtual or ridge or predict or full_config" 2>&1 | grep -E "^E  |passed|failed" | head -30
