TAG=fixed timeout 300 python tools/qr_debug2.py
timeout 600 python tools/qr_variants.py 2>&1 | tail -12
timeout 300 python tools/tc_check.py 2>&1 | tail -12
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -4
