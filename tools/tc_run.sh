#!/bin/bash
set -o pipefail
timeout 900 python tools/qr3.py 24,32 4,5 2>&1
