#!/bin/bash
set -o pipefail
timeout 900 python tools/qr3.py 32,64 2,3,4 2>&1
