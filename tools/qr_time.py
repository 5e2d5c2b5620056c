"""Time the TSQR solve under Tune variants (ELMRNN_TESTING=1 + knobs), one
subprocess per variant: python tools/qr_time.py M N '{"ELMRNN_PW_MODE": "0"}' ..."""
import json
import os
import subprocess
import sys

M, N = sys.argv[1], sys.argv[2]
variants = [json.loads(v) for v in sys.argv[3:]] or [{}]
for v in variants:
    env = dict(os.environ, ELMRNN_TESTING="1", **v)
    out = subprocess.run([sys.executable, "tools/prof.py", "qr", M, N], env=env, capture_output=True, text=True)
    print(json.dumps(v), out.stdout.strip() or out.stderr[-400:], flush=True)
