"""Parse a WY-leaf trace (tools/qr_trace.sh): per panel step p, cycles of
  LA  = step start -> panel warp released by the look-ahead barrier
  pan = panel factorisation of panel p+1 (panel warp)
  wait= panel end -> step barrier exit
  t0la= trailing warp 0: step start -> its look-ahead columns done
  t0  = trailing warp 0: step start -> all its trailing columns done
  step= step start -> next step start"""
import sys
import numpy as np
d = np.loadtxt(sys.argv[1], delimiter=',', dtype=np.int64)
d = d[np.argsort(d[:, 0])]
print(" p   LA    pan   wait  t0la    t0   step")
tot = np.zeros(6)
for k in range(len(d) - 1):
    p, c = d[k, 0], d[k, 1:]
    nxt = d[k + 1, 1]
    v = [c[1] - c[0], c[5] - c[1], c[2] - c[5], c[3] - c[0], c[4] - c[0], nxt - c[0]]
    tot += v
    print(f"{p:3d} " + " ".join(f"{x:6d}" for x in v))
print("sum " + " ".join(f"{x:6.0f}" for x in tot))
