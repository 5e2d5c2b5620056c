"""Parse a look-ahead WY trace: per panel step p: warp-0 trailing(next panel cols) / panel / wait-at-barrier / G."""
import sys, numpy as np
d = np.loadtxt(sys.argv[1], delimiter=',', dtype=np.int64)
d = d[d[:, 0] % 16 == 0]
tot = 0
for row in d:
    p, c = row[0], row[1:]
    if not c[2]:
        continue
    t = c[3] - c[0] if c[3] > c[0] else 0
    tot += t
    print(f"p={p:3d} w0-trail {c[1]-c[0]:6d} panel {c[5]-c[1]:6d} barrier-wait {c[2]-c[5]:6d} G {c[3]-c[2] if c[3] else 0:5d} step {t:6d}")
print("sum", tot)
