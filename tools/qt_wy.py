"""Parse a WY-fold trace (ELM_QR_TRACE build): per panel p, cycles of panel / G / trailing, and clock MHz."""
import sys, numpy as np
d = np.loadtxt(sys.argv[1], delimiter=',', dtype=np.int64)
d = d[d[:, 0] % 16 == 0]
p = d[:, 0]; t = d[:, 1:]
for i in range(len(p)):
    c = t[i]
    tot = c[3] - c[0] if c[3] else 0
    mhz = (c[3] - c[0]) / max(1, (c[6] - c[4])) * 1e3 if c[3] and c[6] else 0
    print(f"p={p[i]:3d} panel {c[1]-c[0]:6d} G {c[2]-c[1] if c[2] else 0:6d} trailing(t0) {c[5]-c[2] if c[5] else 0:6d} "
          f"barrier {c[3]-c[5] if c[3] else 0:6d} total {tot:7d} cyc  ~{mhz:.0f} MHz")
