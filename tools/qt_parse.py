"""Parse an 8-slot TSQR trace (ELM_QR_TRACE build): per-phase median cycles."""
import sys, numpy as np
d = np.loadtxt(sys.argv[1], delimiter=',', dtype=np.int64)
k = d[:, 0]; t = d[:, 1:]
step = np.diff(t[:, 0])
print("cols", len(k), "median step", np.median(step))
names = {1: "top->crit start", 2: "apply LC", 4: "reflector", 5: "apply rest", 3: "crit end->barrier exit"}
for lo, hi in ((0, 64), (64, 128), (128, 192), (192, 256)):
    m = (k[:-1] >= lo) & (k[:-1] < hi)
    r = lambda a, b: np.median((t[:-1, b] - t[:-1, a])[m])
    if t[:, 1].any():
        print(f" k {lo:3d}-{hi:3d}: step {np.median(step[m]):6.0f} | wait-top->crit {r(0,1):5.0f} applyLC {r(1,2):5.0f} "
              f"refl {r(2,4):5.0f} rest {r(4,5):5.0f} crit->barrier-exit {r(5,3):5.0f} | t0: top->pre-ld {r(0,6):5.0f}")
    else:
        print(f" k {lo:3d}-{hi:3d}: step {np.median(step[m]):6.0f}")
