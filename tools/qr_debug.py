import os, subprocess, sys
code = r'''
import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_1911_13252_b200 import ELMRNN
M, N = int(sys.argv[1]), int(sys.argv[2])
e = ELMRNN('lstm', 1, M, 4, 1, force_path=1)
g = torch.Generator(device='cuda').manual_seed(0)
H = torch.rand(N, M, device='cuda', generator=g); Y = torch.rand(N, device='cuda', generator=g)
Rpk = e.solve_local(H, Y).cpu().numpy()
n = M + 1
R = np.zeros((n, n)); off = 0
for k in range(n):
    R[k, k:] = Rpk[off: off + n - k]; off += n - k
Rn = np.linalg.qr(np.column_stack([H.double().cpu().numpy(), Y.double().cpu().numpy()]), mode='r')
d = np.abs(np.abs(R) - np.abs(Rn[:n]))
bad = np.argwhere(~np.isfinite(R))
print(f"M={M} N={N} var={sys.argv[3]} max|dR|={np.nanmax(d):.2e} nonfinite={len(bad)} first={bad[:3].tolist()}", flush=True)
'''
for M, N in ((8, 48), (8, 49), (8, 100), (8, 1000), (40, 200), (64, 256), (256, 1024), (256, 8000)):
    for v in (0, 3, 1, 2):
        if v in (0, 3) and M + 1 > 288: continue
        env = dict(os.environ, ELMRNN_TSQR_VAR=str(v))
        r = subprocess.run([sys.executable, "-c", code, str(M), str(N), str(v)], env=env, capture_output=True, text=True, timeout=300)
        print(r.stdout.strip() or r.stderr[-400:], flush=True)
