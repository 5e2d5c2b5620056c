import os, sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_1911_13252_b200 import ELMRNN
def run(M, N, v):
    os.environ['ELMRNN_TSQR_VAR'] = str(v)
    e = ELMRNN('lstm', 1, M, 4, 1, force_path=1)
    g = torch.Generator(device='cuda').manual_seed(0)
    H = torch.rand(N, M, device='cuda', generator=g); Y = torch.rand(N, device='cuda', generator=g)
    Rpk = e.solve_local(H, Y).cpu().numpy()
    n = M + 1; R = np.zeros((n, n)); off = 0
    for k in range(n):
        R[k, k:] = Rpk[off: off + n - k]; off += n - k
    Rn = np.linalg.qr(np.column_stack([H.double().cpu().numpy(), Y.double().cpu().numpy()]), mode='r')
    d = np.abs(np.abs(R) - np.abs(Rn[:n]))
    bad = np.argwhere(~np.isfinite(R))
    print(f"{os.environ.get('TAG','')} M={M} N={N} var={v} max|dR|={np.nanmax(d):.2e} nonfinite={len(bad)} first={bad[:3].tolist()}", flush=True)
for M, N in ((64, 256), (256, 1024), (256, 8000)):
    for v in (4, 0, 3, 1, 2):
        if v in (0, 3, 4) and M + 1 > 288: continue
        run(M, N, v)
