import os, sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_1911_13252_b200 import ELMRNN
M, N, v = 256, 1024, 3
os.environ['ELMRNN_TSQR_VAR'] = str(v)
g = torch.Generator(device='cuda').manual_seed(0)
H = torch.rand(N, M, device='cuda', generator=g); Y = torch.rand(N, device='cuda', generator=g)
n = M + 1
for L in range(0, 6):
    os.environ['ELMRNN_TSQR_LEVELS'] = str(L)
    e = ELMRNN('lstm', 1, M, 4, 1, force_path=1)
    Rpk = e.solve_local(H, Y).cpu().numpy()
    R = np.zeros((n, n)); off = 0
    for k in range(n):
        R[k, k:] = Rpk[off: off + n - k]; off += n - k
    bad = np.argwhere(~np.isfinite(R))
    diag = np.abs(np.diag(R))
    print(f"levels={L}: nonfinite={len(bad)} first={bad[:2].tolist()} maxabs={np.nanmax(np.abs(R[np.isfinite(R)])):.3e} "
          f"diag[40:56]={np.array2string(diag[40:56], precision=1)}", flush=True)
    print("   diag[90:100]", np.array2string(diag[90:100], precision=1), " diag[140:150]", np.array2string(diag[140:150], precision=1),
          " rows>=96 max", np.nanmax(np.abs(R[96:, :])) if np.isfinite(R[96:]).any() else None, flush=True)
