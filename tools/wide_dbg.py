import os, sys, numpy as np, torch
from paper_1911_13252_b200 import ELMRNN
def R_of(pk, n):
    R = np.zeros((n, n)); off = 0
    for k in range(n):
        R[k, k:] = pk[off: off + n - k]; off += n - k
    return R
for M, N in [(256, 3001), (511, 3001), (600, 3001), (1000, 3001), (1024, 3001), (1024, 1025), (1024, 20000)]:
    g = torch.Generator(device="cuda").manual_seed(M + N)
    H = torch.rand(N, M, device="cuda", generator=g) - 0.5
    Y = torch.rand(N, device="cuda", generator=g) - 0.5
    n = M + 1
    Rn = np.abs(np.linalg.qr(np.column_stack([H.double().cpu().numpy(), Y.double().cpu().numpy()]), mode="r"))
    e = ELMRNN("lstm", 1, M, 4, 1)
    R = np.abs(R_of(e.solve_local(H, Y).cpu().numpy(), n))
    bad = ~np.isfinite(R)
    d = np.abs(R - Rn); d[bad] = np.inf
    rows, cols = np.nonzero(d > 1e-10 * Rn.max())
    print(M, N, os.environ.get("ELMRNN_TSQR_WY_ROWS"), "err", np.nanmax(np.where(bad, np.nan, d)), "nbad", bad.sum(),
          "first bad rows", rows[:5], cols[:5], "last diag", R[-1, -1], Rn[-1, -1], flush=True)
