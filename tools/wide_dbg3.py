import os, sys, numpy as np, torch
from paper_1911_13252_b200 import ELMRNN
def R_of(pk, n):
    R = np.zeros((n, n)); off = 0
    for k in range(n):
        R[k, k:] = pk[off: off + n - k]; off += n - k
    return R
os.environ["ELMRNN_TSQR_WY"] = "1"
for rows in ("16", "32"):
    os.environ["ELMRNN_TSQR_WY_ROWS"] = rows
    for M in (63, 127, 200, 300, 511):
        out = []
        for N in (16, 32, 48, 64, 100, 300, 600):
            g = torch.Generator(device="cuda").manual_seed(M + N)
            H = torch.rand(N, M, device="cuda", generator=g) - 0.5
            Y = torch.rand(N, device="cuda", generator=g) - 0.5
            n = M + 1
            Rn = np.abs(np.linalg.qr(np.column_stack([H.double().cpu().numpy(), Y.double().cpu().numpy()]), mode="r"))
            e = ELMRNN("lstm", 1, M, 4, 1, force_path=1)
            R = np.abs(R_of(e.solve_local(H, Y).cpu().numpy(), n))[:Rn.shape[0]]
            d = np.abs(R - Rn); d[~np.isfinite(d)] = 1e9
            rws, cls = np.nonzero(d > 1e-10 * Rn.max())
            out.append(f"N={N}:{'ok' if len(rws)==0 else 'BAD@%d,%d' % (rws[0], cls[0])}")
        print("rows", rows, "M", M, " ".join(out), flush=True)
