import os, sys, numpy as np, torch
from paper_1911_13252_b200 import ELMRNN
def R_of(pk, n):
    R = np.zeros((n, n)); off = 0
    for k in range(n):
        R[k, k:] = pk[off: off + n - k]; off += n - k
    return R
cases = [(511, 600), (511, 3001), (300, 600), (300, 3001)]
for rows in ("16", "32"):
    for warps in ("2", "4", "6", "8"):
        os.environ["ELMRNN_TSQR_WY_ROWS"] = rows; os.environ["ELMRNN_TSQR_WY_WARPS"] = warps
        out = []
        for M, N in cases:
            g = torch.Generator(device="cuda").manual_seed(M + N)
            H = torch.rand(N, M, device="cuda", generator=g) - 0.5
            Y = torch.rand(N, device="cuda", generator=g) - 0.5
            n = M + 1
            Rn = np.abs(np.linalg.qr(np.column_stack([H.double().cpu().numpy(), Y.double().cpu().numpy()]), mode="r"))
            e = ELMRNN("lstm", 1, M, 4, 1)
            R = np.abs(R_of(e.solve_local(H, Y).cpu().numpy(), n))
            d = np.abs(R - Rn); d[~np.isfinite(d)] = 1e9
            rws, cls = np.nonzero(d > 1e-10 * Rn.max())
            out.append(f"M={M} N={N}: {'OK' if len(rws)==0 else 'BAD@'+str(rws[0])}")
        print("rows", rows, "warps", warps, " | ".join(out), flush=True)
