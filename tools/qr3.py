"""WY TSQR sweep: correctness once, then C4/C3/C2-size solve timing per (ROWS, warps) setting."""
import os, sys, numpy as np, torch
sys.path.insert(0, '.')
os.environ['ELMRNN_TSQR_WY'] = '1'
from paper_1911_13252_b200 import ELMRNN


def check(M, N):
    e = ELMRNN('lstm', 1, M, 4, 1, force_path=1)
    g = torch.Generator(device='cuda').manual_seed(M + N)
    H = torch.rand(N, M, device='cuda', generator=g); Y = torch.rand(N, device='cuda', generator=g)
    Rpk = e.solve_local(H, Y).cpu().numpy()
    n = M + 1; R = np.zeros((n, n)); off = 0
    for k in range(n):
        R[k, k:] = Rpk[off: off + n - k]; off += n - k
    Rn = np.linalg.qr(np.column_stack([H.double().cpu().numpy(), Y.double().cpu().numpy()]), mode='r')
    return np.nanmax(np.abs(np.abs(R) - np.abs(Rn[:n])) / np.abs(Rn[:n]).max()), int((~np.isfinite(R)).sum())


def timeit(M, N):
    e = ELMRNN('lstm', 1, M, 4, 1, force_path=1)
    H = torch.rand(N, M, device='cuda'); Y = torch.rand(N, device='cuda')
    b, _ = e.solve_beta(H, Y); torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True); t1 = torch.cuda.Event(enable_timing=True)
    t0.record(); e.solve_beta(H, Y, b, info=False); t1.record(); torch.cuda.synchronize()
    return t0.elapsed_time(t1)


for rows in sys.argv[1].split(','):
    for warps in sys.argv[2].split(','):
        os.environ['ELMRNN_TSQR_WY_ROWS'] = rows
        os.environ['ELMRNN_TSQR_WY_WARPS'] = warps
        worst, nf = 0.0, 0
        for M, N in ((1, 100), (5, 77), (16, 300), (64, 256), (127, 5000), (200, 999), (256, 20000), (263, 4000), (511, 3000)):
            d, f = check(M, N); worst = max(worst, d); nf += f
        t = [timeit(256, 4_000_000), timeit(128, 1_000_000), timeit(64, 100_000)]
        print(f"rows={rows} warps={warps}: worst|dR|={worst:.1e} nonfinite={nf}  C4 {t[0]:.1f} ms  C3 {t[1]:.2f} ms  C2 {t[2]:.2f} ms", flush=True)
