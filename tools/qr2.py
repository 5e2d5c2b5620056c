"""2D-tiled TSQR leaf/merge check: R vs numpy QR on random matrices, C4-size timing vs the 1D fold."""
import os, sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_1911_13252_b200 import ELMRNN


def run(M, N, d2):
    os.environ['ELMRNN_TSQR_2D'] = str(d2)
    e = ELMRNN('lstm', 1, M, 4, 1, force_path=1)
    g = torch.Generator(device='cuda').manual_seed(M + N)
    H = torch.rand(N, M, device='cuda', generator=g); Y = torch.rand(N, device='cuda', generator=g)
    Rpk = e.solve_local(H, Y).cpu().numpy()
    n = M + 1; R = np.zeros((n, n)); off = 0
    for k in range(n):
        R[k, k:] = Rpk[off: off + n - k]; off += n - k
    Rn = np.linalg.qr(np.column_stack([H.double().cpu().numpy(), Y.double().cpu().numpy()]), mode='r')
    d = np.abs(np.abs(R) - np.abs(Rn[:n])) / np.abs(Rn[:n]).max()
    print(f"2d={d2} M={M} N={N} rel max|dR|={np.nanmax(d):.2e} nonfinite={int((~np.isfinite(R)).sum())}", flush=True)


for M, N in ((1, 100), (5, 77), (64, 256), (127, 5000), (128, 3000), (200, 999), (256, 1024), (256, 20000), (263, 4000)):
    run(M, N, 1)
for d2 in (1, 0):
    os.environ['ELMRNN_TSQR_2D'] = str(d2)
    for M in (256, 128):
        e = ELMRNN('lstm', 1, M, 4, 1, force_path=1)
        N = 4_000_000 if M == 256 else 1_000_000
        H = torch.rand(N, M, device='cuda'); Y = torch.rand(N, device='cuda')
        b, _ = e.solve_beta(H, Y); torch.cuda.synchronize()
        t0 = torch.cuda.Event(enable_timing=True); t1 = torch.cuda.Event(enable_timing=True)
        t0.record(); e.solve_beta(H, Y, b, info=False); t1.record(); torch.cuda.synchronize()
        print(f"solve 2d={d2} M={M} N={N}: {t0.elapsed_time(t1):.2f} ms", flush=True)
