"""TSQR variant check: R vs numpy QR on random matrices, and C4/C3-size solve timing.
usage: python tools/qr2.py ENVVAR=VAL [...]   (each arg is one variant; '-' = defaults)"""
import os, sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_1911_13252_b200 import ELMRNN

variants = sys.argv[1:] or ['-']


def setenv(v):
    for k in ('ELMRNN_TSQR_2D', 'ELMRNN_TSQR_WY', 'ELMRNN_TSQR_VAR'):
        os.environ.pop(k, None)
    if v != '-':
        for kv in v.split(','):
            k, val = kv.split('=')
            os.environ[k] = val


def run(M, N):
    e = ELMRNN('lstm', 1, M, 4, 1, force_path=1)
    g = torch.Generator(device='cuda').manual_seed(M + N)
    H = torch.rand(N, M, device='cuda', generator=g); Y = torch.rand(N, device='cuda', generator=g)
    Rpk = e.solve_local(H, Y).cpu().numpy()
    n = M + 1; R = np.zeros((n, n)); off = 0
    for k in range(n):
        R[k, k:] = Rpk[off: off + n - k]; off += n - k
    Rn = np.linalg.qr(np.column_stack([H.double().cpu().numpy(), Y.double().cpu().numpy()]), mode='r')
    d = np.abs(np.abs(R) - np.abs(Rn[:n])) / np.abs(Rn[:n]).max()
    return np.nanmax(d), int((~np.isfinite(R)).sum())


for v in variants:
    setenv(v)
    worst = 0.0
    for M, N in ((1, 100), (5, 77), (15, 300), (16, 300), (64, 256), (127, 5000), (128, 3000), (200, 999),
                 (256, 1024), (256, 20000), (263, 4000), (511, 3000)):
        d, nf = run(M, N)
        worst = max(worst, d)
        if d > 1e-12 or nf:
            print(f"  {v} M={M} N={N}: rel max|dR|={d:.2e} nonfinite={nf}", flush=True)
    print(f"{v}: worst rel |dR| = {worst:.2e}", flush=True)
    for M, N in ((256, 4_000_000), (128, 1_000_000), (64, 100_000)):
        e = ELMRNN('lstm', 1, M, 4, 1, force_path=1)
        H = torch.rand(N, M, device='cuda'); Y = torch.rand(N, device='cuda')
        b, _ = e.solve_beta(H, Y); torch.cuda.synchronize()
        t0 = torch.cuda.Event(enable_timing=True); t1 = torch.cuda.Event(enable_timing=True)
        t0.record(); e.solve_beta(H, Y, b, info=False); t1.record(); torch.cuda.synchronize()
        print(f"{v}: solve M={M} N={N}: {t0.elapsed_time(t1):.2f} ms", flush=True)
