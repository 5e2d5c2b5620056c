"""TSQR variant sweep: correctness vs oracle (small N) and timing (large N)."""
import os, subprocess, sys
code = r'''
import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_1911_13252_b200 import ELMRNN
from oracle import oracle as orc
M, Nbig = int(sys.argv[1]), int(sys.argv[2])
e = ELMRNN('lstm', 1, M, 4, 1, force_path=1)
g = torch.Generator(device='cuda').manual_seed(0)
H = torch.rand(4 * M, M, device='cuda', generator=g); Y = torch.rand(4 * M, device='cuda', generator=g)
b, info = e.solve_beta(H, Y)
bo, _ = orc.lstsq(H.double().cpu().numpy(), Y.double().cpu().numpy())
err = np.linalg.norm(b.cpu().numpy() - bo) / np.linalg.norm(bo)
H = torch.rand(Nbig, M, device='cuda', generator=g); Y = torch.rand(Nbig, device='cuda', generator=g)
e.solve_beta(H, Y, b, info=False); torch.cuda.synchronize()
t0 = torch.cuda.Event(enable_timing=True); t1 = torch.cuda.Event(enable_timing=True)
t0.record(); e.solve_beta(H, Y, b, info=False); t1.record(); torch.cuda.synchronize()
print(f"M={M} var={sys.argv[3]} rel_err={err:.2e} N={Nbig} ms={t0.elapsed_time(t1):.2f}", flush=True)
'''
for M, N, vs in ((256, 4_000_000, (0, 3, 1, 2)), (511, 200_000, (1, 2)), (64, 100_000, (0, 3, 1, 2)), (20, 1000, (0, 3, 1, 2))):
    for v in vs:
        env = dict(os.environ, ELMRNN_TSQR_VAR=str(v))
        r = subprocess.run([sys.executable, "-c", code, str(M), str(N), str(v)], env=env, capture_output=True, text=True, timeout=300)
        print(r.stdout.strip() or r.stderr[-300:], flush=True)
