"""TSQR timing at C4 size + quick parity vs oracle on a small case."""
import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_1911_13252_b200 import ELMRNN
from oracle import oracle as orc
for M, N in ((256, 4_000_000), (64, 100_000), (20, 1000)):
    e = ELMRNN('lstm', 1, M, 4, 1, force_path=1)
    g = torch.Generator(device='cuda').manual_seed(0)
    H = torch.rand(N, M, device='cuda', generator=g)
    Y = torch.rand(N, device='cuda', generator=g)
    b, info = e.solve_beta(H, Y)
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True); t1 = torch.cuda.Event(enable_timing=True)
    t0.record()
    for _ in range(3): e.solve_beta(H, Y, b, info=False)
    t1.record(); torch.cuda.synchronize()
    ms = t0.elapsed_time(t1) / 3
    fl = 2.0 * (M + 1) ** 2 * N
    print(f"M={M} N={N}: solve {ms:.2f} ms  {fl/ms/1e9:.2f} TFLOP/s fp64", flush=True)
    if N <= 100_000:
        bo, io = orc.lstsq(H.double().cpu().numpy(), Y.double().cpu().numpy())
        print("   rel dbeta vs oracle (same H):", np.linalg.norm(b.cpu().numpy() - bo) / np.linalg.norm(bo))
