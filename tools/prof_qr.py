"""One TSQR solve for ncu: python tools/prof_qr.py M N."""
import sys, torch
sys.path.insert(0, '.')
from paper_1911_13252_b200 import ELMRNN
M, N = int(sys.argv[1]), int(sys.argv[2])
e = ELMRNN('lstm', 1, M, 4, 1, force_path=1)
H = torch.rand(N, M, device='cuda'); Y = torch.rand(N, device='cuda')
b, _ = e.solve_beta(H, Y)
b, _ = e.solve_beta(H, Y)
torch.cuda.synchronize()
