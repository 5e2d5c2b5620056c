"""Run build_H once (after a warm-up) for ncu: python tools/prof_build.py ARCH M Q N [force_path]."""
import sys
import torch
sys.path.insert(0, '.')
from paper_1911_13252_b200 import ELMRNN
arch, M, Q, N = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
fp = int(sys.argv[5]) if len(sys.argv) > 5 else 0
S = 4 if arch in ("gru", "fc") else 1
X = torch.randn(N, Q, S, device='cuda') * 0.5
e = ELMRNN(arch, S, M, Q, 1, force_path=fp)
H = e.build_H(X)
H = e.build_H(X, None, H)
torch.cuda.synchronize()
print("path", e.path)
