"""FC tensor-core builder check on the GPU: parity vs oracle and FMA path, C3fc timing."""
import sys
import numpy as np, torch
sys.path.insert(0, '.')
from paper_1911_13252_b200 import build, ELMRNN
build.build()
from oracle import oracle as orc
from synth import series as sy


def check(N, Q, S, L=-1, act=0, seed=3):
    s = sy.series('sin4', N + Q + 1)
    s = np.tile(s, (1, S))[:, :S] if S > s.shape[1] else s[:, :S]
    X, Y, _ = sy.windows(s, N, Q)
    Xd = torch.from_numpy(X).cuda()
    et = ELMRNN('fc', S, 128, Q, seed, force_path=2, fc_lags=L, act=act)
    Ht = et.build_H(Xd).cpu().numpy().astype(np.float64)
    net = orc.Net('fc', S=S, M=128, Q=Q, fc_lags=L, act=act)
    rows = np.arange(min(N, 400))
    Ho = orc.build_H(net, orc.gen_weights(net, seed), X[rows], threads=16)
    print(f"fc N={N} Q={Q} S={S} L={L} act={act} path={et.path}: |Htc-Ho|={np.abs(Ht[rows]-Ho).max():.3e} "
          f"nan={np.isnan(Ht).sum()}", flush=True)


for a in [(300, 2, 1), (1000, 10, 2), (333, 30, 4), (129, 1, 1), (700, 12, 2, 3), (300, 9, 1, 1, 1)]:
    check(*a)
N, Q, M = 1_000_000, 30, 128
X = torch.randn(N, Q, 4, device='cuda') * 0.5
e = ELMRNN('fc', 4, M, Q, 1)
H = torch.empty(N, M, device='cuda')
e.build_H(X, None, H); torch.cuda.synchronize()
t0 = torch.cuda.Event(enable_timing=True); t1 = torch.cuda.Event(enable_timing=True)
t0.record(); e.build_H(X, None, H); t1.record(); torch.cuda.synchronize()
ms = t0.elapsed_time(t1)
fl = 2 * M * M * sum(min(t - 1, Q) for t in range(1, Q + 1)) * N
print(f"C3 FC build_H: {ms:.2f} ms  {fl/ms/1e9:.1f} TFLOP/s (fp32-equivalent, lag contraction) path={e.path}", flush=True)
