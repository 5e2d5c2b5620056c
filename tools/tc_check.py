"""Quick tensor-core builder check on the GPU: parity vs oracle and FMA path, timing."""
import sys, time
import numpy as np, torch
sys.path.insert(0, '.')
from paper_1911_13252_b200 import build, ELMRNN
build.build()
from oracle import oracle as orc
from synth import series as sy

def check(M, N, Q, S=1, seed=3, arch='lstm'):
    s = sy.series('mg' if S == 1 else 'sin4', N + Q, noise=0.01)
    X, Y, _ = sy.windows(s[:, :S], N, Q)
    Xd = torch.from_numpy(X).cuda()
    et = ELMRNN(arch, S, M, Q, seed, force_path=2)
    ef = ELMRNN(arch, S, M, Q, seed, force_path=1)
    Ht = et.build_H(Xd).cpu().numpy().astype(np.float64)
    Hf = ef.build_H(Xd).cpu().numpy().astype(np.float64)
    net = orc.Net(arch, S=S, M=M, Q=Q)
    rows = np.arange(min(N, 512))
    Ho = orc.build_H(net, orc.gen_weights(net, seed), X[rows], threads=16)
    print(f"{arch} M={M} N={N} Q={Q} S={S} path={et.path}: |Htc-Ho|={np.abs(Ht[rows]-Ho).max():.3e} "
          f"|Hfma-Ho|={np.abs(Hf[rows]-Ho).max():.3e} |Htc-Hfma|all={np.abs(Ht-Hf).max():.3e} "
          f"nan={np.isnan(Ht).sum()}", flush=True)

for args in [(256, 300, 2), (256, 1000, 10), (128, 1000, 10), (256, 777, 50), (128, 500, 30, 4), (256, 129, 1)]:
    check(*args)
for args in [(128, 300, 2, 1), (128, 1000, 30, 4), (128, 129, 1, 1)]:
    check(*args, arch='gru')
# GRU C3 timing
N, Q, M = 1_000_000, 30, 128
X = torch.randn(N, Q, 4, device='cuda') * 0.5
e = ELMRNN('gru', 4, M, Q, 1)
H = torch.empty(N, M, device='cuda')
e.build_H(X, None, H); torch.cuda.synchronize()
t0 = torch.cuda.Event(enable_timing=True); t1 = torch.cuda.Event(enable_timing=True)
t0.record(); e.build_H(X, None, H); t1.record(); torch.cuda.synchronize()
ms = t0.elapsed_time(t1)
fl = Q * (6 * 4 * M + 6 * M * M + 5 * M) * N
print(f"C3 GRU build_H tc: {ms:.2f} ms  {fl/ms/1e9:.1f} TFLOP/s (fp32-equivalent) path={e.path}", flush=True)

# timing at C4 size
N, Q, M = 4_000_000, 50, 256
X = torch.randn(N, Q, 1, device='cuda') * 0.5
e = ELMRNN('lstm', 1, M, Q, 1)
H = torch.empty(N, M, device='cuda')
e.build_H(X, None, H); torch.cuda.synchronize()
t0 = torch.cuda.Event(enable_timing=True); t1 = torch.cuda.Event(enable_timing=True)
t0.record(); e.build_H(X, None, H); t1.record(); torch.cuda.synchronize()
ms = t0.elapsed_time(t1)
fl = Q * (8 * M + 8 * M * M + 6 * M) * N
print(f"C4 build_H tc: {ms:.1f} ms  {fl/ms/1e9:.1f} TFLOP/s (fp32-equivalent)", flush=True)
