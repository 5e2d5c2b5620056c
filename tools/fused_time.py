"""Time elmrnn_train (fused build -> leaf) against build_H + solve_beta on a config (dev tool)."""
import sys
import torch
sys.path.insert(0, ".")
from paper_1911_13252_b200 import ELMRNN  # noqa: E402
from synth import series as sy  # noqa: E402

cfg = sys.argv[1]
c = sy.CONFIGS[cfg]
X, Y, _ = sy.config_inputs(cfg)
e = ELMRNN(c["arch"], c["S"], c["M"], c["Q"], 1)
Xd, Yd = torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda()
H = torch.empty(X.shape[0], c["M"], device="cuda")
beta = torch.empty(c["M"], dtype=torch.float64, device="cuda")


def t(fn, reps=50):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3


def unfused():
    e.build_H(Xd, None, H)
    e.solve_beta(H, Yd, beta, info=False)


print(cfg, "fused" if e.train_fused else "not fused", "train us", t(lambda: e.train_direct(Xd, Yd, beta=beta, info=False)),
      "build+solve us", t(unfused))
