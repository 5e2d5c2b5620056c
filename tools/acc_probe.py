"""Accuracy probe of an H builder (dev tool, GPU box): max|dH|, the
||H_gpu - H_o||_F / ||fp32(H_o) - H_o||_F ratio and the beta deviation in units
of the fp32-rounding floor (oracle/parity_rule.py) on ill-conditioned cases.
Select a library variant with ELMRNN_LIB=tools/dbg/libelmrnn_<name>.so."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle import oracle as orc  # noqa: E402
from oracle import parity_rule as pr  # noqa: E402
from paper_1911_13252_b200 import ELMRNN  # noqa: E402
from synth import series as sy  # noqa: E402

CASES = {"lstm256mg": ("lstm", 8000, 1, 256, 50, "mg", 0.01), "lstm512ar": ("lstm", 10277, 1, 512, 4, "ar5", 0.0),
         "lstm128mg": ("lstm", 6000, 1, 128, 30, "mg", 0.01), "gru128mg": ("gru", 6000, 1, 128, 30, "mg", 0.01),
         "fc128sin": ("fc", 3000, 4, 128, 30, "sin4", 0.0), "gru512ar": ("gru", 10277, 1, 512, 4, "ar5", 0.0)}
for name in sys.argv[1:] or list(CASES):
    arch, N, S, M, Q, kind, noise = CASES[name]
    s = sy.series(kind, N + Q, seed=11, noise=noise)
    X, Y, _ = sy.windows(s[:, :S], N, Q)
    e = ELMRNN(arch, S, M, Q, 5)
    H, beta, info = e.train(torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda())
    Hg = H.cpu().numpy().astype(np.float64)
    net = orc.Net(arch, S=S, M=M, Q=Q)
    Ho = orc.build_H(net, orc.gen_weights(net, 5), X, threads=os.cpu_count())
    d = Hg - Ho
    bd = pr.bounds(Ho, Y)
    rel = np.linalg.norm(beta.cpu().numpy() - bd.b_ref) / np.linalg.norm(bd.b_ref)
    H32 = Ho.astype(np.float32).astype(np.float64)
    ratio = np.linalg.norm(d) / np.linalg.norm(H32 - Ho)
    print(f"{os.environ.get('ELMRNN_LIB', 'default')} {name} path={e.path}: max|dH|={np.abs(d).max():.2e} "
          f"mean dH={d.mean():.2e} ratio={ratio:.1f} cond={bd.cond:.1e} dbeta={rel:.2e} = {rel / bd.floor_b:.1f} floor",
          flush=True)
