"""Developer timing / profiling driver (not product code; run on the GPU box).

  python tools/prof.py qr M N [reps]          time the TSQR solve of a random N x M [H | Y]
  python tools/prof.py build ARCH M Q N [S]   time elmrnn_build_H on random windows
Both print one JSON line (CUDA events on the current stream, after warm-up).
Variants: export ELMRNN_TESTING=1 plus the knobs of csrc/common.cuh `Tune`.
Under ncu (`-k regex:<kernel> -c 1`) use reps = 1.
"""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_1911_13252_b200 import ELMRNN  # noqa: E402


def timed(fn, reps):
    for _ in range(2 if reps > 1 else 0):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def main():
    cmd = sys.argv[1]
    g = torch.Generator(device="cuda").manual_seed(0)
    if cmd == "qr":
        M, N = int(sys.argv[2]), int(sys.argv[3])
        reps = int(sys.argv[4]) if len(sys.argv) > 4 else 5
        e = ELMRNN("lstm", 1, M, 4, 1, force_path=1)
        H = torch.rand(N, M, device="cuda", generator=g) - 0.5
        Y = torch.rand(N, device="cuda", generator=g) - 0.5
        beta = torch.empty(M, dtype=torch.float64, device="cuda")
        ms = timed(lambda: e.solve_beta(H, Y, beta, info=False), reps)
        floor = 2.0 * N * (M + 1) ** 2 / 37.2e12 * 1e3
        print(json.dumps({"op": "qr", "M": M, "N": N, "ms": ms, "fp64_floor_ms": floor, "frac": floor / ms}))
    elif cmd == "build":
        arch, M, Q, N = sys.argv[2], int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5])
        S = int(sys.argv[6]) if len(sys.argv) > 6 else 1
        reps = int(sys.argv[7]) if len(sys.argv) > 7 else 5
        e = ELMRNN(arch, S, M, Q, 1)
        X = torch.randn(N, Q, S, device="cuda", generator=g)
        H = torch.empty(N, M, device="cuda")
        ms = timed(lambda: e.build_H(X, None, H), reps)
        print(json.dumps({"op": "build", "arch": arch, "M": M, "Q": Q, "N": N, "S": S, "path": e.path, "ms": ms}))
    else:
        raise SystemExit(__doc__)


if __name__ == "__main__":
    main()
