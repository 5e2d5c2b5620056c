"""e2e experiment: plain copy-then-build vs chunked build_H_from_host (C4 shape)."""
import sys, torch
sys.path.insert(0, '.')
from paper_1911_13252_b200 import ELMRNN
N, Q, M = 4_000_000, 50, 256
Xh = (torch.rand(N, Q, 1) * 0.5).pin_memory()
Xd = torch.empty(N, Q, 1, device='cuda'); H = torch.empty(N, M, device='cuda')
e = ELMRNN('lstm', 1, M, Q, 1)
cs = torch.cuda.Stream()
def t(fn, K=3):
    fn(); torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(K): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / K
print("build only", t(lambda: e.build_H(Xd, None, H)), flush=True)
print("copy only", t(lambda: Xd.copy_(Xh, non_blocking=True)), flush=True)
print("copy then build", t(lambda: (Xd.copy_(Xh, non_blocking=True), e.build_H(Xd, None, H))), flush=True)
for c in (1, 2, 4, 8, 16):
    print(f"chunks={c}", t(lambda: e.build_H_from_host(Xh, Xd, H, chunks=c, copy_stream=cs)), flush=True)
for c in (2, 8):
    def seq():
        cuts = [N * k // c for k in range(c + 1)]
        for a, b in zip(cuts[:-1], cuts[1:]):
            e.build_H(Xd[a:b], None, H[a:b])
    print(f"build in {c} chunks (no copy)", t(seq), flush=True)
