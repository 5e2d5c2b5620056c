import os, sys, torch
sys.path.insert(0, '.')
from paper_1911_13252_b200 import ELMRNN
for v in (4, 3, 0):
    os.environ['ELMRNN_TSQR_VAR'] = str(v)
    e = ELMRNN('lstm', 1, 256, 4, 1, force_path=1)
    H = torch.rand(4_000_000, 256, device='cuda'); Y = torch.rand(4_000_000, device='cuda')
    b, _ = e.solve_beta(H, Y); torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True); t1 = torch.cuda.Event(enable_timing=True)
    t0.record(); e.solve_beta(H, Y, b, info=False); t1.record(); torch.cuda.synchronize()
    print("C4-size solve var", v, "ms", t0.elapsed_time(t1), flush=True)
