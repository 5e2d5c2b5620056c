"""Time the TSQR solve at the C4 shape under env variants: python tools/qr_time.py [M N]."""
import os, sys, subprocess, json
sys.path.insert(0, '.')
if len(sys.argv) > 1 and sys.argv[1] == "child":
    import torch
    from paper_1911_13252_b200 import ELMRNN
    M, N = int(sys.argv[2]), int(sys.argv[3])
    e = ELMRNN('lstm', 1, M, 4, 1, force_path=1)
    g = torch.Generator(device='cuda').manual_seed(0)
    H = torch.rand(N, M, device='cuda', generator=g) - 0.5
    Y = torch.rand(N, device='cuda', generator=g) - 0.5
    beta = torch.empty(M, dtype=torch.float64, device='cuda')
    for _ in range(2):
        e.solve_beta(H, Y, beta, info=False)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5):
        e.solve_beta(H, Y, beta, info=False)
    b.record(); torch.cuda.synchronize()
    print(a.elapsed_time(b) / 5)
    sys.exit(0)
M, N = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (256, 4_000_000)
variants = [json.loads(v) for v in os.environ.get("QR_VARIANTS", "").split(";") if v] or [
    {}, {"ELMRNN_TSQR_LEVELS": "0"}, {"ELMRNN_TSQR_WY_ROWS": "64"}, {"ELMRNN_TSQR_WY_ROWS": "96"},
    {"ELMRNN_TSQR_WY_ROWS": "16"}, {"ELMRNN_TSQR_WY_WARPS": "8"}, {"ELMRNN_TSQR_WY_WARPS": "2"},
    {"ELMRNN_TSQR_WY": "0"}]
for v in variants:
    env = dict(os.environ, **v)
    out = subprocess.run([sys.executable, __file__, "child", str(M), str(N)], env=env, capture_output=True, text=True)
    print(json.dumps(v), out.stdout.strip() or out.stderr[-300:], flush=True)
