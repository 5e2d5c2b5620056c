"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle.

Tolerances (BASELINE.json north_star):
  H       max |H_gpu - H_oracle| <= 1e-5 (fp32 arithmetic vs fp64)
  beta    ||beta_gpu - beta_ref|| / ||beta_ref|| <= max(1e-3, 8 floor_b) end to end, floor_b =
          the deviation fp32 rounding of the oracle's own H alone causes (fixed rule, reading
          R26, tests/parity_rule.py); the literal 1e-3 on the well-conditioned cases (one per
          builder path); <= 1e-12 cond(R) when both solvers factor the identical fp32 H
  RMSE    relative difference <= max(1e-4, 8 floor_r); literal 1e-4 on the well-conditioned cases
  weights bit-exact (integer RNG, identical rounding)
"""
import numpy as np
import pytest
import torch

from oracle import oracle as orc
from synth import series as sy
from oracle import parity_rule as pr

pytestmark = pytest.mark.gpu

H_TOL = 1e-5


@pytest.fixture(scope="module", autouse=True)
def _lib():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1911_13252_b200 import build
    build.build()


def E(*a, **k):
    from paper_1911_13252_b200 import ELMRNN
    return ELMRNN(*a, **k)


def oracle_net(arch, S, M, Q, **o):
    return orc.Net(arch, S=S, M=M, Q=Q, **{k: v for k, v in o.items() if k in
                                           ("F", "R", "act", "fc_lags", "rec_scale", "weight_grid")})


def inputs(N, Q, S, seed=0, kind=None):
    if kind is None:
        kind = "sin4" if S == 4 else "mg"
    s = sy.series(kind, N + Q + 1, seed=seed)
    if S > s.shape[1]:
        s = np.tile(s, (1, S))[:, :S]
    X, Y, Yfb = sy.windows(s[:, :S], N, Q)
    return X, Y, Yfb


def gpu_H(arch, S, M, Q, seed, X, Yfb=None, **o):
    e = E(arch, S, M, Q, seed, **o)
    Xd = torch.from_numpy(X).cuda()
    Yd = torch.from_numpy(Yfb).cuda() if Yfb is not None else None
    H = e.build_H(Xd, Yd)
    torch.cuda.synchronize()
    return e, H.cpu().numpy().astype(np.float64)


# ------------------------------------------------------------------------- weights
@pytest.mark.parametrize("arch,M,Q,o", [
    ("elman", 20, 10, {}), ("jordan", 7, 5, {}), ("narmax", 9, 6, {"F": 3, "R": 2}), ("fc", 12, 4, {}),
    ("fc", 12, 4, {"fc_lags": 1, "weight_grid": 1}), ("lstm", 33, 3, {}), ("lstm", 16, 3, {"weight_grid": 1}),
    ("gru", 40, 3, {"weight_grid": 2}), ("gru", 8, 2, {"rec_scale": 1}),
    ("lstm_diag", 21, 4, {}), ("gru_diag", 17, 3, {"rec_scale": 1}), ("fc_eq8", 12, 5, {"fc_lags": 3})])
def test_weights_bitwise(arch, M, Q, o):
    S = 3
    e = E(arch, S, M, Q, 12345, **o)
    ref = orc.gen_weights(oracle_net(arch, S, M, Q, **o), 12345)
    for k, w in enumerate(ref):
        g = e.get_weights(k).numpy()
        np.testing.assert_array_equal(g.view(np.uint32), w.reshape(-1).view(np.uint32))


# ------------------------------------------------------------------------- H parity grid
GRID = [
    # arch, N, S, M, Q, opts, use_yfb
    ("elman", 1000, 1, 20, 10, {}, False),          # C1 shape
    ("elman", 333, 4, 50, 1, {}, False),            # Q = 1, S = 4
    ("elman", 77, 1, 3, 50, {"act": 1}, False),
    ("elman", 64, 2, 37, 100, {}, False),
    ("jordan", 1000, 1, 64, 20, {}, False),         # C2 shape, Yfb derived from X
    ("jordan", 515, 1, 64, 20, {}, True),
    ("narmax", 1000, 1, 64, 20, {}, True),
    ("narmax", 300, 4, 5, 10, {"F": 3, "R": 7}, True),
    ("narmax", 200, 1, 5, 10, {"F": 0, "R": 0}, False),
    ("fc", 300, 4, 128, 30, {}, False),             # C3 shape (ring in global memory)
    ("fc", 261, 1, 50, 10, {}, False),
    ("fc", 100, 2, 3, 5, {"fc_lags": 1, "act": 1}, False),
    ("fc", 65, 1, 1, 9, {}, False),
    ("gru", 300, 4, 128, 30, {}, False),            # C3 shape
    ("gru", 257, 1, 50, 10, {}, False),
    ("gru", 100, 1, 1, 10, {}, False),
    ("lstm", 200, 1, 256, 50, {}, False),           # C4 shape
    ("lstm", 301, 4, 50, 10, {}, False),
    ("lstm", 129, 1, 3, 1, {}, False),
    ("lstm", 64, 1, 32, 100, {"weight_grid": 1}, False),
    # paper-literal per-cell variants
    ("lstm_diag", 300, 4, 128, 30, {}, False),      # C3 shape
    ("lstm_diag", 257, 1, 50, 100, {}, False),
    ("lstm_diag", 99, 7, 3, 1, {}, False),           # S > 4: runtime-S loop
    ("gru_diag", 300, 4, 128, 30, {}, False),
    ("gru_diag", 129, 2, 33, 50, {"rec_scale": 1}, False),
    ("fc_eq8", 300, 4, 128, 30, {}, False),
    ("fc_eq8", 200, 1, 20, 12, {"fc_lags": 3, "act": 1}, False),
    ("fc_eq8", 50, 1, 1, 9, {}, False),
]


@pytest.mark.parametrize("arch,N,S,M,Q,o,yfb", GRID)
def test_H_parity(arch, N, S, M, Q, o, yfb):
    X, Y, Yfb = inputs(N, Q, S, seed=N + M)
    Yfb = Yfb if yfb else None
    _, Hg = gpu_H(arch, S, M, Q, 7, X, Yfb, **o)
    net = oracle_net(arch, S, M, Q, **o)
    Ho = orc.build_H(net, orc.gen_weights(net, 7), X, Yfb, threads=8)
    err = np.abs(Hg - Ho).max()
    assert err <= H_TOL, f"max |dH| = {err:.3e}"


# tcgen05 LSTM builder (3-pass fp16 hi/lo split): ragged tiles, Q = 1, S padded 3 -> 4
TC_CASES = [("lstm", 256, 333, 50, 1), ("lstm", 256, 129, 1, 1), ("lstm", 128, 1000, 10, 3),
            ("lstm", 128, 257, 30, 4), ("lstm", 256, 2100, 20, 2), ("lstm", 128, 64, 7, 1),
            ("gru", 128, 333, 30, 4), ("gru", 128, 129, 1, 1), ("gru", 128, 1000, 10, 2), ("gru", 128, 300, 50, 3),
            ("fc", 128, 333, 30, 4), ("fc", 128, 129, 1, 1), ("fc", 128, 1000, 10, 2), ("fc", 128, 300, 2, 3)]


@pytest.mark.parametrize("arch,M,N,Q,S", TC_CASES)
def test_tc_parity(arch, M, N, Q, S):
    X, Y, _ = inputs(N, Q, S, seed=M + Q)
    e, Hg = gpu_H(arch, S, M, Q, 4, X, force_path=2)
    assert e.path == 2
    net = orc.Net(arch, S=S, M=M, Q=Q)
    Ho = orc.build_H(net, orc.gen_weights(net, 4), X, threads=8)
    err = np.abs(Hg - Ho).max()
    assert err <= H_TOL, f"max |dH| = {err:.3e}"
    _, Hf = gpu_H(arch, S, M, Q, 4, X, force_path=1)
    assert np.abs(Hf - Ho).max() <= H_TOL


@pytest.mark.parametrize("L,act,N,Q", [(3, 0, 700, 12), (1, 1, 300, 9), (5, 1, 520, 40), (40, 0, 260, 20)])
def test_fc_tc_lag_ring(L, act, N, Q):
    """FC tensor path with a lag window shorter than Q (ring wrap-around,
    S2.2.4 prose reading R9), longer than Q, and tanh activations."""
    X, _, _ = inputs(N, Q, 2, seed=L + Q)
    e, Hg = gpu_H("fc", 2, 128, Q, 6, X, force_path=2, fc_lags=L, act=act)
    assert e.path == 2
    net = oracle_net("fc", 2, 128, Q, fc_lags=L, act=act)
    Ho = orc.build_H(net, orc.gen_weights(net, 6), X, threads=8)
    err = np.abs(Hg - Ho).max()
    assert err <= H_TOL, f"max |dH| = {err:.3e}"


@pytest.mark.parametrize("arch,M,N,Q,S", [("lstm", 256, 700, 20, 1), ("lstm", 128, 300, 9, 2),
                                           ("gru", 128, 500, 30, 4), ("fc", 128, 400, 12, 3)])
def test_tc_two_pass_fp16_grid(arch, M, N, Q, S):
    """weight_grid = 1 (fp16-representable U / A_k, SURVEY 8(c) "2xFP16 A-split"):
    the tensor path drops the hi.lo pass; parity against the oracle run on the
    same grid-rounded weights."""
    X, _, _ = inputs(N, Q, S, seed=M + Q + 1)
    e, Hg = gpu_H(arch, S, M, Q, 8, X, force_path=2, weight_grid=1)
    assert e.path == 2
    net = oracle_net(arch, S, M, Q, weight_grid=1)
    Ho = orc.build_H(net, orc.gen_weights(net, 8), X, threads=8)
    err = np.abs(Hg - Ho).max()
    assert err <= H_TOL, f"max |dH| = {err:.3e}"


def test_H_written_once_and_ld_respected():
    N, M, Q = 100, 20, 10
    X, _, _ = inputs(N, Q, 1)
    e = E("elman", 1, M, Q, 3)
    Xp = torch.zeros((N, 16), dtype=torch.float32, device="cuda")   # padded ldx = 16
    Xp[:, :Q] = torch.from_numpy(X.reshape(N, Q)).cuda()
    H = torch.full((N, 24), 7.0, device="cuda")                      # ldh = 24
    e.build_H(Xp, None, H[:, :M])
    torch.cuda.synchronize()
    assert torch.all(H[:, M:] == 7.0)
    ref = orc.build_H(orc.Net("elman", 1, M, Q), orc.gen_weights(orc.Net("elman", 1, M, Q), 3), X)
    assert np.abs(H[:, :M].cpu().numpy() - ref).max() <= H_TOL


@pytest.mark.parametrize("arch,M,Q", [("lstm", 512, 4), ("gru", 512, 4), ("lstm", 1024, 2), ("gru", 256, 3)])
def test_wide_pair_units_match_single(arch, M, Q, monkeypatch):
    """Wide builders: MMA units of two chunks (N = 256, default) against single-chunk
    units (N = 128, ELMRNN_WIDE_PAIR=0 through the testing knob read at init): the
    same per-element K order, so H agrees to rounding (asserted 1e-6) on a ragged N."""
    N = 2 * 128 + 77
    X, _, _ = inputs(N, Q, 1, seed=M)
    Xd = torch.from_numpy(X).cuda()
    H1 = E(arch, 1, M, Q, 7).build_H(Xd)
    monkeypatch.setenv("ELMRNN_TESTING", "1")
    monkeypatch.setenv("ELMRNN_WIDE_PAIR", "0")
    H0 = E(arch, 1, M, Q, 7).build_H(Xd)
    torch.cuda.synchronize()
    assert float((H1 - H0).abs().max()) <= 1e-6


@pytest.mark.parametrize("arch,M,Q,S", [("lstm", 256, 12, 1), ("lstm", 128, 10, 2), ("gru", 128, 10, 4),
                                        ("lstm", 512, 4, 1), ("gru", 256, 4, 1), ("fc", 128, 6, 1)])
def test_x_staging_layouts_bitwise(arch, M, Q, S):
    """a1 window staging (one cp.async.bulk of each full tile's X block): a padded
    row stride (ldx > Q*d, the padding travels with the block) and an X that is not
    16-byte aligned (staging off, x(t) through L1) give bitwise the H of the
    contiguous, aligned X; N is ragged so the partial last tile is read directly."""
    N = 3 * 128 + 45
    X, _, _ = inputs(N, Q, S, seed=M + Q)
    e = E(arch, S, M, Q, 6)
    assert e.path == 2
    Xd = torch.from_numpy(X).cuda()
    H0 = e.build_H(Xd)
    pad = torch.full((N, Q * S + 5), float("nan"), device="cuda")
    pad[:, :Q * S] = Xd.reshape(N, Q * S)
    H1 = e.build_H(pad[:, :Q * S])
    flat = torch.zeros(N * Q * S + 1, device="cuda")
    flat[1:] = Xd.reshape(-1)
    H2 = e.build_H(flat[1:].view(N, Q * S))
    torch.cuda.synchronize()
    assert torch.equal(H0, H1) and torch.equal(H0, H2)


@pytest.mark.parametrize("arch,M", [("lstm", 128), ("gru", 32), ("elman", 20)])
def test_build_H_from_host_chunked(arch, M):
    """The chunked, copy-overlapped build from pinned host X equals build_H."""
    N, Q = 3001, 9
    X, _, _ = inputs(N, Q, 1)
    e = E(arch, 1, M, Q, 5)
    Xd = torch.from_numpy(X).cuda()
    H1 = e.build_H(Xd)
    Xh = torch.from_numpy(X).pin_memory()
    Xs = torch.empty_like(Xd)
    H2 = torch.empty_like(H1)
    e.build_H_from_host(Xh, Xs, H2, chunks=7)
    torch.cuda.synchronize()
    assert torch.equal(H1, H2)


def test_empty_and_errors():
    from paper_1911_13252_b200 import ElmrnnError
    e = E("gru", 1, 8, 4, 1)
    H = e.build_H(torch.empty((0, 4, 1), device="cuda"))
    assert H.shape == (0, 8)
    with pytest.raises(ElmrnnError, match="ERR_SHAPE"):
        e.build_H(torch.zeros((5, 3), device="cuda"))
    with pytest.raises(ElmrnnError, match="ERR_UNDERDETERMINED"):
        e.solve_beta(torch.zeros((5, 8), device="cuda"), torch.zeros(5, device="cuda"))
    with pytest.raises(ElmrnnError, match="ERR_ARG"):
        E("lstm", 0, 8, 4, 1)
    with pytest.raises(ElmrnnError, match="ERR_UNSUPPORTED"):
        E("lstm", 1, 1025, 4, 1)


# ------------------------------------------------------------------------- solve parity
# beta / RMSE rule: tests/parity_rule.py (R26) -- max(1e-3, 8 floor_b) and
# max(1e-4, 8 floor_r) with floor = the deviation the fp32 rounding of the oracle's own
# H alone causes; fixed, independent of the GPU's H error.
SOLVE_CASES = [("elman", 1000, 1, 20, 10, "mg", 0.0), ("jordan", 5000, 1, 64, 20, "ar5", 0.0),
               ("narmax", 5000, 1, 64, 20, "ar5", 0.0), ("gru", 3000, 4, 128, 30, "sin4", 0.0),
               ("fc", 2000, 4, 128, 30, "sin4", 0.0), ("lstm", 8000, 1, 256, 50, "mg", 0.01),
               ("lstm", 10277, 1, 512, 4, "ar5", 0.0), ("lstm", 6000, 1, 128, 30, "mg", 0.01),
               ("gru", 6000, 1, 128, 30, "mg", 0.01), ("gru", 10277, 1, 512, 4, "ar5", 0.0),
               ("lstm_diag", 3000, 4, 128, 30, "sin4", 0.0), ("gru_diag", 3000, 4, 128, 30, "sin4", 0.0),
               ("fc_eq8", 3000, 4, 128, 30, "sin4", 0.0)]


@pytest.mark.parametrize("arch,N,S,M,Q,kind,noise", SOLVE_CASES)
def test_solve_parity(arch, N, S, M, Q, kind, noise):
    s = sy.series(kind, N + Q, seed=11, noise=noise)
    X, Y, _ = sy.windows(s[:, :S], N, Q)
    e, Hg = gpu_H(arch, S, M, Q, 5, X)
    Hd = torch.from_numpy(Hg.astype(np.float32)).cuda()
    Yd = torch.from_numpy(Y).cuda()
    beta, info = e.solve_beta(Hd, Yd)
    beta = beta.cpu().numpy()
    # (a) solver isolation: oracle QR of the identical fp32 H (both fp64)
    b_iso, i_iso = orc.lstsq(Hg.astype(np.float32).astype(np.float64), Y)
    cond = np.linalg.cond(i_iso.R[:M, :M])
    assert np.linalg.norm(beta - b_iso) / np.linalg.norm(b_iso) <= 1e-12 * max(1.0, cond), cond
    assert abs(info.rmse - i_iso.rmse) / i_iso.rmse <= 1e-12 * max(1.0, cond)
    # (b) end to end against the oracle's own fp64 H (fixed rule R26)
    net = orc.Net(arch, S=S, M=M, Q=Q)
    Ho = orc.build_H(net, orc.gen_weights(net, 5), X, threads=8)
    pr.check(f"{arch} N={N} M={M} path={e.path}", beta, info.rmse, Hg, Ho, Y)
    assert info.status == 0 and info.n_total == N


# Well-conditioned end-to-end cases, one per H-builder path: four lagged channels of
# an AR(5) series (synth.lagged_channels), N >= 20 M rows plus a ragged tail, so
# cond(R) is 1e2-2e3 and the fp32-H floor ~1e-7: the north star's LITERAL bounds
# (1e-3 beta, 1e-4 RMSE) are what is tested, on the intended kernel.
WELL_COND = [
    # arch, M, Q, S, forced path (0 auto), expected path, kernel
    ("lstm", 128, 10, 4, 0, 2, "k_lstm_tc M=128"),
    ("lstm", 256, 10, 4, 0, 2, "k_lstm_tc M=256"),
    ("lstm", 512, 3, 4, 0, 2, "k_lstm_wide M=512"),
    ("lstm", 1024, 2, 4, 0, 2, "k_lstm_wide M=1024"),
    ("gru", 128, 10, 4, 0, 2, "k_gru_tc M=128"),
    ("gru", 256, 6, 4, 0, 2, "k_gru_wide M=256"),
    ("gru", 512, 3, 4, 0, 2, "k_gru_wide M=512"),
    ("gru", 384, 3, 4, 0, 2, "k_gru_wide M=384 (odd phase-2 chunk count: N = 128 units)"),
    ("fc", 128, 10, 4, 0, 2, "k_fc_tc M=128"),
    ("lstm", 64, 10, 4, 0, 1, "k_dense_fma LSTM"),
    ("gru", 32, 10, 4, 0, 1, "k_dense_fma GRU"),
    ("lstm", 256, 10, 4, 1, 1, "k_dense_fma LSTM M=256 (forced)"),
]


def well_cond_inputs(M, Q, S, seed=3):
    N = 20 * M + 37
    s = sy.lagged_channels(sy.series("ar5", N + Q + S + 1, seed=seed), S)
    X, Y, _ = sy.windows(s, N, Q)
    return X, Y


@pytest.mark.parametrize("arch,M,Q,S,force,path,kern", WELL_COND)
def test_solve_parity_well_conditioned(arch, M, Q, S, force, path, kern):
    X, Y = well_cond_inputs(M, Q, S)
    e = E(arch, S, M, Q, 5, force_path=force)
    assert e.path == path, kern
    Xd, Yd = torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda()
    H, beta, info = e.train(Xd, Yd)
    Hg = H.cpu().numpy().astype(np.float64)
    net = orc.Net(arch, S=S, M=M, Q=Q)
    Ho = orc.build_H(net, orc.gen_weights(net, 5), X, threads=16)
    assert np.abs(Hg - Ho).max() <= H_TOL
    _, _, bd = pr.check(f"{kern} N={X.shape[0]}", beta.cpu().numpy(), info.rmse, Hg, Ho, Y, literal=True)
    assert bd.floor_b < 1e-5, "case is meant to be well conditioned"
    assert info.status == 0


def test_virtual_ranks_merge_equals_single():
    N, M, Q = 4000, 64, 20
    X, Y, _ = inputs(N, Q, 1, kind="ar5")
    e, Hg = gpu_H("jordan", 1, M, Q, 2, X)
    Hd = torch.from_numpy(Hg.astype(np.float32)).cuda()
    Yd = torch.from_numpy(Y).cuda()
    b1, i1 = e.solve_beta(Hd, Yd)
    for P in (2, 3, 8):
        cuts = np.linspace(0, N, P + 1).astype(int)
        parts = [e.solve_local(Hd[a:b], Yd[a:b]).clone() for a, b in zip(cuts[:-1], cuts[1:])]
        bP, iP = e.solve_merge(torch.stack(parts), P, N)
        rel = (bP - b1).norm() / b1.norm()
        assert rel <= 1e-10, (P, float(rel))
        assert abs(iP.rmse - i1.rmse) <= 1e-10 * i1.rmse
    # an empty shard contributes R = 0
    parts = [e.solve_local(Hd, Yd).clone(), e.solve_local(Hd[:0], Yd[:0]).clone()]
    b2, _ = e.solve_merge(torch.stack(parts), 2, N)
    assert (b2 - b1).norm() / b1.norm() <= 1e-12


def _packed_to_R(Rpk, n):
    R = np.zeros((n, n))
    off = 0
    for k in range(n):
        R[k, k:] = Rpk[off: off + n - k]
        off += n - k
    return R


@pytest.mark.parametrize("M,N", [(200, 1001), (256, 20011), (300, 5003), (511, 3001), (129, 777), (256, 40),
                                 (400, 70000), (1024, 9000)])
def test_tsqr_wy_and_fold_agree(M, N, monkeypatch):
    """The blocked compact-WY TSQR (k_tsqr_leaf_wy, UT-transform trailing update on
    f64 tensor cores) and the per-column fold produce the same R of [H | Y] as
    numpy's Householder QR (LAPACK geqrf), up to row signs (reading R18)."""
    g = torch.Generator(device="cuda").manual_seed(M + N)
    H = torch.rand(N, M, device="cuda", generator=g) - 0.5
    Y = torch.rand(N, device="cuda", generator=g) - 0.5
    n = M + 1
    Rq = np.abs(np.linalg.qr(np.column_stack([H.double().cpu().numpy(), Y.double().cpu().numpy()]), mode="r"))
    Rn = np.zeros((n, n))
    Rn[: Rq.shape[0]] = Rq   # N < n: the trailing rows of R are zero
    scale = Rn.max()
    # blocked WY (two-phase pipelined leaf, forced for n <= 320 too, and the single-chain
    # leaf), per-column fold
    for wy, two in (("1", "2"), ("1", "0"), ("0", "1")):
        monkeypatch.setenv("ELMRNN_TESTING", "1")
        monkeypatch.setenv("ELMRNN_TSQR_WY", wy)
        monkeypatch.setenv("ELMRNN_WY_2PHASE", two)
        e = E("lstm", 1, M, 4, 1, force_path=1)
        R = _packed_to_R(e.solve_local(H, Y).cpu().numpy(), n)
        assert np.isfinite(R).all()
        assert np.abs(np.abs(R) - Rn).max() <= 1e-12 * scale, (wy, two)


@pytest.mark.parametrize("rows,M,N", [("16", 511, 600), ("16", 300, 3001), ("32", 1000, 1500)])
def test_tsqr_wy_deep_noise_cascade(rows, M, N, monkeypatch):
    """A leaf that folds many short tiles before reaching full rank drives the
    noise rows of its partial R into subnormals (DESIGN 6.3); the WY panel must
    treat t = x0^2 + |x|^2 <= 1e-280 as H = I (else rsqrt.approx.ftz gives NaN)."""
    monkeypatch.setenv("ELMRNN_TESTING", "1")
    monkeypatch.setenv("ELMRNN_TSQR_WY", "1")
    monkeypatch.setenv("ELMRNN_TSQR_WY_ROWS", rows)
    g = torch.Generator(device="cuda").manual_seed(M + N)
    H = torch.rand(N, M, device="cuda", generator=g) - 0.5
    Y = torch.rand(N, device="cuda", generator=g) - 0.5
    Rn = np.abs(np.linalg.qr(np.column_stack([H.double().cpu().numpy(), Y.double().cpu().numpy()]), mode="r"))
    e = E("lstm", 1, M, 4, 1, force_path=1)
    R = _packed_to_R(e.solve_local(H, Y).cpu().numpy(), M + 1)
    assert np.isfinite(R).all()
    assert np.abs(np.abs(R) - Rn).max() <= 1e-12 * Rn.max()


def test_ridge_and_nonfinite():
    from paper_1911_13252_b200 import ElmrnnError
    e = E("elman", 1, 4, 3, 1)
    H = np.ones((50, 4), np.float32)
    H[:, 1] = np.linspace(0, 1, 50)
    Y = np.linspace(-1, 2, 50).astype(np.float32)
    beta, info = e.solve_beta(torch.from_numpy(H).cuda(), torch.from_numpy(Y).cuda())
    assert info.status == 1 and info.rank_flag == 1
    b_ref, i_ref = orc.lstsq(H.astype(np.float64), Y.astype(np.float64))
    assert i_ref.status == 1
    np.testing.assert_allclose(beta.cpu().numpy(), b_ref, rtol=1e-6, atol=1e-9)
    assert info.ridge_lambda == pytest.approx(i_ref.ridge_lambda, rel=1e-12)
    Hn = H.copy()
    Hn[17, 2] = np.nan
    with pytest.raises(ElmrnnError, match="NONFINITE"):
        e.solve_beta(torch.from_numpy(Hn).cuda(), torch.from_numpy(Y).cuda())


def test_nonfinite_async_reported_by_sync():
    """An asynchronous solve (info == NULL) cannot return ERR_NONFINITE; the device
    flag is accumulated and elmrnn_sync reports it (then clears it)."""
    from paper_1911_13252_b200 import ElmrnnError
    for M in (4, 200):   # per-column fold and blocked-WY leaf
        e = E("elman", 1, M, 3, 1) if M < 10 else E("lstm", 1, M, 3, 1, force_path=1)
        H = torch.rand(3 * M, M, device="cuda")
        Y = torch.rand(3 * M, device="cuda")
        e.solve_beta(H, Y, info=False)
        e.sync()
        Hn = H.clone()
        Hn[5, 1] = float("nan")
        e.solve_beta(Hn, Y, info=False)
        e.solve_beta(H, Y, info=False)        # a later clean solve does not clear it
        with pytest.raises(ElmrnnError, match="NONFINITE"):
            e.sync()
        e.sync()                               # cleared by the check
        e.solve_local(Hn, Y)                   # row-sharded step 1 reports too
        with pytest.raises(ElmrnnError, match="NONFINITE"):
            e.sync()


@pytest.mark.parametrize("arch,N,S,M,Q,yfb,o", [("elman", 1000, 1, 20, 10, False, {}), ("jordan", 20000, 1, 64, 20, False, {}),
                                                ("narmax", 5000, 1, 64, 20, True, {"F": 3, "R": 7}),
                                                ("elman", 777, 2, 37, 25, False, {"act": 1}), ("gru", 3000, 1, 32, 10, False, {}),
                                                ("lstm", 3000, 4, 128, 10, False, {})])
def test_train_fused(arch, N, S, M, Q, yfb, o):
    """elmrnn_train: the fused build -> TSQR leaf (H never in
    memory) gives bitwise the beta of elmrnn_build_H + elmrnn_solve_beta; archs
    without the fused path take the workspace route and agree as well; the
    row-sharded elmrnn_train_local + merge equals the single call."""
    X, Y, Yfb = inputs(N, Q, S, seed=N + M, kind="ar5" if arch in ("jordan", "narmax") else None)
    e = E(arch, S, M, Q, 3, fused_train=1, **o)
    assert e.train_fused == (arch in ("elman", "jordan", "narmax"))
    assert not E(arch, S, M, Q, 3, **o).train_fused     # default route: build_H + solve (measured faster)
    Xd, Yd = torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda()
    Yfbd = torch.from_numpy(Yfb).cuda() if yfb else None
    b1, i1 = e.train_direct(Xd, Yd, Yfbd)
    H = e.build_H(Xd, Yfbd)
    b2, i2 = e.solve_beta(H, Yd)
    assert torch.equal(b1, b2), float((b1 - b2).norm() / b2.norm())
    assert i1.rmse == i2.rmse and i1.status == i2.status
    cuts = [0, N // 3, N]
    parts = [e.train_local(Xd[a:b], Yd[a:b], Yfbd[a:b] if yfb else None).clone() for a, b in zip(cuts[:-1], cuts[1:])]
    b3, _ = e.solve_merge(torch.stack(parts), 2, N)
    bo, io = orc.lstsq(H.double().cpu().numpy(), Y.astype(np.float64))
    cond = np.linalg.cond(io.R[:M, :M])
    assert float((b3 - b2).norm() / b2.norm()) <= 1e-12 * max(1.0, cond)
    # and against the oracle's own H (R26 rule)
    net = oracle_net(arch, S, M, Q, **o)
    Ho = orc.build_H(net, orc.gen_weights(net, 3), X, Yfb if yfb else None, threads=8)
    pr.check(f"train {arch} fused={e.train_fused}", b1.cpu().numpy(), i1.rmse, H.double().cpu().numpy(), Ho, Y)


def test_predict_parity():
    N, S, M, Q = 700, 1, 32, 10
    X, Y, _ = inputs(N, Q, S)
    e = E("gru", S, M, Q, 9)
    Xd = torch.from_numpy(X).cuda()
    H, beta, info = e.train(Xd, torch.from_numpy(Y).cuda())
    yhat = e.predict(Xd, beta).cpu().numpy()
    net = orc.Net("gru", S=S, M=M, Q=Q)
    Ho = orc.build_H(net, orc.gen_weights(net, 9), X)
    ref = orc.predict(Ho, beta.cpu().numpy())
    assert np.abs(yhat - ref).max() <= 1e-5 * max(1.0, np.abs(beta.cpu().numpy()).sum())
    assert np.sqrt(np.mean((yhat - Y) ** 2)) == pytest.approx(info.rmse, rel=1e-4)


# ------------------------------------------------------------------------- full-size configs
@pytest.mark.parametrize("cfg", ["C1", "C2j", "C2n"])
def test_full_config_end_to_end(cfg):
    c = sy.CONFIGS[cfg]
    X, Y, Yfb = sy.config_inputs(cfg)
    e = E(c["arch"], c["S"], c["M"], c["Q"], 1)
    H, beta, info = e.train(torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda())
    net = orc.Net(c["arch"], S=c["S"], M=c["M"], Q=c["Q"])
    Ho = orc.build_H(net, orc.gen_weights(net, 1), X, threads=8)
    Hg = H.cpu().numpy().astype(np.float64)
    assert np.abs(Hg - Ho).max() <= H_TOL
    pr.check(cfg, beta.cpu().numpy(), info.rmse, Hg, Ho, Y)


def oracle_R_chunked(H: torch.Tensor, Y: np.ndarray, chunk: int = 250_000, threads: int = 16):
    """The oracle's Householder R of the full [H | Y] (H the GPU's fp32 H, widened
    exactly): R factors of row chunks in parallel (ctypes releases the GIL), then the
    oracle's lstsq of their stack -- a TSQR tree of the oracle's own QR, which the
    oracle pins equal to the direct R (test_oracle_weights_solve)."""
    from concurrent.futures import ThreadPoolExecutor
    N, M = H.shape

    def one(a):
        b = min(N, a + chunk)
        Hc = H[a:b].cpu().numpy().astype(np.float64)
        return orc.lstsq(Hc, Y[a:b].astype(np.float64))[1].R

    with ThreadPoolExecutor(threads) as ex:
        Rs = list(ex.map(one, range(0, N, chunk)))
    S = np.concatenate(Rs, axis=0)
    return orc.lstsq(S[:, :M], S[:, M])


@pytest.mark.parametrize("cfg", ["C3gru", "C3fc", "C4"])
def test_full_config_sampled(cfg):
    """Full N in the bench launch configuration: sampled rows of H against the
    oracle (computed row by row); solver isolation at full N -- beta and the RMSE
    against the oracle's Householder solve of the GPU's own full fp32 H (chunked
    oracle TSQR); the normal-equation residual of beta in fp64."""
    c = sy.CONFIGS[cfg]
    X, Y, _ = sy.config_inputs(cfg)
    e = E(c["arch"], c["S"], c["M"], c["Q"], 1)
    Xd = torch.from_numpy(X).cuda()
    Yd = torch.from_numpy(Y).cuda()
    H, beta, info = e.train(Xd, Yd)
    rows = np.sort(np.random.default_rng(0).choice(c["N"], 96, replace=False))
    rows[-1] = c["N"] - 1
    net = orc.Net(c["arch"], S=c["S"], M=c["M"], Q=c["Q"])
    Ho = orc.build_H(net, orc.gen_weights(net, 1), X[rows], threads=8)
    assert np.abs(H[torch.from_numpy(rows).cuda()].cpu().numpy() - Ho).max() <= H_TOL
    b_iso, i_iso = oracle_R_chunked(H, Y)
    M = c["M"]
    cond = float(np.linalg.cond(i_iso.R[:M, :M]))
    rel = float(np.linalg.norm(beta.cpu().numpy() - b_iso) / np.linalg.norm(b_iso))
    drm = abs(info.rmse - i_iso.rho / np.sqrt(c["N"])) / (i_iso.rho / np.sqrt(c["N"]))
    print(f"{cfg} full N={c['N']}: solver isolation cond(R)={cond:.2e} rel dbeta={rel:.2e} rel drmse={drm:.2e}")
    assert rel <= 1e-12 * max(1.0, cond)
    assert drm <= 1e-10
    H64 = H.double()
    r = H64 @ beta - Yd.double()
    g = H64.T @ r
    assert float(g.abs().max()) <= 1e-8 * max(1.0, float((H64.T @ Yd.double()).abs().max()))
    rmse = float(r.norm()) / np.sqrt(c["N"])
    assert info.rmse == pytest.approx(rmse, rel=1e-6)


# ------------------------------------------------------------------------- C5 sweep (BASELINE configs[4])
# LSTM/GRU, M in {32, 128, 512, 1024}, Q in {10, 50, 100}, univariate MG+noise.
# N per case keeps the oracle (8 M^2 Q fp64 flop per LSTM sample) to seconds
# while spanning several tiles of the chosen builder plus a ragged tail
# (FMA tiles are 8-64 rows, tensor-core tiles 128).
def _c5_rows(M, Q):
    return {32: 300, 128: 300, 512: 45, 1024: 21}[M] if Q <= 10 else {32: 200, 128: 140, 512: 21, 1024: 11}[M]


C5_GRID = [(a, M, Q) for a in ("lstm", "gru") for M in (32, 128, 512, 1024) for Q in (10, 50, 100)]


@pytest.mark.parametrize("arch,M,Q", C5_GRID)
def test_c5_sweep_H_parity(arch, M, Q):
    N = _c5_rows(M, Q)
    s = sy.series("mg", N + Q + 1, seed=M + Q, noise=0.01)
    X, Y, _ = sy.windows(s[:, :1], N, Q)
    e, Hg = gpu_H(arch, 1, M, Q, 3, X)
    net = orc.Net(arch, S=1, M=M, Q=Q)
    Ho = orc.build_H(net, orc.gen_weights(net, 3), X, threads=8)
    err = np.abs(Hg - Ho).max()
    assert err <= H_TOL, f"path {e.path}: max |dH| = {err:.3e}"


# tcgen05 LSTM builder for wide layers (hbuild_lstm_wide.cu, 256 < M <= 1024):
# several 128-row tiles, ragged tail, more tiles than... S = 1, 2, 3 (padded to 4)
WIDE_CASES = [("lstm", 512, 300, 10, 1), ("lstm", 1024, 260, 3, 1), ("lstm", 384, 333, 7, 2),
              ("lstm", 640, 129, 5, 3), ("lstm", 512, 1000, 2, 1),
              # GRU (hbuild_gru_wide.cu, 128 < M <= 1024, M % 128 == 0): both phases streamed
              ("gru", 256, 300, 10, 1), ("gru", 1024, 260, 3, 1), ("gru", 384, 333, 7, 2), ("gru", 640, 129, 5, 3),
              ("gru", 512, 1000, 2, 4), ("gru", 256, 129, 1, 1)]


@pytest.mark.parametrize("arch,M,N,Q,S", WIDE_CASES)
def test_wide_tc_parity(arch, M, N, Q, S):
    X, Y, _ = inputs(N, Q, S, seed=M + Q)
    e, Hg = gpu_H(arch, S, M, Q, 4, X)
    assert e.path == 2
    net = orc.Net(arch, S=S, M=M, Q=Q)
    Ho = orc.build_H(net, orc.gen_weights(net, 4), X, threads=8)
    err = np.abs(Hg - Ho).max()
    assert err <= H_TOL, f"max |dH| = {err:.3e}"


@pytest.mark.parametrize("arch", ["lstm", "gru"])
def test_wide_tc_two_pass_and_many_tiles(arch):
    """fp16-grid weights (2-pass MMA) and more tiles than SMs (persistent CTAs
    loop over tiles: the history slots and c state are reused across tiles)."""
    M, Q, S = 512, 4, 1
    N = 128 * 148 + 77
    X, Y, _ = inputs(N, Q, S, seed=5)
    e, Hg = gpu_H(arch, S, M, Q, 4, X, weight_grid=1)
    assert e.path == 2
    rows = np.r_[0:130, N - 300:N]
    net = orc.Net(arch, S=S, M=M, Q=Q, weight_grid=1)
    Ho = orc.build_H(net, orc.gen_weights(net, 4), X[rows], threads=8)
    assert np.abs(Hg[rows] - Ho).max() <= H_TOL


@pytest.mark.parametrize("M,N", [(1024, 3001), (1000, 1201), (1024, 1025)])
def test_tsqr_wide_matches_lapack(M, N):
    """n = M+1 > 1024 columns (more than a CTA's threads): WY leaf/merge and
    the wide solve.  R of [H | Y] against numpy's Householder QR (LAPACK
    geqrf) up to row signs, beta against the oracle's lstsq of the same H."""
    g = torch.Generator(device="cuda").manual_seed(M + N)
    H = torch.rand(N, M, device="cuda", generator=g) - 0.5
    Y = torch.rand(N, device="cuda", generator=g) - 0.5
    n = M + 1
    Hn, Yn = H.double().cpu().numpy(), Y.double().cpu().numpy()
    Rn = np.abs(np.linalg.qr(np.column_stack([Hn, Yn]), mode="r"))
    e = E("lstm", 1, M, 4, 1)
    R = _packed_to_R(e.solve_local(H, Y).cpu().numpy(), n)
    assert np.abs(np.abs(R) - Rn).max() <= 1e-12 * Rn.max()
    beta, info = e.solve_beta(H, Y)
    b_ref, i_ref = orc.lstsq(Hn, Yn)
    cond = np.linalg.cond(i_ref.R[:M, :M])
    assert np.linalg.norm(beta.cpu().numpy() - b_ref) / np.linalg.norm(b_ref) <= 1e-12 * cond
    assert info.rmse == pytest.approx(i_ref.rmse, rel=1e-10 * cond)
    assert info.status == 0 and info.n_total == N
    # virtual ranks: solve_local x 3 + solve_merge equals the single solve
    cuts = np.linspace(0, N, 4).astype(int)
    parts = [e.solve_local(H[a:b], Y[a:b]).clone() for a, b in zip(cuts[:-1], cuts[1:])]
    b3, _ = e.solve_merge(torch.stack(parts), 3, N)
    assert float((b3 - beta).norm() / beta.norm()) <= 1e-12 * cond


def test_tsqr_wide_ridge():
    """Rank-deficient H at n > 1024: the wide solve takes the ridge path (R19)
    like the oracle (duplicated columns)."""
    M, N = 1024, 2000
    g = torch.Generator(device="cuda").manual_seed(5)
    H = torch.rand(N, M, device="cuda", generator=g) - 0.5
    H[:, 700:] = H[:, :M - 700]
    Y = torch.rand(N, device="cuda", generator=g) - 0.5
    e = E("gru", 1, M, 4, 1)
    beta, info = e.solve_beta(H, Y)
    b_ref, i_ref = orc.lstsq(H.double().cpu().numpy(), Y.double().cpu().numpy())
    assert info.status == 1 and info.rank_flag == 1 and i_ref.status == 1
    assert info.ridge_lambda == pytest.approx(i_ref.ridge_lambda, rel=1e-10)
    assert info.rmse == pytest.approx(i_ref.rmse, rel=1e-6)
    np.testing.assert_allclose(beta.cpu().numpy(), b_ref, rtol=1e-5, atol=1e-6 * np.abs(b_ref).max())


@pytest.mark.parametrize("arch", ["lstm", "gru"])
def test_c5_m1024_train_sampled(arch):
    """C5 widest shape end to end (M = 1024, Q = 10, N = 4096 rows on one GPU):
    sampled H rows against the oracle; beta and the RMSE against the oracle's
    Householder lstsq of the same fp32 H (n = 1025: WY leaf + wide solve)."""
    N, M, Q = 4096, 1024, 10
    s = sy.series("mg", N + Q + 1, seed=1, noise=0.01)
    X, Y, _ = sy.windows(s[:, :1], N, Q)
    e = E(arch, 1, M, Q, 1)
    Xd, Yd = torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda()
    H, beta, info = e.train(Xd, Yd)
    rows = np.array([0, 1, 777, 2049, N - 1])
    net = orc.Net(arch, S=1, M=M, Q=Q)
    Ho = orc.build_H(net, orc.gen_weights(net, 1), X[rows], threads=8)
    assert np.abs(H[torch.from_numpy(rows).cuda()].cpu().numpy() - Ho).max() <= H_TOL
    # solver isolation at n = 1025: the oracle's Householder lstsq of the same fp32 H
    b_iso, i_iso = orc.lstsq(H.double().cpu().numpy(), Y.astype(np.float64))
    assert info.status == i_iso.status
    cond = np.linalg.cond(i_iso.R[:M, :M])
    rel = np.linalg.norm(beta.cpu().numpy() - b_iso) / np.linalg.norm(b_iso)
    print(f"{arch} M=1024: cond(R)={cond:.2e} status={info.status} rel dbeta={rel:.2e}")
    assert rel <= (1e-4 if info.status else max(1e-10, 1e-12 * cond))
    assert info.rmse == pytest.approx(i_iso.rmse, rel=1e-6)


# ------------------------------------------------------------------------- NARMAX error feedback (8(f) row 4)
@pytest.mark.parametrize("N,S,M,Q,o", [(1000, 1, 64, 20, {}), (333, 4, 37, 10, {"F": 3, "R": 7, "act": 1}),
                                       (100, 1, 5, 1, {}), (257, 2, 16, 12, {"F": 0, "R": 12})])
def test_narmax_error_window_build_parity(N, S, M, Q, o):
    """elmrnn_build_H_ef against the oracle's Eq.-7 t-loop on the same error window."""
    X, Y, Yfb = inputs(N, Q, S, seed=N, kind="ar5")
    Ef = np.random.default_rng(N).standard_normal((N, Q)).astype(np.float32)
    e = E("narmax", S, M, Q, 6, **o)
    Hg = e.build_H(torch.from_numpy(X).cuda(), torch.from_numpy(Yfb).cuda(),
                   Ef=torch.from_numpy(Ef).cuda()).cpu().numpy().astype(np.float64)
    net = oracle_net("narmax", S, M, Q, **o)
    Ho = orc.build_H(net, orc.gen_weights(net, 6), X, Yfb, threads=8, Ef=Ef)
    assert np.abs(Hg - Ho).max() <= H_TOL
    # Ef = 0 is exactly the one-pass build
    H0 = e.build_H(torch.from_numpy(X).cuda(), torch.from_numpy(Yfb).cuda()).cpu().numpy()
    Hz = e.build_H(torch.from_numpy(X).cuda(), torch.from_numpy(Yfb).cuda(),
                   Ef=torch.zeros(N, Q, device="cuda")).cpu().numpy()
    np.testing.assert_array_equal(H0, Hz)


def test_narmax_error_windows_parity():
    """elmrnn_error_windows against the oracle's definition on the same fp32 H and beta."""
    N, M, Q = 5000, 64, 20
    g = torch.Generator(device="cuda").manual_seed(3)
    H = torch.rand(N, M, device="cuda", generator=g)
    Y = torch.randn(N, device="cuda", generator=g)
    beta = torch.randn(M, device="cuda", dtype=torch.float64, generator=g)
    e = E("narmax", 1, M, Q, 1)
    Ef = e.error_windows(H, Y, beta).cpu().numpy()
    ref = orc.error_windows(H.double().cpu().numpy(), Y.double().cpu().numpy(), beta.cpu().numpy(), Q)
    scale = np.abs(ref).max()
    assert np.abs(Ef - ref).max() <= 4e-7 * scale
    assert (Ef[:Q][np.arange(Q)[:, None] + np.arange(Q)[None, :] < Q - 1] == 0).all()   # k < 0 entries


def test_narmax_two_pass_train_parity():
    """Two-pass NARMAX training end to end (C2 shape, 20k rows) against the oracle's two-pass method."""
    N, M, Q = 20000, 64, 20
    s = sy.series("ar5", N + Q + 1, seed=4)
    X, Y, Yfb = sy.windows(s[:, :1], N, Q)
    e = E("narmax", 1, M, Q, 1)
    Xd, Yd, Yfbd = (torch.from_numpy(a).cuda() for a in (X, Y, Yfb))
    H1, b1, i1, b0, i0 = e.train_narmax_ef(Xd, Yd, Yfbd)
    net = orc.Net("narmax", S=1, M=M, Q=Q)
    Ho1, bo1, io1, bo0, io0 = orc.train_narmax_ef(net, orc.gen_weights(net, 1), X, Y, Yfb, threads=8)
    Hg1 = H1.cpu().numpy().astype(np.float64)
    assert np.abs(Hg1 - Ho1).max() <= H_TOL
    print(f"narmax-ef: rmse pass0 {i0.rmse:.6f} pass1 {i1.rmse:.6f}")
    pr.check("narmax-ef pass 1", b1.cpu().numpy(), i1.rmse, Hg1, Ho1, Y)
    assert abs(i0.rmse - io0.rmse) / io0.rmse <= 1e-4


# ------------------------------------------------------------------------- forecasting (8(f) row 3)
FC_ARCHS = [("elman", 20, 10), ("jordan", 64, 20), ("narmax", 64, 20), ("fc", 50, 10), ("lstm", 32, 10),
            ("lstm", 128, 30), ("gru", 128, 30), ("gru", 40, 12), ("lstm_diag", 33, 10), ("gru_diag", 33, 10),
            ("fc_eq8", 20, 12)]


@pytest.mark.parametrize("arch,M,Q", FC_ARCHS)
def test_forecast_per_step_parity(arch, M, Q):
    """Each forecast step k against the oracle's Eq. 4 on the window the GPU
    itself fed back (w_k = X shifted by the GPU's own fp32 predictions), so
    the check does not compound; then the whole trajectory against the
    oracle's forecast for a contractive beta."""
    N, K = 300, 6
    X, Y, _ = inputs(N, Q, 1, seed=M + Q)
    beta = np.random.default_rng(M).standard_normal(M) / M
    e = E(arch, 1, M, Q, 8)
    bd = torch.from_numpy(beta).cuda()
    Yh = e.forecast(torch.from_numpy(X).cuda(), bd, K).cpu().numpy()
    net = orc.Net(arch, S=1, M=M, Q=Q)
    bl = orc.gen_weights(net, 8)
    tol = 1e-5 * max(1.0, np.abs(beta).sum())
    W = X[:, :, 0].copy()
    for k in range(K):
        ref = orc.predict(orc.build_H(net, bl, W[:, :, None], threads=8), beta)
        assert np.abs(Yh[:, k] - ref).max() <= tol, k
        W = np.concatenate([W[:, 1:], Yh[:, k:k + 1]], axis=1)
    full = orc.forecast(net, bl, X, beta, K, threads=8)
    assert np.abs(Yh - full).max() <= 10 * tol


READOUT_CASES = [  # (arch, M, Q, S, force_path): one per builder kernel and its readout-slot layout
    ("lstm", 256, 12, 1, 0), ("lstm", 128, 12, 2, 0), ("lstm", 512, 4, 1, 0), ("gru", 128, 12, 4, 0),
    ("gru", 256, 6, 1, 0), ("fc", 128, 10, 4, 0), ("lstm", 48, 10, 1, 0), ("gru", 40, 10, 2, 0), ("fc", 50, 10, 1, 0),
    ("elman", 20, 10, 1, 0), ("elman", 64, 40, 1, 0), ("jordan", 64, 20, 1, 0), ("narmax", 33, 20, 1, 0),
    ("lstm_diag", 33, 10, 2, 0), ("gru_diag", 96, 10, 1, 0), ("fc_eq8", 20, 12, 1, 0)]


@pytest.mark.parametrize("arch,M,Q,S,fp", READOUT_CASES)
def test_fused_readout_every_builder(arch, M, Q, S, fp):
    """elmrnn_predict through the fused readout epilogue (no H(Q) is written:
    each builder emits fp64 partial products H_i . beta per row segment, summed
    in a fixed slot order) against the oracle's Eq. 4 on every row of a ragged N
    (partial last tile / warp group), and bitwise repeatable."""
    N = 1000 + 37
    X, Y, _ = inputs(N, Q, S, seed=M + Q + S, kind="ar5")
    beta = np.random.default_rng(M + Q).standard_normal(M) / np.sqrt(M)
    e = E(arch, S, M, Q, 4, force_path=fp)
    Xd, bd = torch.from_numpy(X).cuda(), torch.from_numpy(beta).cuda()
    y1 = e.predict(Xd, bd)
    y2 = e.predict(Xd, bd)
    assert torch.equal(y1, y2)
    net = orc.Net(arch, S=S, M=M, Q=Q)
    ref = orc.predict(orc.build_H(net, orc.gen_weights(net, 4), X, threads=8), beta)
    tol = 1e-5 * max(1.0, np.abs(beta).sum())
    err = np.abs(y1.cpu().numpy() - ref).max()
    assert err <= tol, (arch, M, e.path, err, tol)


def test_fused_readout_large_n():
    """Fused readout / forecast at 140000 rows (M = 64, Elman: a row spans up to
    three 32-cell warp groups, slot layout kRoCellSlots): first, middle and last
    rows against the oracle's Eq. 4 and free-running forecast."""
    N, M, Q, K = 140000, 64, 10, 2
    X, Y, _ = inputs(N, Q, 1, seed=5, kind="ar5")
    beta = np.random.default_rng(2).standard_normal(M) / M
    e = E("elman", 1, M, Q, 8)
    Xd, bd = torch.from_numpy(X).cuda(), torch.from_numpy(beta).cuda()
    yp = e.predict(Xd, bd).cpu().numpy()
    Yh = e.forecast(Xd, bd, K).cpu().numpy()
    rows = np.r_[0:50, 131000:131200, N - 50:N]
    net = orc.Net("elman", S=1, M=M, Q=Q)
    bl = orc.gen_weights(net, 8)
    tol = 1e-5 * max(1.0, np.abs(beta).sum())
    assert np.abs(yp[rows] - orc.predict(orc.build_H(net, bl, X[rows], threads=8), beta)).max() <= tol
    assert np.abs(Yh[rows] - orc.forecast(net, bl, X[rows], beta, K, threads=8)).max() <= 10 * tol


def test_forecast_errors_and_empty():
    from paper_1911_13252_b200 import ElmrnnError
    e = E("gru", 2, 8, 4, 1)
    with pytest.raises(ElmrnnError, match="UNSUPPORTED"):
        e.forecast(torch.zeros(5, 4, 2, device="cuda"), torch.zeros(8, dtype=torch.float64, device="cuda"), 3)
    e1 = E("gru", 1, 8, 4, 1)
    assert e1.forecast(torch.zeros(0, 4, 1, device="cuda"), torch.zeros(8, dtype=torch.float64, device="cuda"),
                       3).shape == (0, 3)


@pytest.mark.parametrize("arch,M,Q,S", [("gru", 32, 10, 1), ("lstm", 256, 20, 1), ("narmax", 64, 20, 1),
                                        ("fc", 128, 10, 4)])
def test_test_rmse_parity(arch, M, Q, S):
    """Held-out RMSE of a beta trained on the first windows, evaluated on later ones."""
    Ntr, Nte = 3000, 1000
    kind = "sin4" if S == 4 else ("ar5" if arch == "narmax" else "mg")
    s = sy.series(kind, Ntr + Nte + Q + 1, seed=9)
    X, Y, _ = sy.windows(s[:, :S], Ntr + Nte, Q)
    e = E(arch, S, M, Q, 2)
    Xd, Yd = torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda()
    _, beta, _ = e.train(Xd[:Ntr], Yd[:Ntr])
    r = e.test_rmse(Xd[Ntr:], Yd[Ntr:], beta)
    b = beta.cpu().numpy()
    net = orc.Net(arch, S=S, M=M, Q=Q)
    ref = orc.test_rmse(net, orc.gen_weights(net, 2), X[Ntr:], Y[Ntr:], b, threads=8)
    assert abs(r - ref) <= 1e-5 * max(1.0, np.abs(b).sum()), (r, ref)


# ------------------------------------------------------------------------- multi-output Y (8(f) row 3)
@pytest.mark.parametrize("M,N,P", [(64, 5000, 3), (20, 1000, 1), (256, 20011, 2), (1024, 3001, 4), (129, 777, 5)])
def test_solve_beta_multi_parity(M, N, P):
    """One TSQR of [H | Y_1..Y_P] against the oracle's P independent Householder
    solves of the same fp32 H, and against elmrnn_solve_beta column by column."""
    g = torch.Generator(device="cuda").manual_seed(M + N + P)
    H = torch.rand(N, M, device="cuda", generator=g) - 0.5
    Y = torch.rand(N, P, device="cuda", generator=g) - 0.5
    e = E("lstm", 1, M, 4, 1, force_path=1)
    B, rmse, info = e.solve_beta_multi(H, Y)
    Bo, io = orc.lstsq_multi(H.double().cpu().numpy(), Y.double().cpu().numpy())
    cond = np.linalg.cond(io[0].R[:M, :M])
    tol = 1e-12 * max(1.0, cond)
    for p in range(P):
        rel = np.linalg.norm(B[p].cpu().numpy() - Bo[p]) / np.linalg.norm(Bo[p])
        assert rel <= tol, (p, rel, cond)
        assert rmse[p] == pytest.approx(io[p].rmse, rel=tol)
        b1, i1 = e.solve_beta(H, Y[:, p].contiguous())
        assert float((b1 - B[p]).norm() / b1.norm()) <= tol
    assert info.status == 0 and info.rmse == pytest.approx(rmse[0], rel=1e-14)


@pytest.mark.parametrize("M,N,P,ranks", [(64, 5000, 3, 2), (256, 20011, 2, 4), (20, 1000, 2, 3), (129, 3777, 5, 8)])
def test_multi_output_virtual_ranks(M, N, P, ranks):
    """Row-sharded multi-output solve on one GPU: elmrnn_solve_local_multi on each
    row block, elmrnn_solve_merge_multi of the stacked factors equals the single
    elmrnn_solve_beta_multi and the oracle's P Householder solves."""
    g = torch.Generator(device="cuda").manual_seed(M + N + P)
    H = torch.rand(N, M, device="cuda", generator=g) - 0.5
    Y = torch.rand(N, P, device="cuda", generator=g) - 0.5
    e = E("lstm", 1, M, 4, 1, force_path=1)
    B1, rm1, _ = e.solve_beta_multi(H, Y)
    cuts = np.linspace(0, N, ranks + 1).astype(int)
    parts = [e.solve_local_multi(H[a:b], Y[a:b]).clone() for a, b in zip(cuts[:-1], cuts[1:])]
    BP, rmP, info = e.solve_merge_multi(torch.stack(parts), ranks, P, N)
    Bo, io = orc.lstsq_multi(H.double().cpu().numpy(), Y.double().cpu().numpy())
    cond = np.linalg.cond(io[0].R[:M, :M])
    tol = 1e-12 * max(1.0, cond)
    assert info.status == 0
    for p in range(P):
        assert float((BP[p] - B1[p]).norm() / B1[p].norm()) <= tol
        assert np.linalg.norm(BP[p].cpu().numpy() - Bo[p]) / np.linalg.norm(Bo[p]) <= tol
        assert rmP[p] == pytest.approx(io[p].rmse, rel=tol)


def test_solve_beta_multi_ridge_and_trained():
    """Rank-deficient H: the ridge path (R19) is shared by all outputs; and a real
    GRU H with two targets (y(t+1) and y(t+2))."""
    M, N = 32, 600
    g = torch.Generator(device="cuda").manual_seed(3)
    H = torch.rand(N, M, device="cuda", generator=g)
    H[:, 20:] = H[:, :12]
    Y = torch.rand(N, 2, device="cuda", generator=g)
    e = E("gru", 1, M, 4, 1)
    B, rmse, info = e.solve_beta_multi(H, Y)
    Bo, io = orc.lstsq_multi(H.double().cpu().numpy(), Y.double().cpu().numpy())
    assert info.status == 1 and io[0].status == 1
    for p in range(2):
        np.testing.assert_allclose(B[p].cpu().numpy(), Bo[p], rtol=1e-5, atol=1e-6 * np.abs(Bo[p]).max())
        assert rmse[p] == pytest.approx(io[p].rmse, rel=1e-6)
    Q, S, M2, N2 = 10, 1, 64, 3000
    s = sy.series("mg", N2 + Q + 2, seed=4)
    X, Y1, _ = sy.windows(s[:, :1], N2, Q)
    Y2 = s[Q + 1: Q + 1 + N2, 0].astype(np.float32)
    e2 = E("gru", S, M2, Q, 2)
    Hg = e2.build_H(torch.from_numpy(X).cuda())
    Yd = torch.from_numpy(np.stack([Y1, Y2], axis=1)).cuda()
    B2, rm2, _ = e2.solve_beta_multi(Hg, Yd)
    Bo2, io2 = orc.lstsq_multi(Hg.double().cpu().numpy(), Yd.double().cpu().numpy())
    cond = np.linalg.cond(io2[0].R[:M2, :M2])
    for p in range(2):
        assert np.linalg.norm(B2[p].cpu().numpy() - Bo2[p]) / np.linalg.norm(Bo2[p]) <= 1e-12 * cond


@pytest.mark.parametrize("M,P", [(256, 2), (256, 5), (300, 8), (128, 3)])
def test_virtual_ranks_wy_pipelined_merge(M, P):
    """Row-sharded solve on one GPU through the WY path: P local TSQRs, then
    elmrnn_solve_merge (unpack + pipelined merge tree + solve) equals the single
    solve, and both match the oracle's Householder lstsq of the same H."""
    N = 6000 + 37 * P
    g = torch.Generator(device="cuda").manual_seed(M * P)
    H = torch.rand(N, M, device="cuda", generator=g) - 0.5
    Y = torch.rand(N, device="cuda", generator=g) - 0.5
    e = E("lstm", 1, M, 4, 1, force_path=1)
    b1, i1 = e.solve_beta(H, Y)
    cuts = np.linspace(0, N, P + 1).astype(int)
    parts = [e.solve_local(H[a:b], Y[a:b]).clone() for a, b in zip(cuts[:-1], cuts[1:])]
    bP, iP = e.solve_merge(torch.stack(parts), P, N)
    bo, io = orc.lstsq(H.double().cpu().numpy(), Y.double().cpu().numpy())
    cond = np.linalg.cond(io.R[:M, :M])
    assert float((bP - b1).norm() / b1.norm()) <= 1e-12 * cond
    assert np.linalg.norm(bP.cpu().numpy() - bo) / np.linalg.norm(bo) <= 1e-12 * cond
    assert iP.rmse == pytest.approx(io.rmse, rel=1e-10)
