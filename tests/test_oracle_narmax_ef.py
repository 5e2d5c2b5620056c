"""Pins for the oracle's NARMAX with real error feedback.

Eq. 7 with e(t) = y(t) - yhat(t), reading R30:
the rows are consecutive stride-1 windows of one series, so window i's e(tau)
is the residual of window k = i + tau - Q (0 for k < 0).  Pins: the e == 0
reduction to the one-pass NARMAX (already pinned in test_oracle_hbuild.py),
R = 0 inertness, the one-step collapse written out in numpy, the residual
windows against numpy's matmul residual windowed by synth.windows (independent
code), and the exact-fit fixed point of the two-pass method.
"""
import numpy as np
import pytest

from oracle import oracle as orc
from synth import series as sy


def _setup(N=40, Q=7, S=2, M=6, seed=3, **kw):
    net = orc.Net("narmax", S=S, M=M, Q=Q, **kw)
    bl = orc.gen_weights(net, seed=seed)
    rng = np.random.default_rng(seed)
    X = rng.standard_normal((N, Q, S)).astype(np.float32)
    Yfb = rng.standard_normal((N, Q)).astype(np.float32)
    Ef = rng.standard_normal((N, Q)).astype(np.float32)
    return net, bl, X, Yfb, Ef


def test_zero_error_window_is_one_pass_narmax():
    net, bl, X, Yfb, _ = _setup()
    np.testing.assert_array_equal(orc.build_H(net, bl, X, Yfb, Ef=np.zeros_like(Yfb)),
                                  orc.build_H(net, bl, X, Yfb))


def test_error_lags_zero_is_inert():
    net, bl, X, Yfb, Ef = _setup(R=0)
    np.testing.assert_array_equal(orc.build_H(net, bl, X, Yfb, Ef=Ef), orc.build_H(net, bl, X, Yfb))


def test_error_window_changes_H():
    net, bl, X, Yfb, Ef = _setup()
    assert np.abs(orc.build_H(net, bl, X, Yfb, Ef=Ef) - orc.build_H(net, bl, X, Yfb)).max() > 1e-3


@pytest.mark.parametrize("F,R,act", [(-1, -1, 0), (3, 5, 1), (9, 2, 0)])
def test_tloop_equals_onestep_with_error(F, R, act):
    """H(Q) = g(W x(Q) + b + sum_{l<=min(F,Q-1)} W'[:,l] y(Q-l)
                 + sum_{l<=min(R,Q-1)} W''[:,l] e(Q-l)), written out in numpy."""
    net, bl, X, Yfb, Ef = _setup(F=F, R=R, act=act)
    Q = net.Q
    H = orc.build_H(net, bl, X, Yfb, Ef=Ef)
    W, b, W1, W2 = (x.astype(np.float64) for x in bl)
    a = X[:, Q - 1, :].astype(np.float64) @ W + b
    for l in range(1, min(net.F, Q - 1) + 1):
        a += np.outer(Yfb[:, Q - l - 1].astype(np.float64), W1[:, l - 1])
    for l in range(1, min(net.R, Q - 1) + 1):
        a += np.outer(Ef[:, Q - l - 1].astype(np.float64), W2[:, l - 1])
    ref = np.tanh(a) if act else 1 / (1 + np.exp(-a))
    np.testing.assert_allclose(H, ref, rtol=0, atol=4e-16)


def test_error_windows_are_windows_of_the_residual_series():
    N, M, Q = 57, 5, 9
    rng = np.random.default_rng(7)
    H = rng.standard_normal((N, M))
    Y = rng.standard_normal(N)
    beta = rng.standard_normal(M)
    Ef = orc.error_windows(H, Y, beta, Q)
    r = Y - H @ beta                                  # numpy residual (Eq. 4)
    e_series = np.concatenate([np.zeros(Q), r, [0.0]])   # e at global time g = r[g - Q]
    _, _, Eref = sy.windows(e_series.astype(np.float64), N, Q)   # Eref[i][tau-1] = e_series[i + tau]
    np.testing.assert_allclose(Ef, Eref, rtol=2e-7, atol=1e-30)
    assert Ef.dtype == np.float32


def test_two_pass_exact_fit_is_fixed_point():
    """Y in span(H0): the residual is ~0, so pass 1 reproduces pass 0."""
    net, bl, X, Yfb, _ = _setup(N=80, M=6)
    H0 = orc.build_H(net, bl, X, Yfb)
    Y = H0 @ np.linspace(-1, 1, net.M)
    H1, b1, i1, b0, i0 = orc.train_narmax_ef(net, bl, X, Y, Yfb)
    assert i0.rmse < 1e-13
    np.testing.assert_allclose(H1, H0, rtol=0, atol=1e-12)
    np.testing.assert_allclose(b1, b0, rtol=0, atol=1e-9)


def test_two_pass_on_ar5_series():
    """The second pass solves the least-squares problem of the rebuilt H (its
    normal-equation residual vanishes) and its e windows are pass 0's residuals."""
    N, Q, M = 600, 10, 16
    s = sy.series("ar5", N + Q + 1, seed=2)
    X, Y, Yfb = sy.windows(s[:, :1], N, Q)
    net = orc.Net("narmax", S=1, M=M, Q=Q)
    bl = orc.gen_weights(net, seed=4)
    H1, b1, i1, b0, i0 = orc.train_narmax_ef(net, bl, X, Y, Yfb)
    r1 = H1 @ b1 - Y
    assert np.abs(H1.T @ r1).max() <= 1e-10 * np.abs(H1.T @ Y).max()
    assert i1.rmse == pytest.approx(np.sqrt(np.mean(r1 ** 2)), rel=1e-10)
    H0 = orc.build_H(net, bl, X, Yfb)
    assert not np.allclose(H0, H1)
