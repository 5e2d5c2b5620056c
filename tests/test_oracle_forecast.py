"""Pins for the oracle's held-out RMSE and free-running forecast.

Reading R31: a K-step free-running forecast of a univariate
autoregressive window feeds each prediction back as the next observation
(fp32, the input type).  Pins: K = 1 is Eq. 4 on the window; a constant model
(all weights zero except the bias) forecasts the closed form sigma(b).beta at
every step; the semigroup property (a K-step forecast continues as the
(K-1)-step forecast of the shifted window); agreement with a forecast of a
linear AR model when H is the window itself (identity features, built by hand
in numpy); the held-out RMSE against numpy.
"""
import numpy as np
import pytest

from oracle import oracle as orc
from synth import series as sy


def _win(N=30, Q=8, seed=0):
    s = sy.series("mg", N + Q + 1, seed=seed)
    X, Y, _ = sy.windows(s[:, :1], N, Q)
    return X, Y


@pytest.mark.parametrize("arch", ["elman", "jordan", "narmax", "lstm", "gru", "fc"])
def test_one_step_forecast_is_predict(arch):
    X, Y = _win()
    net = orc.Net(arch, S=1, M=7, Q=8)
    bl = orc.gen_weights(net, 2)
    beta = np.linspace(-1, 1, 7)
    f = orc.forecast(net, bl, X, beta, 1)
    np.testing.assert_array_equal(f[:, 0], orc.predict(orc.build_H(net, bl, X), beta))


def test_constant_model_closed_form():
    X, Y = _win()
    net = orc.Net("elman", S=1, M=5, Q=8)
    bl = [np.zeros_like(b) for b in orc.gen_weights(net, 2)]
    bl[1] = np.linspace(-2, 2, 5).astype(np.float32)
    beta = np.array([0.5, -1.0, 2.0, 0.25, 1.0])
    f = orc.forecast(net, bl, X, beta, 6)
    c = (1 / (1 + np.exp(-bl[1].astype(np.float64)))) @ beta
    np.testing.assert_allclose(f, c, rtol=1e-15, atol=0)


@pytest.mark.parametrize("arch", ["jordan", "gru"])
def test_semigroup(arch):
    X, Y = _win(N=12)
    net = orc.Net(arch, S=1, M=9, Q=8)
    bl = orc.gen_weights(net, 5)
    beta = np.random.default_rng(1).standard_normal(9) * 0.3
    f = orc.forecast(net, bl, X, beta, 5)
    X1 = np.concatenate([X[:, 1:, 0], f[:, :1].astype(np.float32)], axis=1)[:, :, None]
    f1 = orc.forecast(net, bl, X1, beta, 4)
    np.testing.assert_array_equal(f[:, 1:], f1)


def test_forecast_follows_the_window_dynamics():
    """Jordan with zero input weight W, zero bias and tanh: H_j = tanh(sum_k alpha[j,k] y(Q-k)).
    Checked against the recursion written out independently over the raw series
    values (numpy, explicit time index instead of shifted windows)."""
    X, Y = _win(N=5, Q=6)
    net = orc.Net("jordan", S=1, M=4, Q=6, act=1)
    bl = orc.gen_weights(net, 3)
    bl[0][:] = 0
    bl[1][:] = 0
    beta = np.array([0.3, -0.2, 0.5, 0.1])
    K = 7
    f = orc.forecast(net, bl, X, beta, K)
    al = bl[2].astype(np.float64)            # [M][Q], alpha[j][k-1]
    for i in range(X.shape[0]):
        s = list(X[i, :, 0].astype(np.float32))   # s[0..Q-1] observed, then forecasts appended
        Q = 6
        for k in range(K):
            T = len(s)                              # window is s[T-Q .. T-1]; y(tau) = s[T-Q+tau]
            a = np.zeros(4)
            for kk in range(1, Q):                  # y(Q-kk), kk = 1..Q-1 (y(0) = 0)
                a += al[:, kk - 1] * np.float64(s[T - Q + (Q - kk)])
            yh = np.tanh(a) @ beta
            assert f[i, k] == pytest.approx(yh, rel=1e-13, abs=1e-15)
            s.append(np.float32(yh))


def test_test_rmse_matches_numpy():
    X, Y = _win(N=200, Q=10)
    net = orc.Net("lstm", S=1, M=6, Q=10)
    bl = orc.gen_weights(net, 4)
    H = orc.build_H(net, bl, X)
    beta = np.linalg.lstsq(H, Y.astype(np.float64), rcond=None)[0]
    r = orc.test_rmse(net, bl, X, Y, beta)
    assert r == pytest.approx(np.sqrt(np.mean((H @ beta - Y) ** 2)), rel=1e-12)
