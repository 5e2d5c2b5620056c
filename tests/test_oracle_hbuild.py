"""Pins for the oracle's H build (CPU only, -m "not gpu").

Each test ties oracle.build_H to something other than itself: worked examples
(tests/golden/spec_examples.json, each cited), library reductions to
torch.nn.LSTM / GRU / RNN in fp64, collapse identities between independently
written oracle functions, and equivariance properties.  A dropped term, wrong
gate order, transposed U or off-by-one lag fails at least one of them.
"""
import json
import math
import os

import numpy as np
import pytest
import torch

from oracle import oracle as orc

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def zeros_like_blocks(net):
    return [np.zeros(orc.block_shape(net, b), np.float32) for b in range(orc.num_blocks(net.arch))]


def rand_X(N, Q, S, seed=0, scale=1.0):
    return (np.random.default_rng(seed).standard_normal((N, Q, S)) * scale).astype(np.float32)


# ---------------------------------------------------------------- special values
@pytest.mark.parametrize("arch", ["elman", "jordan", "narmax", "fc"])
@pytest.mark.parametrize("act,expect", [(0, 0.5), (1, 0.0)])
def test_zero_weights_sigma0(arch, act, expect):
    net = orc.Net(arch, S=2, M=5, Q=6, act=act)
    H = orc.build_H(net, zeros_like_blocks(net), rand_X(7, 6, 2))
    assert np.all(H == expect)


@pytest.mark.parametrize("arch", ["lstm", "gru"])
def test_zero_weights_gated(arch):
    net = orc.Net(arch, S=2, M=5, Q=6)
    H = orc.build_H(net, zeros_like_blocks(net), rand_X(7, 6, 2))
    assert np.all(H == 0.0)


def test_spec_elman_t1():
    net = orc.Net("elman", S=1, M=1, Q=1)
    bl = zeros_like_blocks(net)
    bl[0][:] = 1.0
    H = orc.build_H(net, bl, np.array([[[2.0]]], np.float32))
    assert H[0, 0] == pytest.approx(GOLD["sigmoid_2"]["value"], abs=1e-16)


def test_spec_elman_two_step():
    net = orc.Net("elman", S=1, M=1, Q=2)
    bl = zeros_like_blocks(net)
    bl[2][0, 0] = 1.0          # alpha[j,1] (lag 1)
    bl[2][0, 1] = 123.0        # alpha[j,2]: never used inside a 2-step window (R4)
    H = orc.build_H(net, bl, np.zeros((1, 2, 1), np.float32))
    assert H[0, 0] == pytest.approx(GOLD["elman_two_step"]["value"], abs=1e-16)


def test_spec_jordan_two_step():
    net = orc.Net("jordan", S=1, M=1, Q=2)
    bl = zeros_like_blocks(net)
    bl[2][0, 0] = 2.0
    Yfb = np.array([[0.25, 99.0]], np.float32)   # y(1) = 0.25; y(2) is the target, unused
    H = orc.build_H(net, bl, np.zeros((1, 2, 1), np.float32), Yfb)
    assert H[0, 0] == pytest.approx(GOLD["jordan_two_step"]["value"], abs=1e-16)
    # Yfb == NULL convention: y(tau) = X[i][tau][0]
    X = np.array([[[7.0], [0.25]]], np.float32)
    bl[0][:] = 0.0
    H2 = orc.build_H(net, bl, X)
    assert H2[0, 0] == pytest.approx(GOLD["jordan_two_step"]["value"], abs=1e-16)


def test_spec_narmax_two_step_and_e_inert():
    net = orc.Net("narmax", S=1, M=1, Q=2, F=1, R=2)
    bl = zeros_like_blocks(net)
    bl[2][0, 0] = 1.0
    bl[3][:] = 55.0            # W'' multiplies e == 0 (R8)
    H = orc.build_H(net, bl, np.zeros((1, 2, 1), np.float32), np.array([[0.3, 0.0]], np.float32))
    # the fp32 input 0.3 is 0.30000001192...: the golden sigma(0.3) holds to 3e-9
    assert H[0, 0] == pytest.approx(GOLD["narmax_two_step"]["value"], abs=5e-9)
    assert H[0, 0] == pytest.approx(1 / (1 + math.exp(-float(np.float32(0.3)))), abs=1e-16)


def test_fc_prose_distinguishing_pin():
    net = orc.Net("fc", S=1, M=2, Q=2)
    bl = zeros_like_blocks(net)
    bl[1][:] = [1.0, -1.0]
    bl[2][0, 0, 1] = 1.0       # A_1[m=0][j=1]
    H = orc.build_H(net, bl, np.zeros((1, 2, 1), np.float32))
    np.testing.assert_allclose(H[0], GOLD["fc_prose_pin"]["value"], rtol=0, atol=1e-16)
    assert abs(H[0, 1] - GOLD["fc_prose_pin"]["literal_eq8_value_1"]) > 0.1


def test_spec_lstm_t1():
    net = orc.Net("lstm", S=1, M=1, Q=1)
    bl = zeros_like_blocks(net)
    for g in range(4):
        bl[3 * g][:] = 1.0
    H = orc.build_H(net, bl, np.ones((1, 1, 1), np.float32))
    assert H[0, 0] == pytest.approx(GOLD["lstm_t1"]["h"], abs=1e-16)


def test_spec_gru_t1():
    net = orc.Net("gru", S=1, M=1, Q=1)
    bl = zeros_like_blocks(net)
    for g in range(3):
        bl[3 * g][:] = 1.0
    H = orc.build_H(net, bl, np.ones((1, 1, 1), np.float32))
    assert H[0, 0] == pytest.approx(GOLD["gru_t1"]["h"], abs=1e-16)


def _pin_params(arch):
    net = orc.Net(arch, S=1, M=2, Q=2)
    bl = zeros_like_blocks(net)
    for g in range(4 if arch == "lstm" else 3):
        bl[3 * g][:] = 0.5
        bl[3 * g + 1][:] = [[0.1, 0.2], [0.3, 0.4]]
    X = np.array([[[1.0], [-0.5]]], np.float32)
    return net, bl, X


def test_dense_lstm_pin():
    net, bl, X = _pin_params("lstm")
    H = orc.build_H(net, bl, X)
    # golden uses exact 0.1..0.4; the fp32 weights differ by <1e-8 -> |dH| ~ 5e-10
    np.testing.assert_allclose(H[0], GOLD["lstm_dense_pin"]["value"], rtol=0, atol=2e-9)


def test_dense_gru_pin():
    net, bl, X = _pin_params("gru")
    H = orc.build_H(net, bl, X)
    np.testing.assert_allclose(H[0], GOLD["gru_dense_pin"]["value"], rtol=0, atol=2e-9)


# ---------------------------------------------------------------- library reductions
def test_lstm_equals_torch_lstm():
    """Dense LSTM == torch.nn.LSTM (fp64): gates (o,c,lambda,in) -> torch (i,f,g,o)."""
    S, M, Q, N = 3, 7, 9, 11
    net = orc.Net("lstm", S=S, M=M, Q=Q)
    bl = orc.gen_weights(net, seed=5)
    X = rand_X(N, Q, S, seed=1)
    H = orc.build_H(net, bl, X)
    lstm = torch.nn.LSTM(S, M, batch_first=True).double()
    W = {g: bl[3 * k].astype(np.float64) for k, g in enumerate(("o", "c", "l", "i"))}
    U = {g: bl[3 * k + 1].astype(np.float64) for k, g in enumerate(("o", "c", "l", "i"))}
    b = {g: bl[3 * k + 2].astype(np.float64) for k, g in enumerate(("o", "c", "l", "i"))}
    order = ("i", "l", "c", "o")
    with torch.no_grad():
        lstm.weight_ih_l0.copy_(torch.from_numpy(np.concatenate([W[g].T for g in order])))
        lstm.weight_hh_l0.copy_(torch.from_numpy(np.concatenate([U[g].T for g in order])))
        lstm.bias_ih_l0.copy_(torch.from_numpy(np.concatenate([b[g] for g in order])))
        lstm.bias_hh_l0.zero_()
        out, _ = lstm(torch.from_numpy(X.astype(np.float64)))
    np.testing.assert_allclose(H, out[:, -1].numpy(), rtol=0, atol=1e-14)


def test_diag_gru_equals_torch_gru():
    """Diagonal-U GRU == torch.nn.GRU with the z weights negated (1-sigma(a) = sigma(-a))."""
    S, M, Q, N = 2, 6, 8, 9
    net = orc.Net("gru", S=S, M=M, Q=Q)
    bl = orc.gen_weights(net, seed=3)
    for g in range(3):
        bl[3 * g + 1] = np.diag(np.diag(bl[3 * g + 1])).astype(np.float32)
    X = rand_X(N, Q, S, seed=2)
    H = orc.build_H(net, bl, X)
    gru = torch.nn.GRU(S, M, batch_first=True).double()
    Wz, Uz, bz = (bl[i].astype(np.float64) for i in (0, 1, 2))
    Wr, Ur, br = (bl[i].astype(np.float64) for i in (3, 4, 5))
    Wf, Uf, bf = (bl[i].astype(np.float64) for i in (6, 7, 8))
    with torch.no_grad():
        gru.weight_ih_l0.copy_(torch.from_numpy(np.concatenate([Wr.T, -Wz.T, Wf.T])))
        gru.weight_hh_l0.copy_(torch.from_numpy(np.concatenate([Ur.T, -Uz.T, Uf.T])))
        gru.bias_ih_l0.copy_(torch.from_numpy(np.concatenate([br, -bz, bf])))
        gru.bias_hh_l0.zero_()
        out, _ = gru(torch.from_numpy(X.astype(np.float64)))
    np.testing.assert_allclose(H, out[:, -1].numpy(), rtol=0, atol=1e-14)


def test_fc_lag1_tanh_equals_torch_rnn():
    S, M, Q, N = 3, 5, 7, 6
    net = orc.Net("fc", S=S, M=M, Q=Q, act=1, fc_lags=1)
    bl = orc.gen_weights(net, seed=9)
    X = rand_X(N, Q, S, seed=4)
    H = orc.build_H(net, bl, X)
    rnn = torch.nn.RNN(S, M, nonlinearity="tanh", batch_first=True).double()
    with torch.no_grad():
        rnn.weight_ih_l0.copy_(torch.from_numpy(bl[0].astype(np.float64).T))
        rnn.weight_hh_l0.copy_(torch.from_numpy(bl[2][0].astype(np.float64).T))
        rnn.bias_ih_l0.copy_(torch.from_numpy(bl[1].astype(np.float64)))
        rnn.bias_hh_l0.zero_()
        out, _ = rnn(torch.from_numpy(X.astype(np.float64)))
    np.testing.assert_allclose(H, out[:, -1].numpy(), rtol=0, atol=1e-14)


def test_elman_q2_tanh_equals_torch_rnn_diag():
    """Elman with Q=2 is an RNN with diagonal W_hh = diag(alpha[:,0])."""
    S, M, N = 2, 4, 5
    net = orc.Net("elman", S=S, M=M, Q=2, act=1)
    bl = orc.gen_weights(net, seed=2)
    X = rand_X(N, 2, S, seed=6)
    H = orc.build_H(net, bl, X)
    rnn = torch.nn.RNN(S, M, nonlinearity="tanh", batch_first=True).double()
    with torch.no_grad():
        rnn.weight_ih_l0.copy_(torch.from_numpy(bl[0].astype(np.float64).T))
        rnn.weight_hh_l0.copy_(torch.from_numpy(np.diag(bl[2][:, 0].astype(np.float64))))
        rnn.bias_ih_l0.copy_(torch.from_numpy(bl[1].astype(np.float64)))
        rnn.bias_hh_l0.zero_()
        out, _ = rnn(torch.from_numpy(X.astype(np.float64)))
    np.testing.assert_allclose(H, out[:, -1].numpy(), rtol=0, atol=1e-14)


# ---------------------------------------------------------------- collapse identities
def test_fc_M1_equals_elman():
    Q, S, N = 9, 2, 6
    fc = orc.Net("fc", S=S, M=1, Q=Q)
    el = orc.Net("elman", S=S, M=1, Q=Q)
    blf = orc.gen_weights(fc, seed=4)
    ble = [blf[0], blf[1], blf[2][:, 0, 0].reshape(1, Q).copy()]
    X = rand_X(N, Q, S, seed=3)
    np.testing.assert_array_equal(orc.build_H(fc, blf, X), orc.build_H(el, ble, X))


@pytest.mark.parametrize("arch", ["jordan", "narmax"])
def test_teacher_forced_tloop_equals_onestep(arch):
    """Under teacher forcing H(Q) depends only on step Q: compare the oracle's
    t-loop with the one-step formula written out in numpy."""
    S, M, Q, N = 2, 6, 8, 10
    net = orc.Net(arch, S=S, M=M, Q=Q)
    bl = orc.gen_weights(net, seed=11)
    X = rand_X(N, Q, S, seed=8)
    Yfb = np.random.default_rng(1).standard_normal((N, Q)).astype(np.float32)
    H = orc.build_H(net, bl, X, Yfb)
    W, b, al = (x.astype(np.float64) for x in bl[:3])
    a = X[:, Q - 1, :].astype(np.float64) @ W + b
    y = Yfb.astype(np.float64)
    for k in range(1, Q):              # y(Q-k) = Yfb[:, Q-k-1]
        a += np.outer(y[:, Q - k - 1], al[:, k - 1])
    np.testing.assert_allclose(H, 1 / (1 + np.exp(-a)), rtol=0, atol=2e-16)


def test_narmax_FQ_equals_jordan():
    S, M, Q, N = 1, 5, 7, 8
    nn = orc.Net("narmax", S=S, M=M, Q=Q)
    jj = orc.Net("jordan", S=S, M=M, Q=Q)
    bl = orc.gen_weights(nn, seed=1)
    X = rand_X(N, Q, S, seed=5)
    np.testing.assert_array_equal(orc.build_H(nn, bl, X), orc.build_H(jj, bl[:3], X))


@pytest.mark.parametrize("arch", ["jordan", "narmax"])
def test_no_feedback_is_feedforward(arch):
    S, M, Q, N = 3, 4, 5, 6
    net = orc.Net(arch, S=S, M=M, Q=Q, F=0, R=0) if arch == "narmax" else orc.Net(arch, S=S, M=M, Q=Q)
    bl = orc.gen_weights(net, seed=2)
    if arch == "jordan":
        bl[2][:] = 0.0
    X = rand_X(N, Q, S, seed=1)
    ff = 1 / (1 + np.exp(-(X[:, -1].astype(np.float64) @ bl[0].astype(np.float64) + bl[1])))
    np.testing.assert_allclose(orc.build_H(net, bl, X), ff, rtol=0, atol=2e-16)


@pytest.mark.parametrize("arch", ["elman", "jordan", "narmax", "fc"])
def test_Q1_is_feedforward(arch):
    S, M, N = 3, 4, 6
    net = orc.Net(arch, S=S, M=M, Q=1)
    bl = orc.gen_weights(net, seed=7)
    X = rand_X(N, 1, S, seed=1)
    ff = 1 / (1 + np.exp(-(X[:, 0].astype(np.float64) @ bl[0].astype(np.float64) + bl[1])))
    np.testing.assert_allclose(orc.build_H(net, bl, X), ff, rtol=0, atol=2e-16)


# ---------------------------------------------------------------- equivariance
@pytest.mark.parametrize("arch", ["elman", "jordan", "narmax", "fc", "lstm", "gru"])
def test_row_independence(arch):
    S, M, Q, N = 2, 5, 6, 9
    net = orc.Net(arch, S=S, M=M, Q=Q)
    bl = orc.gen_weights(net, seed=3)
    X = rand_X(N, Q, S, seed=2)
    perm = np.random.default_rng(0).permutation(N)
    np.testing.assert_array_equal(orc.build_H(net, bl, X)[perm], orc.build_H(net, bl, X[perm]))


@pytest.mark.parametrize("arch", ["elman", "jordan", "narmax", "fc", "lstm", "gru"])
def test_neuron_permutation_equivariance(arch):
    S, M, Q, N = 2, 6, 5, 7
    net = orc.Net(arch, S=S, M=M, Q=Q)
    bl = orc.gen_weights(net, seed=4)
    X = rand_X(N, Q, S, seed=3)
    p = np.random.default_rng(1).permutation(M)
    pb = []
    for k, w in enumerate(bl):
        shp = orc.block_shape(net, k)
        if arch in ("lstm", "gru"):
            w = {0: lambda a: a[:, p], 1: lambda a: a[p][:, p], 2: lambda a: a[p]}[k % 3](w)
        elif arch == "fc" and k == 2:
            w = w[:, p][:, :, p]
        elif shp == (S, M):
            w = w[:, p]
        else:
            w = w[p]
        pb.append(np.ascontiguousarray(w))
    H = orc.build_H(net, bl, X)
    Hp = orc.build_H(net, pb, X)
    np.testing.assert_allclose(Hp, H[:, p], rtol=0, atol=1e-15)


def test_thread_count_bitwise():
    net = orc.Net("lstm", S=1, M=9, Q=7)
    bl = orc.gen_weights(net, seed=2)
    X = rand_X(37, 7, 1)
    np.testing.assert_array_equal(orc.build_H(net, bl, X, threads=1), orc.build_H(net, bl, X, threads=4))
