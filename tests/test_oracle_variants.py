"""Pins for the oracle's paper-literal per-cell variants:
diagonal-U LSTM / GRU (consistent with Alg. 2's cell independence
P:250 and Table 2's per-cell counts P:367-368) and FC by the letter of Eq. 8
(SPEC S:231).

Each variant is pinned against something other than itself: torch.nn.LSTM /
torch.nn.GRU in fp64 (library reductions), the dense oracle functions run with
diagonal U (an independently written code path), the SURVEY's distinguishing
FC pin, hand-evaluated closed forms, and Elman (collapse identity).
"""
import math

import numpy as np
import pytest
import torch

from oracle import oracle as orc


def rand_X(N, Q, S, seed=0, scale=1.0):
    return (np.random.default_rng(seed).standard_normal((N, Q, S)) * scale).astype(np.float32)


def sig(a):
    return 1.0 / (1.0 + math.exp(-a))


# ---------------------------------------------------------------- diagonal LSTM
def test_lstm_diag_equals_torch_lstm():
    """Diagonal-U LSTM == torch.nn.LSTM with W_hh = diag(u) (gates (o,c,lambda,in) -> torch (i,f,g,o))."""
    S, M, Q, N = 3, 7, 9, 11
    net = orc.Net("lstm_diag", S=S, M=M, Q=Q)
    bl = orc.gen_weights(net, seed=5)
    X = rand_X(N, Q, S, seed=1)
    H = orc.build_H(net, bl, X)
    lstm = torch.nn.LSTM(S, M, batch_first=True).double()
    W = {g: bl[3 * k].astype(np.float64) for k, g in enumerate(("o", "c", "l", "i"))}
    u = {g: bl[3 * k + 1].astype(np.float64) for k, g in enumerate(("o", "c", "l", "i"))}
    b = {g: bl[3 * k + 2].astype(np.float64) for k, g in enumerate(("o", "c", "l", "i"))}
    order = ("i", "l", "c", "o")
    with torch.no_grad():
        lstm.weight_ih_l0.copy_(torch.from_numpy(np.concatenate([W[g].T for g in order])))
        lstm.weight_hh_l0.copy_(torch.from_numpy(np.concatenate([np.diag(u[g]) for g in order])))
        lstm.bias_ih_l0.copy_(torch.from_numpy(np.concatenate([b[g] for g in order])))
        lstm.bias_hh_l0.zero_()
        out, _ = lstm(torch.from_numpy(X.astype(np.float64)))
    np.testing.assert_allclose(H, out[:, -1].numpy(), rtol=0, atol=1e-14)


def test_lstm_diag_equals_dense_with_diagonal_U():
    """The per-cell function equals the dense-U oracle function fed diag(u)."""
    S, M, Q, N = 2, 6, 7, 5
    nd = orc.Net("lstm_diag", S=S, M=M, Q=Q)
    bd = orc.gen_weights(nd, seed=9)
    dense = [np.diag(x).astype(np.float32) if k % 3 == 1 else x for k, x in enumerate(bd)]
    X = rand_X(N, Q, S, seed=3)
    np.testing.assert_allclose(orc.build_H(nd, bd, X), orc.build_H(orc.Net("lstm", S=S, M=M, Q=Q), dense, X),
                               rtol=0, atol=1e-15)


def test_lstm_diag_spec_t1_and_two_steps():
    """SPEC S:202 worked value at t = 1 (x = 1, every W = 1, u = b = 0; corrected
    reading R23), then a hand-evaluated second step with u_o = 0.5."""
    net = orc.Net("lstm_diag", S=1, M=1, Q=2)
    bl = [np.zeros(orc.block_shape(net, k), np.float32) for k in range(12)]
    for g in range(4):
        bl[3 * g][:] = 1.0
    X = np.ones((1, 2, 1), np.float32)
    c1 = sig(1) * math.tanh(1)
    h1 = sig(1) * math.tanh(c1)
    assert abs(orc.build_H(orc.Net("lstm_diag", S=1, M=1, Q=1), bl, X[:, :1])[0, 0] - 0.36960635293570576) < 1e-15
    assert abs(h1 - 0.36960635293570576) < 1e-15
    bl[1][:] = 0.5            # u_o
    c2 = sig(1) * c1 + sig(1) * math.tanh(1)
    h2 = sig(1 + 0.5 * h1) * math.tanh(c2)
    assert abs(orc.build_H(net, bl, X)[0, 0] - h2) < 1e-15


# ---------------------------------------------------------------- diagonal GRU
def test_gru_diag_equals_torch_gru():
    """Diagonal-U GRU == torch.nn.GRU with the z weights negated (1 - sigma(a) = sigma(-a));
    u_f (r h) = r (u_f h) for a diagonal U_f (reset-before equals reset-after)."""
    S, M, Q, N = 2, 6, 8, 9
    net = orc.Net("gru_diag", S=S, M=M, Q=Q)
    bl = orc.gen_weights(net, seed=3)
    X = rand_X(N, Q, S, seed=2)
    H = orc.build_H(net, bl, X)
    gru = torch.nn.GRU(S, M, batch_first=True).double()
    Wz, uz, bz = (bl[k].astype(np.float64) for k in (0, 1, 2))
    Wr, ur, br = (bl[k].astype(np.float64) for k in (3, 4, 5))
    Wf, uf, bf = (bl[k].astype(np.float64) for k in (6, 7, 8))
    with torch.no_grad():
        gru.weight_ih_l0.copy_(torch.from_numpy(np.concatenate([Wr.T, -Wz.T, Wf.T])))
        gru.weight_hh_l0.copy_(torch.from_numpy(np.concatenate([np.diag(ur), -np.diag(uz), np.diag(uf)])))
        gru.bias_ih_l0.copy_(torch.from_numpy(np.concatenate([br, -bz, bf])))
        gru.bias_hh_l0.zero_()
        out, _ = gru(torch.from_numpy(X.astype(np.float64)))
    np.testing.assert_allclose(H, out[:, -1].numpy(), rtol=0, atol=1e-14)


def test_gru_diag_spec_t1_and_gate_closed():
    """SPEC S:211 worked value at t = 1 (x = 1, W = 1, u = b = 0 -> 0.5568...), and
    the update gate closed (b_z -> -inf) keeps h at 0 for all t."""
    net = orc.Net("gru_diag", S=1, M=1, Q=1)
    bl = [np.zeros(orc.block_shape(net, k), np.float32) for k in range(9)]
    for g in range(3):
        bl[3 * g][:] = 1.0
    X = np.ones((1, 1, 1), np.float32)
    assert abs(orc.build_H(net, bl, X)[0, 0] - sig(1) * math.tanh(1)) < 1e-15
    net5 = orc.Net("gru_diag", S=1, M=1, Q=5)
    bl[2][:] = -1e4            # b_z
    assert orc.build_H(net5, bl, np.ones((1, 5, 1), np.float32))[0, 0] == 0.0


# ---------------------------------------------------------------- FC by Eq. 8
def test_fc_eq8_distinguishing_pin():
    """M = 2, Q = 2, x = W = 0, b = (1, -1), A_1[0][1] = 1.  The prose
    reading gives h(2) = (sigma(1), 0.4331669929794054); Eq. 8 by the letter scales
    each neuron's own history by sum_l alpha[j,l,1] = (0, 1): (sigma(1), 0.3249624726231763)."""
    net = orc.Net("fc_eq8", S=1, M=2, Q=2)
    bl = [np.zeros(orc.block_shape(net, k), np.float32) for k in range(3)]
    bl[1][:] = (1.0, -1.0)
    bl[2][0, 0, 1] = 1.0
    H = orc.build_H(net, bl, np.zeros((1, 2, 1), np.float32))
    np.testing.assert_allclose(H[0], [sig(1.0), 0.3249624726231763], rtol=0, atol=1e-15)
    Hp = orc.build_H(orc.Net("fc", S=1, M=2, Q=2), bl, np.zeros((1, 2, 1), np.float32))
    np.testing.assert_allclose(Hp[0], [sig(1.0), 0.4331669929794054], rtol=0, atol=1e-15)


def test_fc_eq8_spec_example():
    """alpha[j,.,1] = [0.5, 0.5], prior h = 1.0, W.x + b = 0 -> sigma(1.0).
    A prior h(1) close to 1 comes from a huge bias at t = 1 only; with x(2) = -b/W
    the pre-activation at t = 2 is exactly sum_l alpha h(1) = h(1)."""
    net = orc.Net("fc_eq8", S=1, M=2, Q=2)
    bl = [np.zeros(orc.block_shape(net, k), np.float32) for k in range(3)]
    bl[0][:] = 64.0            # W: x(1) = 1 -> a(1) = 64 + b
    bl[1][:] = 0.0
    bl[2][0, :, :] = 0.5       # alpha[j, l, 1] = A[0][l][j] = 0.5
    X = np.array([[[1.0], [0.0]]], np.float32)
    h1 = sig(64.0)
    H = orc.build_H(net, bl, X)
    np.testing.assert_allclose(H[0], [sig(h1), sig(h1)], rtol=0, atol=1e-15)
    assert abs(sig(h1) - sig(1.0)) < 1e-12


def test_fc_eq8_equals_elman_with_summed_alpha():
    """Collapse identity: Eq. 8 == Elman (Eq. 5) with alpha[j,k] = sum_l A[k-1][l][j]
    (lags > L zero), an independently written oracle function."""
    S, M, Q, N, L = 2, 5, 7, 6, 4
    n8 = orc.Net("fc_eq8", S=S, M=M, Q=Q, fc_lags=L)
    bl = orc.gen_weights(n8, seed=4)
    X = rand_X(N, Q, S, seed=5)
    al = np.zeros((M, Q), np.float64)
    al[:, :L] = bl[2].astype(np.float64).sum(axis=1).T     # [L][M_l][M_j] -> [j][k]
    ne = orc.Net("elman", S=S, M=M, Q=Q)
    He = orc.build_H(ne, [bl[0], bl[1], al.astype(np.float32)], X)
    # the Elman block is fp32: compare with the column sums rounded the same way
    al32 = al.astype(np.float32).astype(np.float64)
    assert np.abs(al32 - al).max() < 1e-6
    H8 = orc.build_H(n8, bl, X)
    np.testing.assert_allclose(H8, He, rtol=0, atol=5e-6)


def test_fc_eq8_M1_equals_elman_exactly():
    """M = 1: the inner sum has one term, so Eq. 8 == Eq. 5 with alpha[0,k] = A[k-1][0][0]."""
    S, Q, N = 1, 6, 4
    n8 = orc.Net("fc_eq8", S=S, M=1, Q=Q)
    bl = orc.gen_weights(n8, seed=2)
    X = rand_X(N, Q, S, seed=1)
    He = orc.build_H(orc.Net("elman", S=S, M=1, Q=Q), [bl[0], bl[1], bl[2][:, 0, 0].reshape(1, Q).copy()], X)
    np.testing.assert_array_equal(orc.build_H(n8, bl, X), He)


@pytest.mark.parametrize("arch", ["lstm_diag", "gru_diag", "fc_eq8"])
def test_cell_independence(arch):
    """h_ij depends only on row i's window, column-j weights and its own
    history -- permuting neurons (weights) permutes H's columns, any row order works."""
    S, M, Q, N = 2, 6, 5, 7
    net = orc.Net(arch, S=S, M=M, Q=Q)
    bl = orc.gen_weights(net, seed=8)
    X = rand_X(N, Q, S, seed=6)
    H = orc.build_H(net, bl, X)
    perm = np.random.default_rng(0).permutation(M)
    if arch == "fc_eq8":
        pb = [bl[0][:, perm], bl[1][perm], bl[2][:, :, perm]]
    else:
        pb = [x[:, perm] if x.ndim == 2 else x[perm] for x in bl]
    np.testing.assert_allclose(orc.build_H(net, pb, X), H[:, perm], rtol=0, atol=1e-15)
    rows = np.random.default_rng(1).permutation(N)
    np.testing.assert_array_equal(orc.build_H(net, bl, X[rows]), H[rows])
