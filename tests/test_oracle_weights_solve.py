"""Pins for the oracle's weight generator and least-squares solver (CPU only).

Weights: SplitMix64 known-answer values, determinism, range and scale, and
grid rounding against numpy's float16 cast / a bit-level TF32 RNA rounding.
Solver (S4.2): closed forms from tests/golden, numpy lstsq / pinv
(LAPACK SVD) on tiny problems, numpy QR's R up to row signs, normal-equation
residual, exact fit, perturbation optimality, ridge == (H^T H + lambda I)^-1 H^T Y.
"""
import json
import math
import os

import numpy as np
import pytest

from oracle import oracle as orc

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


# ---------------------------------------------------------------- weights
def test_splitmix64_known_answers():
    golden = GOLD["splitmix64_seed0"]["values"]
    g = 0x9E3779B97F4A7C15
    for k, v in enumerate(golden):
        assert orc.rng_u64((k * g) % 2**64) == int(v, 16)


def test_weights_deterministic_and_seed_sensitive():
    net = orc.Net("lstm", S=2, M=16, Q=5)
    a = orc.gen_weights(net, 1)
    b = orc.gen_weights(net, 1)
    c = orc.gen_weights(net, 2)
    for x, y, z in zip(a, b, c):
        np.testing.assert_array_equal(x, y)
        assert not np.array_equal(x, z)


@pytest.mark.parametrize("arch,M,Q", [("elman", 20, 10), ("fc", 16, 6), ("lstm", 64, 5), ("gru", 64, 5),
                                      ("jordan", 8, 20), ("narmax", 8, 20)])
def test_weight_ranges_and_scales(arch, M, Q):
    net = orc.Net(arch, S=3, M=M, Q=Q)
    blocks = orc.gen_weights(net, 7)
    unit = orc.gen_weights(orc.Net(arch, S=3, M=M, Q=Q, rec_scale=1), 7)
    for k, (w, u) in enumerate(zip(blocks, unit)):
        assert np.all(np.abs(u) <= 1.0) and u.min() < -0.5 and u.max() > 0.5
        ratio = np.abs(w).max() / np.abs(u).max()
        if arch in ("lstm", "gru") and k % 3 == 1:
            expect = 1 / math.sqrt(M)
        elif arch == "fc" and k == 2:
            expect = 1 / math.sqrt(M * Q)
        elif arch == "elman" and k == 2:
            expect = 1 / math.sqrt(Q)
        else:
            expect = 1.0
        assert ratio == pytest.approx(expect, rel=1e-6)
        if u.size > 1000:
            assert abs(float(u.mean())) < 0.05 and float(u.std()) == pytest.approx(1 / math.sqrt(3), rel=0.05)


def test_fp16_grid_matches_numpy_cast():
    net = orc.Net("lstm", S=1, M=64, Q=3)
    w32 = orc.gen_weights(net, 3)
    w16 = orc.gen_weights(orc.Net("lstm", S=1, M=64, Q=3, weight_grid=1), 3)
    for k in range(12):
        if k % 3 == 1:
            np.testing.assert_array_equal(w16[k], w32[k].astype(np.float16).astype(np.float32))
        else:
            np.testing.assert_array_equal(w16[k], w32[k])


def test_tf32_grid_matches_bit_rounding():
    net = orc.Net("gru", S=1, M=32, Q=3)
    w32 = orc.gen_weights(net, 4)
    wtf = orc.gen_weights(orc.Net("gru", S=1, M=32, Q=3, weight_grid=2), 4)
    for k in range(9):
        if k % 3 == 1:
            bits = w32[k].view(np.uint32).astype(np.uint64)
            rna = ((bits + 0x1000) & 0xFFFFE000).astype(np.uint32).view(np.float32)
            np.testing.assert_array_equal(wtf[k], rna)


# ---------------------------------------------------------------- solver closed forms
def test_qr_3_4():
    beta, info = orc.lstsq(np.array([[3.0], [4.0]]), np.array([0.6 * 5, 0.8 * 5]))
    assert abs(info.R[0, 0]) == pytest.approx(GOLD["qr_3_4"]["R"], abs=1e-15)
    assert beta[0] == pytest.approx(1.0, abs=1e-15)


def test_backsub_closed_form():
    g = GOLD["backsub"]
    R = np.zeros((3, 3))
    R[:2, :2] = g["R"]
    R[:2, 2] = g["z"]
    beta, info = orc.solve_from_R(R, 2, 10)
    np.testing.assert_allclose(beta, g["beta"], rtol=0, atol=1e-15)
    assert info.rho == 0.0


def test_identity_design():
    g = GOLD["identity_design"]
    beta, info = orc.lstsq(np.array(g["H"], float), np.array(g["Y"], float))
    np.testing.assert_allclose(beta, g["beta"], atol=1e-15)
    assert info.status == 0 and info.rho == pytest.approx(0.0, abs=1e-15)


def test_exact_single_column():
    g = GOLD["exact_1col"]
    beta, info = orc.lstsq(np.array(g["H"], float), np.array(g["Y"], float))
    assert beta[0] == pytest.approx(1.0, abs=1e-15) and info.rho == pytest.approx(0.0, abs=1e-15)


def test_rank_deficient_ridge():
    H = np.ones((3, 2))
    beta, info = orc.lstsq(H, np.array([1.0, 2.0, 3.0]))
    assert info.status == 1 and info.rank_flag == 1 and np.all(np.isfinite(beta))
    lam = info.ridge_lambda
    assert lam == pytest.approx(1e-8 * np.trace(H.T @ H) / 2, rel=1e-12)
    ref = np.linalg.solve(H.T @ H + lam * np.eye(2), H.T @ np.array([1.0, 2.0, 3.0]))
    np.testing.assert_allclose(beta, ref, rtol=1e-6)


def test_underdetermined_and_nonfinite():
    assert orc.lstsq(np.ones((2, 3)), np.ones(2))[1].status == -3
    H = np.ones((5, 2)); H[3, 1] = np.nan
    assert orc.lstsq(H, np.ones(5))[1].status == -4
    assert orc.lstsq(np.eye(5)[:, :2], np.array([1, 2, np.inf, 0, 0.0]))[1].status == -4


# ---------------------------------------------------------------- solver vs libraries
@pytest.mark.parametrize("seed", range(10))
def test_matches_numpy_lstsq_and_pinv(seed):
    rng = np.random.default_rng(seed)
    N, M = rng.integers(9, 64), rng.integers(1, 8)
    H = rng.standard_normal((N, M))
    Y = rng.standard_normal(N)
    beta, info = orc.lstsq(H, Y)
    ref = np.linalg.lstsq(H, Y, rcond=None)[0]
    np.testing.assert_allclose(beta, ref, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(beta, np.linalg.pinv(H) @ Y, rtol=1e-10, atol=1e-12)
    rmse = np.linalg.norm(H @ ref - Y) / math.sqrt(N)
    assert info.rmse == pytest.approx(rmse, rel=1e-12)
    assert info.rho == pytest.approx(rmse * math.sqrt(N), rel=1e-12)
    Rnp = np.linalg.qr(np.column_stack([H, Y]), mode="r")
    Rnp = Rnp * np.sign(np.diag(Rnp))[:, None]
    np.testing.assert_allclose(info.R, Rnp, rtol=0, atol=1e-12 * np.abs(Rnp).max())


def test_normal_equation_residual_50_instances():
    rng = np.random.default_rng(1911)
    for _ in range(50):
        H = rng.standard_normal((200, 20))
        Y = rng.standard_normal(200)
        beta, _ = orc.lstsq(H, Y)
        r = H.T @ (H @ beta - Y)
        assert np.abs(r).max() <= 1e-8 * max(1.0, np.abs(H.T @ Y).max())


def test_exact_fit_and_perturbation_optimality():
    rng = np.random.default_rng(3)
    H = 1 / (1 + np.exp(-rng.standard_normal((300, 12))))
    bstar = rng.standard_normal(12)
    beta, info = orc.lstsq(H, H @ bstar)
    np.testing.assert_allclose(beta, bstar, rtol=1e-9, atol=1e-9)
    assert info.rho <= 1e-9 * np.linalg.norm(H @ bstar)
    Y = H @ bstar + 0.1 * rng.standard_normal(300)
    beta, _ = orc.lstsq(H, Y)
    f0 = np.sum((H @ beta - Y) ** 2)
    for _ in range(20):
        d = rng.standard_normal(12)
        d *= 1e-3 / np.linalg.norm(d)
        assert np.sum((H @ (beta + d) - Y) ** 2) >= f0


def test_tsqr_tree_equals_direct_R():
    """R of stacked partial R factors equals direct R (sign-normalised): the
    identity the GPU row-sharded / multi-rank merge relies on."""
    rng = np.random.default_rng(5)
    H = rng.standard_normal((400, 9)); Y = rng.standard_normal(400)
    _, full = orc.lstsq(H, Y)
    parts = [orc.lstsq(H[i:i + 100], Y[i:i + 100])[1].R for i in range(0, 400, 100)]
    stacked = np.vstack(parts)
    _, merged = orc.lstsq(stacked[:, :9], stacked[:, 9])
    np.testing.assert_allclose(merged.R, full.R, rtol=0, atol=1e-13 * np.abs(full.R).max())


def test_predict_is_H_beta():
    rng = np.random.default_rng(0)
    H = rng.standard_normal((17, 5)); b = rng.standard_normal(5)
    np.testing.assert_allclose(orc.predict(H, b), H @ b, rtol=1e-14, atol=1e-14)


def test_lstsq_multi_is_per_output_lstsq_and_numpy():
    """Multi-output least squares = P independent problems: each column against
    numpy's lstsq (LAPACK SVD) and the single-output Householder lstsq."""
    rng = np.random.default_rng(17)
    H = rng.standard_normal((120, 9))
    Y = rng.standard_normal((120, 3))
    B, infos = orc.lstsq_multi(H, Y)
    ref = np.linalg.lstsq(H, Y, rcond=None)[0].T
    np.testing.assert_allclose(B, ref, rtol=1e-10, atol=1e-12)
    for p in range(3):
        b1, i1 = orc.lstsq(H, Y[:, p])
        np.testing.assert_array_equal(B[p], b1)
        assert infos[p].rmse == pytest.approx(np.sqrt(np.mean((H @ ref[p] - Y[:, p]) ** 2)), rel=1e-10)
