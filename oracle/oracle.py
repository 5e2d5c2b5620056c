"""TEST INFRASTRUCTURE ONLY -- ctypes front end of the fp64 CPU oracle.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import this module.  The
product path (``paper_1911_13252_b200``) never imports it and shares no code
with it: the oracle regenerates the weights with its own implementation of the
counter-based generator and computes in fp64.

Paper: El Zini, Rizk, Awad, arXiv 1911.13252 ("P:n" = PAPER.md line n).
  * ``build_H``  -- Alg. 1 line 2 with Eqs. 5-10 read as
    DESIGN.md readings R3-R14 state.
  * ``lstsq``    -- S4.2: Householder QR of [H | Y], z = Q^T Y,
    back substitution; rank check + ridge fallback (R19).
  * ``predict``  -- Eq. 4, no output bias (R16).
  * ``error_windows`` / ``train_narmax_ef`` -- Eq. 7 with e = y - yhat,
    two passes (reading R30).
  * ``test_rmse`` / ``forecast`` -- held-out RMSE and the free-running
    recursive forecast (reading R31).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "elm_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

ARCHS = {"elman": 0, "jordan": 1, "narmax": 2, "fc": 3, "lstm": 4, "gru": 5,
         # paper-literal per-cell variants: diagonal-U LSTM/GRU
         # and FC by the letter of Eq. 8
         "lstm_diag": 6, "gru_diag": 7, "fc_eq8": 8}
GATES = {"lstm": ("o", "c", "lambda", "in"), "gru": ("z", "r", "f"),
         "lstm_diag": ("o", "c", "lambda", "in"), "gru_diag": ("z", "r", "f")}


def build(force: bool = False) -> str:
    """Compile the oracle (plain C, -O2 -ffp-contract=off, OpenMP row split)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-ffp-contract=off", "-fopenmp", "-shared", "-fPIC",
               "-o", _LIB + ".tmp", _SRC, "-lm"]
        subprocess.run(cmd, check=True)
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        L = _lib
        i64, i32, u64 = ctypes.c_int64, ctypes.c_int, ctypes.c_uint64
        vp = ctypes.c_void_p
        L.orc_gen_block.argtypes = [i32] * 9 + [u64, i32, vp]
        L.orc_gen_block.restype = i32
        L.orc_block_len.argtypes = [i32] * 8
        L.orc_block_len.restype = i64
        L.orc_num_blocks.argtypes = [i32]
        L.orc_num_blocks.restype = i32
        L.orc_build_H.argtypes = [i32] * 8 + [vp, vp, i64, vp, i64, i64, vp, i64, i32]
        L.orc_build_H.restype = i32
        L.orc_build_H_ef.argtypes = [i32] * 8 + [vp, vp, i64, vp, i64, vp, i64, i64, vp, i64, i32]
        L.orc_build_H_ef.restype = i32
        L.orc_error_windows.argtypes = [vp, i64, vp, i64, i32, i32, vp, vp, i64]
        L.orc_error_windows.restype = None
        L.orc_lstsq.argtypes = [vp, i64, vp, i64, i32, vp, vp, vp]
        L.orc_lstsq.restype = i32
        L.orc_solve_from_R.argtypes = [vp, i32, i64, vp, vp]
        L.orc_solve_from_R.restype = i32
        L.orc_predict.argtypes = [vp, i64, i64, i32, vp, vp]
        L.orc_predict.restype = None
        L.orc_rng_u64.argtypes = [u64]
        L.orc_rng_u64.restype = u64
        L.orc_set_qr_threads.argtypes = [i32]
        L.orc_set_qr_threads.restype = None
        L.orc_max_threads.argtypes = []
        L.orc_max_threads.restype = i32
    return _lib


class _Info(ctypes.Structure):
    _fields_ = [("rho", ctypes.c_double), ("rmse", ctypes.c_double),
                ("rdiag_min_abs", ctypes.c_double), ("rdiag_max_abs", ctypes.c_double),
                ("ridge_lambda", ctypes.c_double), ("rank_flag", ctypes.c_int),
                ("n_total", ctypes.c_int64)]


@dataclass
class Net:
    """Architecture + hyper-parameters (Table 1; opts of DESIGN.md)."""
    arch: str
    S: int
    M: int
    Q: int
    F: int = -1          # NARMAX output lags (default Q, reading R8)
    R: int = -1          # NARMAX error lags (default Q)
    act: int = 0         # 0 sigmoid, 1 tanh for g (Elman/Jordan/NARMAX/FC)
    fc_lags: int = -1    # FC lags (default Q, prose reading R9)
    rec_scale: int = 0   # 0 = 1/sqrt(fan_in) on blocks multiplying h; 1 = unit
    weight_grid: int = 0  # 0 fp32, 1 fp16-grid, 2 tf32-grid (MMA blocks only)

    def __post_init__(self):
        if self.F < 0:
            self.F = self.Q
        if self.R < 0:
            self.R = self.Q
        if self.fc_lags < 0:
            self.fc_lags = self.Q

    @property
    def code(self) -> int:
        return ARCHS[self.arch]

    def _dims(self):
        return (self.code, self.S, self.M, self.Q, self.F, self.R, self.fc_lags)


def num_blocks(arch: str) -> int:
    return lib().orc_num_blocks(ARCHS[arch])


def block_shape(net: Net, block_id: int):
    """Logical shape of a weight block."""
    a, S, M, Q, F, R, L = net.arch, net.S, net.M, net.Q, net.F, net.R, net.fc_lags
    if a in ("elman", "jordan"):
        return [(S, M), (M,), (M, Q)][block_id]
    if a == "narmax":
        return [(S, M), (M,), (M, F), (M, R)][block_id]
    if a in ("fc", "fc_eq8"):
        return [(S, M), (M,), (L, M, M)][block_id]
    if a in ("lstm_diag", "gru_diag"):
        return [(S, M), (M,), (M,)][block_id % 3]
    return [(S, M), (M, M), (M,)][block_id % 3]


def gen_weights(net: Net, seed: int):
    """Regenerate all weight blocks (fp32 numpy arrays in logical layout)."""
    L = lib()
    out = []
    for b in range(num_blocks(net.arch)):
        n = L.orc_block_len(*net._dims(), b)
        arr = np.empty(n, dtype=np.float32)
        rc = L.orc_gen_block(*net._dims(), net.rec_scale, net.weight_grid,
                             ctypes.c_uint64(seed & (2**64 - 1)), b, arr.ctypes.data)
        assert rc == 0
        out.append(arr.reshape(block_shape(net, b)))
    return out


def build_H(net: Net, blocks, X, Yfb=None, threads: int = 1, Ef=None) -> np.ndarray:
    """fp64 H(Q) [N][M] for fp32 X [N][Q][S] (or [N][Q*S]), optional Yfb [N][Q]
    and, for NARMAX, an optional error window Ef [N][Q] (e_i(tau) = Ef[i][tau-1],
    reading R30; None: e == 0, reading R8)."""
    X = np.ascontiguousarray(X, dtype=np.float32)
    N = X.shape[0]
    X2 = X.reshape(N, -1)
    assert X2.shape[1] >= net.Q * net.S
    blks = [np.ascontiguousarray(b, dtype=np.float32) for b in blocks]
    assert len(blks) == num_blocks(net.arch)
    ptrs = (ctypes.c_void_p * len(blks))(*[b.ctypes.data for b in blks])
    H = np.zeros((N, net.M), dtype=np.float64)
    ydata, ldy = None, 0
    if Yfb is not None:
        Yfb = np.ascontiguousarray(Yfb, dtype=np.float32).reshape(N, -1)
        ydata, ldy = Yfb.ctypes.data, Yfb.shape[1]
    edata, lde = None, 0
    if Ef is not None:
        Ef = np.ascontiguousarray(Ef, dtype=np.float32).reshape(N, -1)
        assert Ef.shape[1] >= net.Q
        edata, lde = Ef.ctypes.data, Ef.shape[1]
    if N == 0:
        return H
    rc = lib().orc_build_H_ef(net.code, net.S, net.M, net.Q, net.F, net.R, net.act, net.fc_lags,
                              ctypes.cast(ptrs, ctypes.c_void_p), X2.ctypes.data, X2.shape[1],
                              ydata, ldy, edata, lde, N, H.ctypes.data, net.M, threads)
    assert rc == 0
    return H


@dataclass
class SolveInfo:
    rho: float
    rmse: float
    rdiag_min_abs: float
    rdiag_max_abs: float
    ridge_lambda: float
    rank_flag: int
    n_total: int
    status: int
    R: np.ndarray


def set_qr_threads(t: int) -> None:
    """Threads for the column updates of the Householder QR (bitwise identical
    result for any count: each column is updated by one thread in fixed order)."""
    lib().orc_set_qr_threads(int(t))


def lstsq(H, Y):
    """beta = argmin ||H beta - Y|| by unblocked Householder QR on [H | Y] (fp64).

    Returns (beta, SolveInfo).  status: 0 ok, 1 ridge fallback, -3
    underdetermined (N < M), -4 non-finite input."""
    H = np.ascontiguousarray(H, dtype=np.float64)
    N, M = H.shape
    Y = np.ascontiguousarray(np.asarray(Y, dtype=np.float64).reshape(N))
    beta = np.zeros(M, dtype=np.float64)
    info = _Info()
    R = np.zeros((M + 1, M + 1), dtype=np.float64)
    rc = lib().orc_lstsq(H.ctypes.data, M, Y.ctypes.data, N, M, beta.ctypes.data,
                         ctypes.addressof(info), R.ctypes.data)
    return beta, SolveInfo(info.rho, info.rmse, info.rdiag_min_abs, info.rdiag_max_abs,
                           info.ridge_lambda, info.rank_flag, info.n_total, rc, R)


def error_windows(H, Y, beta, Q: int) -> np.ndarray:
    """NARMAX error-feedback windows (Eq. 7, P:122 e(t) = y(t) - yhat(t); reading
    R30): Ef[i][tau-1] = Y[k] - H[k].beta with k = i + tau - Q (0 when k < 0),
    fp32 [N][Q]."""
    H = np.ascontiguousarray(H, dtype=np.float64)
    N, M = H.shape
    Y = np.ascontiguousarray(np.asarray(Y, dtype=np.float64).reshape(N))
    beta = np.ascontiguousarray(beta, dtype=np.float64).reshape(M)
    Ef = np.zeros((N, Q), dtype=np.float32)
    lib().orc_error_windows(H.ctypes.data, M, Y.ctypes.data, N, M, Q, beta.ctypes.data, Ef.ctypes.data, Q)
    return Ef


def train_narmax_ef(net: Net, blocks, X, Y, Yfb=None, threads: int = 1):
    """Two-pass NARMAX training with real error feedback:
    pass 0 with e == 0 (R8) gives beta0; e = y - yhat(beta0) (R30); pass 1
    rebuilds H with that e and re-solves.  Returns (H1, beta1, info1, beta0, info0)."""
    assert net.arch == "narmax"
    H0 = build_H(net, blocks, X, Yfb, threads=threads)
    b0, i0 = lstsq(H0, Y)
    Ef = error_windows(H0, Y, b0, net.Q)
    H1 = build_H(net, blocks, X, Yfb, threads=threads, Ef=Ef)
    b1, i1 = lstsq(H1, Y)
    return H1, b1, i1, b0, i0


def solve_from_R(R, M: int, n_total: int):
    """beta from an (M+1)x(M+1) upper-triangular R of [H | Y] (sign-normalised in a copy)."""
    Rf = np.array(R, dtype=np.float64, copy=True, order="C")
    beta = np.zeros(M, dtype=np.float64)
    info = _Info()
    rc = lib().orc_solve_from_R(Rf.ctypes.data, M, n_total, beta.ctypes.data, ctypes.addressof(info))
    return beta, SolveInfo(info.rho, info.rmse, info.rdiag_min_abs, info.rdiag_max_abs,
                           info.ridge_lambda, info.rank_flag, info.n_total, rc, Rf)


def predict(H, beta) -> np.ndarray:
    H = np.ascontiguousarray(H, dtype=np.float64)
    N, M = H.shape
    beta = np.ascontiguousarray(beta, dtype=np.float64)
    out = np.zeros(N, dtype=np.float64)
    lib().orc_predict(H.ctypes.data, M, N, M, beta.ctypes.data, out.ctypes.data)
    return out


def train(net: Net, seed: int, X, Y, Yfb=None, threads: int = 1):
    """Alg. 1 end to end: weights -> H(Q) -> beta."""
    blocks = gen_weights(net, seed)
    H = build_H(net, blocks, X, Yfb, threads=threads)
    beta, info = lstsq(H, Y)
    return H, beta, info


def rng_u64(z: int) -> int:
    """splitmix64 mix of DESIGN.md "Weights" (for the known-answer test)."""
    return lib().orc_rng_u64(ctypes.c_uint64(z & (2**64 - 1)))


def max_threads() -> int:
    return lib().orc_max_threads()


def test_rmse(net: Net, blocks, X, Y, beta, Yfb=None, threads: int = 1) -> float:
    """Held-out RMSE (SPEC "rmse_test"): sqrt(mean((yhat - y)^2))
    with yhat = H(Q) beta (Eq. 4) on the evaluation windows."""
    yhat = predict(build_H(net, blocks, X, Yfb, threads=threads), beta)
    d = yhat - np.asarray(Y, dtype=np.float64).reshape(-1)
    return float(np.sqrt(np.mean(d * d)))


def forecast(net: Net, blocks, X, beta, K: int, threads: int = 1) -> np.ndarray:
    """Free-running (recursive) K-step forecast (SPEC "recursive
    self-feedback mode"; reading R31).  Univariate autoregressive windows (d = 1):
    window w_0 = X[i] (s[i..i+Q-1]); step k predicts yhat_k = H(w_k) beta (Eq. 4;
    Jordan/NARMAX feedback y(tau) = w_k[tau], the Yfb = NULL convention, R7), then
    w_{k+1} = (w_k[1:], fp32(yhat_k)): the prediction replaces the next observation.
    Returns fp64 [N][K]."""
    assert net.S == 1
    W = np.ascontiguousarray(np.asarray(X, dtype=np.float32).reshape(X.shape[0], -1)[:, :net.Q])
    out = np.zeros((W.shape[0], K), dtype=np.float64)
    for k in range(K):
        yhat = predict(build_H(net, blocks, W, None, threads=threads), beta)
        out[:, k] = yhat
        W = np.ascontiguousarray(np.concatenate([W[:, 1:], yhat.astype(np.float32)[:, None]], axis=1))
    return out


def lstsq_multi(H, Y):
    """Multi-output least squares (the paper's future work P:655):
    the P outputs are independent problems beta_p = argmin ||H beta - Y[:, p]||, each
    solved by the single-output Householder lstsq above.  Returns (B [P][M], [SolveInfo])."""
    Y = np.asarray(Y, dtype=np.float64)
    if Y.ndim == 1:
        Y = Y[:, None]
    out = [lstsq(H, Y[:, p]) for p in range(Y.shape[1])]
    return np.stack([b for b, _ in out]), [i for _, i in out]
