"""Seeded synthetic time series and windowing (shared input generator).

This module is the ONLY code shared by the oracle side (tests) and the CUDA
side (bench / tests).  It holds none of the ELM method's arithmetic: it draws
series shaped like the paper's ten workloads (Table 3, P:377-405 -- univariate,
S = 1 mostly, Q in {10, 50}) and cuts them into windows with the layout of the
nomenclature (Table 1): X[i][t][c] = s_c[i+t], Y[i] = s_0[i+Q],
Yfb[i][tau-1] = s_0[i+tau] (teacher signal, reading R7).

Series:
  * ``mg``   Mackey-Glass, tau = 17: dx/dt = 0.2 x(t-17)/(1+x(t-17)^10) - 0.1 x(t),
             Euler dt = 0.1, constant history 1.2, every 10th sub-step kept,
             first 1000 samples dropped; optional N(0, noise^2) observation noise.
  * ``ar5``  y_t = 0.4y_{t-1} + 0.2y_{t-2} - 0.1y_{t-3} + 0.1y_{t-4} - 0.05y_{t-5} + e_t.
  * ``sin4`` 4 channels of 3-tone sinusoid mixtures + 0.05 noise.
All are z-scored over the whole series and returned as float32.
"""
from __future__ import annotations

import numpy as np
from scipy.signal import lfilter

DATA_SEED = 1911


def mackey_glass(length: int, seed: int = DATA_SEED, noise: float = 0.0) -> np.ndarray:
    dt, sub, delay_steps, burn = 0.1, 10, 170, 1000
    total = (length + burn) * sub + 1
    x = np.empty(total + delay_steps, dtype=np.float64)
    x[: delay_steps + 1] = 1.2
    # x[n+1] = (1 - 0.1 dt) x[n] + dt * 0.2 x[n-170] / (1 + x[n-170]^10):
    # blocks of 170 sub-steps only read the previous block through the delay,
    # so each block is a first-order linear filter driven by a known input.
    a = 1.0 - 0.1 * dt
    n = delay_steps
    end = total + delay_steps - 1
    while n < end:
        m = min(delay_steps, end - n)
        xd = x[n - delay_steps: n - delay_steps + m]
        u = dt * 0.2 * xd / (1.0 + xd ** 10)
        y, _ = lfilter([1.0], [1.0, -a], u, zi=[a * x[n]])
        x[n + 1: n + 1 + m] = y
        n += m
    s = x[delay_steps::sub][burn: burn + length]
    if noise > 0:
        s = s + np.random.default_rng(seed).normal(0.0, noise, size=s.shape)
    return s[:, None]


def ar5(length: int, seed: int = DATA_SEED) -> np.ndarray:
    burn = 1000
    e = np.random.default_rng(seed).standard_normal(length + burn)
    y = lfilter([1.0], [1.0, -0.4, -0.2, 0.1, -0.1, 0.05], e)
    return y[burn:, None]


def sin4(length: int, seed: int = DATA_SEED) -> np.ndarray:
    rng = np.random.default_rng(seed)
    A = rng.uniform(0.5, 1.5, size=(4, 3))
    f = rng.uniform(1.0 / 200.0, 1.0 / 10.0, size=(4, 3))
    ph = rng.uniform(0.0, 2 * np.pi, size=(4, 3))
    t = np.arange(length, dtype=np.float64)
    out = np.empty((length, 4), dtype=np.float64)
    for c in range(4):
        acc = np.zeros(length)
        for m in range(3):
            acc += A[c, m] * np.sin(2 * np.pi * f[c, m] * t + ph[c, m])
        out[:, c] = acc
    out += 0.05 * rng.standard_normal(out.shape)
    return out


def zscore(s: np.ndarray) -> np.ndarray:
    s = np.asarray(s, dtype=np.float64)
    mu = s.mean(axis=0, keepdims=True)
    sd = s.std(axis=0, keepdims=True)
    sd[sd == 0] = 1.0
    return ((s - mu) / sd).astype(np.float32)


def series(kind: str, length: int, seed: int = DATA_SEED, noise: float = 0.0) -> np.ndarray:
    """z-scored float32 series of shape [length][S]."""
    if kind == "mg":
        raw = mackey_glass(length, seed, noise)
    elif kind == "ar5":
        raw = ar5(length, seed)
    elif kind == "sin4":
        raw = sin4(length, seed)
    else:
        raise ValueError(f"unknown series kind {kind!r}")
    return zscore(raw)


def lagged_channels(s: np.ndarray, S: int) -> np.ndarray:
    """[L][1] series -> [L-S+1][S] with channel c = s[t+c] (a multivariate input
    for the well-conditioned parity cases: S-dimensional windows of one AR
    series; pure data shaping, no method arithmetic)."""
    s = np.asarray(s, dtype=np.float32).reshape(len(s), -1)[:, 0]
    L = s.shape[0] - S + 1
    return np.ascontiguousarray(np.stack([s[c:c + L] for c in range(S)], axis=1))


def windows(s: np.ndarray, N: int, Q: int):
    """Cut N windows of Q steps from series s [L][S] (L >= N + Q).

    Returns X float32 [N][Q][S], Y float32 [N], Yfb float32 [N][Q]."""
    s = np.asarray(s, dtype=np.float32)
    if s.ndim == 1:
        s = s[:, None]
    L, S = s.shape
    if L < N + Q:
        raise ValueError("series too short for the requested windows")
    idx = np.arange(N)[:, None] + np.arange(Q)[None, :]
    X = s[idx]                                   # [N][Q][S]
    Y = s[Q: Q + N, 0].copy()
    Yfb = s[idx + 1, 0]                          # Yfb[i][tau-1] = s_0[i+tau]
    return np.ascontiguousarray(X), Y, np.ascontiguousarray(Yfb)


# Benchmark configurations of BASELINE.json (C1..C5), DESIGN.md "Inputs".
CONFIGS = {
    "C1": dict(arch="elman", series="mg", N=1000, Q=10, S=1, M=20, noise=0.0),
    "C2j": dict(arch="jordan", series="ar5", N=100_000, Q=20, S=1, M=64, noise=0.0),
    "C2n": dict(arch="narmax", series="ar5", N=100_000, Q=20, S=1, M=64, noise=0.0),
    "C3fc": dict(arch="fc", series="sin4", N=1_000_000, Q=30, S=4, M=128, noise=0.0),
    "C3gru": dict(arch="gru", series="sin4", N=1_000_000, Q=30, S=4, M=128, noise=0.0),
    "C4": dict(arch="lstm", series="mg", N=4_000_000, Q=50, S=1, M=256, noise=0.01),
    # paper-literal per-cell variants at the C3 shape
    "C3lstm_diag": dict(arch="lstm_diag", series="sin4", N=1_000_000, Q=30, S=4, M=128, noise=0.0),
    "C3gru_diag": dict(arch="gru_diag", series="sin4", N=1_000_000, Q=30, S=4, M=128, noise=0.0),
    "C3fc_eq8": dict(arch="fc_eq8", series="sin4", N=1_000_000, Q=30, S=4, M=128, noise=0.0),
    # NARMAX with real error feedback (two passes) at the C2 shape
    "C2n_ef": dict(arch="narmax", series="ar5", N=100_000, Q=20, S=1, M=64, noise=0.0, mode="ef"),
    # C5 (BASELINE configs[4]) widest point, one GPU's share of N = 16M over 8 GPUs
    "C5lstm1024": dict(arch="lstm", series="mg", N=2_000_000, Q=10, S=1, M=1024, noise=0.01),
    "C5gru1024": dict(arch="gru", series="mg", N=2_000_000, Q=10, S=1, M=1024, noise=0.01),
}
# The full C5 sweep (BASELINE configs[4]): LSTM/GRU x M in {32, 128, 512, 1024} x Q in
# {10, 50, 100}, one GPU's share of N = 16M over 8 GPUs (2M rows): "C5{arch}{M}q{Q}".
for _a in ("lstm", "gru"):
    for _m in (32, 128, 512, 1024):
        for _q in (10, 50, 100):
            CONFIGS[f"C5{_a}{_m}q{_q}"] = dict(arch=_a, series="mg", N=2_000_000, Q=_q, S=1, M=_m, noise=0.01)


def config_inputs(name: str, N: int | None = None, seed: int = DATA_SEED):
    """Windows for a named configuration (optionally truncated to N rows)."""
    c = CONFIGS[name]
    n = c["N"] if N is None else N
    s = series(c["series"], n + c["Q"], seed=seed, noise=c["noise"])
    return windows(s, n, c["Q"])
