"""The beta / RMSE parity rule (reading R26) -- test infrastructure.

North star: ||beta_gpu - beta_ref|| / ||beta_ref|| <= 1e-3 "reported alongside
cond(R)", training RMSE within 1e-4 relative.  beta_ref is the oracle's fp64
Householder solve of the oracle's own fp64 H.

Any implementation that stores H in fp32 (the north star's H tolerance is
fp32-sized: 1e-5 max-abs) perturbs the least-squares problem by at least the
fp32 rounding of H.  On smooth series cond(R) reaches 1e6-1e7 and that
rounding alone moves beta beyond 1e-3 (C1 Elman: 4.7e-4; the smoke's old
M = 512 case: 3.5e-2).  The rule is therefore FIXED and independent of the
GPU's own H error:

    floor_b = ||beta(fp32(H_o)) - beta(H_o)|| / ||beta(H_o)||
    floor_r = |rmse(fp32(H_o)) - rmse(H_o)| / rmse(H_o)
    tol_b   = max(1e-3, K * floor_b)      tol_r = max(1e-4, K * floor_r)     K = 8

(the floors from LAPACK least-squares solves -- a sensitivity measure of the
problem; the reference beta_ref / rmse_ref is the oracle's Householder lstsq).  On well-conditioned cases
(floor_b << 1e-3) this is exactly the north star's literal bound; the
well-conditioned cases of tests/test_gpu_parity.py additionally assert the
literal 1e-3 / 1e-4 directly.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from oracle import oracle as orc

K_FLOOR = 8.0
BETA_TOL = 1e-3
RMSE_TOL = 1e-4


@dataclass
class Bounds:
    tol_b: float
    tol_r: float
    floor_b: float
    floor_r: float
    cond: float
    b_ref: np.ndarray
    i_ref: object


def _np_lstsq(H, Y):
    b = np.linalg.lstsq(H, Y, rcond=None)[0]
    return b, float(np.linalg.norm(H @ b - Y)) / np.sqrt(H.shape[0])


def bounds(Ho: np.ndarray, Y: np.ndarray) -> Bounds:
    """Reference solve of the oracle's fp64 H and the fixed tolerances of R26."""
    Y = np.asarray(Y, dtype=np.float64)
    b_ref, i_ref = orc.lstsq(Ho, Y)
    # the floor is a sensitivity measure of the problem, not a reference value:
    # LAPACK (numpy) solves of H_o and fp32(H_o), compared with each other
    b64, r64 = _np_lstsq(Ho, Y)
    b32, r32 = _np_lstsq(Ho.astype(np.float32).astype(np.float64), Y)
    fb = float(np.linalg.norm(b32 - b64) / np.linalg.norm(b64))
    fr = float(abs(r32 - r64) / r64)
    M = Ho.shape[1]
    cond = float(np.linalg.cond(i_ref.R[:M, :M]))
    return Bounds(max(BETA_TOL, K_FLOOR * fb), max(RMSE_TOL, K_FLOOR * fr), fb, fr, cond, b_ref, i_ref)


def check(tag: str, beta_gpu, rmse_gpu: float, Hg: np.ndarray, Ho: np.ndarray, Y, literal: bool = False):
    """Assert the R26 rule (or, with literal=True, the north star's bare 1e-3 /
    1e-4) and return (rel_dbeta, rel_drmse, Bounds).  Prints cond(R), the floor
    and the ratio ||H_gpu - H_o||_F / ||fp32(H_o) - H_o||_F (reported only)."""
    bd = bounds(Ho, Y)
    beta_gpu = np.asarray(beta_gpu, dtype=np.float64)
    rel = float(np.linalg.norm(beta_gpu - bd.b_ref) / np.linalg.norm(bd.b_ref))
    drm = float(abs(rmse_gpu - bd.i_ref.rmse) / bd.i_ref.rmse)
    H32 = Ho.astype(np.float32).astype(np.float64)
    ratio = float(np.linalg.norm(Hg - Ho) / max(np.linalg.norm(H32 - Ho), 1e-300))
    tb, tr = (BETA_TOL, RMSE_TOL) if literal else (bd.tol_b, bd.tol_r)
    print(f"{tag}: cond(R)={bd.cond:.2e} rel dbeta={rel:.2e} (tol {tb:.1e}, fp32-H floor {bd.floor_b:.2e}) "
          f"rel drmse={drm:.2e} (tol {tr:.1e}, floor {bd.floor_r:.2e}) |dH| ratio {ratio:.1f}")
    assert rel <= tb, f"{tag}: rel dbeta {rel:.3e} > {tb:.3e} (cond {bd.cond:.2e}, floor {bd.floor_b:.2e})"
    assert drm <= tr, f"{tag}: rel drmse {drm:.3e} > {tr:.3e} (floor {bd.floor_r:.2e})"
    return rel, drm, bd
