"""Thin ctypes binding of libelmrnn.so (include/elmrnn.h), same names.

Argument marshalling only: torch tensors -> device pointers + leading
dimensions, the current torch CUDA stream -> the handle's stream.  Every
arithmetic step runs in the library's CUDA kernels.  There is no fallback:
if the shared library is missing or the device is not a CUDA device, calls
raise.  (PAPER.md = arXiv 1911.13252; see the header for the citations.)
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("ELMRNN_LIB") or os.path.join(_HERE, "libelmrnn.so")   # override: testing aid

ARCHS = {"elman": 0, "jordan": 1, "narmax": 2, "fc": 3, "lstm": 4, "gru": 5,
         "lstm_diag": 6, "gru_diag": 7, "fc_eq8": 8}   # paper-literal per-cell variants (elmrnn.h)
STATUS = {0: "OK", 1: "WARN_RIDGE", -1: "ERR_ARG", -2: "ERR_SHAPE", -3: "ERR_UNDERDETERMINED",
          -4: "ERR_NONFINITE", -5: "ERR_UNSUPPORTED", -6: "ERR_CUDA", -7: "ERR_OOM"}

EXPORTED = ("elmrnn_opts_default", "elmrnn_init", "elmrnn_init_ex", "elmrnn_set_stream", "elmrnn_build_H",
            "elmrnn_build_H_ef", "elmrnn_error_windows", "elmrnn_forecast", "elmrnn_test_rmse",
            "elmrnn_solve_beta_multi",
            "elmrnn_solve_beta", "elmrnn_solve_local", "elmrnn_solve_merge", "elmrnn_sync", "elmrnn_packed_r_len",
            "elmrnn_solve_local_multi", "elmrnn_solve_merge_multi", "elmrnn_packed_r_len_multi",
            "elmrnn_train", "elmrnn_train_local", "elmrnn_train_fused",
            "elmrnn_predict", "elmrnn_get_weights", "elmrnn_weight_block_len", "elmrnn_path",
            "elmrnn_launch_count", "elmrnn_last_error", "elmrnn_destroy")


class ElmrnnError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class Opts(ctypes.Structure):
    _fields_ = [("F", ctypes.c_int), ("R", ctypes.c_int), ("act", ctypes.c_int), ("rec_scale", ctypes.c_int),
                ("weight_grid", ctypes.c_int), ("fc_lags", ctypes.c_int), ("force_path", ctypes.c_int),
                ("fused_train", ctypes.c_int)]


class _Info(ctypes.Structure):
    _fields_ = [("rho", ctypes.c_double), ("rmse", ctypes.c_double), ("rdiag_min_abs", ctypes.c_double),
                ("rdiag_max_abs", ctypes.c_double), ("ridge_lambda", ctypes.c_double), ("rank_flag", ctypes.c_int),
                ("n_total", ctypes.c_int64)]


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


_lib = None


def lib() -> ctypes.CDLL:
    """Load libelmrnn.so (build it first with paper_1911_13252_b200.build)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built: run `python -m paper_1911_13252_b200.build`")
        L = ctypes.CDLL(LIB_PATH)
        vp, i64, i32, u64 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_uint64
        L.elmrnn_opts_default.argtypes = [vp]
        L.elmrnn_opts_default.restype = None
        L.elmrnn_init.argtypes = [vp, i32, i32, i32, i32, u64]
        L.elmrnn_init_ex.argtypes = [vp, i32, i32, i32, i32, u64, vp]
        L.elmrnn_set_stream.argtypes = [vp, vp]
        L.elmrnn_build_H.argtypes = [vp, vp, i64, vp, i64, i64, vp, i64]
        L.elmrnn_build_H_ef.argtypes = [vp, vp, i64, vp, i64, vp, i64, i64, vp, i64]
        L.elmrnn_error_windows.argtypes = [vp, vp, i64, vp, i64, vp, vp, i64]
        L.elmrnn_forecast.argtypes = [vp, vp, i64, i64, vp, i32, vp, i64]
        L.elmrnn_test_rmse.argtypes = [vp, vp, i64, vp, i64, vp, i64, vp, vp]
        L.elmrnn_solve_beta.argtypes = [vp, vp, i64, vp, i64, vp, vp]
        L.elmrnn_solve_beta_multi.argtypes = [vp, vp, i64, vp, i64, i32, i64, vp, vp, vp]
        L.elmrnn_solve_local.argtypes = [vp, vp, i64, vp, i64, vp]
        L.elmrnn_solve_merge.argtypes = [vp, vp, i32, i64, vp, vp]
        L.elmrnn_sync.argtypes = [vp]
        L.elmrnn_train.argtypes = [vp, vp, i64, vp, i64, vp, i64, vp, vp]
        L.elmrnn_train_local.argtypes = [vp, vp, i64, vp, i64, vp, i64, vp]
        L.elmrnn_train_fused.argtypes = [vp]
        L.elmrnn_solve_local_multi.argtypes = [vp, vp, i64, vp, i64, i32, i64, vp]
        L.elmrnn_solve_merge_multi.argtypes = [vp, vp, i32, i32, i64, vp, vp, vp]
        L.elmrnn_packed_r_len_multi.argtypes = [vp, i32]
        L.elmrnn_packed_r_len_multi.restype = i64
        L.elmrnn_packed_r_len.argtypes = [vp]
        L.elmrnn_packed_r_len.restype = i64
        L.elmrnn_predict.argtypes = [vp, vp, i64, vp, i64, i64, vp, vp]
        L.elmrnn_get_weights.argtypes = [vp, i32, vp, i64]
        L.elmrnn_weight_block_len.argtypes = [vp, i32]
        L.elmrnn_weight_block_len.restype = i64
        L.elmrnn_path.argtypes = [vp]
        L.elmrnn_launch_count.argtypes = [vp]
        L.elmrnn_launch_count.restype = i64
        L.elmrnn_last_error.argtypes = [vp]
        L.elmrnn_last_error.restype = ctypes.c_char_p
        L.elmrnn_destroy.argtypes = [vp]
        L.elmrnn_destroy.restype = None
        for f in ("elmrnn_init", "elmrnn_init_ex", "elmrnn_set_stream", "elmrnn_build_H", "elmrnn_build_H_ef",
                  "elmrnn_error_windows", "elmrnn_forecast", "elmrnn_test_rmse", "elmrnn_solve_beta",
                  "elmrnn_solve_beta_multi",
                  "elmrnn_solve_local", "elmrnn_solve_merge", "elmrnn_sync", "elmrnn_predict", "elmrnn_get_weights",
                  "elmrnn_solve_local_multi", "elmrnn_solve_merge_multi", "elmrnn_train", "elmrnn_train_local",
                  "elmrnn_train_fused",
                  "elmrnn_path"):
            getattr(L, f).restype = i32
        _lib = L
    return _lib


def _ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


def _dev_check(t: torch.Tensor, name: str, dtype: torch.dtype):
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor (no CPU path)")
    if t.dtype != dtype:
        raise ValueError(f"{name} must be {dtype}")


def _vec(t: torch.Tensor, name: str, dtype: torch.dtype, n: int):
    """A contiguous CUDA vector of at least n elements (the library reads/writes n)."""
    _dev_check(t, name, dtype)
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    if t.numel() < n:
        raise ValueError(f"{name} has {t.numel()} elements, needs >= {n}")


def _need_rows(rows: int, N: int, name: str):
    if rows < N:
        raise ValueError(f"{name} has {rows} rows, needs >= {N}")


def _rows(t: torch.Tensor, name: str):
    """(leading dimension, rows) of a 2-D view with unit inner stride."""
    t2 = t.reshape(t.shape[0], -1) if t.dim() != 2 else t
    if t2.dim() != 2 or t2.stride(1) != 1:
        raise ValueError(f"{name} must have unit inner stride")
    return t2.stride(0) if t2.shape[0] > 1 else t2.shape[1], t2.shape[0]


class ELMRNN:
    """Handle of one ELM-RNN (fixed random weights) on the current CUDA device.

    ELMRNN(arch, d, M, Q, seed, F=-1, R=-1, act=0, rec_scale=0, weight_grid=0,
    fc_lags=-1, force_path=0, fused_train=0) -- elmrnn_init_ex."""

    def __init__(self, arch, d: int, M: int, Q: int, seed: int = 1, **opts):
        L = lib()
        o = Opts()
        L.elmrnn_opts_default(ctypes.byref(o))
        for k, v in opts.items():
            if not hasattr(o, k):
                raise TypeError(f"unknown option {k}")
            setattr(o, k, int(v))
        self.arch = arch if isinstance(arch, str) else [k for k, v in ARCHS.items() if v == arch][0]
        self.d, self.M, self.Q = d, M, Q
        self.opts = {f: getattr(o, f) for f, _ in Opts._fields_}
        h = ctypes.c_void_p()
        st = L.elmrnn_init_ex(ctypes.byref(h), ARCHS[self.arch], d, M, Q, ctypes.c_uint64(seed & (2**64 - 1)),
                              ctypes.byref(o))
        if st != 0:
            raise ElmrnnError(st, L.elmrnn_last_error(None).decode())
        self._h = h

    # -- plumbing
    def _check(self, st: int) -> int:
        if st < 0:
            raise ElmrnnError(st, lib().elmrnn_last_error(self._h).decode())
        return st

    def _stream(self):
        lib().elmrnn_set_stream(self._h, ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))

    def close(self):
        if getattr(self, "_h", None):
            lib().elmrnn_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:   # interpreter shutdown: module globals may already be gone
            pass

    def sync(self) -> None:
        """elmrnn_sync: wait for the handle's stream; raises ERR_NONFINITE when an
        asynchronous solve since the last check met NaN/Inf."""
        self._check(lib().elmrnn_sync(self._h))

    @property
    def path(self) -> int:
        return lib().elmrnn_path(self._h)

    @property
    def launch_count(self) -> int:
        return lib().elmrnn_launch_count(self._h)

    @property
    def packed_r_len(self) -> int:
        return lib().elmrnn_packed_r_len(self._h)

    # -- API
    def build_H(self, X: torch.Tensor, Yfb: torch.Tensor | None = None, H: torch.Tensor | None = None,
                Ef: torch.Tensor | None = None):
        """elmrnn_build_H (elmrnn_build_H_ef when a NARMAX error window Ef [N][Q] is
        given): X [N][Q][d] (or [N][ldx]) fp32 CUDA -> H [N][M] fp32."""
        _dev_check(X, "X", torch.float32)
        N = X.shape[0]
        ldx, _ = _rows(X, "X") if N else (self.Q * self.d, 0)
        ldy = 0
        if Yfb is not None:
            _dev_check(Yfb, "Yfb", torch.float32)
            ldy, ry = _rows(Yfb, "Yfb")
            _need_rows(ry, N, "Yfb")
        if H is None:
            H = torch.empty((N, self.M), dtype=torch.float32, device=X.device)
        _dev_check(H, "H", torch.float32)
        ldh, rh = _rows(H, "H") if N else (self.M, 0)
        _need_rows(rh, N, "H")
        if N and H.shape[-1] < self.M:
            raise ValueError(f"H needs >= {self.M} columns")
        self._stream()
        if Ef is None:
            self._check(lib().elmrnn_build_H(self._h, _ptr(X), ldx, _ptr(Yfb), ldy, N, _ptr(H), ldh))
        else:
            _dev_check(Ef, "Ef", torch.float32)
            lde, re_ = _rows(Ef, "Ef") if N else (self.Q, 0)
            _need_rows(re_, N, "Ef")
            self._check(lib().elmrnn_build_H_ef(self._h, _ptr(X), ldx, _ptr(Yfb), ldy, _ptr(Ef), lde, N,
                                                _ptr(H), ldh))
        return H

    def error_windows(self, H: torch.Tensor, Y: torch.Tensor, beta: torch.Tensor, Ef: torch.Tensor | None = None):
        """elmrnn_error_windows: NARMAX error window Ef [N][Q] fp32 from the
        residuals Y - H beta of consecutive windows (reading R30)."""
        _dev_check(H, "H", torch.float32)
        N = H.shape[0]
        _vec(Y, "Y", torch.float32, N)
        _vec(beta, "beta", torch.float64, self.M)
        if Ef is None:
            Ef = torch.empty((N, self.Q), dtype=torch.float32, device=H.device)
        _dev_check(Ef, "Ef", torch.float32)
        ldh = _rows(H, "H")[0] if N else self.M
        lde, re_ = _rows(Ef, "Ef") if N else (self.Q, 0)
        _need_rows(re_, N, "Ef")
        self._stream()
        self._check(lib().elmrnn_error_windows(self._h, _ptr(H), ldh, _ptr(Y), N, _ptr(beta), _ptr(Ef), lde))
        return Ef

    def build_H_from_host(self, Xh: torch.Tensor, Xd: torch.Tensor, H: torch.Tensor, chunks: int = 8,
                          copy_stream: torch.cuda.Stream | None = None):
        """elmrnn_build_H over row chunks of a pinned host X: the host->device copy
        of chunk k+1 (on `copy_stream`) overlaps the build of chunk k (current
        stream).  Rows are independent (every sample's window runs on its own),
        so this is only copy scheduling; Xd is the device staging buffer."""
        N = Xh.shape[0]
        cs = copy_stream or torch.cuda.Stream()
        cur = torch.cuda.current_stream()
        cs.wait_stream(cur)   # Xd / H may still be in use by earlier work on this stream
        cuts = [N * k // chunks for k in range(chunks + 1)]
        for a, b in zip(cuts[:-1], cuts[1:]):
            if b <= a:
                continue
            with torch.cuda.stream(cs):
                Xd[a:b].copy_(Xh[a:b], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(cs)
            cur.wait_event(ev)
            self.build_H(Xd[a:b], None, H[a:b])
        return H

    def solve_beta(self, H: torch.Tensor, Y: torch.Tensor, beta: torch.Tensor | None = None, info: bool = True):
        """elmrnn_solve_beta -> (beta fp64 [M], SolveInfo or None)."""
        _dev_check(H, "H", torch.float32)
        N = H.shape[0]
        _vec(Y, "Y", torch.float32, N)
        ldh, _ = _rows(H, "H")
        if beta is None:
            beta = torch.empty(self.M, dtype=torch.float64, device=H.device)
        _vec(beta, "beta", torch.float64, self.M)
        self._stream()
        inf = _Info()
        st = self._check(lib().elmrnn_solve_beta(self._h, _ptr(H), ldh, _ptr(Y), N, _ptr(beta),
                                                 ctypes.byref(inf) if info else None))
        return beta, (self._info(inf, st) if info else None)

    def solve_beta_multi(self, H: torch.Tensor, Y: torch.Tensor):
        """elmrnn_solve_beta_multi: Y [N][P] -> (B fp64 [P][M], rmse list [P], SolveInfo of output 0)."""
        _dev_check(H, "H", torch.float32)
        _dev_check(Y, "Y", torch.float32)
        N = H.shape[0]
        if Y.shape[0] != N:
            raise ValueError(f"Y has {Y.shape[0]} rows, needs {N}")
        Y2 = Y.reshape(N, -1)
        P = Y2.shape[1]
        ldh, _ = _rows(H, "H")
        ldy = Y2.stride(0) if N > 1 else P
        if Y2.stride(1) != 1:
            raise ValueError("Y must have unit inner stride")
        B = torch.empty((P, self.M), dtype=torch.float64, device=H.device)
        rm = (ctypes.c_double * P)()
        inf = _Info()
        self._stream()
        st = self._check(lib().elmrnn_solve_beta_multi(self._h, _ptr(H), ldh, _ptr(Y2), ldy, P, N, _ptr(B), rm,
                                                       ctypes.byref(inf)))
        return B, list(rm), self._info(inf, st)

    def solve_local(self, H: torch.Tensor, Y: torch.Tensor, Rpk: torch.Tensor | None = None):
        """elmrnn_solve_local -> packed R fp64 [(M+1)(M+2)/2]."""
        _dev_check(H, "H", torch.float32)
        N = H.shape[0]
        _vec(Y, "Y", torch.float32, N)
        ldh = _rows(H, "H")[0] if N else self.M
        if Rpk is None:
            Rpk = torch.empty(self.packed_r_len, dtype=torch.float64, device=H.device)
        _vec(Rpk, "Rpk", torch.float64, self.packed_r_len)
        self._stream()
        self._check(lib().elmrnn_solve_local(self._h, _ptr(H), ldh, _ptr(Y), N, _ptr(Rpk)))
        return Rpk

    def packed_r_len_multi(self, P: int) -> int:
        return lib().elmrnn_packed_r_len_multi(self._h, P)

    def solve_local_multi(self, H: torch.Tensor, Y: torch.Tensor, Rpk: torch.Tensor | None = None):
        """elmrnn_solve_local_multi: Y [N][P] -> packed R fp64 [(M+P)(M+P+1)/2]."""
        _dev_check(H, "H", torch.float32)
        _dev_check(Y, "Y", torch.float32)
        N = H.shape[0]
        if Y.shape[0] != N:
            raise ValueError(f"Y has {Y.shape[0]} rows, needs {N}")
        Y2 = Y.reshape(N, -1)
        P = Y2.shape[1]
        if N and Y2.stride(1) != 1:
            raise ValueError("Y must have unit inner stride")
        ldy = Y2.stride(0) if N > 1 else P
        ldh = _rows(H, "H")[0] if N else self.M
        L = self.packed_r_len_multi(P)
        if Rpk is None:
            Rpk = torch.empty(L, dtype=torch.float64, device=H.device)
        _vec(Rpk, "Rpk", torch.float64, L)
        self._stream()
        self._check(lib().elmrnn_solve_local_multi(self._h, _ptr(H), ldh, _ptr(Y2), ldy, P, N, _ptr(Rpk)))
        return Rpk

    def solve_merge_multi(self, Rpk_all: torch.Tensor, ranks: int, P: int, N_total: int, B: torch.Tensor | None = None,
                          info: bool = True):
        """elmrnn_solve_merge_multi -> (B fp64 [P][M], rmse list [P] or None, SolveInfo or None)."""
        _vec(Rpk_all, "Rpk_all", torch.float64, ranks * self.packed_r_len_multi(P))
        if B is None:
            B = torch.empty((P, self.M), dtype=torch.float64, device=Rpk_all.device)
        _vec(B, "B", torch.float64, P * self.M)
        self._stream()
        rm = (ctypes.c_double * P)()
        inf = _Info()
        st = self._check(lib().elmrnn_solve_merge_multi(self._h, _ptr(Rpk_all), ranks, P, N_total, _ptr(B),
                                                        rm if info else None, ctypes.byref(inf) if info else None))
        return B, (list(rm) if info else None), (self._info(inf, st) if info else None)

    def solve_merge(self, Rpk_all: torch.Tensor, P: int, N_total: int, beta: torch.Tensor | None = None,
                    info: bool = True):
        """elmrnn_solve_merge on P stacked packed R factors."""
        _vec(Rpk_all, "Rpk_all", torch.float64, P * self.packed_r_len)
        if beta is None:
            beta = torch.empty(self.M, dtype=torch.float64, device=Rpk_all.device)
        _vec(beta, "beta", torch.float64, self.M)
        self._stream()
        inf = _Info()
        st = self._check(lib().elmrnn_solve_merge(self._h, _ptr(Rpk_all), P, N_total, _ptr(beta),
                                                  ctypes.byref(inf) if info else None))
        return beta, (self._info(inf, st) if info else None)

    def predict(self, X: torch.Tensor, beta: torch.Tensor, Yfb: torch.Tensor | None = None):
        """elmrnn_predict -> Yhat fp32 [N]."""
        _dev_check(X, "X", torch.float32)
        _vec(beta, "beta", torch.float64, self.M)
        N = X.shape[0]
        ldx = _rows(X, "X")[0] if N else self.Q * self.d
        ldy = 0
        if Yfb is not None:
            _dev_check(Yfb, "Yfb", torch.float32)
            ldy, ry = _rows(Yfb, "Yfb")
            _need_rows(ry, N, "Yfb")
        out = torch.empty(N, dtype=torch.float32, device=X.device)
        self._stream()
        self._check(lib().elmrnn_predict(self._h, _ptr(X), ldx, _ptr(Yfb), ldy, N, _ptr(beta), _ptr(out)))
        return out

    def forecast(self, X: torch.Tensor, beta: torch.Tensor, K: int):
        """elmrnn_forecast: free-running K-step forecast of univariate windows -> fp32 [N][K]."""
        _dev_check(X, "X", torch.float32)
        _vec(beta, "beta", torch.float64, self.M)
        N = X.shape[0]
        ldx = _rows(X, "X")[0] if N else self.Q
        out = torch.empty((N, K), dtype=torch.float32, device=X.device)
        self._stream()
        self._check(lib().elmrnn_forecast(self._h, _ptr(X), ldx, N, _ptr(beta), K, _ptr(out), max(K, 1)))
        return out

    def test_rmse(self, X: torch.Tensor, Y: torch.Tensor, beta: torch.Tensor, Yfb: torch.Tensor | None = None) -> float:
        """elmrnn_test_rmse: held-out RMSE of beta on evaluation windows."""
        _dev_check(X, "X", torch.float32)
        N = X.shape[0]
        _vec(Y, "Y", torch.float32, N)
        _vec(beta, "beta", torch.float64, self.M)
        ldx = _rows(X, "X")[0] if N else self.Q * self.d
        ldy = 0
        if Yfb is not None:
            _dev_check(Yfb, "Yfb", torch.float32)
            ldy, ry = _rows(Yfb, "Yfb")
            _need_rows(ry, N, "Yfb")
        r = ctypes.c_double()
        self._stream()
        self._check(lib().elmrnn_test_rmse(self._h, _ptr(X), ldx, _ptr(Yfb), ldy, _ptr(Y), N, _ptr(beta),
                                           ctypes.byref(r)))
        return r.value

    def get_weights(self, block_id: int):
        """elmrnn_get_weights: logical weight block as a flat float32 CPU tensor."""
        n = lib().elmrnn_weight_block_len(self._h, block_id)
        if n < 0:
            raise ValueError("block id out of range")
        out = torch.empty(n, dtype=torch.float32)
        self._stream()
        self._check(lib().elmrnn_get_weights(self._h, block_id, out.data_ptr(), n))
        return out

    @property
    def train_fused(self) -> bool:
        return bool(lib().elmrnn_train_fused(self._h))

    def train_direct(self, X: torch.Tensor, Y: torch.Tensor, Yfb: torch.Tensor | None = None,
                     beta: torch.Tensor | None = None, info: bool = True):
        """elmrnn_train: beta (and SolveInfo) straight from the windows, without
        returning H (fused build -> TSQR leaf where supported)."""
        _dev_check(X, "X", torch.float32)
        N = X.shape[0]
        _vec(Y, "Y", torch.float32, N)
        ldx = _rows(X, "X")[0] if N else self.Q * self.d
        ldy = 0
        if Yfb is not None:
            _dev_check(Yfb, "Yfb", torch.float32)
            ldy, ry = _rows(Yfb, "Yfb")
            _need_rows(ry, N, "Yfb")
        if beta is None:
            beta = torch.empty(self.M, dtype=torch.float64, device=X.device)
        _vec(beta, "beta", torch.float64, self.M)
        self._stream()
        inf = _Info()
        st = self._check(lib().elmrnn_train(self._h, _ptr(X), ldx, _ptr(Yfb), ldy, _ptr(Y), N, _ptr(beta),
                                            ctypes.byref(inf) if info else None))
        return beta, (self._info(inf, st) if info else None)

    def train_local(self, X: torch.Tensor, Y: torch.Tensor, Yfb: torch.Tensor | None = None,
                    Rpk: torch.Tensor | None = None):
        """elmrnn_train_local: this shard's packed R of [H | Y] straight from its windows."""
        _dev_check(X, "X", torch.float32)
        N = X.shape[0]
        _vec(Y, "Y", torch.float32, N)
        ldx = _rows(X, "X")[0] if N else self.Q * self.d
        ldy = 0
        if Yfb is not None:
            _dev_check(Yfb, "Yfb", torch.float32)
            ldy, ry = _rows(Yfb, "Yfb")
            _need_rows(ry, N, "Yfb")
        if Rpk is None:
            Rpk = torch.empty(self.packed_r_len, dtype=torch.float64, device=X.device)
        _vec(Rpk, "Rpk", torch.float64, self.packed_r_len)
        self._stream()
        self._check(lib().elmrnn_train_local(self._h, _ptr(X), ldx, _ptr(Yfb), ldy, _ptr(Y), N, _ptr(Rpk)))
        return Rpk

    def train(self, X, Y, Yfb=None):
        """Alg. 1 lines 2-3: H(Q) then beta."""
        H = self.build_H(X, Yfb)
        beta, info = self.solve_beta(H, Y)
        return H, beta, info

    def train_narmax_ef(self, X, Y, Yfb=None):
        """NARMAX with real error feedback (reading R30): pass 0
        with e == 0, e = y - yhat(beta0) as error windows, pass 1 rebuilds H with
        them and re-solves.  Returns (H1, beta1, info1, beta0, info0)."""
        if self.arch != "narmax":
            raise ValueError("error feedback is a NARMAX method")
        H0, b0, i0 = self.train(X, Y, Yfb)
        Ef = self.error_windows(H0, Y, b0)
        H1 = self.build_H(X, Yfb, H0, Ef=Ef)
        b1, i1 = self.solve_beta(H1, Y)
        return H1, b1, i1, b0, i0

    @staticmethod
    def _info(i: _Info, st: int) -> SolveInfo:
        return SolveInfo(i.rho, i.rmse, i.rdiag_min_abs, i.rdiag_max_abs, i.ridge_lambda, i.rank_flag, i.n_total, st)
