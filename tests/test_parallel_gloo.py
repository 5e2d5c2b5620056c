"""World-size-2 gloo test of the row-sharded driver's host logic (CPU).

The CUDA solve is replaced by a CPU stand-in built on the oracle (tests may
use it); what is exercised is the product's sharding, all-gather of packed R
factors, merge on the root and broadcast of beta (paper_1911_13252_b200/parallel.py).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class CpuStandIn:
    """build_H / solve_local / solve_merge with the oracle (packed R layout of elmrnn.h)."""

    def __init__(self, arch, S, M, Q, seed):
        from oracle import oracle as orc
        self.orc, self.M = orc, M
        self.net = orc.Net(arch, S=S, M=M, Q=Q)
        self.blocks = orc.gen_weights(self.net, seed)

    @property
    def packed_r_len(self):
        return (self.M + 1) * (self.M + 2) // 2

    def build_H(self, X, Yfb=None):
        return torch.from_numpy(self.orc.build_H(self.net, self.blocks, X.numpy()))

    def solve_local(self, H, Y):
        n = self.M + 1
        R = np.zeros((n, n))
        if H.shape[0]:
            A = np.column_stack([H.numpy(), Y.numpy().astype(np.float64)])
            r = np.linalg.qr(A, mode="r")
            R[: r.shape[0]] = r
        return torch.from_numpy(np.concatenate([R[k, k:] for k in range(n)]))

    def packed_r_len_multi(self, P):
        return (self.M + P) * (self.M + P + 1) // 2

    def _local(self, H, Y2):
        n = self.M + Y2.shape[1]
        R = np.zeros((n, n))
        if H.shape[0]:
            r = np.linalg.qr(np.column_stack([H.numpy(), Y2.numpy().astype(np.float64)]), mode="r")
            R[: r.shape[0]] = r
        return torch.from_numpy(np.concatenate([R[k, k:] for k in range(n)]))

    def solve_local_multi(self, H, Y):
        return self._local(H, Y.reshape(H.shape[0], -1))

    def solve_merge_multi(self, Rall, ranks, P, N_total, B, info=True):
        n = self.M + P
        rows = []
        for p in range(ranks):
            R = np.zeros((n, n))
            off = 0
            for k in range(n):
                R[k, k:] = Rall[p, off: off + n - k].numpy()
                off += n - k
            rows.append(R)
        S = np.vstack(rows)
        Bo, infos = self.orc.lstsq_multi(S[:, :self.M], S[:, self.M:])
        B.copy_(torch.from_numpy(Bo))
        return B, [i.rho / np.sqrt(N_total) for i in infos], infos[0]

    def solve_merge(self, Rall, P, N_total, beta, info=True):
        n = self.M + 1
        rows = []
        for p in range(P):
            R = np.zeros((n, n))
            off = 0
            for k in range(n):
                R[k, k:] = Rall[p, off: off + n - k].numpy()
                off += n - k
            rows.append(R)
        S = np.vstack(rows)
        b, inf = self.orc.lstsq(S[:, :-1], S[:, -1])
        inf.rmse = inf.rho / np.sqrt(N_total)
        beta.copy_(torch.from_numpy(b))
        return beta, inf


def _worker(rank, world, port, out, root):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1911_13252_b200 import parallel as par
    from synth import series as sy
    N, Q, M = 900, 10, 12
    lo, hi = par.shard_rows(N, world, rank)
    X, Y, _ = sy.windows(sy.series("mg", N + Q), N, Q)
    model = CpuStandIn("gru", 1, M, Q, 3)
    H, beta, info = par.train_sharded(model, torch.from_numpy(X[lo:hi]), torch.from_numpy(Y[lo:hi]), N, root=root)
    out[rank] = beta.numpy().copy()
    if info is not None:
        out[f"rmse{rank}"] = info.rmse
    # two outputs (y(t+1), y(t+2)): the multi-output sharded solve
    s = sy.series("mg", N + Q + 1)
    Y2 = np.stack([s[Q:Q + N, 0], s[Q + 1:Q + 1 + N, 0]], axis=1).astype(np.float32)
    B, info2 = par.solve_sharded(model, H, torch.from_numpy(Y2[lo:hi]), N, root=root, info=True)
    out[f"B{rank}"] = B.numpy().copy()
    dist.destroy_process_group()


@pytest.mark.parametrize("root", [None, 0])
def test_sharded_solve_matches_single_process(root):
    """root=None: every rank merges (no broadcast); root=0: merge on rank 0 + broadcast.
    Either way both ranks hold identical bits equal to the single-process oracle solve,
    for one output and for two outputs (multi-output sharded path)."""
    from oracle import oracle as orc
    from synth import series as sy
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out, root), nprocs=world, join=True)
    N, Q, M = 900, 10, 12
    X, Y, _ = sy.windows(sy.series("mg", N + Q), N, Q)
    net = orc.Net("gru", S=1, M=M, Q=Q)
    H = orc.build_H(net, orc.gen_weights(net, 3), X)
    b, inf = orc.lstsq(H, Y)
    for r in range(world):
        np.testing.assert_allclose(out[r], b, rtol=1e-9, atol=1e-12)
    np.testing.assert_array_equal(out[0], out[1])       # identical bits on every rank
    assert out["rmse0"] == pytest.approx(inf.rmse, rel=1e-10)
    if root is None:
        assert out["rmse1"] == out["rmse0"]
    s = sy.series("mg", N + Q + 1)
    Y2 = np.stack([s[Q:Q + N, 0], s[Q + 1:Q + 1 + N, 0]], axis=1)
    Bo, _ = orc.lstsq_multi(H, Y2)
    for r in range(world):
        np.testing.assert_allclose(out[f"B{r}"], Bo, rtol=1e-9, atol=1e-12)
    np.testing.assert_array_equal(out["B0"], out["B1"])


def test_shard_rows_cover_exactly():
    from paper_1911_13252_b200 import parallel as par
    for N in (0, 1, 7, 1000, 4_000_000):
        for w in (1, 2, 3, 8):
            parts = [par.shard_rows(N, w, r) for r in range(w)]
            assert parts[0][0] == 0 and parts[-1][1] == N
            assert all(parts[i][1] == parts[i + 1][0] for i in range(w - 1))
