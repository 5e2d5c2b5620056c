"""Row-sharded multi-GPU driver (one process per GPU, torch.distributed).

The ELM solve shards naturally over samples (rows of H): each rank builds its
own H block and factors [H | Y] into an (M+1)x(M+1) R (elmrnn_solve_local);
the only exchange is an all-gather of the packed R factors (265 KB per rank at
M = 256) over NCCL / NVLink, then a final small QR of their stack
(elmrnn_solve_merge) -- on every rank by default (identical bits, no broadcast),
or on a root rank followed by a broadcast of beta, the north-star decomposition
(SURVEY 8(e)).  Householder QR of stacked R factors equals the QR of the
stacked rows (tests/test_oracle_weights_solve.py::test_tsqr_tree_equals_direct_R).

The functions are written against a tiny interface (build_H / solve_local /
solve_merge / packed_r_len / M) so the collective plumbing can be exercised on
CPU with the gloo backend in tests; the product passes an ELMRNN handle.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard_rows(N_total: int, world: int, rank: int):
    """Contiguous, balanced row range [lo, hi) of rank (depends only on N_total, world)."""
    return N_total * rank // world, N_total * (rank + 1) // world


def _all_gather_rows(Rpk: torch.Tensor, group=None) -> torch.Tensor:
    world = dist.get_world_size(group)
    out = torch.empty((world, Rpk.numel()), dtype=Rpk.dtype, device=Rpk.device)
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(out, Rpk.contiguous(), group=group)
    else:
        dist.all_gather(list(out.unbind(0)), Rpk.contiguous(), group=group)
    return out


def solve_sharded(model, H: torch.Tensor, Y: torch.Tensor, N_total: int, beta: torch.Tensor | None = None,
                  group=None, root: int | None = None, info: bool = False):
    """beta for the row-sharded [H | Y]: local TSQR, all-gather of the packed R factors,
    merge + solve.  Y [N] (one output) or [N][P] (P outputs, SURVEY 8(f) row 3,
    P:655; beta then [P][M]).

    root=None (default): EVERY rank merges the identical all-gathered factors with
    the same deterministic kernels, so all ranks hold bitwise-identical beta and
    no broadcast is needed (SURVEY 8(e) alternative; the merge is ~1 ms).
    root=r: merge on rank r only, then broadcast beta (the north-star form)."""
    multi = Y.dim() == 2 and Y.shape[1] > 1
    P = Y.shape[1] if multi else 1
    Rpk = model.solve_local_multi(H, Y) if multi else model.solve_local(H, Y.reshape(-1))
    Rall = _all_gather_rows(Rpk, group)
    rank = dist.get_rank(group)
    if beta is None:
        beta = torch.empty((P, model.M) if multi else (model.M,), dtype=torch.float64, device=H.device)
    sinfo = None
    if root is None or rank == root:
        if multi:
            _, rm, sinfo = model.solve_merge_multi(Rall, Rall.shape[0], P, N_total, beta, info=info)
            if sinfo is not None:
                sinfo.rmse_all = rm
        else:
            _, sinfo = model.solve_merge(Rall, Rall.shape[0], N_total, beta, info=info)
    if root is not None:
        dist.broadcast(beta, src=root, group=group)
    return beta, sinfo


def train_sharded(model, X_local: torch.Tensor, Y_local: torch.Tensor, N_total: int, Yfb_local=None, group=None,
                  root: int | None = None, info: bool = True):
    """Alg. 1 on this rank's rows: H(Q) block, then the sharded solve."""
    H = model.build_H(X_local, Yfb_local)
    beta, sinfo = solve_sharded(model, H, Y_local, N_total, group=group, root=root, info=info)
    return H, beta, sinfo
