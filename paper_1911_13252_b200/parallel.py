"""Row-sharded multi-GPU driver (one process per GPU, torch.distributed).

The ELM solve shards naturally over samples (rows of H): each rank builds its
own H block and factors [H | Y] into an (M+1)x(M+1) R (elmrnn_solve_local);
the only exchange is an all-gather of the packed R factors (265 KB per rank at
M = 256) over NCCL / NVLink, a final small QR of their stack on rank 0
(elmrnn_solve_merge) and a broadcast of beta -- the north-star decomposition
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
                  group=None, root: int = 0, info: bool = False):
    """beta for the row-sharded [H | Y]: local TSQR, all-gather R, merge on root, broadcast."""
    Rpk = model.solve_local(H, Y)
    Rall = _all_gather_rows(Rpk, group)
    rank = dist.get_rank(group)
    if beta is None:
        beta = torch.empty(model.M, dtype=torch.float64, device=H.device)
    sinfo = None
    if rank == root:
        _, sinfo = model.solve_merge(Rall, Rall.shape[0], N_total, beta, info=info)
    dist.broadcast(beta, src=root, group=group)
    return beta, sinfo


def train_sharded(model, X_local: torch.Tensor, Y_local: torch.Tensor, N_total: int, Yfb_local=None, group=None,
                  root: int = 0, info: bool = True):
    """Alg. 1 on this rank's rows: H(Q) block, then the sharded solve."""
    H = model.build_H(X_local, Yfb_local)
    beta, sinfo = solve_sharded(model, H, Y_local, N_total, group=group, root=root, info=info)
    return H, beta, sinfo
