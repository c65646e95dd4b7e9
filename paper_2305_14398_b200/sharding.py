"""Row-block sharding of the accumulated unitary over G GPUs.

Rank r owns rows [r*B, r*B + B) of U = L_last ... L_first. It computes
V = L_last[rows, :] and then V <- V * L for every further layer, regenerating
each operator tile locally from the replicated descriptor — no communication
during the chain. The only exchange is the final all-gather of the psi row
slices (16 * B bytes per rank): ``dist.all_gather_into_tensor`` over NCCL on
GPUs, and the very same call over gloo in the CPU tests. (The C ABI has its own
NCCL all-gather for C++ hosts and the in-process multi-device handle:
qsb_plan_allgather_state / qsb_simulate_full_state with n_devices > 1.)
"""
from __future__ import annotations

from typing import Tuple


def block_rows(N: int, world: int) -> int:
    """Rows per rank: N / world for power-of-two worlds, else the next power of
    two >= ceil(N / world) (trailing ranks then own no rows)."""
    if world < 1:
        raise ValueError("world size must be >= 1")
    b = -(-N // world)
    p = 1
    while p < b:
        p <<= 1
    return min(p, N)


def row_shard(N: int, world: int, rank: int) -> Tuple[int, int]:
    """(row_begin, row_count) of `rank`; row_count may be 0."""
    b = block_rows(N, world)
    begin = min(rank * b, N)
    return begin, max(0, min(b, N - begin))


def gather_rows(local_re, local_im, N: int, world: int):
    """All-gather equal row blocks (padded to block_rows) into full psi planes.
    One code path for every backend: each rank contributes a flat [re | im]
    buffer of 2 * block_rows doubles, gathered rank-major into one flat tensor
    (CUDA tensors over NCCL, CPU tensors over gloo)."""
    import torch
    import torch.distributed as dist

    b = block_rows(N, world)
    local = torch.zeros(2 * b, dtype=local_re.dtype, device=local_re.device)
    n = local_re.numel()
    if n:
        local[:n].copy_(local_re)
        local[b:b + n].copy_(local_im)
    out = torch.empty(world * 2 * b, dtype=local.dtype, device=local.device)
    dist.all_gather_into_tensor(out, local)
    full = out.view(world, 2, b).permute(1, 0, 2).reshape(2, world * b)[:, :N]
    return full[0], full[1]


def gather_state(plan, psi_re, psi_im, begin: int, count: int, world: int, stream: int = 0) -> None:
    """Fill psi_re/psi_im (length N, CUDA) with the full state: the local plan's
    rows, all-gathered across ranks when world > 1. Row-block plans only: a
    column-block plan's state is a full-length share that must be summed."""
    import torch

    if plan is not None and getattr(plan, "columns", False):
        raise ValueError("gather_state needs row-block plans; column-block shares are summed, not gathered")
    N = psi_re.numel()
    if world == 1:
        plan.copy_state(psi_re.data_ptr(), psi_im.data_ptr(), stream)
        return
    lr = torch.empty(count, dtype=torch.float64, device=psi_re.device)
    li = torch.empty(count, dtype=torch.float64, device=psi_re.device)
    if plan is not None and count:
        plan.copy_state(lr.data_ptr(), li.data_ptr(), stream)
    re, im = gather_rows(lr, li, N, world)
    psi_re.copy_(re)
    psi_im.copy_(im)
