"""Multi-GPU plumbing: one process per GPU, torch.distributed
process groups (NCCL over NVLink/NVSwitch on the GPU box, gloo in CPU tests).

Two data-parallel strategies, both with the paper's per-column independence
(K̂V for a batch of directions touches no other column):
  * scenario sharding — independent load scenarios per rank, no collective
    on the hot path (config 5);
  * direction sharding — rank r owns columns [r·c, min((r+1)c, n_u)),
    c = ⌈n_u / world⌉ rounded up to the handle's direction-tile width (so
    every rank's first column starts a canonical tile and its forward sweep
    keeps the sparse-RHS reach lists); network, point and LU are replicated (every rank
    refactorizes G_x, which avoids a factor broadcast) and ONE all-gather of
    equal-count column slabs assembles K̂ (configs 3–4).
"""
from __future__ import annotations


def column_partition(n_u: int, world: int, rank: int, align: int = 8):
    """(col0, ncols, c) of the rank's equal-count slab; the last may be short
    (or empty).  c is a multiple of `align` (the tile width of the handles)."""
    c = -(-n_u // world)
    c = -(-c // align) * align
    col0 = min(rank * c, n_u)
    return col0, max(0, min(c, n_u - col0)), c


def scenario_partition(n_total: int, world: int, rank: int):
    """(first, count) of the rank's contiguous scenario block."""
    per = -(-n_total // world)
    first = min(rank * per, n_total)
    return first, max(0, min(per, n_total - first))


def allgather_columns(KV_local, n_u: int, group=None):
    """All-gather the ranks' column slabs into K̂ (column-major, [S][n_u][n_u]).

    KV_local: [S][c][n_u] with c = ⌈n_u/world⌉ (rows past the rank's real
    columns are padding and are dropped).  One collective call per K̂."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    S, c, nu = KV_local.shape
    assert nu == n_u
    parts = [torch.empty_like(KV_local) for _ in range(world)]
    dist.all_gather(parts, KV_local.contiguous(), group=group)
    return assemble_columns(parts, n_u)


def assemble_columns(parts, n_u: int):
    """Concatenate the ranks' equal-count slabs [S][c][n_u] in rank order and
    drop the padding past column n_u (the all-gather's output layout)."""
    import torch
    return torch.cat(list(parts), dim=1)[:, :n_u, :].contiguous()
