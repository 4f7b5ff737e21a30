"""Multi-GPU partition of the minor index j (SURVEY §8 e).

The n minors are independent, so rank r of P owns the contiguous block
j in [r n / P, (r+1) n / P) — in the reference layout out[j*n+i] that block is
contiguous rows, and the only collective is one all-gather of those rows
(NCCL over NVLink on the GPU box; gloo in the CPU tests).  lambda(A) is
recomputed on every rank (1/n of the work) instead of broadcast.  Each
(i, j) product depends only on (i, j, n), so the gathered matrix is
bit-identical for every P.
"""
from __future__ import annotations


def shard_range(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced block of minor indices owned by `rank`."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of {world}")
    return rank * n // world, (rank + 1) * n // world


def rows_per_rank(n: int, world: int) -> list[int]:
    return [shard_range(n, world, r)[1] - shard_range(n, world, r)[0]
            for r in range(world)]


def gather_rows(local_rows, n: int, world: int, dist_mod, group=None):
    """All-gathers every rank's (rows x n) block into the full n x n matrix.

    Uses all_gather_into_tensor when all blocks have the same height (n % P
    == 0, the benchmark case) and a padded all_gather otherwise.
    """
    import torch
    counts = rows_per_rank(n, world)
    if len(set(counts)) == 1:
        full = torch.empty((n, n), dtype=local_rows.dtype, device=local_rows.device)
        dist_mod.all_gather_into_tensor(full, local_rows.contiguous(), group=group)
        return full
    h = max(counts)
    pad = torch.zeros((h, n), dtype=local_rows.dtype, device=local_rows.device)
    pad[: local_rows.shape[0]] = local_rows
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist_mod.all_gather(parts, pad, group=group)
    return torch.cat([p[:c] for p, c in zip(parts, counts)], dim=0)
