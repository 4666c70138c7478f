"""Image-tile partitioning across GPUs.

Every step is per-pixel independent given replicated weights, so the frame is
split into 16-row stripes dealt round-robin to the ranks (interleaving evens
out where the objects fall on screen).  Each rank renders its rows with the
same scene and replicated models; the only exchange is one gather of the
colour / depth / id tiles to rank 0 (NCCL over NVLink on GPUs, gloo in the
CPU tests).
"""

from __future__ import annotations

import numpy as np

STRIPE = 16


def stripe_rows(height: int, rank: int, world: int, stripe: int = STRIPE) -> np.ndarray:
    """Camera rows owned by `rank`: stripes k with k % world == rank."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    rows = [r for r in range(height) if (r // stripe) % world == rank]
    return np.asarray(rows, dtype=np.int32)


def max_rows(height: int, world: int, stripe: int = STRIPE) -> int:
    return max(len(stripe_rows(height, r, world, stripe)) for r in range(world))


def gather_tiles(tile: dict, height: int, width: int, rank: int, world: int, group=None,
                 stripe: int = STRIPE, dst: int = 0):
    """Gather per-rank row tiles {name: tensor (n_rows, width, ...)} into full
    frames on `dst` (returns dict there, None elsewhere).  Tiles are padded to
    the largest rank's row count so one all_gather per buffer suffices."""
    import torch
    import torch.distributed as dist
    mr = max_rows(height, world, stripe)
    out = {} if rank == dst else None
    for name in sorted(tile):
        t = tile[name]
        pad_shape = (mr,) + tuple(t.shape[1:])
        buf = torch.zeros(pad_shape, dtype=t.dtype, device=t.device)
        buf[: t.shape[0]] = t
        parts = [torch.empty_like(buf) for _ in range(world)]
        dist.all_gather(parts, buf, group=group)
        if rank == dst:
            full = torch.empty((height,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
            for r in range(world):
                rows = torch.as_tensor(stripe_rows(height, r, world, stripe), dtype=torch.long, device=t.device)
                full[rows] = parts[r][: rows.numel()]
            out[name] = full
    return out
