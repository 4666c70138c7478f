"""Image-tile partitioning across GPUs.

Every step is per-pixel independent given replicated weights, so the frame is
split into 16-row stripes dealt round-robin to the ranks (interleaving evens
out where the objects fall on screen).  Each rank renders its rows with the
same scene and replicated models; the only exchange is one collective per
frame: the colour / depth / id tiles packed into one byte tile and
all-gathered (NCCL over NVLink on GPUs, gloo in the CPU tests).
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


_PERM = {}


def _row_permutation(height: int, world: int, stripe: int, mr: int, device):
    """perm[y] = position of camera row y in the all-gathered (world * mr)-row buffer (cached)."""
    import torch
    key = (height, world, stripe, mr, str(device))
    p = _PERM.get(key)
    if p is None:
        perm = np.empty(height, dtype=np.int64)
        for r in range(world):
            rows = stripe_rows(height, r, world, stripe)
            perm[rows] = r * mr + np.arange(len(rows))
        p = _PERM[key] = torch.as_tensor(perm, device=device)
    return p


def gather_tiles(tile: dict, height: int, width: int, rank: int, world: int, group=None,
                 stripe: int = STRIPE, dst: int = 0):
    """Gather per-rank row tiles {name: tensor (n_rows, width, ...)} into full
    frames on `dst` (returns dict there, None elsewhere).  One collective per
    frame: every buffer's rows are packed side by side as bytes into one
    (rows, bytes) tile, padded to the largest rank's row count, and
    all-gathered; `dst` then reorders the rows with one cached permutation."""
    import torch
    import torch.distributed as dist
    mr = max_rows(height, world, stripe)
    names = sorted(tile)
    dev = tile[names[0]].device
    widths = []
    for name in names:
        t = tile[name].contiguous()
        b = t.view(torch.uint8).reshape(t.shape[0], -1)
        widths.append(b.shape[1])
    packed = torch.zeros((mr, sum(widths)), dtype=torch.uint8, device=dev)
    off = 0
    for name, w in zip(names, widths):
        t = tile[name].contiguous()
        packed[: t.shape[0], off:off + w] = t.view(torch.uint8).reshape(t.shape[0], -1)
        off += w
    gathered = torch.empty((world * mr, packed.shape[1]), dtype=torch.uint8, device=dev)
    dist.all_gather_into_tensor(gathered, packed, group=group)
    if rank != dst:
        return None
    full = gathered.index_select(0, _row_permutation(height, world, stripe, mr, dev))
    out = {}
    off = 0
    for name, w in zip(names, widths):
        t = tile[name]
        out[name] = full[:, off:off + w].contiguous().view(t.dtype).reshape((height,) + tuple(t.shape[1:]))
        off += w
    return out
