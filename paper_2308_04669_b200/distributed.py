"""Image-tile partitioning across GPUs.

Every step is per-pixel independent given replicated weights, so the frame is
split by camera rows: row y belongs to rank y % world (a 1-row interleave).
Adjacent rows cross the same objects at almost the same places, so every rank
gets an equal share of the STEP 1 (pixel, object) box hits and of the STEP 3
shadow rays wherever the objects fall on screen; `partition_balance` measures
it.  Each rank renders its rows with the same scene and replicated models; the
only exchange is one collective per frame: the colour / depth / id rows packed
into one byte tile per rank and gathered to rank 0 (NCCL over NVLink on GPUs,
gloo in the CPU tests), where one transpose puts the rows back in camera order.
"""

from __future__ import annotations

import numpy as np


def interleave_rows(height: int, rank: int, world: int, stripe: int = 1) -> np.ndarray:
    """Camera rows owned by `rank`: stripes of `stripe` rows, stripe k to rank k % world."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    if stripe < 1 or height < 0:
        raise ValueError("bad stripe/height")
    y = np.arange(height)
    return np.asarray(y[(y // stripe) % world == rank], dtype=np.int32)


def max_rows(height: int, world: int, stripe: int = 1) -> int:
    return max(len(interleave_rows(height, r, world, stripe)) for r in range(world))


def partition_balance(work_per_row, world: int, stripe: int = 1) -> float:
    """max over ranks / mean over ranks of the per-row work (e.g. box hits per row)."""
    w = np.asarray(work_per_row, dtype=np.float64)
    per = np.array([w[interleave_rows(len(w), r, world, stripe)].sum() for r in range(world)])
    return float(per.max() / per.mean()) if per.mean() > 0 else 1.0


def _tile_layout(tile: dict, mr: int):
    """(name, dtype, per-row shape, bytes per row) for each buffer, in a fixed order."""
    out = []
    for name in sorted(tile):
        t = tile[name]
        row_shape = tuple(t.shape[1:])
        n = int(np.prod(row_shape)) if row_shape else 1
        out.append((name, t.dtype, row_shape, n * t.element_size()))
    return out


def pack_tile(tile: dict, mr: int):
    """One contiguous byte tile per rank: each buffer's rows (padded to `mr` rows)
    one after another: [name0: mr x bytes0][name1: mr x bytes1]..."""
    import torch
    layout = _tile_layout(tile, mr)
    dev = tile[layout[0][0]].device
    total = sum(mr * b for _, _, _, b in layout)
    packed = torch.empty(total, dtype=torch.uint8, device=dev)
    off = 0
    for name, _, _, b in layout:
        t = tile[name].contiguous()
        rows = t.shape[0]
        if rows:
            packed[off:off + rows * b].copy_(t.reshape(-1).view(torch.uint8))
        if rows < mr:
            packed[off + rows * b:off + mr * b].zero_()
        off += mr * b
    return packed, layout


def unpack_gathered(gathered, layout, mr: int, height: int, world: int, stripe: int = 1) -> dict:
    """Inverse of pack_tile over all ranks (gathered: (world, tile bytes)): full
    frames with rows in camera order.  For a 1-row interleave row y = i * world + r
    is local row i of rank r, so camera order is one transpose of (rank, row)."""
    import torch
    out = {}
    off = 0
    for name, dtype, row_shape, b in layout:
        part = gathered[:, off:off + mr * b].reshape(world, mr, b)
        off += mr * b
        if stripe == 1:
            rows = part.transpose(0, 1).reshape(world * mr, b)[:height]
        else:
            order = np.empty(height, dtype=np.int64)
            for r in range(world):
                ys = interleave_rows(height, r, world, stripe)
                order[ys] = r * mr + np.arange(len(ys))
            rows = part.reshape(world * mr, b).index_select(
                0, torch.as_tensor(order, device=gathered.device))
        out[name] = rows.contiguous().view(dtype).reshape((height,) + row_shape)
    return out


def gather_tiles(tile: dict, height: int, width: int, rank: int, world: int, group=None,
                 stripe: int = 1, dst: int = 0):
    """Gather per-rank row tiles {name: tensor (n_rows, width, ...)} into full
    frames on `dst` (returns the dict there, None elsewhere).  One collective per
    frame: a gather of one packed byte tile per rank to `dst` (NCCL implements it
    as grouped point-to-point sends, so only `dst` receives: (world - 1) tiles,
    not world^2 as an all-gather would move).  A rank may own no rows."""
    import torch
    import torch.distributed as dist
    del width
    mr = max(1, max_rows(height, world, stripe))
    packed, layout = pack_tile(tile, mr)
    if rank == dst:
        gathered = torch.empty((world, packed.numel()), dtype=torch.uint8, device=packed.device)
        dist.gather(packed, gather_list=list(gathered.unbind(0)), dst=dst, group=group)
        return unpack_gathered(gathered, layout, mr, height, world, stripe)
    dist.gather(packed, gather_list=None, dst=dst, group=group)
    return None

