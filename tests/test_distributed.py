"""Multi-GPU image-tile partition + gather to rank 0, exercised with gloo on
CPU (world sizes 2, 3 and 4, including ranks that own no rows), and the
partition's load balance on the config-4 headline scene."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2308_04669_b200 import configs as CF
from paper_2308_04669_b200 import distributed as D


def test_interleave_partitions_rows():
    for h in (0, 1, 3, 15, 16, 17, 800, 801):
        for world in (1, 2, 3, 4, 8):
            for stripe in (1, 4, 16):
                parts = [D.interleave_rows(h, r, world, stripe) for r in range(world)]
                allr = np.sort(np.concatenate(parts))
                np.testing.assert_array_equal(allr, np.arange(h))
                assert max(len(p) for p in parts) == D.max_rows(h, world, stripe)
    with pytest.raises(ValueError):
        D.interleave_rows(10, 2, 2)
    with pytest.raises(ValueError):
        D.interleave_rows(10, 0, 2, stripe=0)


def test_config4_partition_balance():
    """every rank gets an equal share of the STEP 1 (pixel, object)
    box hits -- the network work -- on the headline scene at N = 2, 4, 8 (counted
    with the oracle's slab clip over all 1.6M camera rays)."""
    from oracle import nedf_oracle as O
    from tests.helpers import oracle_scene
    spec = CF.config4()
    objs, cam, _, _ = oracle_scene(spec)
    o, d = O.primary_rays(cam)
    hits = np.zeros(cam.width * cam.height)
    for ob in objs:
        lo = ((o - ob.T) @ ob.R) / ob.s
        ld = d @ ob.R
        _, _, hit = O.slab_clip(lo, ld, ob.model.box_min, ob.model.box_max)
        hits += hit
    per_row = hits.reshape(cam.height, cam.width).sum(axis=1)
    for world in (2, 4, 8):
        bal = D.partition_balance(per_row, world)
        assert bal <= 1.03, (world, bal)
    # the round-1 16-row stripes were worse: the interleave is the better split
    assert D.partition_balance(per_row, 8, stripe=16) > D.partition_balance(per_row, 8)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, h, w, stripe, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rows = D.interleave_rows(h, rank, world, stripe)
    # a tile whose content encodes (row, col, rank) so the assembled frame is checkable
    r = torch.as_tensor(rows, dtype=torch.float64)[:, None]
    c = torch.arange(w, dtype=torch.float64)[None, :]
    n = len(rows)
    tile = {"depth": (r * 1000 + c).reshape(n, w),
            "id": (r * 10 + rank).to(torch.int32).expand(n, w).contiguous(),
            "image": torch.stack([r.expand(n, w), c.expand(n, w), torch.full((n, w), rank, dtype=torch.float64)],
                                 dim=-1).float()}
    out = D.gather_tiles(tile, h, w, rank, world, stripe=stripe)
    if rank == 0:
        rr = torch.arange(h, dtype=torch.float64)[:, None]
        ok = bool(torch.equal(out["depth"], rr * 1000 + torch.arange(w, dtype=torch.float64)[None, :]))
        owner = torch.as_tensor([(i // stripe) % world for i in range(h)], dtype=torch.float32)
        ok &= bool(torch.equal(out["image"][..., 2], owner[:, None].expand(-1, w)))
        ok &= bool(torch.equal(out["image"][..., 0], rr.float().expand(-1, w)))
        ok &= bool(torch.equal(out["id"][:, 0], (torch.arange(h) * 10 + owner.long()).int()))
        ok &= out["id"].shape == (h, w) and out["image"].shape == (h, w, 3)
        q.put(ok)
    else:
        assert out is None
    dist.destroy_process_group()


@pytest.mark.parametrize("world,h,w,stripe", [(2, 40, 7, 1), (3, 50, 5, 1), (4, 3, 5, 1), (3, 50, 5, 16)])
def test_gather_tiles_gloo(world, h, w, stripe):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, h, w, stripe, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    assert all(p.exitcode == 0 for p in procs)
    assert q.get(timeout=5) is True
