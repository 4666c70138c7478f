"""Multi-GPU image-tile partition + gather, exercised with gloo on CPU
(world_size 2 and 3)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2308_04669_b200 import distributed as D


def test_stripes_partition_rows():
    for h in (1, 15, 16, 17, 800, 801):
        for world in (1, 2, 3, 4, 8):
            parts = [D.stripe_rows(h, r, world) for r in range(world)]
            allr = np.sort(np.concatenate(parts))
            np.testing.assert_array_equal(allr, np.arange(h))
            assert max(len(p) for p in parts) == D.max_rows(h, world)
    with pytest.raises(ValueError):
        D.stripe_rows(10, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, h, w, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rows = D.stripe_rows(h, rank, world)
    # a tile whose content encodes (row, col) so the assembled frame is checkable
    r = torch.as_tensor(rows, dtype=torch.float64)[:, None]
    c = torch.arange(w, dtype=torch.float64)[None, :]
    tile = {"depth": r * 1000 + c, "id": (r * 10 + rank).to(torch.int32).expand(-1, w).contiguous(),
            "image": torch.stack([r.expand(-1, w), c.expand(len(rows), -1), torch.full((len(rows), w), rank,
                                                                                     dtype=torch.float64)],
                                 dim=-1).float()}
    out = D.gather_tiles(tile, h, w, rank, world)
    if rank == 0:
        rr = torch.arange(h, dtype=torch.float64)[:, None]
        ok = bool(torch.equal(out["depth"], rr * 1000 + torch.arange(w, dtype=torch.float64)[None, :]))
        owner = torch.as_tensor([(i // D.STRIPE) % world for i in range(h)], dtype=torch.float32)
        ok &= bool(torch.equal(out["image"][..., 2], owner[:, None].expand(-1, w)))
        ok &= bool(torch.equal(out["id"][:, 0], (torch.arange(h) * 10 + owner.long()).int()))
        q.put(ok)
    else:
        assert out is None
    dist.destroy_process_group()


@pytest.mark.parametrize("world,h,w", [(2, 40, 7), (3, 50, 5)])
def test_gather_tiles_gloo(world, h, w):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, h, w, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    assert all(p.exitcode == 0 for p in procs)
    assert q.get(timeout=5) is True
