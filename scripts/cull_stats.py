#!/usr/bin/env python3
"""How many network evaluations of a frame provably cannot change its output?
(analysis only: GPU planes from the product, geometry from the oracle)

STEP 1: a NeDF pair's depth is |(o-T).d| - s mu with mu <= mu_max (model.py:89-92,
301-319), so a pair whose lower bound exceeds the pixel's winning depth cannot win.
'front-first' = evaluate each pixel's pair with the smallest bound, then only the
rest whose bound is <= that result.  STEP 3 (point light): a pair with
bound + eps >= |x - light| cannot shadow."""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from oracle import nedf_oracle as O  # noqa: E402
from paper_2308_04669_b200 import configs as CF, pipeline, scenes  # noqa: E402
from tests import helpers  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "config4"
spec = getattr(CF, which)()
objs, ocam, olights, ocfg = helpers.oracle_scene(spec)
scene, cam, lights, cfg = scenes.build(spec)
buf = pipeline.FrameBuffers(cam.width, cam.height, keep_planes=True)
pipeline.nedf_generation_step(scene, cam, buf)
torch.cuda.synchronize()
planes = np.stack([buf.per_object_depth[inst.id].cpu().numpy().ravel() for inst in scene])
depth = buf.depth.cpu().numpy().ravel()
ids = buf.id.cpu().numpy().ravel()
o, d = O.primary_rays(ocam)
n = o.shape[0]


def bounds(ob, ro, rd):
    m = ob.model
    lo = ((ro - ob.T) @ ob.R) / ob.s
    _, _, hit = O.slab_clip(lo, rd @ ob.R, m.box_min, m.box_max)
    mu_max = O.decode_mu(m, m.n_coarse - 1, m.n_fine - 1)
    lower = np.abs(np.einsum("ij,ij->i", ro - ob.T, rd)) - ob.s * mu_max
    return hit, lower


hits, lows = zip(*(bounds(ob, o, d) for ob in objs))
hits = np.stack(hits)
lows = np.where(hits, np.stack(lows), np.inf)
pairs = int(hits.sum())
covered = int(hits.any(0).sum())
front = np.argmin(lows, axis=0)
best1 = np.where(hits.any(0), planes[front, np.arange(n)], np.inf)
second = hits.copy()
second[front, np.arange(n)] = False
pass2 = int((second & (lows.astype(np.float32) <= best1.astype(np.float32)[None, :])).sum())
ideal = int((hits & (lows.astype(np.float32) <= depth.astype(np.float32)[None, :])).sum())
print(f"STEP 1: {pairs} pairs over {covered} pixels; front-first {covered} + {pass2} = {covered + pass2} "
      f"({100 * (covered + pass2) / pairs:.1f}%); oracle-ordered lower bound {ideal} ({100 * ideal / pairs:.1f}%)")
# STEP 3
eps = O.default_eps(objs)
valid = (ids >= 0) & np.isfinite(depth)
for L in olights:
    if L.kind != "point":
        continue
    x = o[valid] + depth[valid, None] * d[valid]
    to_x = x - L.vec[None, :]
    dist = np.linalg.norm(to_x, axis=1)
    rd = to_x / dist[:, None]
    ro = np.broadcast_to(L.vec, x.shape).copy()
    tot = cut = 0
    for ob in objs:
        h, lw = bounds(ob, ro, rd)
        tot += int(h.sum())
        cut += int((h & (lw + eps >= dist)).sum())
    print(f"STEP 3: {tot} pairs over {int(valid.sum())} lit pixels; {cut} cannot shadow ({100 * cut / max(tot, 1):.1f}%)")
