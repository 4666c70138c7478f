"""Test helpers: build oracle-side scenes from the shared config specs.

Test infrastructure only (imports the oracle)."""

from __future__ import annotations

import functools

import numpy as np

from oracle import nedf_oracle as O
from paper_2308_04669_b200 import configs as C


@functools.lru_cache(maxsize=None)
def oracle_model(seed: int, kind: str, d_feat: int = 256, n_blocks: int = 16):
    return O.new_paper_model(seed, kind, d_feat, n_blocks)


def oracle_scene(spec: C.SceneSpec):
    objs = []
    for o in spec.objects:
        m = oracle_model(o.seed, o.kind, spec.d_feat, spec.n_blocks)
        objs.append(O.Obj(o.id, np.asarray(o.R, dtype=np.float64), np.asarray(o.T, dtype=np.float64),
                          float(o.s), C.CANONICAL_PRIMS[o.kind], model=m))
    c = spec.camera
    cam = O.Cam(np.asarray(c.position, dtype=np.float64), O.look_at(c.position, c.look_at, c.up),
                c.fov_y, c.width, c.height)
    lights = [O.Light(L.kind, np.asarray(L.vec, dtype=np.float64), L.beta) for L in spec.lights]
    cfg = O.Config(shadows=spec.shadows, resample=spec.resample)
    return objs, cam, lights, cfg


def psnr(a, b, peak=1.0):
    mse = float(np.mean((np.asarray(a, dtype=np.float64) - np.asarray(b, dtype=np.float64)) ** 2))
    if mse == 0:
        return float("inf")
    return 10.0 * np.log10(peak * peak / mse)
