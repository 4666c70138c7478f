#!/usr/bin/env python3
"""Timeline of the tcgen05 guard kernel (cluster 0, CTA 0, first tile) while
rendering the config-4 frame's STEP 1 (the guard re-evaluates its near-tie rays)."""
import ctypes as C
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2308_04669_b200 import _lib, configs as CF, pipeline, scenes  # noqa: E402

lib = _lib.load_library()
tr = lib.nedf_diag_guard_trace
tr.restype = C.c_int
tr.argtypes = [C.c_int, C.POINTER(C.c_ulonglong), C.c_int]
scene, cam, lights, cfg = scenes.build(CF.config4())
buf = pipeline.FrameBuffers(cam.width, cam.height)
pipeline.nedf_generation_step(scene, cam, buf)
torch.cuda.synchronize()
tr(1, None, 0)
pipeline.nedf_generation_step(scene, cam, buf)
torch.cuda.synchronize()
out = (C.c_ulonglong * 320)()
tr(0, out, 320)
t = list(out)
b = min(x for x in t if x)
r = lambda k: (t[k] - b) if t[k] else -1   # noqa: E731
print("stage issue times (first 12):", [r(240 + q) for q in range(12)])
print("stage issue deltas body:", [t[240 + q + 1] - t[240 + q] for q in range(8, 30)])
L33 = 33
print(" L   mma_start  issued  epi_has   sent  landed  bready | layer  mma  epi  stores  send  xfer  split")
for L in range(34):
    nxt = t[L + 1] if L + 1 < 34 else 0
    print(f"{L:2d} {r(L):9d} {r(40 + L):7d} {r(80 + L):7d} {r(120 + L):7d} {r(160 + L):7d} {r(200 + L):7d} | "
          f"{(nxt - t[L]) if nxt else -1:6d} {t[40 + L] - t[L]:4d} {t[80 + L] - t[40 + L]:4d} "
          f"{(t[280 + L] - t[80 + L]) if t[280 + L] else -1:6d} {t[120 + L] - t[80 + L]:5d} {t[160 + L] - t[120 + L]:5d} {(t[200 + L] - t[160 + L]) if t[200 + L] else -1:5d}")
