#!/usr/bin/env python3
"""Timeline of the cluster-split fp32 guard kernel (cluster 0, CTA 0) while
rendering the config-4 frame."""
import ctypes as C
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2308_04669_b200 import _lib, configs as CF, pipeline, scenes  # noqa: E402

lib = _lib.load_library()
tr = lib.nedf_diag_cl_trace
tr.restype = C.c_int
tr.argtypes = [C.c_int, C.POINTER(C.c_ulonglong), C.c_int]
scene, cam, lights, cfg = scenes.build(CF.config4())
buf = pipeline.FrameBuffers(cam.width, cam.height)
pipeline.nedf_generation_step(scene, cam, buf)
torch.cuda.synchronize()
tr(1, None, 0)
pipeline.nedf_generation_step(scene, cam, buf)
torch.cuda.synchronize()
out = (C.c_ulonglong * 256)()
tr(0, out, 256)
t = list(out)
for i in range(4):
    b = t[64 * i]
    if not b:
        break
    rel = lambda k: (t[64 * i + k] - b) if t[64 * i + k] else None
    layers = [rel(3 + L) for L in range(34)]
    print(f"tile {i}: setup {rel(1)} features {rel(2)} head {layers[0]} L1 {layers[1]} L2 {layers[2]} "
          f"L33 {layers[33]} decoded {rel(40)}")
    d = [layers[L + 1] - layers[L] for L in range(33) if layers[L + 1] and layers[L]]
    print("   per-layer cycles:", d[:8], "...", d[-4:])
    print("   layer 5: MMAs", t[64 * i + 41] - t[64 * i + 3 + 4], "(of which weight-ring waits", t[64 * i + 43], ")",
          "epilogue + sends", t[64 * i + 42] - t[64 * i + 41], "wait for peers", t[64 * i + 3 + 5] - t[64 * i + 42])
print("layer 5 FMA end per warp (tile 0, rel. to layer start):", [t[200 + w] - t[3 + 4] if t[200 + w] else None for w in range(16)])
