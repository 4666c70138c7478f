#!/usr/bin/env python3
"""Wait accounting of one steady-state 256-ray tile of the CTA-pair tcgen05
kernel (cluster 0, its second tile) while rendering STEP 1 of config 4."""

import ctypes as C
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2308_04669_b200 import _lib, configs as CF, pipeline, scenes  # noqa: E402

lib = _lib.load_library()
tr = lib.nedf_diag_tc2_trace
tr.restype = C.c_int
tr.argtypes = [C.c_int, C.POINTER(C.c_ulonglong), C.c_int]
_lib.context().set_option(_lib.OPT_TC_KERNEL, _lib.TC_PAIR)
scene, cam, lights, cfg = scenes.build(CF.config4())
buf = pipeline.FrameBuffers(cam.width, cam.height)
pipeline.nedf_generation_step(scene, cam, buf)
torch.cuda.synchronize()
tr(1, None, 0)
pipeline.nedf_generation_step(scene, cam, buf)
torch.cuda.synchronize()
out = (C.c_ulonglong * 64)()
tr(0, out, 64)
t = list(out)
print(f"MMA tile {t[4]} cycles; waits full {t[0]} peer_full {t[1]} epi_done {t[2]} enc_full {t[3]}")
for r in (0, 1):
    print(f"CTA{r}: producer empty-wait {t[8 + r]}  encoder wait {t[12 + r]} / {t[14 + r]}  "
          f"epilogue wait {t[16 + r]} / {t[18 + r]}")
print(f"relay full-wait {t[10]}")
print(f"cluster 0: {t[6]} tiles, {t[5]} cycles ({t[5] / max(1, t[6]):.0f}/tile), {t[7] / 1e3:.1f} us -> {t[5] / max(1, t[7]):.3f} GHz")
import ctypes
cnt = ctypes.c_int(0)
print("device SMs", torch.cuda.get_device_properties(0).multi_processor_count)
out = (C.c_ulonglong * 512)()
tr(0, out, 512)
t = [int(v) for v in out]
t0 = t[63]
rel = lambda v: v - t0 if v else None
print("head mma", rel(t[64]), "..", rel(t[100]))
for L in range(1, 34):
    print(f"L{L:2d} mma {rel(t[64 + L])}..{rel(t[100 + L])} ({t[100 + L] - t[64 + L]})  "
          f"epi ready {[rel(t[136 + 2 * L + s]) for s in (0, 1)]} done {[rel(t[204 + 2 * L + s]) for s in (0, 1)]}")
