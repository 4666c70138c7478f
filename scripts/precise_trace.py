#!/usr/bin/env python3
"""Timeline of the guard's throughput kernel (mlp_precise.cu), CTA 0, first tile, run on
every ray of a 16k-ray sweep through nedf_diag_ray_logits."""
import ctypes as C
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2308_04669_b200 import _lib, configs as CF, scenes  # noqa: E402
from scripts.tc_calibrate import logits  # noqa: E402

lib = _lib.load_library()
tr = lib.nedf_diag_precise_trace
tr.restype = C.c_int
tr.argtypes = [C.c_int, C.POINTER(C.c_ulonglong), C.c_int]
m = scenes.paper_model(0, "sphere")
o, d = CF.sweep_rays(16384, m.relaxed_box.min, m.relaxed_box.max, seed=1)
o = torch.as_tensor(o, device="cuda")
d = torch.as_tensor(d, device="cuda")
logits(m, o, d, 16 + 3)
tr(1, None, 0)
torch.cuda.synchronize()
logits(m, o, d, 16 + 3)
torch.cuda.synchronize()
out = (C.c_ulonglong * 200)()
tr(0, out, 200)
t = list(out)
b = t[0]
print("ray setup done:", t[192] - b)
print("group 0 point: encode start / done:", [(t[176 + p] - b, t[160 + p] - b) for p in range(0, 16, 4)])
print("head points encoded:", [t[160 + p] - b for p in range(16)])
print(" L  mma_start issued epi_has epi_done | mma epi layer")
for L in range(34):
    nxt = t[L + 1] - t[L] if L < 33 else -1
    print(f"{L:2d} {t[L] - b:9d} {t[40 + L] - b:7d} {t[80 + L] - b:7d} {t[120 + L] - b:8d} | {t[40 + L] - t[L]:5d} "
          f"{t[120 + L] - t[80 + L]:5d} {nxt:6d}")
