#!/usr/bin/env python3
"""Print the per-role timeline of one steady-state tile of the tcgen05 kernel
(CTA 0, its second tile) while rendering STEP 1 of the config-4 frame.

The instrumentation is compiled in only with -DNEDF_TC_TRACE=1:
    python scripts/build_variant.py trace mlp_tc.cu -DNEDF_TC_TRACE=1
    NEDF_LIB=_exp/trace.so python scripts/tc_trace.py 3 3
"""

import ctypes as C
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2308_04669_b200 import _lib, configs as CF, pipeline, scenes  # noqa: E402

lib = _lib.load_library()
tr = lib.nedf_diag_tc_trace
tr.restype = C.c_int
tr.argtypes = [C.c_int, C.POINTER(C.c_ulonglong), C.c_int]

# tc kernel variant (argv[2]): 1 single CTA (default), 3 cluster-multicast pair, 4 multicast x4
_lib.context().set_option(_lib.OPT_TC_KERNEL, int(sys.argv[2]) if len(sys.argv) > 2 else _lib.TC_SINGLE)
spec = CF.config4()
scene, cam, lights, cfg = scenes.build(spec)
buf = pipeline.FrameBuffers(cam.width, cam.height)
pipeline.nedf_generation_step(scene, cam, buf)
torch.cuda.synchronize()
TILE = int(sys.argv[1]) if len(sys.argv) > 1 else 2
tr(TILE, None, 0)
pipeline.nedf_generation_step(scene, cam, buf)
torch.cuda.synchronize()
out = (C.c_ulonglong * 1024)()
tr(0, out, 1024)
t = np.array(out[:], dtype=np.int64)
t0 = t[0]
rel = lambda i: int(t[i] - t0) if t[i] else None
print("producer layer starts:", [rel(450 + L) for L in range(34)])
print("encoder point computed:     ", [rel(500 + p) for p in range(16)])
print("encoder point slot acquired:", [rel(420 + p) for p in range(16)])
print("encoder point written:      ", [rel(400 + p) for p in range(16)])
prev_end = None
for L in range(34):
    ms, me = rel(L), rel(40 + L)
    ready = [rel(100 + 8 * L + s) for s in range(4)]
    done = [rel(104 + 8 * L + s) for s in range(4)]
    print(f"L{L:2d} mma {ms}..{me} (issue {me - ms if ms is not None and me is not None else None})  "
          f"epi ready {ready} done {done}  epi[s3] {done[3] - ready[3] if done[3] and ready[3] else None}")
print("tile cycles (MMA start L0 -> epi done tail):", rel(104 + 8 * 33 + 3))
print("MMA waits in this tile: full", int(t[600]), "(head", int(t[603]), ") epi_done", int(t[601]), "enc_full", int(t[602]))
print("MMA head: epi_done(tail) passed at", rel(80), "; point c ready at", [rel(81 + c) for c in range(16)])
