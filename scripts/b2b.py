#!/usr/bin/env python3
"""Per-frame CUDA-event time of the headline frame back to back vs with an L2
flush between frames, and the wall-clock rate of back-to-back frames."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2308_04669_b200 import configs as CF, pipeline, scenes  # noqa: E402

scene, cam, lights, cfg = scenes.build(CF.config4())
rnd = pipeline.FrameRenderer(scene, cam, lights, cfg)
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
for _ in range(5):
    rnd.render()
torch.cuda.synchronize()
for mode in ("flush", "b2b", "flush", "b2b"):
    n = 30
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
    t0 = time.perf_counter()
    for a, b in evs:
        if mode == "flush":
            flush.zero_()
        a.record()
        rnd.render()
        b.record()
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) * 1e3 / n
    ms = [a.elapsed_time(b) for a, b in evs]
    print(mode, "event mean", round(float(np.mean(ms)), 3), "min", round(float(np.min(ms)), 3), "wall/frame", round(wall, 3))
