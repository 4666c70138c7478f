#!/usr/bin/env python3
"""Back-to-back device time per frame, same box and process: FrameRenderer.render (pre-marshalled
scene) vs compose_frame (the reference's API: scene tables marshalled per call, step events,
stats snapshot), with and without an L2 flush between frames."""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2308_04669_b200 import configs as CF, pipeline, scenes  # noqa: E402

scene, cam, lights, cfg = scenes.build(CF.config4())
buf = pipeline.FrameBuffers(cam.width, cam.height)
rnd = pipeline.FrameRenderer(scene, cam, lights, cfg, buffers=buf)
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
N = 20


def timed(fn, do_flush):
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(N)]
    for a, b in ev:
        if do_flush:
            flush.zero_()
        a.record()
        fn()
        b.record()
    torch.cuda.synchronize()
    return np.array([a.elapsed_time(b) for a, b in ev])


fns = {"render": lambda: rnd.render(), "compose": lambda: pipeline.compose_frame(scene, cam, lights, cfg, buffers=buf)}
for f in fns.values():
    for _ in range(3):
        f()
torch.cuda.synchronize()
for r in range(3):
    for name, f in fns.items():
        for fl in (True, False):
            ms = timed(f, fl)
            print(f"{name:8s} flush={fl!s:5s} mean {ms.mean():.3f} median {np.median(ms):.3f} min {ms.min():.3f}")
