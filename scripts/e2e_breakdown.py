#!/usr/bin/env python3
"""Where the end-to-end frame time goes (config 4, one GPU): back-to-back compose_frame
calls with and without the result copies, against event-timed single frames."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2308_04669_b200 import configs as CF, pipeline, scenes  # noqa: E402

scene, cam, lights, cfg = scenes.build(CF.config4())
bufs = [pipeline.FrameBuffers(cam.width, cam.height) for _ in range(2)]
hosts = [(torch.empty(b.image.shape, dtype=torch.float32).pin_memory(),
          torch.empty(b.depth.shape, dtype=torch.float64).pin_memory(),
          torch.empty(b.id.shape, dtype=torch.int32).pin_memory()) for b in bufs]
cs = torch.cuda.Stream()
N = int(sys.argv[1]) if len(sys.argv) > 1 else 20


def run(copies, n=N):
    copied = [None, None]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    host_ms = []
    for i in range(n):
        k = i & 1
        if copied[k] is not None:
            torch.cuda.current_stream().wait_event(copied[k])
        h0 = time.perf_counter()
        res = pipeline.compose_frame(scene, cam, lights, cfg, buffers=bufs[k])
        host_ms.append((time.perf_counter() - h0) * 1e3)
        if copies:
            done = torch.cuda.Event()
            done.record()
            cs.wait_event(res.events[2])
            with torch.cuda.stream(cs):
                hosts[k][1].copy_(bufs[k].depth, non_blocking=True)
                hosts[k][2].copy_(bufs[k].id, non_blocking=True)
            cs.wait_event(done)
            with torch.cuda.stream(cs):
                hosts[k][0].copy_(bufs[k].image, non_blocking=True)
                copied[k] = torch.cuda.Event()
                copied[k].record(cs)
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) * 1e3 / n, float(np.median(host_ms))


def events_b2b(n=N):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(n + 1)]
    ev[0].record()
    for i in range(n):
        pipeline.compose_frame(scene, cam, lights, cfg, buffers=bufs[i & 1])
        ev[i + 1].record()
    torch.cuda.synchronize()
    return [ev[i].elapsed_time(ev[i + 1]) for i in range(n)]


for _ in range(3):
    run(True, 3)
for r in range(2):
    w, h = run(False)
    print(f"b2b no copies: {w:.3f} ms/frame wall, host per call {h:.3f} ms")
    w, h = run(True)
    print(f"b2b with copies: {w:.3f} ms/frame wall, host per call {h:.3f} ms")
    d = events_b2b()
    print(f"b2b device events: mean {np.mean(d):.3f} first {d[0]:.3f} last {d[-1]:.3f}")
t = time.perf_counter()
torch.cuda.synchronize()
x = torch.empty(bufs[0].image.shape, dtype=torch.float32).pin_memory()
t0 = time.perf_counter()
x.copy_(bufs[0].image)
dt = time.perf_counter() - t0
print(f"one image D2H ({bufs[0].image.numel() * 4 / 1e6:.1f} MB): {dt * 1e3:.3f} ms")
