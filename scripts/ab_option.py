#!/usr/bin/env python3
"""A/B of one context option on the headline frame, same process and box: alternates
blocks of flushed, event-timed config-4 frames with the option at each value.
usage: ab_option.py OPT_NAME v0 v1 [rounds] [frames]"""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "scripts"))
from paper_2308_04669_b200 import _lib, configs as CF, pipeline, scenes  # noqa: E402
from bench_configs import _flush_buf, time_frames  # noqa: E402

name, v0, v1 = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
rounds = int(sys.argv[4]) if len(sys.argv) > 4 else 4
frames = int(sys.argv[5]) if len(sys.argv) > 5 else 10
key = getattr(_lib, name)
scene, cam, lights, cfg = scenes.build(CF.config4())
rnd = pipeline.FrameRenderer(scene, cam, lights, cfg)
flush = _flush_buf()
ctx = _lib.context()
res = {v0: [], v1: []}
for r in range(rounds):
    for v in (v0, v1) if r % 2 == 0 else (v1, v0):
        ctx.set_option(key, v)
        ms, _ = time_frames(rnd, frames, flush)
        res[v] += ms
ctx.set_option(key, v0)
for v, ms in res.items():
    print(f"{name}={v}: mean {np.mean(ms):.3f} median {np.median(ms):.3f} min {np.min(ms):.3f} ms ({len(ms)} frames)")
