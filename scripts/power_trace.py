#!/usr/bin/env python3
"""SM clock and board power while rendering the headline frame back to back (nvidia-smi at
100 ms), with the per-frame event time: how the sustained frame rate follows the power cap."""
import subprocess
import sys
import tempfile
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2308_04669_b200 import configs as CF, pipeline, scenes  # noqa: E402

scene, cam, lights, cfg = scenes.build(CF.config4())
rnd = pipeline.FrameRenderer(scene, cam, lights, cfg)
for _ in range(3):
    rnd.render()
torch.cuda.synchronize()
f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
p = subprocess.Popen(["nvidia-smi", "--query-gpu=timestamp,clocks.sm,power.draw,power.limit,temperature.gpu,"
                      "clocks_event_reasons.active", "--format=csv,noheader,nounits", "-i", "0", "-lms", "100"],
                     stdout=f, stderr=subprocess.DEVNULL)
time.sleep(1.0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 600
ev = [torch.cuda.Event(enable_timing=True) for _ in range(n + 1)]
ev[0].record()
for i in range(n):
    rnd.render()
    ev[i + 1].record()
torch.cuda.synchronize()
time.sleep(0.5)
p.terminate()
p.wait()
ms = np.array([ev[i].elapsed_time(ev[i + 1]) for i in range(n)])
for k in range(0, n, n // 10):
    print(f"frames {k:4d}-{k + n // 10 - 1:4d}: mean {ms[k:k + n // 10].mean():.3f} ms")
rows = [ln.split(",") for ln in Path(f.name).read_text().splitlines() if ln.count(",") >= 5]
for r in rows[:: max(1, len(rows) // 15)]:
    print(",".join(x.strip() for x in r))
