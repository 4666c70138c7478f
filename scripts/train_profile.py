#!/usr/bin/env python3
"""A few steady-state training iterations of the paper profile (batch 4096), for
an ncu launch list of the trainer's kernels."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2308_04669_b200 import fields, geometry, model, train  # noqa: E402

oracle = fields.AnalyticOracle(fields.Sphere(geometry.vec3(0, 0, 0), 1.0))
m = model.new_model(oracle, np.random.default_rng(0), model.PROFILES["paper"])
tr = train.Trainer(m, max_batch=4096)
sampler = train.RaySampler(box=m.relaxed_box, mode="direct")
rng = np.random.default_rng(1)
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 3):
    train.build_training_batch(oracle, sampler, tr, rng, 4096)
    tr.loss_and_grads()
    tr.adam_step()
torch.cuda.synchronize()
