#!/usr/bin/env python3
"""fp16 tcgen05 logits vs the fp32 path for the GPU-distilled models
(tests/golden/trained_*.nedm): error distribution against candidate per-ray
scales, and how many rays a guard at each scale would flag vs how many
decisions actually flip."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2308_04669_b200 import _lib, configs as CF, model  # noqa: E402
from scripts.tc_calibrate import logits  # noqa: E402

ROOT = Path(__file__).resolve().parent.parent
for kind in ("sphere", "box", "torus"):
    m = model.load_nedf(ROOT / "tests" / "golden" / f"trained_{kind}.nedm")
    o, d = CF.sweep_rays(131072, m.relaxed_box.min, m.relaxed_box.max, seed=3)
    o = torch.as_tensor(o, device="cuda")
    d = torch.as_tensor(d, device="cuda")
    t = logits(m, o, d, _lib.PREC_TENSOR)
    f = logits(m, o, d, _lib.PREC_FP32)
    ok = ~torch.isnan(f[2])
    tc, tf, ta = t[0][ok], t[1][ok], t[2][ok]
    fc, ff, fa = f[0][ok], f[1][ok], f[2][ok]
    err_c = (tc - fc).abs().amax(1)
    err_f = (tf - ff).abs().amax(1)
    err = torch.maximum(err_c, err_f)
    S_max = torch.maximum(torch.maximum(fc.abs().amax(1), ff.abs().amax(1)), fa.abs())
    S_fine = ff.abs().amax(1)
    S_rng = (ff.amax(1) - ff.amin(1))
    def q(x):
        return [float(torch.quantile(x.float(), p)) for p in (0.5, 0.99, 0.999)] + [float(x.max())]
    print(kind, "rays", int(ok.sum()))
    print("  max|logit| median", float(S_max.median()), " err abs quantiles", q(err))
    print("  err / max|logit|", q(err / S_max))
    print("  err / max|fine|", q(err / S_fine), " err / fine range", q(err / S_rng))
    top2c = fc.topk(2, 1).values
    top2f = ff.topk(2, 1).values
    mc = top2c[:, 0] - top2c[:, 1]
    mf = top2f[:, 0] - top2f[:, 1]
    flips = (tc.argmax(1) != fc.argmax(1)) | (tf.argmax(1) != ff.argmax(1))
    print("  flips", int(flips.sum()), "fine margin / max|logit| quantiles", q(mf / S_max), "coarse", q(mc / S_max))
    for tau in (3e-3, 1e-3, 3e-4, 1e-4):
        flag = (mc < tau * S_max) | (mf < tau * S_max)
        print(f"  tau {tau:g}: flagged {float(flag.float().mean()):.4f}, flips missed {int((flips & ~flag).sum())}")
