#!/usr/bin/env python3
"""Compare the tcgen05 fp16 network's logits with the fp32 path on sweep rays
and report the error distribution that sets the near-tie guard threshold."""

import ctypes as C
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2308_04669_b200 import _lib, configs as CF, scenes  # noqa: E402

lib = _lib.load_library()
fn = lib.nedf_diag_ray_logits
fn.restype = C.c_int
fn.argtypes = [C.c_void_p] * 4 + [C.c_int64] + [C.c_void_p] * 3 + [C.c_int, C.c_void_p]


def logits(m, o, d, prec):
    n = o.shape[0]
    lc = torch.full((n, 64), float("nan"), device="cuda")
    lf = torch.full((n, 128), float("nan"), device="cuda")
    la = torch.full((n,), float("nan"), device="cuda")
    _lib.check(fn(m._ctx.handle, m.handle, o.data_ptr(), d.data_ptr(), n, lc.data_ptr(), lf.data_ptr(),
                  la.data_ptr(), prec, None))
    torch.cuda.synchronize()
    return lc, lf, la


def main(n=int(sys.argv[1]) if len(sys.argv) > 1 else 65536):
    out = {}
    for seed, kind in [(0, "sphere"), (1, "box"), (5, "torus"), (2, "sphere")]:
        m = scenes.paper_model(seed, kind)
        o, d = CF.sweep_rays(n, m.relaxed_box.min, m.relaxed_box.max, seed=seed)
        o = torch.as_tensor(o, device="cuda")
        d = torch.as_tensor(d, device="cuda")
        t = logits(m, o, d, _lib.PREC_TENSOR)
        f = logits(m, o, d, _lib.PREC_FP32)
        ok = ~torch.isnan(f[2])
        S = torch.maximum(torch.maximum(f[0].abs().amax(1), f[1].abs().amax(1)), f[2].abs())[ok]
        rel = {}
        for name, a, b in [("coarse", t[0], f[0]), ("fine", t[1], f[1])]:
            e = (a[ok] - b[ok]).abs().amax(1) / S
            rel[name] = (float(e.median()), float(torch.quantile(e.float(), 0.999)), float(e.max()))
        ea = (t[2][ok] - f[2][ok]).abs() / S
        rel["alpha"] = (float(ea.median()), float(torch.quantile(ea.float(), 0.999)), float(ea.max()))
        # decision agreement
        ct, cf = t[0][ok].argmax(1), f[0][ok].argmax(1)
        ft, ff = t[1][ok].argmax(1), f[1][ok].argmax(1)
        at, af = t[2][ok] > 0, f[2][ok] > 0
        flips = {"coarse": float((ct != cf).float().mean()), "fine": float((ft != ff).float().mean()),
                 "alpha": float((at != af).float().mean())}
        # guard coverage: fraction flagged at tau, and flips missed by the guard
        top2c = f[0][ok].topk(2, 1).values
        top2f = f[1][ok].topk(2, 1).values
        flagged = {}
        for tau in (1e-3, 2e-3, 3e-3, 5e-3):
            thr = tau * S
            fl = ((top2c[:, 0] - top2c[:, 1]) < thr) | ((top2f[:, 0] - top2f[:, 1]) < thr) | (f[2][ok].abs() < thr)
            bad = ((ct != cf) | (ft != ff) | (at != af)) & ~fl
            flagged[tau] = (float(fl.float().mean()), int(bad.sum()))
        out[f"{seed}:{kind}"] = {"n": int(ok.sum()), "rel_err(med,p999,max)": rel, "flip_rate": flips,
                                 "flagged(frac,missed)": flagged, "alpha_rate": float(af.float().mean())}
        print(json.dumps({f"{seed}:{kind}": out[f"{seed}:{kind}"]}), flush=True)
    return out


if __name__ == "__main__":
    main()
