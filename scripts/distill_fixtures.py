#!/usr/bin/env python3
"""Distil paper-profile NeDFs on the GPU (the trainer, csrc/train.cu) into the
trained fixtures `tests/golden/trained_{sphere,box,torus}.nedm`, then report how
the tcgen05 path's near-tie guard behaves on them (the calibration of
scripts/tc_calibrate.py, with the model's own alpha threshold).

Random-init paper models put the argmax in 1-2 bins with alpha all-on or
all-off; trained ones use many bins and switch alpha inside
the box, so they stress argmax / alpha parity where random init cannot.

    python scripts/distill_fixtures.py train [iterations]     # on a B200
    python scripts/distill_fixtures.py calibrate [n_rays]
"""

import ctypes as C
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2308_04669_b200 import _lib, configs as CF, fields, model as M, scenes, train as T  # noqa: E402

GOLDEN = ROOT / "tests" / "golden"
KINDS = (("sphere", 0), ("box", 1), ("torus", 5))


def with_alpha_threshold(raw: bytes, thr: float) -> bytes:
    """The same weights with another trailer alpha threshold (model.py:354-361)."""
    import struct
    return raw[:-4] + struct.pack("<f", thr)


def train_all(iterations: int):
    out = {}
    for kind, seed in KINDS:
        oracle = fields.AnalyticOracle(scenes.canonical_geometry(kind))
        m = M.new_model(oracle, np.random.default_rng(seed))
        t = time.time()
        losses = T.train(m, oracle, np.random.default_rng(1000 + seed), iterations=iterations, batch_size=4096,
                         lr=5e-4, progress_every=max(1, iterations // 10))
        torch.cuda.synchronize()
        dt = time.time() - t
        (GOLDEN / f"trained_{kind}.nedm").write_bytes(m.nedm_bytes())
        out[kind] = {"seed": seed, "iterations": iterations, "batch": 4096, "lr": 5e-4, "seconds": dt,
                     "loss_first": losses[0], "loss_last": float(np.mean(losses[-50:]))}
        print(json.dumps({kind: out[kind]}), flush=True)
    (GOLDEN / "trained_models.json").write_text(json.dumps(out, indent=1) + "\n")


def _logits(fn, m, o, d, prec):
    n = o.shape[0]
    lc = torch.full((n, 64), float("nan"), device="cuda")
    lf = torch.full((n, 128), float("nan"), device="cuda")
    la = torch.full((n,), float("nan"), device="cuda")
    _lib.check(fn(m._ctx.handle, m.handle, o.data_ptr(), d.data_ptr(), n, lc.data_ptr(), lf.data_ptr(),
                  la.data_ptr(), prec, None))
    torch.cuda.synchronize()
    return lc, lf, la


def calibrate(n: int):
    lib = _lib.load_library()
    fn = lib.nedf_diag_ray_logits
    fn.restype = C.c_int
    fn.argtypes = [C.c_void_p] * 4 + [C.c_int64] + [C.c_void_p] * 3 + [C.c_int, C.c_void_p]
    ctx = _lib.context()
    for kind, _ in KINDS:
        raw = (GOLDEN / f"trained_{kind}.nedm").read_bytes()
        for thr in (0.5, 0.625):
            m = M.loads_nedf(with_alpha_threshold(raw, thr))
            zthr = float(np.log(thr) - np.log1p(-thr))
            o, d = CF.sweep_rays(n, m.relaxed_box.min, m.relaxed_box.max, seed=3)
            o = torch.as_tensor(o, device="cuda")
            d = torch.as_tensor(d, device="cuda")
            t = _logits(fn, m, o, d, _lib.PREC_TENSOR)
            f = _logits(fn, m, o, d, _lib.PREC_FP32)
            ok = ~torch.isnan(f[2])
            S = torch.maximum(torch.maximum(f[0].abs().amax(1), f[1].abs().amax(1)), f[2].abs())[ok]
            err = {k: float(((a[ok] - b[ok]).abs().reshape(int(ok.sum()), -1).amax(1) / S).max())
                   for k, a, b in (("coarse", t[0], f[0]), ("fine", t[1], f[1]), ("alpha", t[2], f[2]))}
            ct, cf = t[0][ok].argmax(1), f[0][ok].argmax(1)
            ft, ff = t[1][ok].argmax(1), f[1][ok].argmax(1)
            at, af = t[2][ok] > zthr, f[2][ok] > zthr
            flips = (ct != cf) | (ft != ff) | (at != af)
            # the kernel's guard: top-2 margins and |z - z*| against tau * max|logit| (tensor logits)
            tc2, tf2 = t[0][ok].topk(2, 1).values, t[1][ok].topk(2, 1).values
            St = torch.maximum(torch.maximum(t[0].abs().amax(1), t[1].abs().amax(1)), t[2].abs())[ok]
            tau = ctx.get_option(_lib.OPT_GUARD_PPM) * 1e-6
            g = tau * St
            flag = ((tc2[:, 0] - tc2[:, 1]) < g) | ((tf2[:, 0] - tf2[:, 1]) < g) | ((t[2][ok] - zthr).abs() < g)
            # end to end: query_rays in AUTO vs FP32 (the guard re-evaluates the flagged rays)
            ctx.set_option(_lib.OPT_PRECISION, _lib.PREC_AUTO)
            mu_a, al_a = M.query_rays(m, o, d)
            ctx.set_option(_lib.OPT_PRECISION, _lib.PREC_FP32)
            mu_f, al_f = M.query_rays(m, o, d)
            ctx.set_option(_lib.OPT_PRECISION, _lib.PREC_AUTO)
            hit = ~torch.isnan(mu_f)
            rep = {"model": kind, "alpha_threshold": thr, "n": int(ok.sum()), "max_rel_err": err,
                   "max_abs_logit_median": float(S.median()),
                   "coarse_bins_used": int(cf.unique().numel()), "fine_bins_used": int(ff.unique().numel()),
                   "alpha_rate": float(af.float().mean()), "tensor_flips": int(flips.sum()),
                   "guard_flagged_frac": float(flag.float().mean()), "unflagged_flips": int((flips & ~flag).sum()),
                   "auto_vs_fp32_mu_mismatch": int((mu_a[hit] != mu_f[hit]).sum()),
                   "auto_vs_fp32_alpha_mismatch": int((al_a[hit] != al_f[hit]).sum())}
            print(json.dumps(rep), flush=True)


if __name__ == "__main__":
    what = sys.argv[1] if len(sys.argv) > 1 else "train"
    if what == "train":
        train_all(int(sys.argv[2]) if len(sys.argv) > 2 else 6000)
    else:
        calibrate(int(sys.argv[2]) if len(sys.argv) > 2 else 65536)
