#!/usr/bin/env python3
"""Calibrate the CPU baseline: the REAL reference (`/root/reference/pkg/src/nedf`)
against the float64 oracle port that `bench.py --impl reference` times on the
GPU box (which has no /root/reference), on the same host and core count.

Build container only:

    PYTHONPATH=/root/reference/pkg/src python scripts/cpu_calibrate.py [--out profiles/r2_cpu_calibration.json]

Measures (1) config 4 at 250x100 through `pipeline.compose_frame` (reference) vs
`oracle.render` (port), checking the id buffers agree, and (2) CPU NeDF rays/s at
B = 16,384: `model.query_rays` (encode + MLP + decode, ref
model.py:277-293) vs the port's `query_rays`, on `RaySampler` rays (seed 0).
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests" / "golden"))
THREADS = os.cpu_count() or 1
os.environ.setdefault("OPENBLAS_NUM_THREADS", str(THREADS))

import numpy as np  # noqa: E402

import make_golden as MG  # noqa: E402  (imports the reference; asserts it is /root/reference)
from nedf import model as RM, pipeline as RP  # noqa: E402
from oracle import nedf_oracle as O  # noqa: E402
from paper_2308_04669_b200 import configs as CF  # noqa: E402
from tests.helpers import oracle_scene, oracle_model  # noqa: E402


def best_of(fn, reps):
    ts = []
    out = None
    for _ in range(reps):
        t0 = time.perf_counter()
        out = fn()
        ts.append(time.perf_counter() - t0)
    return min(ts), out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=str(ROOT / "profiles" / "r2_cpu_calibration.json"))
    ap.add_argument("--width", type=int, default=250)
    ap.add_argument("--height", type=int, default=100)
    ap.add_argument("--reps", type=int, default=2)
    a = ap.parse_args()
    RP.set_thread_count(THREADS)

    spec = CF.config4(a.width, a.height)
    scene, cam, lights, cfg = MG.ref_scene(spec)
    RP.compose_frame(scene, cam, lights, cfg)                      # warm (model load, BLAS init)
    t_ref, res = best_of(lambda: RP.compose_frame(scene, cam, lights, cfg), a.reps)
    objs, ocam, olights, ocfg = oracle_scene(spec)
    O.render(objs, ocam, olights, ocfg, threads=THREADS)
    t_port, out = best_of(lambda: O.render(objs, ocam, olights, ocfg, threads=THREADS), a.reps)
    id_equal = bool(np.array_equal(res.buffers.id, out.id.reshape(res.buffers.id.shape)))

    # CPU NeDF rays/s at B = 16,384 (encode + MLP + decode)
    B = 16384
    m_ref, _ = MG.paper_model(0, "sphere")
    o, d = RM.RaySampler(box=m_ref.relaxed_box).sample(np.random.default_rng(0), B)
    RM.query_rays(m_ref, o[:256], d[:256])
    t_qr, (mu_r, al_r) = best_of(lambda: RM.query_rays(m_ref, o, d), a.reps)
    m_port = oracle_model(0, "sphere")
    O.query_local(m_port, o[:256], d[:256])
    t_qp, (mu_p, al_p) = best_of(lambda: O.query_local(m_port, o, d), a.reps)
    hits = int(np.isfinite(mu_r).sum())

    rep = {
        "host_threads": THREADS,
        "env": {"OPENBLAS_NUM_THREADS": os.environ.get("OPENBLAS_NUM_THREADS"), "nedf_threads": THREADS},
        "frame": {"workload": f"config4 at {a.width}x{a.height}, compose_frame (STEP 1-3 + composite)",
                  "reference_s": t_ref, "port_s": t_port, "reference_over_port": t_ref / t_port,
                  "id_buffers_equal": id_equal, "timing": f"best of {a.reps}"},
        "query_rays_B16384": {"rays": B, "box_hits": hits,
                              "reference_s": t_qr, "port_s": t_qp,
                              "reference_rays_per_s": B / t_qr, "port_rays_per_s": B / t_qp,
                              "reference_evals_per_s": hits / t_qr, "port_evals_per_s": hits / t_qp,
                              "mu_equal": bool(np.array_equal(mu_r, mu_p, equal_nan=True)),
                              "alpha_equal": bool(np.array_equal(al_r, al_p))},
        "note": "bench.py's CPU arm times the port (the GPU box has no /root/reference); "
                "multiply its ms/frame by frame.reference_over_port for the reference's own time",
    }
    Path(a.out).write_text(json.dumps(rep, indent=1) + "\n")
    print(json.dumps(rep, indent=1))


if __name__ == "__main__":
    main()
