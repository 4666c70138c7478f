"""Parity criteria of BASELINE.json's north star, shared by the GPU tests and
smoke(): depth |err| <= 1e-3 scene units, id identical on >= 99.9% of pixels
(mismatches only where two surfaces lie within tolerance), RGB PSNR >= 45 dB."""

from __future__ import annotations

import numpy as np

DEPTH_TOL = 1e-3
ID_FRACTION = 0.999
PSNR_MIN = 45.0


def psnr(a, b, peak=1.0):
    mse = float(np.mean((np.asarray(a, dtype=np.float64) - np.asarray(b, dtype=np.float64)) ** 2))
    return float("inf") if mse == 0 else 10.0 * np.log10(peak * peak / mse)


def frame_parity(depth, ids, image, ref_depth, ref_id, ref_image=None, ref_planes=None, ref_scene_ids=None,
                 depth_tol=DEPTH_TOL):
    """Returns a dict of measurements and a list of violations."""
    depth = np.asarray(depth, dtype=np.float64)
    ids = np.asarray(ids)
    rep = {}
    bad = []
    same = ids == ref_id
    rep["id_match"] = float(same.mean())
    if rep["id_match"] < ID_FRACTION:
        bad.append(f"id match {rep['id_match']:.5f} < {ID_FRACTION}")
    mism = ~same
    if mism.any() and ref_planes is not None and ref_scene_ids is not None:
        # a mismatch is allowed only where the two surfaces' reference depths are within tolerance
        idx = {int(i): k for k, i in enumerate(ref_scene_ids)}
        flat_m = np.flatnonzero(mism.ravel())
        pl = ref_planes.reshape(len(ref_scene_ids), -1)
        for p in flat_m:
            a, b = int(ref_id.ravel()[p]), int(ids.ravel()[p])
            da = pl[idx[a], p] if a >= 0 else np.inf
            db = pl[idx[b], p] if b >= 0 else np.inf
            if not (np.isfinite(da) and np.isfinite(db) and abs(da - db) <= depth_tol):
                bad.append(f"id mismatch at pixel {p}: ref {a} ({da}) vs {b} ({db})")
                break
    both = same & (ref_id >= 0)
    if both.any():
        err = np.abs(depth[both] - ref_depth[both])
        rep["depth_max_err"] = float(err.max())
        rep["depth_n_over"] = int((err > depth_tol).sum())
        if rep["depth_max_err"] > depth_tol:
            bad.append(f"depth max err {rep['depth_max_err']:.3e} > {depth_tol} on {rep['depth_n_over']} px")
    miss_ok = np.array_equal(np.isinf(depth[same & (ref_id < 0)]), np.ones(int((same & (ref_id < 0)).sum()), bool))
    if not miss_ok:
        bad.append("missed pixels must have depth +inf")
    if ref_image is not None and image is not None:
        rep["psnr"] = psnr(image, ref_image)
        if rep["psnr"] < PSNR_MIN:
            bad.append(f"PSNR {rep['psnr']:.2f} dB < {PSNR_MIN}")
    return rep, bad
