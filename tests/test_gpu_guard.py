"""The near-tie guard's fp32-accurate re-evaluation on tcgen05 (guard_tc.cu:
tf32 + bf16 split products, 4-CTA clusters, M = 64 weights x N = 16 rays)
against the float64 oracle (the reference's nn.forward, nn.py:115-135) and the
warp-level mma.sync kernel it replaces, at the logit level and through the
decisions of query_rays (model.py:277-293)."""

import numpy as np
import pytest

from oracle import nedf_oracle as O
from paper_2308_04669_b200 import configs as CF
from tests.helpers import oracle_model
from tests.test_gpu_scene import _diag_logits

pytestmark = pytest.mark.gpu

GUARD_TC, GUARD_SYNC, GUARD_PRECISE = 16 + 1, 16 + 2, 16 + 3


def _mods():
    from paper_2308_04669_b200 import _lib, model, scenes
    return _lib, model, scenes


@pytest.mark.parametrize("seed,kind", [(0, "sphere"), (1, "box"), (5, "torus")])
@pytest.mark.parametrize("n", [1, 16, 37, 700, 5000])
def test_guard_logits_match_float64(seed, kind, n):
    """Every ray through the guard kernel alone: logits within float32-level error of the
    float64 forward pass (|err| <= 1e-5 max|logit|, the 3xTF32 mma.sync kernel's level);
    1, 16, 37 and 700 rays exercise partial tiles, one tile, tile tails and several rounds."""
    _lib, model, scenes = _mods()
    m = scenes.paper_model(seed, kind)
    o, d = CF.sweep_rays(n, m.relaxed_box.min, m.relaxed_box.max, seed=5 + n)
    om = oracle_model(seed, kind)
    _, _, hit, (rc, rf, ra) = O.query_local(om, o, d, return_logits=True)
    assert hit.sum() > 0
    scale = max(np.abs(rc).max(), np.abs(rf).max(), np.abs(ra).max())
    errs = {}
    for name, prec in (("tcgen05", GUARD_TC), ("mma_sync", GUARD_SYNC), ("precise", GUARD_PRECISE)):
        lc, lf, la = _diag_logits(m, o, d, prec)
        e = max(np.abs(lc[hit] - rc).max(), np.abs(lf[hit] - rf).max(), np.abs(la[hit] - ra.ravel()).max())
        errs[name] = e / scale
        assert np.isnan(lc[~hit]).all()                     # box misses never reach the network
    print(seed, kind, n, errs)
    assert errs["tcgen05"] < 1e-5, errs
    assert errs["tcgen05"] < 4 * errs["mma_sync"] + 2e-6, errs
    assert errs["precise"] < 1e-5, errs


@pytest.mark.parametrize("kernel", ["tcgen05", "mma_sync4", "mma_sync8", "precise", "auto"])
@pytest.mark.parametrize("n_rays", [3000, 300, 60])
def test_guard_kernels_match_fp32_path(n_rays, kernel):
    """With the guard threshold at 100% of max|logit| every ray is re-evaluated by the
    guard kernel; its decisions must match the streaming fp32 kernel's (NEDF_PREC_FP32)
    up to fp32 summation-order ties, and depths to float32 accuracy."""
    _lib, model, scenes = _mods()
    ctx = _lib.context()
    m = scenes.paper_model(1, "box")
    o, d = CF.sweep_rays(n_rays, m.relaxed_box.min, m.relaxed_box.max, seed=11)
    ctx.set_option(_lib.OPT_PRECISION, _lib.PREC_FP32)
    mu32, a32 = model.query_rays(m, o, d)
    ctx.set_option(_lib.OPT_PRECISION, _lib.PREC_AUTO)
    ctx.set_option(_lib.OPT_GUARD_PPM, 1_000_000)
    ctx.set_option(_lib.OPT_GUARD_KERNEL, {"tcgen05": _lib.GUARD_TCGEN05, "precise": _lib.GUARD_PRECISE,
                                           "auto": _lib.GUARD_AUTO}.get(kernel, _lib.GUARD_MMA_SYNC))
    ctx.set_option(_lib.OPT_GUARD_CLUSTER, 8 if kernel == "mma_sync8" else 4)
    try:
        mug, ag = model.query_rays(m, o, d)
    finally:
        ctx.set_option(_lib.OPT_GUARD_PPM, 3000)
        ctx.set_option(_lib.OPT_GUARD_KERNEL, _lib.GUARD_AUTO)
        ctx.set_option(_lib.OPT_GUARD_CLUSTER, 0)
    allowed = max(1, n_rays // 1000)
    assert (ag != a32).sum() <= allowed
    fin = np.isfinite(mu32) & np.isfinite(mug)
    same = np.abs(mug[fin] - mu32[fin]) <= 1e-12
    assert (~same).sum() <= allowed
    fine = 2 * m.config.half_range / m.n_coarse / m.n_fine
    assert np.all(np.abs(mug[fin] - mu32[fin]) <= fine * 1.0001 + 2 * m.config.half_range / m.n_coarse)


def test_frame_guard_kernels_agree():
    """A config-4 frame with each guard kernel: identical ids, depths within float32 error
    of each other (the guarded rays are near-ties by construction, so a rare flip between
    two fp32-accurate kernels is allowed only where the reference planes tie within 1e-3)."""
    import torch
    from paper_2308_04669_b200 import pipeline
    _lib, model, scenes = _mods()
    ctx = _lib.context()
    scene, cam, lights, cfg = scenes.build(CF.config4(400, 160))
    out = {}
    for k in (_lib.GUARD_TCGEN05, _lib.GUARD_MMA_SYNC):
        ctx.set_option(_lib.OPT_GUARD_KERNEL, k)
        r = pipeline.compose_frame(scene, cam, lights, cfg)
        torch.cuda.synchronize()
        out[k] = r.buffers.numpy()
        assert r.timing["guarded_evals"] > 0
    ctx.set_option(_lib.OPT_GUARD_KERNEL, _lib.GUARD_AUTO)
    a, b = out[_lib.GUARD_TCGEN05], out[_lib.GUARD_MMA_SYNC]
    assert (a["id"] != b["id"]).sum() <= 2
    fin = np.isfinite(a["depth"]) & np.isfinite(b["depth"])
    assert (np.abs(a["depth"][fin] - b["depth"][fin]) > 1e-3).sum() <= 2


def test_trained_frame_guard_kernels_agree():
    """The trained config-4 scene (a third of its evaluations are near-ties): the frame with
    the throughput guard (auto picks it for large batches) equals the frame with the
    latency guard up to fp32-level ties, and the auto mode really took the throughput path
    (guarded work finishes far faster than the latency kernel's)."""
    import torch
    from pathlib import Path
    from paper_2308_04669_b200 import pipeline, scene as S
    _lib, model, scenes = _mods()
    ctx = _lib.context()
    desc = S.load_scene(Path(__file__).resolve().parent.parent / "scenes" / "config4_trained.json")
    inst = desc.instantiate()
    cam = desc.camera()
    cam = pipeline.Camera(cam.position, cam.orientation, cam.fov_y, 500, 200)
    out, times = {}, {}
    ctx.set_option(_lib.OPT_PROFILE, 1)
    try:
        for k in (_lib.GUARD_AUTO, _lib.GUARD_TCGEN05):
            ctx.set_option(_lib.OPT_GUARD_KERNEL, k)
            ctx.read_stats(_lib.stream_handle())
            buf = pipeline.FrameBuffers(cam.width, cam.height)
            pipeline.FrameRenderer(inst, cam, desc.build_lights(), desc.render_config(), buffers=buf).render()
            torch.cuda.synchronize()
            st = ctx.read_stats(_lib.stream_handle())
            out[k] = buf.numpy()
            times[k] = st["guard_ms"]
            assert st["guarded"] > 5000, st
    finally:
        ctx.set_option(_lib.OPT_GUARD_KERNEL, _lib.GUARD_AUTO)
        ctx.set_option(_lib.OPT_PROFILE, 0)
    a, b = out[_lib.GUARD_AUTO], out[_lib.GUARD_TCGEN05]
    print("guard ms auto / latency kernel:", times)
    assert (a["id"] != b["id"]).sum() <= 3
    fin = np.isfinite(a["depth"]) & np.isfinite(b["depth"])
    assert (np.abs(a["depth"][fin] - b["depth"][fin]) > 1e-3).sum() <= 0.001 * fin.sum()
    assert times[_lib.GUARD_AUTO] < 0.5 * times[_lib.GUARD_TCGEN05]
