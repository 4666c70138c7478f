"""STEP 1 front-first culling (NEDF_OPT_CULL): each pixel's NeDF pair with the
smallest depth bound |(o - T).d| - s mu_max is evaluated first and the others only
if that bound can still beat the pixel's z-key.  A pair it skips has fp32 depth
above the winner's, so its key could not have won the atomicMin: every output
buffer must equal the all-pairs frame bit for bit, and the evaluations it saves
plus the ones it runs add up to the all-pairs count (model.py:301-319;
pipeline.py:259-268)."""

from pathlib import Path

import numpy as np
import pytest

from paper_2308_04669_b200 import configs as CF

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parent.parent


def _mods():
    from paper_2308_04669_b200 import _lib, fields, geometry, pipeline, scenes
    return _lib, fields, geometry, pipeline, scenes


def _render(scene, cam, lights, cfg, cull, precision=0, keep_planes=False):
    import torch
    _lib, fields, geometry, pipeline, scenes = _mods()
    ctx = _lib.context()
    ctx.set_option(_lib.OPT_PRECISION, precision)
    ctx.set_option(_lib.OPT_CULL, cull)
    try:
        buf = pipeline.FrameBuffers(cam.width, cam.height, keep_planes=keep_planes)
        ctx.read_stats(_lib.stream_handle())
        pipeline.FrameRenderer(scene, cam, lights, cfg, buffers=buf).render()
        torch.cuda.synchronize()
        st = ctx.read_stats(_lib.stream_handle())
    finally:
        ctx.set_option(_lib.OPT_CULL, 1)
        ctx.set_option(_lib.OPT_PRECISION, _lib.PREC_AUTO)
    b = buf.numpy()
    b["image"] = buf.image.cpu().numpy()
    return b, st


def _check(scene, cam, lights, cfg, precision=0, expect_cut=True):
    off, st_off = _render(scene, cam, lights, cfg, 0, precision)
    on, st_on = _render(scene, cam, lights, cfg, 1, precision)
    for k in ("depth", "id", "rgb", "shadow", "image"):
        np.testing.assert_array_equal(on[k], off[k], err_msg=k)
    assert st_off["culled"] == 0
    assert st_on["evals"] + st_on["culled"] == st_off["evals"]
    assert st_on["covered"] == st_off["covered"]
    if expect_cut:
        assert st_on["culled"] > 0
    return st_on["culled"] / max(1, st_off["evals"])


def test_config4_bit_identical_and_fewer_evaluations():
    _lib, fields, geometry, pipeline, scenes = _mods()
    scene, cam, lights, cfg = scenes.build(CF.config4(400, 160))
    share = _check(scene, cam, lights, cfg)
    print("culled share of all evaluations", share)


def test_config3_no_lights():
    _lib, fields, geometry, pipeline, scenes = _mods()
    scene, cam, lights, cfg = scenes.build(CF.config3(320, 128))
    _check(scene, cam, [], cfg)


def test_fp32_network_path():
    _lib, fields, geometry, pipeline, scenes = _mods()
    scene, cam, lights, cfg = scenes.build(CF.config4(160, 64))
    _check(scene, cam, lights, cfg, precision=_lib.PREC_FP32)


def test_trained_models():
    """Distilled networks: many pixels' front pair misses (alpha below the threshold),
    so their deferred pairs must all come back."""
    _lib, fields, geometry, pipeline, scenes = _mods()
    from paper_2308_04669_b200 import scene as S
    desc = S.load_scene(ROOT / "scenes" / "config4_trained.json")
    cam = desc.camera()
    cam = pipeline.Camera(cam.position, cam.orientation, cam.fov_y, 500, 200)
    _check(desc.instantiate(), cam, desc.build_lights(), desc.render_config())


def test_mixed_analytic_objects_and_overlaps():
    """Analytic objects set the key before any network pass (their hits can cut NeDF
    pairs); two NeDF objects overlapping in depth keep both pairs."""
    _lib, fields, geometry, pipeline, scenes = _mods()
    m = scenes.paper_model(0, "sphere")
    m2 = scenes.paper_model(1, "box")
    sph = fields.AnalyticOracle(fields.Sphere(geometry.vec3(0, 0, 0), 0.6))
    wall = fields.AnalyticOracle(fields.BoxPrim(geometry.vec3(0, 0, 0), geometry.vec3(3.0, 3.0, 0.1)))
    scene = [pipeline.SceneInstance(3, geometry.RigidTransform(np.eye(3), geometry.vec3(0, 0, 0), 1.0),
                                    pipeline.NedfDepthBackend(m), sph),
             pipeline.SceneInstance(4, geometry.RigidTransform(np.eye(3), geometry.vec3(0.3, 0.1, 0.4), 0.9),
                                    pipeline.NedfDepthBackend(m2), sph),
             pipeline.SceneInstance(5, geometry.RigidTransform(np.eye(3), geometry.vec3(0.0, 0.0, -2.5), 1.0),
                                    pipeline.OracleDepthBackend(wall), wall),
             pipeline.SceneInstance(7, geometry.RigidTransform(np.eye(3), geometry.vec3(-1.5, 0.0, 2.0), 0.7),
                                    pipeline.NedfDepthBackend(m), sph)]
    cam = pipeline.Camera(geometry.vec3(0.4, 0.8, -6.0), pipeline.look_at([0.4, 0.8, -6.0], [0.0, 0.0, 0.0]),
                          0.9, 160, 120)
    lights = [pipeline.PointLight(geometry.vec3(2.0, 4.0, -3.0), 0.35)]
    _check(scene, cam, lights, pipeline.RenderConfig())


def test_plane_cache_turns_culling_off():
    _lib, fields, geometry, pipeline, scenes = _mods()
    scene, cam, lights, cfg = scenes.build(CF.config4(160, 64))
    b, st = _render(scene, cam, lights, cfg, 1, keep_planes=True)
    ref, st_ref = _render(scene, cam, lights, cfg, 0, keep_planes=True)
    assert st["culled"] == 0 and st["evals"] == st_ref["evals"]
    for k in ("depth", "id", "image"):
        np.testing.assert_array_equal(b[k], ref[k], err_msg=k)


# ---- STEP 3 near-tie certainty (NEDF_OPT_SHADOW_CERT) ----
# A flagged shadow ray is finished by the fast kernel when its pair's decision (shadows or not)
# is the same for every bin within the guard margin of the fast maxima and either alpha; the
# shadow factors and the image must equal the all-guarded frame's, with fewer guarded rays.

def _render_cert(scene, cam, lights, cfg, cert):
    import torch
    _lib, fields, geometry, pipeline, scenes = _mods()
    ctx = _lib.context()
    ctx.set_option(_lib.OPT_SHADOW_CERT, cert)
    try:
        buf = pipeline.FrameBuffers(cam.width, cam.height)
        ctx.read_stats(_lib.stream_handle())
        pipeline.FrameRenderer(scene, cam, lights, cfg, buffers=buf).render()
        torch.cuda.synchronize()
        st = ctx.read_stats(_lib.stream_handle())
    finally:
        ctx.set_option(_lib.OPT_SHADOW_CERT, 1)
    b = buf.numpy()
    b["image"] = buf.image.cpu().numpy()
    return b, st


def _check_cert(scene, cam, lights, cfg):
    off, st_off = _render_cert(scene, cam, lights, cfg, 0)
    on, st_on = _render_cert(scene, cam, lights, cfg, 1)
    for k in ("depth", "id", "rgb", "shadow", "image"):
        np.testing.assert_array_equal(on[k], off[k], err_msg=k)
    assert st_on["evals"] == st_off["evals"]
    assert st_on["guarded"] <= st_off["guarded"]
    return st_off["guarded"], st_on["guarded"]


def test_shadow_certainty_config4_full_frame():
    _lib, fields, geometry, pipeline, scenes = _mods()
    scene, cam, lights, cfg = scenes.build(CF.config4())
    g_off, g_on = _check_cert(scene, cam, lights, cfg)
    print("guarded per frame: all", g_off, "undecided only", g_on)
    assert g_on < g_off


def test_shadow_certainty_directional_and_point():
    _lib, fields, geometry, pipeline, scenes = _mods()
    spec = CF.config4(500, 200)
    spec.lights = [CF.LightSpec("directional", (0.0, -0.9805806756909202, 0.19611613513818404), 0.3),
                   CF.LightSpec("point", (1.0, 5.0, -3.0), 0.5)]
    scene, cam, lights, cfg = scenes.build(spec)
    print(_check_cert(scene, cam, lights, cfg))


def test_shadow_certainty_trained_models():
    _lib, fields, geometry, pipeline, scenes = _mods()
    from paper_2308_04669_b200 import scene as S
    desc = S.load_scene(ROOT / "scenes" / "config4_trained.json")
    cam = desc.camera()
    cam = pipeline.Camera(cam.position, cam.orientation, cam.fov_y, 500, 200)
    print(_check_cert(desc.instantiate(), cam, desc.build_lights(), desc.render_config()))
