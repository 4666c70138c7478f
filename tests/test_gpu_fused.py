"""The fused per-pixel passes of nedf_render_frame (STEP 1 resolve + STEP 2 +
shadow fill + the first light's STEP 3 setup in one kernel; the last light's
resolve + composite in one kernel) and the certified fp32 box test of the
setup kernels.  Both are pure re-arrangements of the same float64 arithmetic,
so every buffer must equal the one-kernel-per-step, all-float64 frame bit for
bit, with the same network work (pipeline.py:430-468; geometry.py:258-280)."""

import numpy as np
import pytest

from paper_2308_04669_b200 import configs as CF

pytestmark = pytest.mark.gpu

MODES = [(0, 1), (1, 0), (0, 0), (1, 1)]          # (fuse, setup_exact); the first is the reference arrangement


def _mods():
    from paper_2308_04669_b200 import _lib, fields, geometry, pipeline, scenes
    return _lib, fields, geometry, pipeline, scenes


def _render_all(scene, cam, lights, cfg, rows=None):
    import torch
    _lib, fields, geometry, pipeline, scenes = _mods()
    ctx = _lib.context()
    ctx.set_option(_lib.OPT_PRECISION, _lib.PREC_AUTO)
    out = {}
    try:
        for fuse, exact in MODES:
            ctx.set_option(_lib.OPT_FUSE, fuse)
            ctx.set_option(_lib.OPT_SETUP_EXACT, exact)
            buf = pipeline.FrameBuffers(cam.width, cam.height, rows=rows)
            ctx.read_stats(_lib.stream_handle())
            pipeline.FrameRenderer(scene, cam, lights, cfg, buffers=buf).render()
            torch.cuda.synchronize()
            st = ctx.read_stats(_lib.stream_handle())
            b = buf.numpy()
            b["image"] = buf.image.cpu().numpy()
            out[(fuse, exact)] = (b, st)
    finally:
        ctx.set_option(_lib.OPT_FUSE, 1)
        ctx.set_option(_lib.OPT_SETUP_EXACT, 0)
    return out


def _check_identical(out, max_exact_share=0.05):
    ref, st_ref = out[MODES[0]]
    for mode in MODES[1:]:
        b, st = out[mode]
        for k in ("depth", "id", "rgb", "shadow", "image"):
            np.testing.assert_array_equal(b[k], ref[k], err_msg=f"{mode} {k}")
        assert st["evals"] == st_ref["evals"], mode
        assert st["covered"] == st_ref["covered"], mode
    # exact=1 counts every box test that passed the bounding-sphere test; the certified
    # fp32 test leaves only a small share of them to float64
    all_tests = out[(0, 1)][1]["exact_clips"]
    left = out[(0, 0)][1]["exact_clips"]
    assert all_tests > 0
    assert left <= max_exact_share * all_tests, (left, all_tests)
    return left / all_tests


def test_config4_point_light():
    _lib, fields, geometry, pipeline, scenes = _mods()
    scene, cam, lights, cfg = scenes.build(CF.config4(320, 128))
    share = _check_identical(_render_all(scene, cam, lights, cfg))
    print("exact share", share)


def test_two_lights_directional_first():
    _lib, fields, geometry, pipeline, scenes = _mods()
    spec = CF.config4(160, 64)
    spec.objects = spec.objects[:5]
    spec.lights = [CF.LightSpec("directional", (0.0, -0.9805806756909202, 0.19611613513818404), 0.3), CF.LightSpec("point", (1.0, 5.0, -3.0), 0.5)]
    scene, cam, lights, cfg = scenes.build(spec)
    _check_identical(_render_all(scene, cam, lights, cfg))


def test_no_lights_and_shadows_off():
    _lib, fields, geometry, pipeline, scenes = _mods()
    scene, cam, lights, cfg = scenes.build(CF.config3(160, 64))
    _check_identical(_render_all(scene, cam, [], cfg))
    scene, cam, lights, cfg = scenes.build(CF.config4(160, 64))
    cfg = pipeline.RenderConfig(shadows=False, clear_color=(0.2, 0.1, 0.05))
    _check_identical(_render_all(scene, cam, lights, cfg))


def test_image_tile_rows():
    _lib, fields, geometry, pipeline, scenes = _mods()
    from paper_2308_04669_b200 import distributed as D
    scene, cam, lights, cfg = scenes.build(CF.config4(200, 80))
    _check_identical(_render_all(scene, cam, lights, cfg, rows=D.interleave_rows(cam.height, 1, 3)))


def test_mixed_analytic_and_nedf_objects():
    """Analytic depth backends go through the same per-pixel passes (sphere tracing
    in the setup kernels) next to NeDF objects; a camera looking along a box face
    makes grazing rays the certified test must hand to float64."""
    _lib, fields, geometry, pipeline, scenes = _mods()
    m = scenes.paper_model(0, "sphere")
    sph = fields.AnalyticOracle(fields.Sphere(geometry.vec3(0, 0, 0), 0.6))
    box = fields.AnalyticOracle(fields.BoxPrim(geometry.vec3(0, 0, 0), geometry.vec3(0.8, 0.5, 0.6)))
    scene = [pipeline.SceneInstance(3, geometry.RigidTransform(np.eye(3), geometry.vec3(0, 0, 0), 1.0),
                                    pipeline.NedfDepthBackend(m), box),
             pipeline.SceneInstance(5, geometry.RigidTransform(np.eye(3), geometry.vec3(1.2, 0.3, -1.5), 1.0),
                                    pipeline.OracleDepthBackend(sph), sph),
             pipeline.SceneInstance(7, geometry.RigidTransform(np.eye(3), geometry.vec3(-1.5, 0.0, 0.0), 0.7),
                                    pipeline.NedfDepthBackend(m), sph)]
    # camera on the plane y = 1.5 (the relaxed box's top face of object 3) looking along it
    cam = pipeline.Camera(geometry.vec3(0.0, 1.5, -6.0), pipeline.look_at([0.0, 1.5, -6.0], [0.0, 1.5, 0.0]),
                          0.9, 96, 64)
    lights = [pipeline.PointLight(geometry.vec3(2.0, 4.0, -3.0), 0.35),
              pipeline.DirectionalLight(geometry.vec3(0.0, -1.0, 0.0), 0.5)]
    _check_identical(_render_all(scene, cam, lights, pipeline.RenderConfig()), max_exact_share=0.5)


def test_compose_frame_matches_renderer_and_reports_steps():
    import torch
    _lib, fields, geometry, pipeline, scenes = _mods()
    scene, cam, lights, cfg = scenes.build(CF.config4(200, 80))
    res = pipeline.compose_frame(scene, cam, lights, cfg)
    a = res.buffers.numpy()
    buf = pipeline.FrameBuffers(cam.width, cam.height)
    pipeline.FrameRenderer(scene, cam, lights, cfg, buffers=buf).render()
    torch.cuda.synchronize()
    b = buf.numpy()
    for k in ("depth", "id", "rgb", "shadow"):
        np.testing.assert_array_equal(a[k], b[k])
    np.testing.assert_array_equal(res.image.cpu().numpy(), buf.image.cpu().numpy())
    t = res.timing
    assert t["step1_depth_id"] > 0 and t["step2_shading"] > 0 and t["step3_shadow"] > 0
    assert t["network_evals"] > 0
