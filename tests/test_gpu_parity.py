"""Parity of the CUDA path (through the C ABI) with the reference's golden
outputs and the oracle.  Needs a B200."""

import numpy as np
import pytest

from oracle import nedf_oracle as O
from paper_2308_04669_b200 import configs as CF
from tests.helpers import oracle_model, oracle_scene
from tests.parity import frame_parity, psnr

pytestmark = pytest.mark.gpu

PRECISIONS = ["fp32", "auto"]


@pytest.fixture(scope="module")
def nedf():
    import paper_2308_04669_b200 as P
    from paper_2308_04669_b200 import _lib, model, pipeline, scenes
    return P, _lib, model, pipeline, scenes


def set_precision(nedf, prec):
    P, _lib, *_ = nedf
    ctx = _lib.context()
    ctx.set_option(_lib.OPT_PRECISION, {"fp32": _lib.PREC_FP32, "auto": _lib.PREC_AUTO,
                                        "tensor": _lib.PREC_TENSOR}[prec])


@pytest.mark.parametrize("name", ["0_sphere", "1_box", "5_torus", "2_sphere"])
def test_forward_logits_fp32(nedf, golden, name):
    P, _lib, model, pipeline, scenes = nedf
    z = golden(f"forward_{name}.npz")
    seed, kind = name.split("_")
    m = scenes.paper_model(int(seed), kind)
    om = oracle_model(int(seed), kind)
    feats, hit = O.encode_rays(z["origins"], z["dirs"], om.box_min, om.box_max)
    lc, lf, la = model.forward(m, feats[hit])
    scale = np.abs(z["logits_c"]).max()
    for got, ref in [(lc, z["logits_c"]), (lf, z["logits_f"]), (la[:, 0], z["logit_a"])]:
        err = np.abs(got - ref).max() / scale
        assert err < 2e-5, err


@pytest.mark.parametrize("prec", PRECISIONS)
@pytest.mark.parametrize("name", ["0_sphere", "1_box", "5_torus", "2_sphere"])
def test_query_rays_and_world(nedf, golden, name, prec):
    P, _lib, model, pipeline, scenes = nedf
    set_precision(nedf, prec)
    z = golden(f"forward_{name}.npz")
    seed, kind = name.split("_")
    m = scenes.paper_model(int(seed), kind)
    mu, alpha = model.query_rays(m, z["origins"], z["dirs"])
    np.testing.assert_array_equal(np.isnan(mu), np.isnan(z["mu"]))
    hit = ~np.isnan(z["mu"])
    np.testing.assert_array_equal(mu[hit], z["mu"][hit])
    np.testing.assert_array_equal(alpha, z["alpha"])
    from paper_2308_04669_b200.geometry import RigidTransform
    g = RigidTransform(z["R"], z["T"], float(z["s"]))
    depth, walpha = model.query_depth_world_batch(m, g, z["world_o"], z["world_d"])
    np.testing.assert_array_equal(walpha, z["world_alpha"])
    ok = np.isfinite(z["world_depth"])
    np.testing.assert_allclose(depth[ok], z["world_depth"][ok], rtol=0, atol=1e-9)
    np.testing.assert_array_equal(np.isnan(depth), np.isnan(z["world_depth"]))


def _render(nedf, spec, prec, planes=False):
    P, _lib, model, pipeline, scenes = nedf
    set_precision(nedf, prec)
    scene, cam, lights, cfg = scenes.build(spec)
    buf = pipeline.FrameBuffers(cam.width, cam.height, keep_planes=planes)
    res = pipeline.compose_frame(scene, cam, lights, cfg, buffers=buf)
    return res, buf.numpy(), res.image.cpu().numpy()


@pytest.mark.parametrize("prec", PRECISIONS)
def test_config1_step1_matches_reference(nedf, golden, prec):
    z = golden("frame_config1.npz")
    P, _lib, model, pipeline, scenes = nedf
    set_precision(nedf, prec)
    spec = CF.config1()
    scene, cam, lights, cfg = scenes.build(spec)
    buf = pipeline.FrameBuffers(cam.width, cam.height)
    pipeline.nedf_generation_step(scene, cam, buf)
    b = buf.numpy()
    rep, bad = frame_parity(b["depth"], b["id"], None, z["depth"], z["id"])
    assert not bad, (rep, bad)


@pytest.mark.parametrize("prec", PRECISIONS)
@pytest.mark.parametrize("fname,spec_fn", [("frame_config4_200x80.npz", lambda: CF.config4(200, 80)),
                                           ("frame_config3_160x64.npz", lambda: CF.config3(160, 64)),
                                           ("frame_config5_f7_100x40.npz", lambda: CF.config5_frame(7, width=100, height=40)),
                                           ("frame_config5_f38_100x40.npz", lambda: CF.config5_frame(38, width=100, height=40))])
def test_small_frames_match_reference(nedf, golden, fname, spec_fn, prec):
    z = golden(fname)
    spec = spec_fn()
    res, b, img = _render(nedf, spec, prec)
    rep, bad = frame_parity(b["depth"], b["id"], img, z["depth"], z["id"], z["image"], z["planes"],
                            [o.id for o in spec.objects])
    assert not bad, (rep, bad)
    np.testing.assert_allclose(b["rgb"], z["rgb"], atol=2e-3)
    assert (np.abs(b["shadow"] - z["shadow"]) > 1e-6).mean() < 1e-3


@pytest.mark.parametrize("prec", PRECISIONS)
def test_two_lights(nedf, golden, prec):
    z = golden("frame_twolights_96x40.npz")
    spec = CF.config4(96, 40)
    spec.objects = spec.objects[:4]
    spec.lights = [CF.LightSpec("point", (0.0, 6.0, -2.0), 0.4), CF.LightSpec("directional", (0.0, -1.0, 0.0), 0.3)]
    res, b, img = _render(nedf, spec, prec)
    rep, bad = frame_parity(b["depth"], b["id"], img, z["depth"], z["id"], z["image"])
    assert not bad, (rep, bad)
    np.testing.assert_allclose(b["shadow"], z["shadow"], atol=1e-6)


def test_analytic_backend(nedf, golden):
    P, _lib, model, pipeline, scenes = nedf
    from paper_2308_04669_b200 import fields as F
    from paper_2308_04669_b200.geometry import RigidTransform, vec3
    z = golden("frame_analytic_48.npz")
    sph = F.AnalyticOracle(F.Sphere(vec3(0, 0, 0), 0.5))
    slab = F.AnalyticOracle(F.BoxPrim(vec3(0, 0, 0), vec3(4.0, 0.5, 4.0)))
    scene = [pipeline.SceneInstance(0, RigidTransform(np.eye(3), vec3(0, -0.5, 0)), pipeline.OracleDepthBackend(slab), slab),
             pipeline.SceneInstance(1, RigidTransform(np.eye(3), vec3(0, 2.5, 0)), pipeline.OracleDepthBackend(sph), sph)]
    cam = pipeline.Camera(vec3(0, 2.5, 5.5), pipeline.look_at([0, 2.5, 5.5], [0, 0.5, 0]), 1.1, 48, 48)
    res = pipeline.compose_frame(scene, cam, [pipeline.PointLight(vec3(0, 5, 0), 0.4)])
    b = res.buffers.numpy()
    np.testing.assert_array_equal(b["id"], z["id"])
    fin = np.isfinite(z["depth"])
    np.testing.assert_allclose(b["depth"][fin], z["depth"][fin], atol=1e-9)
    np.testing.assert_allclose(b["shadow"], z["shadow"], atol=1e-6)
    assert psnr(res.image.cpu().numpy(), z["image"]) > 60
    res2 = pipeline.compose_frame(scene, cam, [pipeline.DirectionalLight(vec3(0, -1, 0), 0.3)])
    np.testing.assert_allclose(res2.buffers.shadow.cpu().numpy(), z["shadow_dir"], atol=1e-6)


def test_empty_scene_and_errors(nedf):
    P, _lib, model, pipeline, scenes = nedf
    from paper_2308_04669_b200.geometry import vec3
    cam = pipeline.Camera(vec3(0, 0, -5), pipeline.look_at([0, 0, -5], [0, 0, 0]), 0.8, 4, 4)
    buf = pipeline.FrameBuffers(4, 4)
    pipeline.nedf_generation_step([], cam, buf)
    assert np.all(np.isinf(buf.depth.cpu().numpy()))
    assert np.all(buf.id.cpu().numpy() == -1)
    with pytest.raises(ValueError):
        pipeline.PointLight(vec3(0, 0, 0), beta=1.5)
    with pytest.raises(P.FormatError):
        model.loads_nedf(b"XXXX" + bytes(100))
