"""Pin the CPU oracle against outputs of the real reference (tests/golden/).

The fixtures were produced by `tests/golden/make_golden.py` running the
unmodified reference; these checks make the oracle a trustworthy checker for
the CUDA path (CPU only)."""

import hashlib
import json
from pathlib import Path

import numpy as np
import pytest

from oracle import nedf_oracle as O
from paper_2308_04669_b200 import configs as C
from tests.conftest import GOLDEN, ROOT
from tests.helpers import oracle_model, oracle_scene


def test_clip_and_encoding(golden):
    z = golden("geometry.npz")
    t0, t1, hit = O.slab_clip(z["origins"], z["dirs"], z["box_min"], z["box_max"])
    np.testing.assert_array_equal(hit, z["hit"])
    np.testing.assert_array_equal(t0[hit], z["t0"][hit])
    np.testing.assert_array_equal(t1[hit], z["t1"][hit])
    feats, h2 = O.encode_rays(z["origins"], z["dirs"], z["box_min"], z["box_max"])
    np.testing.assert_array_equal(h2, z["hit"])
    np.testing.assert_allclose(feats[z["enc_rows"]], z["enc"], rtol=0, atol=1e-12)


def test_primary_rays(golden):
    z = golden("geometry.npz")
    cam = O.Cam(np.array([1.0, 2.0, 3.0]), O.look_at([1, 2, 3], [0, 0, 0]), 0.8, 7, 5)
    o, d = O.primary_rays(cam)
    np.testing.assert_allclose(d, z["cam_dirs"], atol=1e-15)
    np.testing.assert_array_equal(o, z["cam_origins"])
    # pixel subsets are exact
    sub = np.array([0, 5, 34])
    o2, d2 = O.primary_rays(cam, sub)
    np.testing.assert_array_equal(d2, d[sub])


@pytest.mark.parametrize("key", json.loads((GOLDEN / "models.json").read_text()).keys())
def test_random_init_matches_reference_bytes(key):
    ref = json.loads((GOLDEN / "models.json").read_text())[key]
    seed, kind = key.split(":")
    m = oracle_model(int(seed), kind)
    raw = O.nedm_bytes(m)
    assert len(raw) == ref["bytes"]
    assert hashlib.sha256(raw).hexdigest() == ref["sha256"]
    assert m.half_range == ref["half_range"]
    np.testing.assert_array_equal(m.box_min, ref["box_min"])


@pytest.mark.parametrize("name", ["0_sphere", "1_box", "5_torus", "2_sphere"])
def test_forward_and_queries(golden, name):
    z = golden(f"forward_{name}.npz")
    seed, kind = name.split("_")
    m = oracle_model(int(seed), kind)
    mu, alpha, hit, logits = O.query_local(m, z["origins"], z["dirs"], return_logits=True)
    np.testing.assert_array_equal(hit, z["hit"])
    lc, lf, la = logits
    scale = np.abs(z["logits_c"]).max()
    np.testing.assert_allclose(lc, z["logits_c"], rtol=0, atol=1e-9 * scale)
    np.testing.assert_allclose(lf, z["logits_f"], rtol=0, atol=1e-9 * scale)
    np.testing.assert_allclose(la, z["logit_a"], rtol=0, atol=1e-9 * scale)
    np.testing.assert_array_equal(np.isnan(mu), np.isnan(z["mu"]))
    np.testing.assert_array_equal(mu[hit], z["mu"][hit])
    np.testing.assert_array_equal(alpha, z["alpha"])
    depth, walpha = O.world_depth(m, z["R"], z["T"], float(z["s"]), z["world_o"], z["world_d"])
    np.testing.assert_array_equal(walpha, z["world_alpha"])
    ok = np.isfinite(z["world_depth"])
    np.testing.assert_allclose(depth[ok], z["world_depth"][ok], rtol=1e-12, atol=1e-12)


def _check_frame(out, z, shadows=True):
    np.testing.assert_array_equal(out.id, z["id"])
    fin = np.isfinite(z["depth"])
    np.testing.assert_array_equal(np.isfinite(out.depth), fin)
    np.testing.assert_allclose(out.depth[fin], z["depth"][fin], rtol=1e-12, atol=1e-12)
    if "rgb" in z:
        np.testing.assert_allclose(out.rgb, z["rgb"], atol=1e-12)
        np.testing.assert_array_equal(out.shadow, z["shadow"])
        np.testing.assert_allclose(out.image, z["image"], atol=1e-12)


def test_frame_config1(golden):
    objs, cam, lights, cfg = oracle_scene(C.config1())
    out = O.render(objs, cam, [], cfg, threads=4)
    _check_frame(out, golden("frame_config1.npz"))


@pytest.mark.parametrize("fname,spec", [("frame_config4_200x80.npz", C.config4(200, 80)),
                                        ("frame_config3_160x64.npz", C.config3(160, 64)),
                                        ("frame_config5_f7_100x40.npz", C.config5_frame(7, width=100, height=40)),
                                        ("frame_config5_f38_100x40.npz", C.config5_frame(38, width=100, height=40))])
def test_frame_small_configs(golden, fname, spec):
    z = golden(fname)
    objs, cam, lights, cfg = oracle_scene(spec)
    out = O.render(objs, cam, lights, cfg, threads=4)
    _check_frame(out, z)
    for k, ob in enumerate(objs):
        np.testing.assert_allclose(out.planes[ob.id], z["planes"][k], rtol=1e-12, atol=1e-12)


def test_frame_pixel_subset_is_exact(golden):
    z = golden("frame_config4_200x80.npz")
    objs, cam, lights, cfg = oracle_scene(C.config4(200, 80))
    pix = np.random.default_rng(0).choice(200 * 80, size=500, replace=False)
    out = O.render(objs, cam, lights, cfg, pixels=pix, threads=4)
    np.testing.assert_array_equal(out.id, z["id"].ravel()[pix])
    np.testing.assert_allclose(out.image, z["image"].reshape(-1, 3)[pix], atol=1e-12)


def test_frame_two_lights(golden):
    spec = C.config4(96, 40)
    spec.objects = spec.objects[:4]
    spec.lights = [C.LightSpec("point", (0.0, 6.0, -2.0), 0.4),
                   C.LightSpec("directional", (0.0, -1.0, 0.0), 0.3)]
    objs, cam, lights, cfg = oracle_scene(spec)
    out = O.render(objs, cam, lights, cfg, threads=4)
    _check_frame(out, golden("frame_twolights_96x40.npz"))


def test_analytic_backend_frame(golden):
    z = golden("frame_analytic_48.npz")
    slab = ("box", (0.0, 0.0, 0.0), (4.0, 0.5, 4.0))
    sph = ("sphere", (0.0, 0.0, 0.0), 0.5)
    objs = [O.Obj(0, np.eye(3), np.array([0, -0.5, 0.0]), 1.0, slab),
            O.Obj(1, np.eye(3), np.array([0, 2.5, 0.0]), 1.0, sph)]
    cam = O.Cam(np.array([0, 2.5, 5.5]), O.look_at([0, 2.5, 5.5], [0, 0.5, 0]), 1.1, 48, 48)
    out = O.render(objs, cam, [O.Light("point", np.array([0, 5.0, 0]), 0.4)])
    _check_frame(out, z)
    out2 = O.render(objs, cam, [O.Light("directional", np.array([0, -1.0, 0]), 0.3)])
    np.testing.assert_array_equal(out2.shadow, z["shadow_dir"])
    np.testing.assert_allclose(out2.image, z["image_dir"], atol=1e-12)


def test_voxel_sample(golden):
    z = golden("voxel_probe.npz")
    prim = ("voxel", z["density"].shape, z["bmin"], z["bmax"], z["density"], z["color"])
    rgb, sig = O.voxel_sample(prim, z["points"])
    np.testing.assert_allclose(rgb, z["rgb"], atol=1e-14)
    np.testing.assert_allclose(sig, z["sigma"], atol=1e-14)


def test_resample_frame(golden):
    z = golden("frame_resample_100x40.npz")
    spec = C.config4(100, 40)
    spec.resample = True
    objs, cam, lights, cfg = oracle_scene(spec)
    out = O.render(objs, cam, lights, cfg, threads=4)
    _check_frame(out, z)
    assert out.resampled / (100 * 40) == pytest.approx(float(z["resample_ratio"]))


@pytest.mark.parametrize("tag,resample", [("plain", False), ("rs", True)])
def test_voxel_mixed_frame(golden, tag, resample):
    z = golden("frame_voxel_mixed_64x48.npz")
    vox = ("voxel", z["density"].shape, z["bmin"], z["bmax"], z["density"], z["color"])
    sph = ("sphere", (0.0, 0.0, 0.0), 0.6)
    objs = [O.Obj(3, np.eye(3), np.zeros(3), 1.0, vox, model=oracle_model(0, "sphere")),
            O.Obj(5, np.eye(3), np.array([1.2, 0.3, -1.5]), 1.0, sph)]
    cam = O.Cam(np.array([0.5, 1.0, -5.0]), O.look_at([0.5, 1.0, -5.0], [0, 0, 0]), 0.9, 64, 48)
    out = O.render(objs, cam, [O.Light("point", np.array([2.0, 4.0, -3.0]), 0.35)],
                   O.Config(resample=resample, clear_color=(0.1, 0.2, 0.3)), threads=4)
    np.testing.assert_array_equal(out.id, z[f"id_{tag}"])
    fin = np.isfinite(z[f"depth_{tag}"])
    np.testing.assert_allclose(out.depth[fin], z[f"depth_{tag}"][fin], rtol=1e-12, atol=1e-12)
    np.testing.assert_array_equal(out.shadow, z[f"shadow_{tag}"])
    np.testing.assert_allclose(out.image, z[f"image_{tag}"], atol=1e-12)


def test_nedm_format_errors():
    m = oracle_model(0, "sphere")
    raw = O.nedm_bytes(m)
    with pytest.raises(ValueError):
        O.parse_nedm(b"XXXX" + raw[4:])
    with pytest.raises(ValueError):
        O.parse_nedm(raw[:-1])
    with pytest.raises(ValueError):
        O.parse_nedm(raw[:20])


@pytest.fixture(scope="module")
def trained():
    return {k: O.parse_nedm((GOLDEN / f"trained_{k}.nedm").read_bytes()) for k in ("sphere", "box", "torus")}


def test_hazard_rays(golden, trained):
    """Slab-clip hazards (NaN slabs, edges, grazing edge / corner, signed zeros,
    inside origins) on the trained sphere: clip bit-equal, logits to 1e-9, decisions
    equal to the reference's query_rays."""
    z = golden("hazard_rays.npz")
    m = trained["sphere"]
    t0, t1, hit = O.slab_clip(z["origins"], z["dirs"], m.box_min, m.box_max)
    np.testing.assert_array_equal(hit, z["hit"])
    np.testing.assert_array_equal(t0[hit], z["t0"][hit])
    np.testing.assert_array_equal(t1[hit], z["t1"][hit])
    mu, alpha, h2, (lc, lf, la) = O.query_local(m, z["origins"], z["dirs"], return_logits=True)
    np.testing.assert_array_equal(h2, z["hit"])
    scale = np.abs(z["logits_f"]).max()
    np.testing.assert_allclose(lf, z["logits_f"], rtol=0, atol=1e-9 * scale)
    np.testing.assert_allclose(lc, z["logits_c"], rtol=0, atol=1e-9 * scale)
    np.testing.assert_allclose(la, z["logit_a"], rtol=0, atol=1e-9 * scale)
    np.testing.assert_array_equal(mu[hit], z["mu"][hit])
    np.testing.assert_array_equal(alpha, z["alpha"])


def _desc_objs(desc, models, time=None):
    """Oracle objects for a scene.SceneDescription (scene file -> oracle)."""
    from paper_2308_04669_b200 import scene as S
    objs = []
    for spec in desc.objects:
        g = desc.pose(spec, time)
        geo = spec.geometry
        prim = {"sphere": lambda: ("sphere", tuple(geo["center"]), geo["radius"]),
                "box": lambda: ("box", tuple(geo["center"]), tuple(geo["half_extents"])),
                "torus": lambda: ("torus", tuple(geo["center"]), geo["major_r"], geo["minor_r"])}[geo["type"]]()
        key = str((desc.base_dir / spec.nedf_model).resolve())
        if key not in models:
            models[key] = O.parse_nedm(Path(key).read_bytes())
        objs.append(O.Obj(spec.id, np.asarray(g.rotation), np.asarray(g.translation), float(g.scale), prim,
                          model=models[key]))
    c = desc.camera()
    cam = O.Cam(np.asarray(c.position), np.asarray(c.orientation), c.fov_y, c.width, c.height)
    return objs, cam


def test_trained_frame_pixels(golden):
    """The oracle on the trained fixtures through scenes/config4_trained.json:
    a pixel sample of the reference's 1000x400 frame."""
    from paper_2308_04669_b200 import scene as S
    g = golden("frame_trained_1000x400.npz")
    desc = S.load_scene(ROOT / "scenes" / "config4_trained.json")
    desc.camera_spec["width"], desc.camera_spec["height"] = 1000, 400
    objs, cam = _desc_objs(desc, {})
    lights = [O.Light("point", np.asarray(L["position"], dtype=np.float64), L["beta"]) for L in desc.lights]
    pix = np.random.default_rng(1).choice(1000 * 400, size=1500, replace=False)
    out = O.render(objs, cam, lights, O.Config(), pixels=pix, threads=8)
    np.testing.assert_array_equal(out.id, g["id"].ravel()[pix])
    fin = np.isfinite(out.depth)
    np.testing.assert_allclose(out.depth[fin], g["depth"].ravel()[pix][fin], rtol=2e-7)
    np.testing.assert_allclose(out.image, g["image_u16"].reshape(-1, 3)[pix] / 65535.0, atol=1e-5)


@pytest.mark.parametrize("frame", [7, 38])
def test_scene_file_config5_frames(golden, frame):
    """config 5 posed by the keyframe tracks of scenes/config5.json (reference
    load_scene + evaluate_animation) -- the oracle reproduces the frames."""
    from paper_2308_04669_b200 import scene as S
    S.ensure_random_init_models(ROOT / "scenes" / "models", [("sphere", 0), ("box", 1), ("torus", 5)])
    z = golden(f"frame_config5json_f{frame}_100x40.npz")
    desc = S.load_scene(ROOT / "scenes" / "config5.json")
    desc.camera_spec["width"], desc.camera_spec["height"] = 100, 40
    objs, cam = _desc_objs(desc, {}, time=frame / C.CONFIG5_FPS)
    L = C.config5_light(frame)
    out = O.render(objs, cam, [O.Light("point", np.asarray(L.vec, dtype=np.float64), L.beta)], O.Config(), threads=4)
    _check_frame(out, z)
