"""Scene files and keyframe animation, host side: the
schema's validation behaviour (the reference's tests/test_scene.py cases), the
animation math, and agreement with the REAL reference's load_scene /
evaluate_animation / dumps_scene on the committed scene files
(tests/golden/scene_poses.npz, make_golden.py gen_scenes)."""

import hashlib
import json
from pathlib import Path

import numpy as np
import pytest

from paper_2308_04669_b200 import configs as CF
from paper_2308_04669_b200 import scene as S
from paper_2308_04669_b200.errors import SceneValidationError

ROOT = Path(__file__).resolve().parent.parent

BASE = {
    "version": 1,
    "camera": {"position": [0, 0, -5], "look_at": [0, 0, 0], "fov_deg": 45, "width": 32, "height": 32},
    "clear_color": [0, 0, 0],
    "lights": [{"type": "point", "position": [0, 5, 0], "beta": 0.4}],
    "objects": [{"id": 0, "geometry": {"type": "sphere", "center": [0, 0, 0], "radius": 1.0},
                 "transform": {"translation": [0, 0, 0], "rotation_quat": [1, 0, 0, 0], "scale": 1.0}}],
}


def doc(**kw):
    d = json.loads(json.dumps(BASE))
    d.update(kw)
    return d


def rot_z(a):
    c, s = np.cos(a), np.sin(a)
    return np.array([[c, -s, 0.0], [s, c, 0.0], [0.0, 0.0, 1.0]])


def track(*keys):
    return S.AnimationTrack(tuple((t, S.QuatTransform(np.asarray(tr, dtype=np.float64),
                                                      np.asarray(q, dtype=np.float64), s)) for t, tr, q, s in keys))


# --- quaternions ---------------------------------------------------------

def test_quaternion_identity_and_round_trip():
    np.testing.assert_allclose(S.quat_to_matrix([1.0, 0, 0, 0]), np.eye(3))
    rng = np.random.default_rng(4)
    for _ in range(200):
        q, _ = np.linalg.qr(rng.normal(size=(3, 3)))
        if np.linalg.det(q) < 0:
            q[:, 0] *= -1
        np.testing.assert_allclose(S.quat_to_matrix(S.matrix_to_quat(q)), q, atol=1e-12)
        assert S.matrix_to_quat(q)[0] >= 0                       # canonical sign


def test_slerp_halfway_and_near_parallel():
    mid = S.quat_to_matrix(S.quat_slerp([1.0, 0, 0, 0], S.matrix_to_quat(rot_z(np.pi / 2)), 0.5))
    np.testing.assert_allclose(mid, rot_z(np.pi / 4), atol=1e-12)
    q = S.matrix_to_quat(rot_z(1e-3))                            # cos > 0.9995: normalised lerp
    np.testing.assert_allclose(S.quat_to_matrix(S.quat_slerp([1.0, 0, 0, 0], q, 0.5)), rot_z(5e-4), atol=1e-9)
    # shortest arc: the negated key is the same rotation
    qb = S.matrix_to_quat(rot_z(2.0))
    np.testing.assert_allclose(S.quat_slerp([1.0, 0, 0, 0], -qb, 0.5), S.quat_slerp([1.0, 0, 0, 0], qb, 0.5))


# --- loading / validation --------------------------------------------------

def test_minimal_scene_defaults():
    d = S.loads_scene(json.dumps(doc()))
    assert len(d.objects) == 1 and d.objects[0].nedf_model is None
    cam = d.camera()
    assert (cam.width, cam.height) == (32, 32) and cam.fov_y == pytest.approx(np.pi / 4)
    assert d.render_config().clear_color == (0.0, 0.0, 0.0)
    assert len(d.build_lights()) == 1


@pytest.mark.parametrize("mutate,where", [
    (lambda d: d["objects"].append(dict(d["objects"][0])), "objects[1].id"),
    (lambda d: d["objects"][0]["transform"].update(rotation_quat=[1, 0, 0]), "objects[0].transform.rotation_quat"),
    (lambda d: d["objects"][0]["transform"].update(rotation_quat=[2, 0, 0, 0]), "not unit length"),
    (lambda d: d["objects"][0]["transform"].update(scale=0.0), "objects[0].transform.scale"),
    (lambda d: d["objects"][0]["transform"].update(translation=[0, 0]), "objects[0].transform.translation"),
    (lambda d: d["objects"][0].update(geometry={"type": "blob"}), "objects[0].geometry"),
    (lambda d: d["objects"][0].update(geometry={"type": "sphere"}), "objects[0].geometry"),
    (lambda d: d["objects"][0].pop("geometry"), "objects[0].geometry: missing"),
    (lambda d: d["objects"][0].pop("id"), "objects[0].id: missing"),
    (lambda d: d["objects"][0].update(id=-3), "objects[0].id: must be non-negative"),
    (lambda d: d.update(version=99), "version"),
    (lambda d: d["camera"].pop("look_at"), "camera"),
    (lambda d: d["lights"].append({"type": "spot"}), "lights[1].type"),
    (lambda d: d["lights"].append({"type": "directional", "direction": [0, 0, 0]}), "lights[1].direction"),
    (lambda d: d["objects"][0].update(animation={"keyframes": []}), "objects[0].animation.keyframes"),
    (lambda d: d["objects"][0].update(animation={"keyframes": [{"transform": {}}]}),
     "objects[0].animation.keyframes[0].time"),
    (lambda d: d["objects"][0].update(animation={"keyframes": [{"time": 1.0}, {"time": 1.0}]}),
     "objects[0].animation"),
])
def test_invalid_fields_are_named(mutate, where):
    d = doc()
    mutate(d)
    with pytest.raises(SceneValidationError) as e:
        S.loads_scene(json.dumps(d))
    assert where in str(e.value)


def test_duplicate_id_names_both_and_bad_json():
    d = doc()
    d["objects"].append(dict(d["objects"][0]))
    with pytest.raises(SceneValidationError) as e:
        S.loads_scene(json.dumps(d))
    assert "objects[1].id" in str(e.value) and "objects[0]" in str(e.value)
    with pytest.raises(SceneValidationError):
        S.loads_scene("{not json")


def test_missing_model_file(tmp_path):
    d = doc()
    d["objects"][0]["nedf_model"] = "missing.nedm"
    (tmp_path / "s.json").write_text(json.dumps(d))
    with pytest.raises(SceneValidationError) as e:
        S.load_scene(tmp_path / "s.json")
    assert "nedf_model" in str(e.value)


def test_composite_geometry_nodes():
    d = doc()
    d["objects"][0]["geometry"] = {"type": "union", "children": [
        {"type": "box", "half_extents": [1, 2, 3]},
        {"type": "transformed", "transform": {"translation": [0, 4, 0]},
         "child": {"type": "torus", "major_r": 1.0, "minor_r": 0.2}}]}
    desc = S.loads_scene(json.dumps(d))
    inst_geom = S.build_oracle(desc.objects[0].geometry, "g", Path("."))
    bb = inst_geom.bounding_box
    np.testing.assert_allclose(bb.min, [-1.2, -2.0, -3.0])
    np.testing.assert_allclose(bb.max, [1.2, 4.2, 3.0])


def test_dump_load_is_a_fixed_point():
    d = doc()
    d["objects"][0]["animation"] = {"keyframes": [{"time": 0.0, "transform": {"translation": [0, 0, 0]}},
                                                  {"time": 1.0, "transform": {"translation": [1, 0, 0]}}]}
    t1 = S.dumps_scene(S.loads_scene(json.dumps(d)))
    assert S.dumps_scene(S.loads_scene(t1)) == t1


# --- animation -------------------------------------------------------------

def test_animation_semantics():
    tr = track((0.0, [0, 0, 0], [1, 0, 0, 0], 1.0), (2.0, [4, 0, 0], [1, 0, 0, 0], 2.0))
    g = S.evaluate_animation(tr, 2.0)
    np.testing.assert_allclose(g.translation, [4, 0, 0])
    assert g.scale == pytest.approx(2.0)
    tr = track((0.0, [0, 0, 0], [1, 0, 0, 0], 1.0), (1.0, [2, 4, -6], [1, 0, 0, 0], 4.0))
    g = S.evaluate_animation(tr, 0.5)
    np.testing.assert_allclose(g.translation, [1, 2, -3])
    assert g.scale == pytest.approx(2.0)                        # log-linear
    tr = track((1.0, [1, 1, 1], [1, 0, 0, 0], 1.0), (2.0, [5, 5, 5], [1, 0, 0, 0], 1.0))
    np.testing.assert_allclose(S.evaluate_animation(tr, 0.0).translation, [1, 1, 1])   # clamped
    np.testing.assert_allclose(S.evaluate_animation(tr, 9.0).translation, [5, 5, 5])
    tr = track((0.0, [0, 0, 0], [1, 0, 0, 0], 1.0), (1.0, [0, 0, 0], S.matrix_to_quat(rot_z(np.pi / 2)), 1.0))
    np.testing.assert_allclose(S.evaluate_animation(tr, 0.5).rotation, rot_z(np.pi / 4), atol=1e-12)
    with pytest.raises(ValueError):
        track((0.0, [0, 0, 0], [1, 0, 0, 0], 1.0), (0.0, [1, 0, 0], [1, 0, 0, 0], 1.0))
    rng = np.random.default_rng(1)
    q, _ = np.linalg.qr(rng.normal(size=(3, 3)))
    if np.linalg.det(q) < 0:
        q[:, 0] *= -1
    tr = track((0.0, [0, 0, 0], [1, 0, 0, 0], 0.5), (1.0, [1, 2, 3], S.matrix_to_quat(q), 3.0))
    for t in np.linspace(-0.5, 1.5, 41):
        R = S.evaluate_animation(tr, t).rotation
        assert np.abs(R.T @ R - np.eye(3)).max() < 1e-12


# --- the committed scene files against the real reference -------------------

def test_scene_files_match_reference_loader(golden):
    """scenes/config5.json through our loader: canonical dump byte-identical to the
    reference's dumps_scene, keyframe poses equal to the reference's
    evaluate_animation (to float64 rounding of the SVD)."""
    g = golden("scene_poses.npz")
    desc = S.load_scene(ROOT / "scenes" / "config5.json")
    assert S.dumps_scene(desc) == bytes(g["dump"]).decode()
    for i, t in enumerate(g["times"]):
        for j, spec in enumerate(desc.objects):
            p = S.evaluate_animation(spec.animation, float(t))
            np.testing.assert_allclose(p.rotation, g["R"][i, j], rtol=0, atol=1e-14)
            np.testing.assert_allclose(p.translation, g["T"][i, j], rtol=0, atol=0)
            assert p.scale == g["s"][i, j]


def test_config5_scene_file_is_the_config5_spin():
    """The keyframe tracks reproduce configs.config5_frame's rotation at every frame."""
    desc = S.load_scene(ROOT / "scenes" / "config5.json")
    for f in (0, 7, 23, 38, 59, 60):
        spec = CF.config5_frame(f)
        for o, so in zip(desc.objects, spec.objects):
            p = S.evaluate_animation(o.animation, f / CF.CONFIG5_FPS)
            np.testing.assert_allclose(p.rotation, so.R, atol=1e-12)
            np.testing.assert_allclose(p.translation, so.T, atol=0)


def test_scene_files_are_up_to_date():
    """scenes/*.json are what scripts/make_scene_files.py writes from configs.py."""
    spec = CF.config4()
    docs = {"config4.json": S.scene_document(spec, lambda o: f"models/{S.model_file_name(o.kind, o.seed)}"),
            "config5.json": S.scene_document(spec, lambda o: f"models/{S.model_file_name(o.kind, o.seed)}",
                                             animation=CF.config5_keyframes()),
            "config4_trained.json": S.scene_document(spec, lambda o: f"../tests/golden/trained_{o.kind}.nedm")}
    for name, d in docs.items():
        assert json.loads((ROOT / "scenes" / name).read_text()) == json.loads(json.dumps(d)), name


def test_random_init_model_files_match_reference(tmp_path):
    """ensure_random_init_models writes the exact bytes of the reference's
    new_model + save_nedf (sha256 from tests/golden/models.json)."""
    ref = json.loads((ROOT / "tests" / "golden" / "models.json").read_text())
    pairs = [("sphere", 0), ("box", 1), ("torus", 5)]
    S.ensure_random_init_models(tmp_path, pairs)
    for kind, seed in pairs:
        raw = (tmp_path / S.model_file_name(kind, seed)).read_bytes()
        assert hashlib.sha256(raw).hexdigest() == ref[f"{seed}:{kind}"]["sha256"]
