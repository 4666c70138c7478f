#!/usr/bin/env python3
"""Generate the golden fixtures under tests/golden/ by running the REAL
reference implementation (`/root/reference/pkg/src/nedf`).

Run in the build container only (the GPU box has no /root/reference):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Every fixture records the reference call that produced it.  The oracle
(`oracle/nedf_oracle.py`) is pinned against these files by
`tests/test_oracle_golden.py`, and the CUDA path is checked against them by
the `-m gpu` tests.
"""

from __future__ import annotations

import hashlib
import importlib.util
import json
import os
import sys
import tempfile
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent

os.environ.setdefault("OPENBLAS_NUM_THREADS", str(os.cpu_count() or 1))

import nedf  # noqa: E402  (the reference, via PYTHONPATH)
from nedf import fields, geometry, model, nn, pipeline  # noqa: E402

assert "/root/reference" in nedf.__file__, nedf.__file__

_spec = importlib.util.spec_from_file_location("cfgs", ROOT / "paper_2308_04669_b200" / "configs.py")
cfgs = importlib.util.module_from_spec(_spec)
sys.modules["cfgs"] = cfgs
_spec.loader.exec_module(cfgs)

pipeline.set_thread_count(os.cpu_count() or 1)

CANON = {
    "sphere": lambda: fields.Sphere(geometry.vec3(0, 0, 0), 1.0),
    "box": lambda: fields.BoxPrim(geometry.vec3(0, 0, 0), geometry.vec3(0.8, 0.5, 0.6)),
    "torus": lambda: fields.Torus(geometry.vec3(0, 0, 0), 0.7, 0.25),
}

_model_cache: dict = {}


def paper_model(seed: int, kind: str):
    """new_model(..., PROFILES['paper']) round-tripped through .nedm."""
    key = (seed, kind)
    if key not in _model_cache:
        oracle = fields.AnalyticOracle(CANON[kind]())
        m = model.new_model(oracle, np.random.default_rng(seed), profile=model.PROFILES["paper"])
        with tempfile.TemporaryDirectory() as td:
            p = Path(td) / "m.nedm"
            model.save_nedf(m, p)
            raw = p.read_bytes()
            m2 = model.load_nedf(p)
        _model_cache[key] = (m2, raw)
    return _model_cache[key]


def ref_scene(spec):
    scene = []
    for o in spec.objects:
        m, _ = paper_model(o.seed, o.kind)
        oracle = fields.AnalyticOracle(CANON[o.kind]())
        g = geometry.RigidTransform(np.asarray(o.R), np.asarray(o.T, dtype=np.float64), o.s)
        scene.append(pipeline.SceneInstance(id=o.id, transform=g,
                                            depth=pipeline.NedfDepthBackend(m), radiance=oracle))
    c = spec.camera
    cam = pipeline.Camera(position=np.asarray(c.position, dtype=np.float64),
                          orientation=pipeline.look_at(c.position, c.look_at, c.up),
                          fov_y=c.fov_y, width=c.width, height=c.height)
    lights = []
    for L in spec.lights:
        if L.kind == "point":
            lights.append(pipeline.PointLight(np.asarray(L.vec, dtype=np.float64), L.beta))
        else:
            lights.append(pipeline.DirectionalLight(np.asarray(L.vec, dtype=np.float64), L.beta))
    cfg = pipeline.RenderConfig(shadows=spec.shadows, resample=spec.resample)
    return scene, cam, lights, cfg


def save(name, **arrays):
    np.savez_compressed(HERE / name, **arrays)
    print("wrote", name, {k: getattr(v, "shape", v) for k, v in arrays.items()})


def gen_geometry():
    rng = np.random.default_rng(11)
    box = geometry.Aabb(geometry.vec3(-1.5, -1.2, -0.9), geometry.vec3(1.5, 1.2, 0.9))
    n = 96
    v = rng.normal(size=(n, 3))
    v /= np.linalg.norm(v, axis=1, keepdims=True)
    o = 4.0 * v
    tgt = rng.uniform(-2.5, 2.5, size=(n, 3))
    d = tgt - o
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    # a few axis-parallel rays with origins on slab planes (NaN slab case)
    o[:4] = [[-1.5, 0.0, -3.0], [0.2, 1.2, -3.0], [3.0, 0.0, 0.9], [0.0, -5.0, 0.0]]
    d[:4] = [[0.0, 0.0, 1.0], [0.0, 0.0, 1.0], [-1.0, 0.0, 0.0], [0.0, 1.0, 0.0]]
    t0, t1, hit = geometry.clip_rays_to_aabb(o, d, box)
    feats, hit2 = geometry.sample_and_encode_rays(o, d, box)
    assert np.array_equal(hit, hit2)
    sel = np.flatnonzero(hit)[:12]
    cam = pipeline.Camera(position=geometry.vec3(1, 2, 3),
                          orientation=pipeline.look_at([1, 2, 3], [0, 0, 0]),
                          fov_y=0.8, width=7, height=5)
    po, pd = pipeline.generate_primary_rays(cam)
    save("geometry.npz", origins=o, dirs=d, box_min=box.min, box_max=box.max,
         t0=t0, t1=t1, hit=hit, enc_rows=sel, enc=feats[sel],
         cam_dirs=pd, cam_origins=po)


def gen_models():
    out = {}
    for seed, kind in [(0, "sphere"), (1, "box"), (5, "torus"), (0, "box"), (1, "sphere"),
                       (0, "torus"), (5, "sphere"), (1, "torus"), (5, "box"), (2, "sphere")]:
        m, raw = paper_model(seed, kind)
        out[f"{seed}:{kind}"] = {"sha256": hashlib.sha256(raw).hexdigest(), "bytes": len(raw),
                                 "half_range": m.config.half_range,
                                 "box_min": list(m.relaxed_box.min), "box_max": list(m.relaxed_box.max)}
    (HERE / "models.json").write_text(json.dumps(out, indent=1) + "\n")
    print("wrote models.json")


def gen_forward():
    for seed, kind in [(0, "sphere"), (1, "box"), (5, "torus"), (2, "sphere")]:
        m, _ = paper_model(seed, kind)
        sampler = model.RaySampler(box=m.relaxed_box)
        o, d = sampler.sample(np.random.default_rng(100 + seed), 64)
        feats, hit = geometry.sample_and_encode_rays(o, d, m.relaxed_box)
        lc, lf, la, _ = nn.forward(m.mlp, feats[hit])
        mu, alpha = model.query_rays(m, o, d)
        # a placed object: world rays through a random rigid transform
        rng = np.random.default_rng(200 + seed)
        R = cfgs.random_rotation(rng)
        T = rng.uniform(-2, 2, size=3)
        s = float(rng.uniform(0.5, 1.5))
        g = geometry.RigidTransform(R, T, s)
        wo = g.apply_points(o)
        wd = d @ R.T
        wdepth, walpha = model.query_depth_world_batch(m, g, wo, wd)
        save(f"forward_{seed}_{kind}.npz", origins=o, dirs=d, hit=hit,
             logits_c=lc, logits_f=lf, logit_a=la[:, 0], mu=mu, alpha=alpha,
             R=R, T=T, s=s, world_o=wo, world_d=wd, world_depth=wdepth, world_alpha=walpha)


def gen_frames():
    # config 1 at full size, STEP 1 only (nedf_generation_step)
    spec = cfgs.config1()
    scene, cam, lights, cfg = ref_scene(spec)
    buf = pipeline.FrameBuffers(cam.width, cam.height)
    pipeline.nedf_generation_step(scene, cam, buf)
    save("frame_config1.npz", depth=buf.depth, id=buf.id)

    # config 4 scene at 1/100 of the pixels (same camera/fov), full compose_frame
    for name, spec in [("frame_config4_200x80.npz", cfgs.config4(200, 80)),
                       ("frame_config3_160x64.npz", cfgs.config3(160, 64))]:
        scene, cam, lights, cfg = ref_scene(spec)
        res = pipeline.compose_frame(scene, cam, lights, cfg)
        b = res.buffers
        planes = np.stack([b.per_object_depth[i.id] for i in scene])
        save(name, depth=b.depth, id=b.id, rgb=b.rgb, shadow=b.shadow, image=res.image,
             planes=planes)

    # a 4-object scene with a directional light and a point light (multi-light)
    spec = cfgs.config4(96, 40)
    spec.objects = spec.objects[:4]
    spec.lights = [cfgs.LightSpec("point", (0.0, 6.0, -2.0), 0.4),
                   cfgs.LightSpec("directional", (0.0, -1.0, 0.0), 0.3)]
    scene, cam, lights, cfg = ref_scene(spec)
    res = pipeline.compose_frame(scene, cam, lights, cfg)
    b = res.buffers
    save("frame_twolights_96x40.npz", depth=b.depth, id=b.id, rgb=b.rgb, shadow=b.shadow,
         image=res.image)


def _frame_compact(res, scene):
    """A full-size frame stored compactly: depth f32 at covered pixels, id int16,
    image u16 (quantised to 1/65535: PSNR contribution > 100 dB), and per pixel the
    second-nearest object plane (f32 depth, id) so a GPU id mismatch can be checked
    against the north star's "two surfaces within tolerance" rule."""
    b = res.buffers
    H, W = b.id.shape
    planes = np.stack([b.per_object_depth[i.id] for i in scene]).reshape(len(scene), -1)
    ids = np.array([i.id for i in scene])
    order = np.argsort(planes, axis=0, kind="stable")
    second = order[1] if len(scene) > 1 else np.zeros(H * W, dtype=np.int64)
    d2 = planes[second, np.arange(H * W)]
    id2 = np.where(np.isfinite(d2), ids[second], -1)
    return dict(depth=b.depth.astype(np.float32), id=b.id.astype(np.int16),
                image_u16=np.round(np.clip(res.image, 0, 1) * 65535).astype(np.uint16),
                shadow_u8=np.round(b.shadow * 250).astype(np.uint8),
                second_depth=np.where(np.isfinite(d2), d2, np.inf).astype(np.float32).reshape(H, W),
                second_id=id2.astype(np.int16).reshape(H, W), scene_ids=ids)


def gen_fullsize():
    """The bench workload itself: config 4 at 2000x800 through the reference's
    compose_frame (about 4 min on 8 cores), stored compactly (_frame_compact)."""
    import time
    spec = cfgs.config4()
    scene, cam, lights, cfg = ref_scene(spec)
    t = time.time()
    res = pipeline.compose_frame(scene, cam, lights, cfg)
    print(f"config4 2000x800 reference frame: {time.time() - t:.1f} s")
    save("frame_config4_2000x800.npz", **_frame_compact(res, scene))


def _scene_models():
    """scenes/models/*.nedm (the random-init files the scene JSONs name), written
    from the reference's own new_model + save_nedf bytes."""
    d = ROOT / "scenes" / "models"
    d.mkdir(parents=True, exist_ok=True)
    for kind, seed in (("sphere", 0), ("box", 1), ("torus", 5)):
        p = d / f"{kind}_seed{seed}.nedm"
        if not p.exists():
            p.write_bytes(paper_model(seed, kind)[1])


def _ref_frame_from_desc(desc, time=None, width=None, height=None, lights=None):
    from nedf import scene as rscene  # noqa: F401
    if width is not None:
        desc.camera_spec["width"], desc.camera_spec["height"] = width, height
    inst = desc.instantiate(time)
    res = pipeline.compose_frame(inst, desc.camera(), lights if lights is not None else desc.build_lights(),
                                 desc.render_config())
    return inst, res


def gen_scenes():
    """Scene files through the reference's load_scene (scene.py:310-366) and
    evaluate_animation (scene.py:128-144): poses of the config-5 keyframe tracks,
    the canonical dump, and frames of config 5 rendered from the JSON."""
    from nedf import scene as rscene
    _scene_models()
    desc = rscene.load_scene(ROOT / "scenes" / "config5.json")
    times = np.concatenate([np.linspace(-0.5, 5.5, 25), np.array([7, 38]) / 12.0])
    R = np.zeros((len(times), len(desc.objects), 3, 3))
    T = np.zeros((len(times), len(desc.objects), 3))
    S = np.zeros((len(times), len(desc.objects)))
    for i, t in enumerate(times):
        for j, spec in enumerate(desc.objects):
            g = rscene.evaluate_animation(spec.animation, float(t))
            R[i, j], T[i, j], S[i, j] = g.rotation, g.translation, g.scale
    dump = rscene.dumps_scene(desc)
    save("scene_poses.npz", times=times, R=R, T=T, s=S,
         dump=np.frombuffer(dump.encode(), dtype=np.uint8))
    for f in (7, 38):
        d = rscene.load_scene(ROOT / "scenes" / "config5.json")
        L = cfgs.config5_light(f)
        inst, res = _ref_frame_from_desc(d, time=f / 12.0, width=100, height=40,
                                         lights=[pipeline.PointLight(np.asarray(L.vec, dtype=np.float64), L.beta)])
        b = res.buffers
        save(f"frame_config5json_f{f}_100x40.npz", depth=b.depth, id=b.id, rgb=b.rgb, shadow=b.shadow,
             image=res.image, planes=np.stack([b.per_object_depth[i.id] for i in inst]))


def gen_trained():
    """Config-4 placements with the GPU-distilled paper-profile fixtures
    (tests/golden/trained_*.nedm, scripts/distill_fixtures.py) through the
    reference's load_scene + compose_frame: at 1000x400 with the stored alpha
    threshold (0.5), and at 400x160 with the same weights under an alpha
    threshold of 0.625 (model.py:354-369)."""
    import shutil
    import struct
    import time
    from nedf import scene as rscene
    src = ROOT / "scenes" / "config4_trained.json"
    t = time.time()
    desc = rscene.load_scene(src)
    inst, res = _ref_frame_from_desc(desc, width=1000, height=400)
    print(f"trained config4 1000x400: {time.time() - t:.1f} s")
    save("frame_trained_1000x400.npz", **_frame_compact(res, inst))
    with tempfile.TemporaryDirectory() as td:
        td = Path(td)
        (td / "scenes").mkdir()
        (td / "tests" / "golden").mkdir(parents=True)
        for kind in ("sphere", "box", "torus"):
            raw = (HERE / f"trained_{kind}.nedm").read_bytes()
            (td / "tests" / "golden" / f"trained_{kind}.nedm").write_bytes(raw[:-4] + struct.pack("<f", 0.625))
        shutil.copy(src, td / "scenes" / src.name)
        desc = rscene.load_scene(td / "scenes" / src.name)
        assert all(abs(desc.shared_model(o.nedf_model).alpha_threshold - 0.625) < 1e-9 for o in desc.objects)
        inst, res = _ref_frame_from_desc(desc, width=400, height=160)
        b = res.buffers
        save("frame_trained_a0625_400x160.npz", depth=b.depth, id=b.id, rgb=b.rgb, shadow=b.shadow,
             image=res.image, planes=np.stack([b.per_object_depth[i.id] for i in inst]))


def gen_hazard():
    """Slab-clip hazards (geometry.py:258-280) through the
    reference's query_rays (model.py:277-293) on the trained sphere fixture (relaxed
    box [-1.5, 1.5]^3): rays on slab planes parallel to an axis (0 * inf = NaN ->
    widened slab), along box edges, grazing an edge / corner (t_exit == t_enter, 16
    identical sample points), signed-zero directions, origins inside the box, boxes
    behind the origin, plus the random rays of geometry.npz."""
    m = model.load_nedf(HERE / "trained_sphere.nedm")
    box = m.relaxed_box
    b = 1.5
    r2 = 1.0 / np.sqrt(2.0)
    rows = [
        ((-b, 0.0, -3.0), (0.0, 0.0, 1.0)),          # on the x = min plane, parallel to it
        ((b, 0.0, -3.0), (0.0, 0.0, 1.0)),           # on the x = max plane
        ((b, b, -3.0), (0.0, 0.0, 1.0)),             # along an edge
        ((-b, -b, -3.0), (0.0, 0.0, 1.0)),
        ((0.0, b, -3.0), (0.0, 0.0, 1.0)),
        ((2.0, 0.0, -3.0), (0.0, 0.0, 1.0)),         # parallel, outside the slab: miss
        ((0.0, -3.0, 0.0), (r2, r2, 0.0)),           # grazes the edge x = b, y = -b (t0 == t1 up to rounding)
        ((0.0, 0.0, -3.0), (0.0, 0.0, 1.0)),         # straight through the centre
        ((0.0, 0.0, 0.0), (0.0, 0.0, 1.0)),          # origin at the centre: t0 clamps to 0
        ((0.3, -0.2, 1.4), (0.1, 0.2, -0.9)),        # origin inside
        ((0.0, 0.0, 3.0), (0.0, 0.0, 1.0)),          # box behind the origin: miss
        ((-0.0, 0.0, -3.0), (-0.0, -0.0, 1.0)),      # signed zeros
        ((-3.0, -3.0, -3.0), (1.0, 1.0, 1.0)),       # through two corners
        ((-3.0, b, b), (1.0, 0.0, 0.0)),             # along the edge y = z = max
        ((b + 1e-12, 0.0, -3.0), (0.0, 0.0, 1.0)),   # just outside a plane: miss
        ((b - 1e-12, 0.0, -3.0), (0.0, 0.0, 1.0)),   # just inside
    ]
    o = np.array([r[0] for r in rows], dtype=np.float64)
    d = np.array([r[1] for r in rows], dtype=np.float64)
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    # corner graze: from outside, aimed exactly at the corner (b, b, b) along a direction that only touches it
    oc = np.array([[b + 1.0, b + 1.0, b - 1.0]])
    dc = np.array([[-1.0, -1.0, 1.0]]) / np.sqrt(3.0)
    g = np.load(HERE / "geometry.npz")
    o = np.concatenate([o, oc, g["origins"]])
    d = np.concatenate([d, dc, g["dirs"]])
    t0, t1, hit = geometry.clip_rays_to_aabb(o, d, box)
    mu, alpha = model.query_rays(m, o, d)
    feats, h2 = geometry.sample_and_encode_rays(o, d, box)
    assert np.array_equal(hit, h2)
    lc, lf, la, _ = nn.forward(m.mlp, feats[hit])
    save("hazard_rays.npz", origins=o, dirs=d, t0=t0, t1=t1, hit=hit, mu=mu, alpha=alpha,
         logits_c=lc, logits_f=lf, logit_a=la[:, 0], n_special=len(rows) + 1)


def gen_dynamic():
    # config 5 (dynamic scene): two frames of the 60-frame sequence -- objects rotated by different
    # amounts about y and the point light elsewhere on its orbit -- at 1/400 of the pixels
    for f in (7, 38):
        spec = cfgs.config5_frame(f, width=100, height=40)
        scene, cam, lights, cfg = ref_scene(spec)
        res = pipeline.compose_frame(scene, cam, lights, cfg)
        b = res.buffers
        planes = np.stack([b.per_object_depth[i.id] for i in scene])
        save(f"frame_config5_f{f}_100x40.npz", depth=b.depth, id=b.id, rgb=b.rgb, shadow=b.shadow,
             image=res.image, planes=planes)


def gen_analytic():
    """Oracle-backend scene (sphere tracing) from the reference's own shadow
    test (test_pipeline.py:211-217), plus a voxel radiance probe."""
    sph = fields.AnalyticOracle(fields.Sphere(geometry.vec3(0, 0, 0), 0.5))
    slab = fields.AnalyticOracle(fields.BoxPrim(geometry.vec3(0, 0, 0), geometry.vec3(4.0, 0.5, 4.0)))
    scene = [pipeline.SceneInstance(0, geometry.RigidTransform(np.eye(3), geometry.vec3(0, -0.5, 0)),
                                    pipeline.OracleDepthBackend(slab), slab),
             pipeline.SceneInstance(1, geometry.RigidTransform(np.eye(3), geometry.vec3(0, 2.5, 0)),
                                    pipeline.OracleDepthBackend(sph), sph)]
    cam = pipeline.Camera(position=geometry.vec3(0, 2.5, 5.5),
                          orientation=pipeline.look_at([0, 2.5, 5.5], [0, 0.5, 0]),
                          fov_y=1.1, width=48, height=48)
    res = pipeline.compose_frame(scene, cam, [pipeline.PointLight(geometry.vec3(0, 5, 0), 0.4)])
    b = res.buffers
    res2 = pipeline.compose_frame(scene, cam, [pipeline.DirectionalLight(geometry.vec3(0, -1, 0), 0.3)])
    save("frame_analytic_48.npz", depth=b.depth, id=b.id, rgb=b.rgb, shadow=b.shadow,
         image=res.image, shadow_dir=res2.buffers.shadow, image_dir=res2.image)

    rng = np.random.default_rng(5)
    res_ = (5, 4, 3)
    dens = rng.uniform(0, 3, size=res_)
    col = rng.uniform(0, 1, size=res_ + (3,))
    vf = fields.VoxelField(res_, geometry.Aabb(geometry.vec3(-1, -1, -1), geometry.vec3(1, 1.5, 1)),
                           dens, col)
    pts = rng.uniform(-1.3, 1.7, size=(200, 3))
    rgb, sig = vf.sample(pts)
    save("voxel_probe.npz", density=dens, color=col, bmin=vf.bounds.min, bmax=vf.bounds.max,
         points=pts, rgb=rgb, sigma=sig)




def gen_extra():
    """Outlier resampling (pipeline.py:336-350) and voxel appearance
    (fields.py:294-319, 477-508) on NeDF-backed objects."""
    spec = cfgs.config4(100, 40)
    spec.resample = True
    scene, cam, lights, cfg = ref_scene(spec)
    res = pipeline.compose_frame(scene, cam, lights, cfg)
    b = res.buffers
    save("frame_resample_100x40.npz", depth=b.depth, id=b.id, rgb=b.rgb, shadow=b.shadow, image=res.image,
         resample_ratio=res.timing["resample_ratio"])

    rng = np.random.default_rng(9)
    res_ = (6, 5, 7)
    vf = fields.VoxelField(res_, geometry.Aabb(geometry.vec3(-1.2, -1.0, -1.1), geometry.vec3(1.1, 1.3, 1.0)),
                           rng.uniform(0, 2, size=res_), rng.uniform(0, 1, size=res_ + (3,)))
    vox = fields.VoxelOracle(vf)
    m, _ = paper_model(0, "sphere")
    sph = fields.AnalyticOracle(fields.Sphere(geometry.vec3(0, 0, 0), 0.6))
    scene = [pipeline.SceneInstance(3, geometry.RigidTransform(np.eye(3), geometry.vec3(0.0, 0.0, 0.0), 1.0),
                                    pipeline.NedfDepthBackend(m), vox),
             pipeline.SceneInstance(5, geometry.RigidTransform(np.eye(3), geometry.vec3(1.2, 0.3, -1.5), 1.0),
                                    pipeline.OracleDepthBackend(sph), sph)]
    cam = pipeline.Camera(position=geometry.vec3(0.5, 1.0, -5.0),
                          orientation=pipeline.look_at([0.5, 1.0, -5.0], [0, 0, 0]), fov_y=0.9, width=64, height=48)
    light = pipeline.PointLight(geometry.vec3(2.0, 4.0, -3.0), 0.35)
    out = {}
    for rs in (False, True):
        r = pipeline.compose_frame(scene, cam, [light], pipeline.RenderConfig(resample=rs, clear_color=(0.1, 0.2, 0.3)))
        tag = "rs" if rs else "plain"
        out[f"depth_{tag}"] = r.buffers.depth
        out[f"id_{tag}"] = r.buffers.id
        out[f"image_{tag}"] = r.image
        out[f"shadow_{tag}"] = r.buffers.shadow
    save("frame_voxel_mixed_64x48.npz", density=vf.density, color=vf.color, bmin=vf.bounds.min, bmax=vf.bounds.max,
         **out)


def gen_imgio():
    """Reference imgio.py conversions (to_u8, depth_to_gray, 16-bit id PNG values) on
    planes with the edge cases: values around the u8 rounding boundaries, out of
    range, misses (+inf), depth ties (round half to even), ids past 65534."""
    from nedf import imgio
    import io as _io
    from PIL import Image
    rng = np.random.default_rng(42)
    rgb = rng.uniform(-0.2, 1.2, size=(16, 24, 3))
    k = rng.integers(0, 256, size=(16, 24, 3))
    rgb[::3] = (k[::3] + 0.5) / 255.0                        # exactly on rounding boundaries
    rgb = rgb.astype(np.float32).astype(np.float64)          # the GPU image is float32
    depth = rng.uniform(0.5, 9.0, size=(16, 24))
    depth[rng.random((16, 24)) < 0.3] = np.inf
    depth[0, :4] = [1.0, 2.0, 3.0, 1.0 + 8.0 * 0.5 / 255.0]
    ids = rng.integers(-1, 70000, size=(16, 24)).astype(np.int32)
    ids[0, :3] = [-1, 65534, 65535]
    u16 = np.asarray(Image.open(_io.BytesIO(imgio.encode_id_png(ids))))
    save("imgio.npz", rgb=rgb, u8=imgio.to_u8(rgb), depth=depth, gray=imgio.depth_to_gray(depth),
         ids=ids, id_u16=u16.astype(np.uint16), depth_raw=np.frombuffer(_raw_depth(imgio, depth), dtype=np.uint8))


def _raw_depth(imgio, depth):
    import tempfile
    with tempfile.NamedTemporaryFile(suffix=".ndpt") as f:
        imgio.write_depth_raw(f.name, depth, 2.5)
        return open(f.name, "rb").read()


def gen_train():
    """One reference training step (model.py:210-248, nn.py:218-232) on a desk-profile
    sphere model (d_feat 64, 4 blocks) with f32-exact weights: the batch drawn by
    RaySampler(seed 7, 256 rays), its targets, the three losses, all gradients and the
    parameters after one Adam step."""
    import tempfile
    from nedf import model as M, nn
    oracle = fields.AnalyticOracle(fields.Sphere(geometry.vec3(0, 0, 0), 1.0))
    nm = M.new_model(oracle, np.random.default_rng(3), M.PROFILES["desk"])
    with tempfile.NamedTemporaryFile(suffix=".nedm") as f:
        M.save_nedf(nm, f.name)
        raw = open(f.name, "rb").read()
        nm = M.load_nedf(f.name)
    sampler = M.RaySampler(box=nm.relaxed_box)
    rng = np.random.default_rng(7)
    origins, dirs = sampler.sample(np.random.default_rng(7), 256)      # the rays the batch draws first
    batch = M.build_training_batch(oracle, sampler, nm.config, rng, batch_size=256)
    total, parts, grads = M.loss_and_grads(nm.mlp, batch)
    params = nm.mlp.parameters()
    state = nn.AdamState.for_params(params, lr=5e-4)
    nn.adam_step(state, params, grads)
    flat = lambda xs: np.concatenate([np.asarray(x, dtype=np.float64).ravel() for x in xs])
    save("train_step.npz", raw=np.frombuffer(raw, dtype=np.uint8), origins=origins, dirs=dirs,
         feats=batch.encoded, coarse=batch.target_coarse.argmax(axis=1), fine=batch.target_fine.argmax(axis=1),
         hit=batch.valid_mu, total=total, parts=np.array(parts), grads=flat(grads), params_after=flat(params))


if __name__ == "__main__":
    which = sys.argv[1:] or ["geometry", "models", "forward", "analytic", "frames", "dynamic", "extra", "imgio",
                             "train"]
    for w in which:
        globals()[f"gen_{w}"]()
