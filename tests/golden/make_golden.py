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
