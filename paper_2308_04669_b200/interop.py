"""Adapters from the reference package's objects (`nedf.*`) to this package.

Duck-typed: nothing here imports the reference.  A reference user keeps
building scenes with `nedf.scene` / `nedf.pipeline` and switches the frame (or
only the depth queries) to the GPU:

    from paper_2308_04669_b200 import interop
    result = interop.render_reference_frame(scene, camera, lights, config)   # numpy, like RenderResult

or, keeping the reference's own CPU pipeline and replacing only its plugin seam
(`SceneInstance.depth`, pipeline.py:116-136):

    inst.depth = interop.B200DepthBackend(inst.depth.model)
"""

from __future__ import annotations

import threading
from dataclasses import dataclass

import numpy as np

from . import fields as F
from .geometry import Aabb, RigidTransform
from .model import NedfModel, nedm_image, query_depth_world_batch
from .pipeline import (Camera, DirectionalLight, FrameBuffers, NedfDepthBackend, OracleDepthBackend, PointLight,
                       RenderConfig, SceneInstance, compose_frame)

_model_cache: dict = {}


def model_from_reference(ref_model, device=None) -> NedfModel:
    """Upload a reference `NedfModel` (model.py:102-117): its float64
    parameters are written as the `.nedm` float32 image the reference itself
    saves (nn.py:235-246), so the GPU sees exactly the weights `load_nedf`
    would give."""
    key = (id(ref_model), device)
    hit = _model_cache.get(key)
    if hit is not None and hit[0] is ref_model:
        return hit[1]
    layers = ref_model.mlp.layers()
    raw = nedm_image([(np.asarray(l.weight), np.asarray(l.bias)) for l in layers], ref_model.config.half_range,
                     ref_model.relaxed_box.min, ref_model.relaxed_box.max, ref_model.alpha_threshold)
    m = NedfModel(raw, device)
    _model_cache[key] = (ref_model, m)
    return m


def _transform(g) -> RigidTransform:
    return RigidTransform(np.asarray(g.rotation), np.asarray(g.translation), float(g.scale))


def _aabb(b) -> Aabb:
    return Aabb(np.asarray(b.min), np.asarray(b.max))


def prim_from_reference(p):
    """Reference SDF primitive (fields.py:64-186) -> device field descriptor."""
    name = type(p).__name__
    if name == "Sphere":
        return F.Sphere(p.center, p.radius)
    if name == "BoxPrim":
        return F.BoxPrim(p.center, p.half_extents)
    if name == "Torus":
        return F.Torus(p.center, p.major_r, p.minor_r)
    if name == "Plane":
        return F.Plane(p.normal, p.offset)
    if name == "Union":
        return F.Union(tuple(prim_from_reference(c) for c in p.children))
    if name == "Transformed":
        return F.Transformed(prim_from_reference(p.child), _transform(p.transform))
    raise TypeError(f"unsupported primitive {name}")


def field_from_reference(o):
    """Reference DepthOracle used as appearance (fields.py:456-508)."""
    name = type(o).__name__
    if name == "AnalyticOracle":
        return F.AnalyticOracle(prim_from_reference(o.prim), getattr(o, "t_max", 100.0))
    if name == "VoxelOracle":
        vf = o.vf
        return F.VoxelOracle(F.VoxelField(tuple(vf.resolution), _aabb(vf.bounds), np.asarray(vf.density),
                                          np.asarray(vf.color)))
    raise TypeError(f"unsupported appearance field {name}")


def scene_from_reference(scene, device=None) -> list:
    out = []
    for inst in scene:
        be = inst.depth
        bname = type(be).__name__
        if isinstance(be, (NedfDepthBackend, OracleDepthBackend)):
            depth = be                                   # already this package's (e.g. scene.load_scene)
        elif bname == "NedfDepthBackend":
            depth = NedfDepthBackend(model_from_reference(be.model, device))
        elif bname == "OracleDepthBackend":
            depth = OracleDepthBackend(field_from_reference(be.oracle))
        else:
            raise TypeError(f"unsupported depth backend {bname}")
        out.append(SceneInstance(int(inst.id), _transform(inst.transform), depth, field_from_reference(inst.radiance)))
    return out


def camera_from_reference(c) -> Camera:
    return Camera(np.asarray(c.position), np.asarray(c.orientation), float(c.fov_y), int(c.width), int(c.height),
                  float(getattr(c, "t_near", 0.05)), float(getattr(c, "t_far", 100.0)))


def lights_from_reference(lights) -> list:
    out = []
    for L in lights:
        name = type(L).__name__
        if name == "PointLight":
            out.append(PointLight(np.asarray(L.position), float(L.beta)))
        elif name == "DirectionalLight":
            out.append(DirectionalLight(np.asarray(L.direction), float(L.beta)))
        else:
            raise TypeError(f"unsupported light type {name}")
    return out


def config_from_reference(cfg) -> RenderConfig:
    if cfg is None:
        return RenderConfig()
    return RenderConfig(cfg.sigma_threshold, bool(cfg.resample), int(cfg.resample_samples), cfg.shadow_epsilon,
                        bool(cfg.shadows), tuple(cfg.clear_color))


@dataclass
class HostBuffers:
    """numpy view of FrameBuffers, laid out like the reference's (pipeline.py:211-232)."""
    width: int
    height: int
    depth: np.ndarray
    id: np.ndarray
    rgb: np.ndarray
    shadow: np.ndarray
    per_object_depth: dict


@dataclass
class HostRenderResult:
    image: np.ndarray
    buffers: HostBuffers
    timing: dict


def render_reference_frame(scene, camera, lights, config=None, device=None) -> HostRenderResult:
    """compose_frame on the GPU for reference objects; returns numpy arrays in
    the reference's dtypes (float64 depth/rgb/shadow/image, int32 id)."""
    sc = scene_from_reference(scene, device)
    cam = camera_from_reference(camera)
    buf = FrameBuffers(cam.width, cam.height, device=device, keep_planes=True)
    res = compose_frame(sc, cam, lights_from_reference(lights), config_from_reference(config), buffers=buf)
    b = buf.numpy()
    hb = HostBuffers(cam.width, cam.height, b["depth"], b["id"], b["rgb"].astype(np.float64),
                     b["shadow"].astype(np.float64),
                     {k: v.cpu().numpy() for k, v in buf.per_object_depth.items()})
    return HostRenderResult(res.image.cpu().numpy().astype(np.float64), hb, res.timing)


class B200DepthBackend:
    """Drop-in for the reference's `NedfDepthBackend` (pipeline.py:116-123):
    `query_world(g, origins, dirs) -> (depth, alpha)` on numpy float64 arrays,
    evaluated on the GPU.  Safe to call from the reference's chunk threads."""

    _lock = threading.Lock()       # one device context: serialise the reference's chunk threads

    def __init__(self, ref_model, device=None):
        self.model = ref_model
        self._dev_model = model_from_reference(ref_model, device)

    def query_world(self, g, origins, dirs):
        with self._lock:
            return query_depth_world_batch(self._dev_model, _transform(g), np.asarray(origins, dtype=np.float64),
                                           np.asarray(dirs, dtype=np.float64))
