"""Instantiate a `configs.SceneSpec` on the device: paper-profile random-init
models (shared per (seed, kind), like scene.py:250-254 shares model files),
scene instances, camera, lights, render config."""

from __future__ import annotations

import numpy as np

from . import configs as CF
from . import fields as F
from .geometry import Aabb, RigidTransform, vec3
from .model import PROFILES, NedfModel, TrainProfile, new_model_bytes
from .pipeline import (Camera, DirectionalLight, NedfDepthBackend, PointLight, RenderConfig, SceneInstance,
                       look_at)

_MODELS: dict = {}


def canonical_geometry(kind: str):
    """cli.py:25-29"""
    if kind == "sphere":
        return F.Sphere(vec3(0, 0, 0), 1.0)
    if kind == "box":
        return F.BoxPrim(vec3(0, 0, 0), vec3(0.8, 0.5, 0.6))
    if kind == "torus":
        return F.Torus(vec3(0, 0, 0), 0.7, 0.25)
    raise ValueError(f"unknown canonical geometry {kind!r}")


def paper_model(seed: int, kind: str, d_feat: int = 256, n_blocks: int = 16, device=None) -> NedfModel:
    import torch
    dev = torch.cuda.current_device() if device is None else int(device)
    key = (seed, kind, d_feat, n_blocks, dev)
    if key not in _MODELS:
        prof = TrainProfile(d_feat, n_blocks)
        raw = new_model_bytes(canonical_geometry(kind).bounding_box(), np.random.default_rng(seed), prof)
        _MODELS[key] = NedfModel(raw, dev)
    return _MODELS[key]


def build(spec: CF.SceneSpec, device=None):
    """-> (scene, camera, lights, config)"""
    scene = []
    for o in spec.objects:
        m = paper_model(o.seed, o.kind, spec.d_feat, spec.n_blocks, device)
        g = RigidTransform(np.asarray(o.R, dtype=np.float64), np.asarray(o.T, dtype=np.float64), float(o.s))
        scene.append(SceneInstance(o.id, g, NedfDepthBackend(m), F.AnalyticOracle(canonical_geometry(o.kind))))
    c = spec.camera
    cam = Camera(np.asarray(c.position, dtype=np.float64), look_at(c.position, c.look_at, c.up), c.fov_y,
                 c.width, c.height)
    lights = []
    for L in spec.lights:
        if L.kind == "point":
            lights.append(PointLight(np.asarray(L.vec, dtype=np.float64), L.beta))
        else:
            lights.append(DirectionalLight(np.asarray(L.vec, dtype=np.float64), L.beta))
    cfg = RenderConfig(shadows=spec.shadows, resample=spec.resample)
    return scene, cam, lights, cfg
