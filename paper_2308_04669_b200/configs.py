"""The BASELINE.json workloads as plain data.

Pure numpy; no device code.  Each config is a `SceneSpec`: NeDF objects
(canonical geometry kind + random-init seed + placement), a look-at camera,
lights, and render-config overrides.  `paper_2308_04669_b200.pipeline.build_scene`
turns a spec into renderable instances; the tests turn the same spec into
oracle objects, so both sides always see the same scene.

Canonical geometries follow the reference CLI (cli.py:25-29): unit sphere,
box (0.8, 0.5, 0.6), torus (0.7, 0.25).  Weights are the paper-profile random
init (model.py:133-150) for the stated seed; seeds 0, 1, 5 give alpha≈1 for
in-box rays, so the objects are visible.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

CANONICAL_PRIMS = {
    "sphere": ("sphere", (0.0, 0.0, 0.0), 1.0),
    "box": ("box", (0.0, 0.0, 0.0), (0.8, 0.5, 0.6)),
    "torus": ("torus", (0.0, 0.0, 0.0), 0.7, 0.25),
}


@dataclass
class ObjSpec:
    id: int
    kind: str            # canonical geometry: sphere | box | torus
    seed: int            # paper-profile random-init seed
    R: np.ndarray        # 3x3 rotation (local -> world)
    T: np.ndarray        # translation
    s: float = 1.0       # uniform scale


@dataclass
class CameraSpec:
    position: tuple
    look_at: tuple
    fov_y: float         # radians
    width: int
    height: int
    up: tuple = (0.0, 1.0, 0.0)


@dataclass
class LightSpec:
    kind: str            # point | directional
    vec: tuple           # position, or unit travel direction
    beta: float = 0.4


@dataclass
class SceneSpec:
    name: str
    objects: list
    camera: CameraSpec
    lights: list = field(default_factory=list)
    shadows: bool = True
    resample: bool = False
    d_feat: int = 256
    n_blocks: int = 16

    def with_resolution(self, width, height):
        cam = CameraSpec(self.camera.position, self.camera.look_at, self.camera.fov_y,
                         width, height, self.camera.up)
        return SceneSpec(self.name + f"@{width}x{height}", self.objects, cam, self.lights,
                         self.shadows, self.resample, self.d_feat, self.n_blocks)


def quat_to_matrix(q) -> np.ndarray:
    """[w, x, y, z] unit quaternion -> rotation (scene.py:51-57)."""
    w, x, y, z = q
    return np.array([
        [1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
        [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
        [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)],
    ])


def random_rotation(rng) -> np.ndarray:
    q = rng.normal(size=4)
    q /= np.linalg.norm(q)
    if q[0] < 0:
        q = -q
    r = quat_to_matrix(q)
    # re-orthonormalise so RigidTransform's 1e-8 checks always pass
    u, _, vt = np.linalg.svd(r)
    return u @ vt


def rotation_y(angle) -> np.ndarray:
    c, s = math.cos(angle), math.sin(angle)
    return np.array([[c, 0.0, s], [0.0, 1.0, 0.0], [-s, 0.0, c]])


def config1(width=128, height=128) -> SceneSpec:
    """Single object, identity transform, STEP 1 depth+id (no lights)."""
    obj = ObjSpec(0, "sphere", 0, np.eye(3), np.zeros(3), 1.0)
    cam = CameraSpec((0.0, 0.5, -4.0), (0.0, 0.0, 0.0), 0.9, width, height)
    return SceneSpec("config1", [obj], cam, [], shadows=False)


def config2(width=800, height=800) -> SceneSpec:
    """Same object, full pipeline (STEP 1 + STEP 2, no lights)."""
    s = config1(width, height)
    s.name = "config2"
    return s


def config3(width=2000, height=800) -> SceneSpec:
    """4 objects (sphere/box/torus/sphere), random rotations, a radius-3 ring,
    s in [0.5, 1.5]; no shadows."""
    rng = np.random.default_rng(3)
    kinds = ["sphere", "box", "torus", "sphere"]
    seeds = [0, 1, 5, 0]
    objs = []
    for k in range(4):
        a = 2 * math.pi * k / 4 + 0.3
        T = np.array([3.0 * math.cos(a), 0.3 * (k - 1.5), 3.0 * math.sin(a)])
        objs.append(ObjSpec(k, kinds[k], seeds[k], random_rotation(rng), T,
                            float(rng.uniform(0.5, 1.5))))
    cam = CameraSpec((0.0, 2.5, -8.0), (0.0, 0.0, 0.0), math.radians(40.0), width, height)
    return SceneSpec("config3", objs, cam, [], shadows=False)


def config4(width=2000, height=800) -> SceneSpec:
    """The headline scene: 8 objects cycling
    sphere/box/torus, seeds [0,1,5,0,1,5,0,1], random rotations
    (default_rng(123)), T = 3.2 (cos 2pi k/8, 0, sin 2pi k/8), s = 0.8,
    camera (0,3,-9) -> origin, fov_y 40 deg, point light (0,6,-2), beta 0.4."""
    rng = np.random.default_rng(123)
    kinds = ["sphere", "box", "torus"]
    seeds = [0, 1, 5, 0, 1, 5, 0, 1]
    objs = []
    for k in range(8):
        a = 2 * math.pi * k / 8
        T = np.array([3.2 * math.cos(a), 0.0, 3.2 * math.sin(a)])
        objs.append(ObjSpec(k, kinds[k % 3], seeds[k], random_rotation(rng), T, 0.8))
    cam = CameraSpec((0.0, 3.0, -9.0), (0.0, 0.0, 0.0), math.radians(40.0), width, height)
    light = LightSpec("point", (0.0, 6.0, -2.0), 0.4)
    return SceneSpec("config4", objs, cam, [light], shadows=True)


CONFIG5_FPS = 12.0                   # scene-file time of frame f is f / CONFIG5_FPS seconds


def config5_angle(frame: float, k: int, n_frames: int = 60) -> float:
    """Rotation of object k about y at frame f: 2 pi f/60 (1 + k/8)."""
    return 2 * math.pi * frame / n_frames * (1 + k / 8)


def config5_light(frame: int, n_frames: int = 60) -> LightSpec:
    """The point light on a radius-4 circle at y = 6 (scene files have no light
    animation, scene.py:274-290, so the harness sets it per frame)."""
    la = 2 * math.pi * frame / n_frames
    return LightSpec("point", (4.0 * math.cos(la), 6.0, 4.0 * math.sin(la)), 0.4)


def config5_keyframes(n_frames: int = 60, every: int = 10) -> dict:
    """Object id -> [(time, R)] keyframes of the config-5 spin (a key every
    `every` frames: at most 0.625 pi of rotation between keys, so slerp follows
    the constant-rate spin about y)."""
    base = config4()
    return {o.id: [(f / CONFIG5_FPS, rotation_y(config5_angle(f, k, n_frames)) @ o.R)
                   for f in range(0, n_frames + 1, every)]
            for k, o in enumerate(base.objects)}


def config5_frame(frame: int, n_frames: int = 60, width=2000, height=800) -> SceneSpec:
    """Dynamic scene: config 4 with object k rotating about y by
    2 pi f/60 (1 + k/8) and the light on a radius-4 circle at y = 6."""
    base = config4(width, height)
    objs = []
    for k, o in enumerate(base.objects):
        objs.append(ObjSpec(o.id, o.kind, o.seed, rotation_y(config5_angle(frame, k, n_frames)) @ o.R, o.T, o.s))
    return SceneSpec(f"config5[{frame}]", objs, base.camera, [config5_light(frame, n_frames)], shadows=True)


def sweep_rays(n: int, box_min, box_max, seed: int = 0):
    """MLP-only sweep rays: origins on a sphere of radius 2.5 l around the
    box, aimed at uniform points inside it (RaySampler.sample,
    model.py:171-186)."""
    rng = np.random.default_rng(seed)
    box_min = np.asarray(box_min, dtype=np.float64)
    box_max = np.asarray(box_max, dtype=np.float64)
    c = 0.5 * (box_min + box_max)
    l = float(np.linalg.norm(0.5 * (box_max - box_min)))
    v = rng.normal(size=(n, 3))
    v /= np.linalg.norm(v, axis=1, keepdims=True)
    o = c + 2.5 * l * v
    tgt = rng.uniform(box_min, box_max, size=(n, 3))
    d = tgt - o
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    return o, d


CONFIGS = {"config1": config1, "config2": config2, "config3": config3, "config4": config4}
