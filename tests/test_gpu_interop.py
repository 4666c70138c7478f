"""Reference-object adapters (interop.py) with stand-in classes named like the
reference's (the reference itself is not on the GPU box)."""

import numpy as np
import pytest

from oracle import nedf_oracle as O
from paper_2308_04669_b200 import configs as CF
from tests.helpers import oracle_model, oracle_scene
from tests.parity import frame_parity

pytestmark = pytest.mark.gpu


class LinearLayer:
    def __init__(self, w, b):
        self.weight, self.bias = w, b


class Mlp:
    def __init__(self, weights):
        self._l = [LinearLayer(w, b) for w, b in weights]

    def layers(self):
        return self._l


class ClassifierConfig:
    def __init__(self, l):
        self.half_range = l


class Aabb:
    def __init__(self, lo, hi):
        self.min, self.max = np.asarray(lo), np.asarray(hi)


class NedfModel:
    def __init__(self, om):
        self.mlp = Mlp(om.weights)
        self.config = ClassifierConfig(om.half_range)
        self.relaxed_box = Aabb(om.box_min, om.box_max)
        self.alpha_threshold = om.alpha_threshold


class NedfDepthBackend:
    def __init__(self, m):
        self.model = m


class Sphere:
    def __init__(self, c, r):
        self.center, self.radius = np.asarray(c, dtype=float), r


class BoxPrim:
    def __init__(self, c, h):
        self.center, self.half_extents = np.asarray(c, dtype=float), np.asarray(h, dtype=float)


class Torus:
    def __init__(self, c, R, r):
        self.center, self.major_r, self.minor_r = np.asarray(c, dtype=float), R, r


class AnalyticOracle:
    def __init__(self, prim):
        self.prim, self.t_max = prim, 100.0


class RigidTransform:
    def __init__(self, R, T, s):
        self.rotation, self.translation, self.scale = np.asarray(R), np.asarray(T), s


class SceneInstance:
    def __init__(self, id, transform, depth, radiance):
        self.id, self.transform, self.depth, self.radiance = id, transform, depth, radiance


class Camera:
    def __init__(self, position, orientation, fov_y, width, height):
        self.position, self.orientation, self.fov_y, self.width, self.height = (
            np.asarray(position), orientation, fov_y, width, height)


class PointLight:
    def __init__(self, position, beta):
        self.position, self.beta = np.asarray(position), beta


class RenderConfig:
    sigma_threshold = None
    resample = False
    resample_samples = 128
    shadow_epsilon = None
    shadows = True
    clear_color = (0.0, 0.0, 0.0)


PRIMS = {"sphere": lambda: Sphere((0, 0, 0), 1.0), "box": lambda: BoxPrim((0, 0, 0), (0.8, 0.5, 0.6)),
         "torus": lambda: Torus((0, 0, 0), 0.7, 0.25)}


def ref_like(spec):
    models = {}
    scene = []
    for o in spec.objects:
        key = (o.seed, o.kind)
        if key not in models:
            models[key] = NedfModel(oracle_model(o.seed, o.kind))
        scene.append(SceneInstance(o.id, RigidTransform(o.R, o.T, o.s), NedfDepthBackend(models[key]),
                                   AnalyticOracle(PRIMS[o.kind]())))
    c = spec.camera
    cam = Camera(c.position, O.look_at(c.position, c.look_at, c.up), c.fov_y, c.width, c.height)
    lights = [PointLight(L.vec, L.beta) for L in spec.lights]
    return scene, cam, lights, RenderConfig()


def test_render_reference_frame(golden):
    from paper_2308_04669_b200 import interop
    z = golden("frame_config4_200x80.npz")
    spec = CF.config4(200, 80)
    scene, cam, lights, cfg = ref_like(spec)
    res = interop.render_reference_frame(scene, cam, lights, cfg)
    assert res.image.dtype == np.float64 and res.image.shape == (80, 200, 3)
    rep, bad = frame_parity(res.buffers.depth, res.buffers.id, res.image, z["depth"], z["id"], z["image"],
                            z["planes"], [o.id for o in spec.objects])
    assert not bad, (rep, bad)
    assert set(res.buffers.per_object_depth) == {o.id for o in spec.objects}


def test_b200_depth_backend_matches_oracle(golden):
    from paper_2308_04669_b200 import interop
    z = golden("forward_1_box.npz")
    om = oracle_model(1, "box")
    be = interop.B200DepthBackend(NedfModel(om))
    depth, alpha = be.query_world(RigidTransform(z["R"], z["T"], float(z["s"])), z["world_o"], z["world_d"])
    np.testing.assert_array_equal(alpha, z["world_alpha"])
    ok = np.isfinite(z["world_depth"])
    np.testing.assert_allclose(depth[ok], z["world_depth"][ok], atol=1e-9)
