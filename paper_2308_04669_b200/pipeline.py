"""The three-step deferred render pipeline on B200 -- a drop-in for the
reference's `nedf.pipeline` hot path (pipeline.py:53-499).

Same names, argument meaning and error behaviour as the reference:
`compose_frame(scene, camera, lights, config, buffers, changed_ids, external)`
returns `RenderResult(image, buffers, timing)`; the steps can be called one at
a time.  Buffers live on the GPU (torch tensors): depth float64 (+inf = miss),
id int32 (-1 = none), rgb/shadow/image float32; `FrameBuffers.numpy()`
copies them to host arrays shaped like the reference's.

Every computation runs in the CUDA library (libnedf_b200.so); nothing here
computes pixels on the CPU.
"""

from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from . import fields as F
from .geometry import Aabb, RigidTransform
from .model import NedfModel, query_depth_world_batch

QUERY_CHUNK = 16384            # pipeline.py:33 (unused on the GPU; kept for API parity)


def set_thread_count(n: int) -> None:
    """API parity with pipeline.py:38-43 (the GPU path has no host threads)."""
    if int(n) < 1:
        raise ValueError("thread count must be >= 1")


@dataclass(frozen=True)
class Camera:
    """Pinhole camera (pipeline.py:53-77); orientation is camera-to-world."""
    position: np.ndarray
    orientation: np.ndarray
    fov_y: float
    width: int
    height: int
    t_near: float = 0.05
    t_far: float = 100.0

    def __post_init__(self):
        object.__setattr__(self, "position", np.asarray(self.position, dtype=np.float64))
        r = np.asarray(self.orientation, dtype=np.float64)
        if not np.allclose(r.T @ r, np.eye(3), atol=1e-8):
            raise ValueError("camera orientation must be orthonormal")
        object.__setattr__(self, "orientation", r)
        if not 0.0 < self.fov_y < np.pi:
            raise ValueError("vertical field of view must be in (0, pi)")
        if self.width < 1 or self.height < 1:
            raise ValueError("image size must be at least 1x1")
        if not 0 < self.t_near < self.t_far:
            raise ValueError("need 0 < t_near < t_far")

    def _c(self):
        c = _lib.NedfCamera()
        c.position[:] = list(self.position)
        c.orientation[:] = list(self.orientation.ravel())
        c.fov_y = float(self.fov_y)
        c.width = int(self.width)
        c.height = int(self.height)
        return c


def look_at(position, target, up=(0.0, 1.0, 0.0)) -> np.ndarray:
    """Camera-to-world rotation (pipeline.py:80-94)."""
    position = np.asarray(position, dtype=np.float64)
    forward = np.asarray(target, dtype=np.float64) - position
    fn = np.linalg.norm(forward)
    if fn == 0:
        raise ValueError("camera target coincides with its position")
    forward = forward / fn
    right = np.cross(forward, np.asarray(up, dtype=np.float64))
    rn = np.linalg.norm(right)
    if rn < 1e-12:
        raise ValueError("camera up vector is parallel to the view direction")
    right /= rn
    true_up = np.cross(right, forward)
    return np.stack([right, true_up, -forward], axis=1)


def generate_primary_rays(camera: Camera):
    """Host helper with the reference's layout (pipeline.py:97-109); the
    render path regenerates these rays on the device in float64."""
    w, h = camera.width, camera.height
    xs = (np.arange(w) + 0.5) / w * 2.0 - 1.0
    ys = 1.0 - (np.arange(h) + 0.5) / h * 2.0
    t = np.tan(camera.fov_y / 2.0)
    gx, gy = np.meshgrid(xs * t * (w / h), ys * t)
    dc = np.stack([gx.ravel(), gy.ravel(), -np.ones(w * h)], axis=1)
    d = dc @ camera.orientation.T
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    return np.broadcast_to(camera.position, (w * h, 3)).copy(), d


# ---------------------------------------------------------------------------
# depth backends (the reference's plugin seam, pipeline.py:116-136)
# ---------------------------------------------------------------------------

class NedfDepthBackend:
    """World-space depth through the device network."""

    def __init__(self, model: NedfModel):
        if not isinstance(model, NedfModel):
            raise TypeError("NedfDepthBackend needs a device NedfModel (see model.load_nedf)")
        self.model = model

    def query_world(self, g: RigidTransform, origins, dirs):
        return query_depth_world_batch(self.model, g, origins, dirs)


class OracleDepthBackend:
    """Exact analytic depth by device sphere tracing (fields.py:194-238)."""

    def __init__(self, oracle):
        if not isinstance(oracle, F.AnalyticOracle):
            raise TypeError("the device oracle backend supports analytic (SDF) geometry")
        self.oracle = oracle


@dataclass
class SceneInstance:
    id: int
    transform: RigidTransform
    depth: object
    radiance: object

    @property
    def sampling_box(self) -> Aabb:
        return self.radiance.bounding_box


@dataclass(frozen=True)
class PointLight:
    position: np.ndarray
    beta: float = 0.4

    def __post_init__(self):
        object.__setattr__(self, "position", np.asarray(self.position, dtype=np.float64))
        if not 0.0 < self.beta < 1.0:
            raise ValueError("shadow intensity beta must be in (0, 1)")


@dataclass(frozen=True)
class DirectionalLight:
    direction: np.ndarray
    beta: float = 0.4

    def __post_init__(self):
        d = np.asarray(self.direction, dtype=np.float64)
        if abs(np.linalg.norm(d) - 1.0) > 1e-9:
            raise ValueError("light direction must be unit length")
        object.__setattr__(self, "direction", d)
        if not 0.0 < self.beta < 1.0:
            raise ValueError("shadow intensity beta must be in (0, 1)")


@dataclass
class RenderConfig:
    sigma_threshold: float | None = None
    resample: bool = False
    resample_samples: int = 128
    shadow_epsilon: float | None = None
    shadows: bool = True
    clear_color: tuple = (0.0, 0.0, 0.0)

    def __post_init__(self):
        if self.sigma_threshold is not None and self.sigma_threshold < 0:
            raise ValueError("sigma threshold must be >= 0")
        if self.shadow_epsilon is not None and self.shadow_epsilon <= 0:
            raise ValueError("shadow epsilon must be positive")

    def _c(self):
        c = _lib.NedfRenderConfig()
        c.sigma_threshold = -1.0 if self.sigma_threshold is None else float(self.sigma_threshold)
        c.resample = int(bool(self.resample))
        c.resample_samples = int(self.resample_samples)
        c.shadow_epsilon = -1.0 if self.shadow_epsilon is None else float(self.shadow_epsilon)
        c.shadows = int(bool(self.shadows))
        c.clear_color[:] = [float(v) for v in self.clear_color]
        return c


def default_shadow_epsilon(scene) -> float:
    """Twice the worst depth quantisation step (pipeline.py:202-208)."""
    eps = 1e-4
    for inst in scene:
        if isinstance(inst.depth, NedfDepthBackend):
            eps = max(eps, 2.0 * inst.transform.scale * inst.depth.model.fine_width)
    return eps


class FrameBuffers:
    """Per-pixel device planes (pipeline.py:211-232).  With `rows`, only those
    camera rows are held (an image tile for multi-GPU rendering)."""

    def __init__(self, width: int, height: int, device=None, rows=None, keep_planes: bool = False):
        import torch
        self.width = int(width)
        self.height = int(height)
        dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        self.device = dev
        self.rows = None if rows is None else np.ascontiguousarray(rows, dtype=np.int32)
        n_rows = self.height if self.rows is None else len(self.rows)
        self.n_rows = n_rows
        self.depth = torch.full((n_rows, self.width), float("inf"), dtype=torch.float64, device=dev)
        self.id = torch.full((n_rows, self.width), -1, dtype=torch.int32, device=dev)
        self.rgb = torch.zeros((n_rows, self.width, 3), dtype=torch.float32, device=dev)
        self.shadow = torch.ones((n_rows, self.width), dtype=torch.float32, device=dev)
        self.image = torch.zeros((n_rows, self.width, 3), dtype=torch.float32, device=dev)
        self.keep_planes = keep_planes
        self.planes = None
        self.plane_ids = None
        self.per_object_depth: dict = {}

    def clear_hit_planes(self):
        self.depth.fill_(float("inf"))
        self.id.fill_(-1)

    def _c(self, n_objs: int = 0):
        import torch
        fb = _lib.NedfFrameBuffers()
        fb.depth_dev = self.depth.data_ptr()
        fb.id_dev = self.id.data_ptr()
        fb.rgb_dev = self.rgb.data_ptr()
        fb.shadow_dev = self.shadow.data_ptr()
        fb.image_dev = self.image.data_ptr()
        if self.keep_planes and n_objs > 0:
            if self.planes is None or self.planes.shape[0] != n_objs:
                self.planes = torch.full((n_objs, self.n_rows, self.width), float("inf"), dtype=torch.float64,
                                         device=self.device)
            fb.planes_dev = self.planes.data_ptr()
        else:
            fb.planes_dev = 0
        if self.rows is not None:
            self._rows_c = (C.c_int32 * len(self.rows))(*self.rows.tolist())
            fb.rows_host = C.cast(self._rows_c, C.POINTER(C.c_int32))
            fb.n_rows = len(self.rows)
        else:
            fb.rows_host = C.POINTER(C.c_int32)()
            fb.n_rows = self.height
        return fb

    def numpy(self) -> dict:
        return {"depth": self.depth.cpu().numpy(), "id": self.id.cpu().numpy(),
                "rgb": self.rgb.cpu().numpy(), "shadow": self.shadow.cpu().numpy()}


@dataclass
class RenderResult:
    image: object
    buffers: FrameBuffers
    timing: dict = field(default_factory=dict)
    # (beyond the reference) CUDA events at the step boundaries of compose_frame: [2] is
    # recorded once depth / id are final, [3] at the end -- a streaming caller can start
    # copying depth / id out while STEP 3 still runs
    events: tuple = ()


# ---------------------------------------------------------------------------
# scene marshalling
# ---------------------------------------------------------------------------

class _SceneTables:
    """ctypes arrays describing a scene for one call (objects, field nodes)."""

    def __init__(self, scene, device):
        nodes: list = []
        objs = (_lib.NedfObject * max(1, len(scene)))()
        self.keep = []
        seen_ids = set()
        for k, inst in enumerate(scene):
            if inst.id in seen_ids:
                raise ValueError(f"duplicate object id {inst.id}")
            seen_ids.add(inst.id)
            o = objs[k]
            g = inst.transform
            o.R[:] = list(np.asarray(g.rotation, dtype=np.float64).ravel())
            o.T[:] = list(np.asarray(g.translation, dtype=np.float64))
            o.s = float(g.scale)
            o.id = int(inst.id)
            o.radiance_field = F.flatten(inst.radiance, nodes, device)
            be = inst.depth
            if isinstance(be, NedfDepthBackend):
                if be.model.device != device.index:
                    raise ValueError("model lives on another device")
                o.depth_kind = _lib.DEPTH_NEDF
                o.model = be.model.handle.value
                o.depth_field = -1
                self.keep.append(be.model)
            elif isinstance(be, OracleDepthBackend):
                o.depth_kind = _lib.DEPTH_ANALYTIC
                o.model = None
                o.depth_field = F.flatten(be.oracle.prim, nodes, device)
            else:
                raise TypeError(f"unsupported depth backend {type(be).__name__}")
        self.objs = objs
        self.n_objs = len(scene)
        self.fields = (_lib.NedfField * max(1, len(nodes)))(*nodes)
        self.n_fields = len(nodes)


def _light_c(light):
    L = _lib.NedfLight()
    if isinstance(light, PointLight):
        L.kind = _lib.LIGHT_POINT
        L.vec[:] = list(light.position)
    elif isinstance(light, DirectionalLight):
        L.kind = _lib.LIGHT_DIRECTIONAL
        L.vec[:] = list(light.direction)
    else:
        raise TypeError(f"unsupported light type {type(light).__name__}")
    L.beta = float(light.beta)
    return L


def _ctx(buffers):
    return _lib.context(buffers.device.index)


def nedf_generation_step(scene, camera: Camera, buffers: FrameBuffers, _tables=None) -> None:
    """STEP 1 (pipeline.py:271-278).  With `buffers.keep_planes` every object's
    alpha-folded depth plane is kept (per_object_depth) and depth/id come from
    the fp64 strict-< recombine of those planes, so later `reuse_buffers` calls
    are bit-identical to this cold render."""
    tb = _tables or _SceneTables(scene, buffers.device)
    fb = buffers._c(tb.n_objs)
    _lib.check(_lib.load_library().nedf_generation_step(
        _ctx(buffers).handle, C.byref(camera._c()), tb.objs, tb.n_objs, tb.fields, tb.n_fields, C.byref(fb),
        _lib.stream_handle()))
    _publish_planes(scene, buffers)


def _publish_planes(scene, buffers: FrameBuffers) -> None:
    if buffers.keep_planes:
        buffers.plane_ids = [inst.id for inst in scene]
        buffers.per_object_depth = {inst.id: buffers.planes[k] for k, inst in enumerate(scene)}


def reuse_buffers(scene, camera: Camera, buffers: FrameBuffers, changed_ids, _tables=None) -> dict:
    """STEP 1 recomputing only the planes of changed objects (pipeline.py:281-305).

    Falls back to a full recompute when an unchanged object has no cached
    plane.  The recombined result is bit-identical to nedf_generation_step."""
    import torch
    changed = set(changed_ids)
    ids = [inst.id for inst in scene]
    cached = set(buffers.per_object_depth) if buffers.keep_planes else set()
    missing = [i for i in ids if i not in changed and i not in cached]
    if missing or not buffers.keep_planes:
        buffers.keep_planes = True
        nedf_generation_step(scene, camera, buffers, _tables)
        return {"recomputed": ids, "fallback": True}
    tb = _tables or _SceneTables(scene, buffers.device)
    if getattr(buffers, "plane_ids", None) != ids:
        # scene membership / order changed: lay the cached planes out in scene order
        old = buffers.per_object_depth
        planes = torch.full((len(ids), buffers.n_rows, buffers.width), float("inf"), dtype=torch.float64,
                            device=buffers.device)
        for k, i in enumerate(ids):
            if i in old and i not in changed:
                planes[k].copy_(old[i])
        buffers.planes = planes
    idx = [k for k, i in enumerate(ids) if i in changed]
    arr = (C.c_int32 * max(1, len(idx)))(*idx)
    fb = buffers._c(tb.n_objs)
    _lib.check(_lib.load_library().nedf_reuse_step(
        _ctx(buffers).handle, C.byref(camera._c()), tb.objs, tb.n_objs, tb.fields, tb.n_fields, arr, len(idx),
        C.byref(fb), _lib.stream_handle()))
    _publish_planes(scene, buffers)
    return {"recomputed": [ids[k] for k in idx], "fallback": False}


def deferred_shading_step(scene, camera: Camera, buffers: FrameBuffers, config: RenderConfig,
                          _tables=None, _stats=True) -> dict:
    """STEP 2 (pipeline.py:315-352); returns {"resampled", "covered"}."""
    tb = _tables or _SceneTables(scene, buffers.device)
    fb = buffers._c(tb.n_objs)
    ctx = _ctx(buffers)
    st = _lib.stream_handle()
    if _stats:
        ctx.read_stats(st)   # reset counters
    _lib.check(_lib.load_library().nedf_shading_step(
        ctx.handle, C.byref(camera._c()), tb.objs, tb.n_objs, tb.fields, tb.n_fields,
        C.byref(config._c()), C.byref(fb), st))
    if not _stats:
        return {}
    s = ctx.read_stats(st)
    return {"resampled": int(s["resampled"]), "covered": int(s["covered"])}


def shadow_step(scene, camera: Camera, buffers: FrameBuffers, light, config: RenderConfig, _tables=None) -> None:
    """STEP 3 for one light (pipeline.py:371-403)."""
    tb = _tables or _SceneTables(scene, buffers.device)
    fb = buffers._c(tb.n_objs)
    _lib.check(_lib.load_library().nedf_shadow_step(
        _ctx(buffers).handle, C.byref(camera._c()), tb.objs, tb.n_objs, tb.fields, tb.n_fields,
        C.byref(_light_c(light)), C.byref(config._c()), C.byref(fb), _lib.stream_handle()))


def import_external_gbuffer(buffers: FrameBuffers, depth_plane, color_image, pseudo_id: int) -> None:
    """Depth-composite an external layer where strictly closer (pipeline.py:406-420)."""
    import torch
    d = torch.as_tensor(depth_plane, dtype=torch.float64, device=buffers.device)
    c = torch.as_tensor(color_image, dtype=torch.float32, device=buffers.device)
    if d.shape != buffers.depth.shape:
        raise ValueError("external depth size does not match the frame")
    if c.shape != buffers.rgb.shape:
        raise ValueError("external color size does not match the frame")
    if pseudo_id < 0:
        raise ValueError("pseudo id must be non-negative")
    closer = d < buffers.depth
    buffers.depth[closer] = d[closer]
    buffers.id[closer] = int(pseudo_id)
    buffers.rgb[closer] = c[closer]


class _LazyTiming(dict):
    """RenderResult.timing without a host sync at the end of compose_frame: the
    host-side entries (kernel_launches, h2d_bytes) are there at once; the first
    access to anything else waits for the frame's last event and fills in the
    step times and the device counters (from a mapped stats slot, valid for the
    next 62 frames).  Behaves as a plain dict afterwards."""

    _EAGER = ("kernel_launches", "h2d_bytes")

    def __init__(self, eager: dict, resolve):
        super().__init__(eager)
        self._resolve = resolve

    def _fill(self):
        if self._resolve is not None:
            r, self._resolve = self._resolve, None
            dict.update(self, r())

    def __getitem__(self, k):
        if k not in self._EAGER:
            self._fill()
        return dict.__getitem__(self, k)

    def get(self, k, default=None):
        if k not in self._EAGER:
            self._fill()
        return dict.get(self, k, default)

    def __contains__(self, k):
        self._fill()
        return dict.__contains__(self, k)

    def __iter__(self):
        self._fill()
        return dict.__iter__(self)

    def __len__(self):
        self._fill()
        return dict.__len__(self)

    def keys(self):
        self._fill()
        return dict.keys(self)

    def items(self):
        self._fill()
        return dict.items(self)

    def values(self):
        self._fill()
        return dict.values(self)

    def copy(self):
        self._fill()
        return dict(self)

    def __eq__(self, other):
        self._fill()
        return dict.__eq__(self, other)

    def __repr__(self):
        self._fill()
        return dict.__repr__(self)


def compose_frame(scene, camera: Camera, lights, config: RenderConfig | None = None,
                  buffers: FrameBuffers | None = None, changed_ids=None, external=None) -> RenderResult:
    """Steps 1-3 and image = rgb * shadow (pipeline.py:430-468).  Timing is
    measured with CUDA events per step (seconds, like the reference).  The call
    returns as soon as the frame is enqueued (no host synchronisation); reading
    the buffers or most timing entries waits for it."""
    import torch
    config = config or RenderConfig()
    if buffers is None:
        buffers = FrameBuffers(camera.width, camera.height)
    tb = _SceneTables(scene, buffers.device)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    ctx = _ctx(buffers)
    st = _lib.stream_handle()
    ctx.reset_stats(st)                    # zero the per-frame counters (no sync)
    if changed_ids is None and external is None:
        # the whole frame in one call (the library fuses the per-pixel passes); events at the step
        # boundaries (the STEP 1 resolve and the first light's shadow-ray setup run in the STEP 2 pass)
        for e in ev:
            e.record()                     # torch creates its events lazily, on first record
        handles = (C.c_void_p * 4)(*[e.cuda_event for e in ev])
        lights = list(lights) if config.shadows else []
        lc = (_lib.NedfLight * max(1, len(lights)))(*[_light_c(L) for L in lights])
        cfg_c = config._c()
        _lib.check(_lib.load_library().nedf_render_frame_timed(
            ctx.handle, C.byref(camera._c()), tb.objs, tb.n_objs, tb.fields, tb.n_fields, lc, len(lights),
            C.byref(cfg_c), C.byref(buffers._c(tb.n_objs)), handles, st))
        _publish_planes(scene, buffers)
    else:
        ev[0].record()
        if changed_ids is None:
            nedf_generation_step(scene, camera, buffers, _tables=tb)
        else:
            reuse_buffers(scene, camera, buffers, changed_ids, _tables=tb)
        ev[1].record()
        if external is not None:
            import_external_gbuffer(buffers, external[0], external[1], external[2])
        deferred_shading_step(scene, camera, buffers, config, _tables=tb, _stats=False)
        ev[2].record()
        buffers.shadow.fill_(1.0)
        if config.shadows:
            for light in lights:
                shadow_step(scene, camera, buffers, light, config, _tables=tb)
        _lib.check(_lib.load_library().nedf_composite(ctx.handle, C.byref(buffers._c(tb.n_objs)), camera.width,
                                                      st))
    if changed_ids is not None or external is not None:
        ev[3].record()
    slot, host = ctx.snapshot_stats(st)
    done = torch.cuda.Event()
    done.record()
    n_pix = float(camera.width * buffers.n_rows)

    def resolve():
        done.synchronize()
        dev = ctx.slot_stats(slot)
        return {
            "step1_depth_id": ev[0].elapsed_time(ev[1]) / 1e3,
            "step2_shading": ev[1].elapsed_time(ev[2]) / 1e3,
            "resample_ratio": dev["resampled"] / n_pix,
            "step3_shadow": ev[2].elapsed_time(ev[3]) / 1e3,
            "network_evals": dev["evals"],
            "guarded_evals": dev["guarded"],
            "culled_evals": dev["culled"],
        }

    timing = _LazyTiming({"kernel_launches": host["launches"], "h2d_bytes": host["h2d_bytes"]}, resolve)
    return RenderResult(image=buffers.image, buffers=buffers, timing=timing, events=tuple(ev))


def step_timing_report(scene, camera: Camera, lights, config: RenderConfig | None = None,
                       repetitions: int = 1) -> dict:
    """Per-step device time over repeated renders (pipeline.py:471-499)."""
    samples = {"step1_depth_id": [], "step2_shading": [], "step3_shadow": []}
    ratio = 0.0
    for _ in range(max(1, repetitions)):
        res = compose_frame(scene, camera, lights, config)
        for k in samples:
            samples[k].append(res.timing[k])
        ratio = res.timing["resample_ratio"]
    total = sum(float(np.mean(v)) for v in samples.values())
    rep = {"width": camera.width, "height": camera.height, "objects": len(scene),
           "repetitions": int(max(1, repetitions)), "resample_ratio": ratio, "total_seconds": total, "steps": {}}
    for k, v in samples.items():
        m = float(np.mean(v))
        rep["steps"][k] = {"mean_seconds": m, "stddev_seconds": float(np.std(v)),
                           "share": m / total if total > 0 else 0.0}
    return rep


class FrameRenderer:
    """Pre-marshalled scene for repeated frames: one `nedf_render_frame` call
    per frame, no host work beyond argument passing (bench / serving loop)."""

    def __init__(self, scene, camera: Camera, lights, config: RenderConfig | None = None,
                 buffers: FrameBuffers | None = None):
        self.scene = scene
        self.camera = camera
        self.config = config or RenderConfig()
        self.buffers = buffers or FrameBuffers(camera.width, camera.height)
        self.tables = _SceneTables(scene, self.buffers.device)
        self._cam = camera._c()
        self._cfg = self.config._c()
        self._lights = (_lib.NedfLight * max(1, len(lights)))(*[_light_c(L) for L in lights])
        self._n_lights = len(lights)
        self._fb = self.buffers._c(self.tables.n_objs)
        self._ctx = _ctx(self.buffers)
        self._lib = _lib.load_library()

    def update_transforms(self, transforms):
        """Per-frame placements (dynamic scenes): list of RigidTransform in scene order."""
        for k, g in enumerate(transforms):
            o = self.tables.objs[k]
            o.R[:] = list(np.asarray(g.rotation, dtype=np.float64).ravel())
            o.T[:] = list(np.asarray(g.translation, dtype=np.float64))
            o.s = float(g.scale)

    def update_lights(self, lights):
        self._lights = (_lib.NedfLight * max(1, len(lights)))(*[_light_c(L) for L in lights])
        self._n_lights = len(lights)

    def render(self, stream=None):
        _lib.check(self._lib.nedf_render_frame(
            self._ctx.handle, C.byref(self._cam), self.tables.objs, self.tables.n_objs, self.tables.fields,
            self.tables.n_fields, self._lights, self._n_lights, C.byref(self._cfg), C.byref(self._fb),
            _lib.stream_handle(stream)))
        return self.buffers
