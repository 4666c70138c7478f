"""Appearance / analytic-geometry field descriptors (fields.py:53-186, 270-357,
439-508 of the reference).

These are host-side descriptions only: `flatten()` turns a primitive tree into
the `NedfField` node array the device evaluates (SDF, procedural colour,
trilinear voxel lookup, sphere tracing).
"""

from __future__ import annotations

import struct
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .errors import FormatError
from .geometry import Aabb, RigidTransform

SURFACE_EPS = 1e-5
SIGMA_SURFACE = 50.0
SURFACE_BAND = 0.02
INTERIOR_STEEPNESS = 1000.0


class SdfPrimitive:
    def bounding_box(self) -> Aabb:
        raise NotImplementedError

    def _leaf(self):
        raise NotImplementedError


@dataclass(frozen=True)
class Sphere(SdfPrimitive):
    center: np.ndarray
    radius: float

    def __post_init__(self):
        object.__setattr__(self, "center", np.asarray(self.center, dtype=np.float64))
        if not self.radius > 0:
            raise ValueError("sphere radius must be positive")

    def bounding_box(self):
        r = np.full(3, self.radius)
        return Aabb(self.center - r, self.center + r)

    def _leaf(self):
        return _lib.FIELD_SPHERE, [*self.center, self.radius]


@dataclass(frozen=True)
class BoxPrim(SdfPrimitive):
    center: np.ndarray
    half_extents: np.ndarray

    def __post_init__(self):
        object.__setattr__(self, "center", np.asarray(self.center, dtype=np.float64))
        object.__setattr__(self, "half_extents", np.asarray(self.half_extents, dtype=np.float64))
        if not np.all(self.half_extents > 0):
            raise ValueError("box half extents must be positive")

    def bounding_box(self):
        return Aabb(self.center - self.half_extents, self.center + self.half_extents)

    def _leaf(self):
        return _lib.FIELD_BOX, [*self.center, *self.half_extents]


@dataclass(frozen=True)
class Torus(SdfPrimitive):
    center: np.ndarray
    major_r: float
    minor_r: float

    def __post_init__(self):
        object.__setattr__(self, "center", np.asarray(self.center, dtype=np.float64))
        if not (self.major_r > 0 and self.minor_r > 0):
            raise ValueError("torus radii must be positive")

    def bounding_box(self):
        r = self.major_r + self.minor_r
        ext = np.array([r, self.minor_r, r])
        return Aabb(self.center - ext, self.center + ext)

    def _leaf(self):
        return _lib.FIELD_TORUS, [*self.center, self.major_r, self.minor_r]


@dataclass(frozen=True)
class Plane(SdfPrimitive):
    normal: np.ndarray
    offset: float

    def __post_init__(self):
        n = np.asarray(self.normal, dtype=np.float64)
        if abs(np.linalg.norm(n) - 1.0) > 1e-9:
            raise ValueError("plane normal must be unit length")
        object.__setattr__(self, "normal", n)

    def bounding_box(self):
        raise ValueError("a plane has no finite bounding box")

    def _leaf(self):
        return _lib.FIELD_PLANE, [*self.normal, self.offset]


@dataclass(frozen=True)
class Union(SdfPrimitive):
    children: tuple

    def __post_init__(self):
        if not self.children:
            raise ValueError("union needs at least one child")
        object.__setattr__(self, "children", tuple(self.children))

    def bounding_box(self):
        boxes = [c.bounding_box() for c in self.children]
        return Aabb(np.minimum.reduce([b.min for b in boxes]), np.maximum.reduce([b.max for b in boxes]))


@dataclass(frozen=True)
class Transformed(SdfPrimitive):
    child: SdfPrimitive
    transform: RigidTransform

    def bounding_box(self):
        b = self.child.bounding_box()
        corners = np.array([[x, y, z] for x in (b.min[0], b.max[0]) for y in (b.min[1], b.max[1])
                            for z in (b.min[2], b.max[2])])
        w = self.transform.apply_points(corners)
        return Aabb(w.min(axis=0), w.max(axis=0))


@dataclass(frozen=True)
class VoxelField:
    """Density/colour at voxel centres (fields.py:270-319); `density` (nx,ny,nz),
    `color` (nx,ny,nz,3)."""

    resolution: tuple
    bounds: Aabb
    density: np.ndarray
    color: np.ndarray
    _dev: dict = field(default_factory=dict, compare=False, repr=False)

    def __post_init__(self):
        nx, ny, nz = self.resolution
        if min(nx, ny, nz) < 1:
            raise ValueError("voxel resolution must be positive")
        if np.asarray(self.density).shape != (nx, ny, nz):
            raise ValueError("density shape does not match resolution")
        if np.asarray(self.color).shape != (nx, ny, nz, 3):
            raise ValueError("color shape does not match resolution")
        if np.any(np.asarray(self.density) < 0):
            raise ValueError("densities must be non-negative")

    def device_arrays(self, device):
        import torch
        key = str(device)
        if key not in self._dev:
            d = torch.as_tensor(np.ascontiguousarray(self.density, dtype=np.float32), device=device)
            c = torch.as_tensor(np.ascontiguousarray(self.color, dtype=np.float32), device=device)
            self._dev[key] = (d, c)
        return self._dev[key]


def load_voxel_field(path) -> VoxelField:
    """NVXF reader (fields.py:322-357)."""
    with open(path, "rb") as f:
        raw = f.read()
    if raw[:4] != b"NVXF":
        raise FormatError(f"{path}: not a voxel field file")
    if len(raw) < 44:
        raise FormatError(f"{path}: truncated header")
    version, nx, ny, nz = struct.unpack_from("<IIII", raw, 4)
    if version != 1:
        raise FormatError(f"{path}: unsupported version {version}")
    b = struct.unpack_from("<6f", raw, 20)
    n = nx * ny * nz
    if len(raw) != 44 + 16 * n:
        raise FormatError(f"{path}: expected {44 + 16 * n} bytes, found {len(raw)}")
    dens = np.frombuffer(raw, dtype="<f4", count=n, offset=44).reshape(nx, ny, nz).astype(np.float64)
    col = np.frombuffer(raw, dtype="<f4", count=3 * n, offset=44 + 4 * n).reshape(nx, ny, nz, 3).astype(np.float64)
    return VoxelField((nx, ny, nz), Aabb(np.array(b[:3], dtype=np.float64), np.array(b[3:], dtype=np.float64)),
                      dens, col)


class DepthOracle:
    bounding_box: Aabb


@dataclass(frozen=True)
class AnalyticOracle(DepthOracle):
    """Analytic appearance (procedural colour + SDF density, fields.py:456-474)."""
    prim: SdfPrimitive
    t_max: float = 100.0

    @property
    def bounding_box(self) -> Aabb:
        return self.prim.bounding_box()


@dataclass(frozen=True)
class VoxelOracle(DepthOracle):
    """Voxel appearance (fields.py:477-508)."""
    vf: VoxelField
    n_samples: int = 192
    alpha_threshold: float = 0.5

    @property
    def bounding_box(self) -> Aabb:
        return self.vf.bounds


def _node(kind, child=0, count=0, p=(), res=(0, 0, 0), dens=None, col=None):
    n = _lib.NedfField()
    n.kind = kind
    n.child = child
    n.count = count
    for i, v in enumerate(res):
        n.res[i] = int(v)
    for i, v in enumerate(p):
        n.p[i] = float(v)
    n.density_dev = dens or 0
    n.color_dev = col or 0
    return n


def _flatten_into(src, nodes: list, slot: int, device):
    if isinstance(src, AnalyticOracle):
        src = src.prim
    if isinstance(src, VoxelOracle):
        src = src.vf
    if isinstance(src, VoxelField):
        d, c = src.device_arrays(device)
        nodes[slot] = _node(_lib.FIELD_VOXEL, p=[*src.bounds.min, *src.bounds.max], res=src.resolution,
                            dens=d.data_ptr(), col=c.data_ptr())
    elif isinstance(src, Union):
        first = len(nodes)
        nodes.extend([None] * len(src.children))
        nodes[slot] = _node(_lib.FIELD_UNION, child=first, count=len(src.children))
        for k, ch in enumerate(src.children):
            _flatten_into(ch, nodes, first + k, device)
    elif isinstance(src, Transformed):
        ci = len(nodes)
        nodes.append(None)
        g = src.transform
        nodes[slot] = _node(_lib.FIELD_TRANSFORMED, child=ci,
                            p=[*g.rotation.ravel(), *g.translation, g.scale])
        _flatten_into(src.child, nodes, ci, device)
    elif isinstance(src, SdfPrimitive):
        kind, p = src._leaf()
        nodes[slot] = _node(kind, p=p)
    else:
        raise TypeError(f"unsupported field type {type(src).__name__}")


def flatten(src, nodes: list, device) -> int:
    """Append `src`'s node tree to `nodes`; returns the root index."""
    root = len(nodes)
    nodes.append(None)
    _flatten_into(src, nodes, root, device)
    return root
