"""Host-side placement and box types with the reference's validation
(geometry.py:78-162).  Pure data; the device computes all ray math."""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

N_RAY_POINTS = 16          # geometry.py:21
ENCODING_LEVELS = 10       # geometry.py:22
ENCODED_DIM = 1008         # geometry.py:24


def vec3(x, y, z) -> np.ndarray:
    return np.array([x, y, z], dtype=np.float64)


@dataclass(frozen=True)
class RigidTransform:
    """v_world = scale * R @ v_local + T, uniform positive scale (geometry.py:78-129)."""

    rotation: np.ndarray
    translation: np.ndarray
    scale: float = 1.0

    def __post_init__(self):
        r = np.asarray(self.rotation, dtype=np.float64)
        t = np.asarray(self.translation, dtype=np.float64)
        if r.shape != (3, 3) or t.shape != (3,):
            raise ValueError("rotation must be 3x3 and translation a 3-vector")
        if not np.allclose(r.T @ r, np.eye(3), atol=1e-8):
            raise ValueError("rotation must be orthonormal")
        if abs(float(np.linalg.det(r)) - 1.0) > 1e-8:
            raise ValueError("rotation must have determinant +1")
        if not (np.isfinite(self.scale) and self.scale > 0):
            raise ValueError("scale must be a positive real")
        object.__setattr__(self, "rotation", r)
        object.__setattr__(self, "translation", t)
        object.__setattr__(self, "scale", float(self.scale))

    @staticmethod
    def identity() -> "RigidTransform":
        return RigidTransform(np.eye(3), np.zeros(3), 1.0)

    def apply_points(self, pts):
        return self.scale * (np.asarray(pts) @ self.rotation.T) + self.translation

    def invert_points(self, pts):
        return ((np.asarray(pts) - self.translation) @ self.rotation) / self.scale


@dataclass(frozen=True)
class Aabb:
    min: np.ndarray
    max: np.ndarray

    def __post_init__(self):
        lo = np.asarray(self.min, dtype=np.float64)
        hi = np.asarray(self.max, dtype=np.float64)
        if lo.shape != (3,) or hi.shape != (3,):
            raise ValueError("box corners must be 3-vectors")
        if np.any(lo > hi):
            raise ValueError("box min must not exceed max")
        object.__setattr__(self, "min", lo)
        object.__setattr__(self, "max", hi)

    @property
    def center(self):
        return 0.5 * (self.min + self.max)

    @property
    def half_extents(self):
        return 0.5 * (self.max - self.min)

    @property
    def half_diagonal(self) -> float:
        return float(np.linalg.norm(self.half_extents))


def relax_aabb(box: Aabb, factor: float) -> Aabb:
    if factor < 1.0:
        raise ValueError("relaxation factor must be >= 1")
    c, h = box.center, box.half_extents
    return Aabb(c - factor * h, c + factor * h)
