"""GPU distillation of a NeDF from an analytic oracle.

Mirrors the reference's training API (model.py:153-274, nn.py:138-232):
`RaySampler`, `build_training_batch`, `loss_and_grads`, `train` and
`TrainingDiverged`, over the C ABI trainer (`nedf_trainer_*`, csrc/train.cu):

  * rays are drawn on the host with the reference's RaySampler code, so a given
    numpy Generator produces the same supervision rays;
  * encoding, oracle sphere tracing, bin targets, forward with cached
    activations, BCE losses, exact backward and Adam run on the GPU (fp32
    arithmetic; the reference is float64).

`train` updates the NedfModel in place (its device weights are rebuilt from the
trained parameters) and returns the per-iteration loss, like the reference.
"""

from __future__ import annotations

import ctypes as C
import struct
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .fields import AnalyticOracle, flatten
from .geometry import Aabb

ALPHA_LOSS_WEIGHT = 0.1                       # model.py:236
_HEADER = 32                                  # .nedm header bytes (nn.py:235-246)


class TrainingDiverged(RuntimeError):
    """Non-finite loss (model.py:262-265)."""


def _lib_trainer():
    return _lib.load_library()


def _check(rc):
    if rc != _lib.NEDF_OK:
        msg = (_lib_trainer().nedf_trainer_last_error() or b"").decode(errors="replace")
        if rc == _lib.NEDF_ERR_INVALID:
            raise ValueError(msg)
        if rc == _lib.NEDF_ERR_UNSUPPORTED:
            raise TypeError(msg)
        raise RuntimeError(f"nedf_b200 trainer error {rc}: {msg}")


@dataclass
class RaySampler:
    """model.py:153-186: origins on a sphere of radius 2.5 l around the box
    (direct) or on a fixed set of viewpoints (views), aimed at uniform points
    in the box.  Host-side, same numpy calls as the reference."""

    box: Aabb
    mode: str = "direct"
    n_views: int = 500
    _views: np.ndarray | None = field(default=None, repr=False)

    def __post_init__(self):
        if self.mode not in ("direct", "views"):
            raise ValueError(f"unknown sampler mode {self.mode!r}")

    def _sphere_points(self, rng, n):
        v = rng.normal(size=(n, 3))
        v /= np.linalg.norm(v, axis=1, keepdims=True)
        center = 0.5 * (self.box.min + self.box.max)
        half_diag = float(np.linalg.norm(0.5 * (self.box.max - self.box.min)))
        return center + 2.5 * half_diag * v

    def sample(self, rng: np.random.Generator, n: int):
        if self.mode == "views":
            if self._views is None:
                self._views = self._sphere_points(rng, self.n_views)
            origins = self._views[rng.integers(0, self.n_views, size=n)]
        else:
            origins = self._sphere_points(rng, n)
        targets = rng.uniform(self.box.min, self.box.max, size=(n, 3))
        dirs = targets - origins
        dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
        return origins, dirs


class Trainer:
    """Device-resident fp32 parameters, Adam moments and activation cache for one model."""

    def __init__(self, model, max_batch: int = 4096, lr: float = 5e-4):
        lib = _lib_trainer()
        raw = model.nedm_bytes()
        info = _lib.NedfModelInfo()
        _lib.check(_lib.load_library().nedf_model_info(model.handle, C.byref(info)))
        self.info = info
        F, NB = info.d_feat, info.n_blocks
        self.n_params = (F * info.d_in + F + NB * (2 * F * F + 2 * F) + (info.n_coarse + 1) * (F + 1)
                         + info.n_fine * (F + 1))
        params = np.frombuffer(raw, dtype="<f4", count=self.n_params, offset=_HEADER).copy()
        self._trailer = raw[_HEADER + 4 * self.n_params:]
        self._header = raw[:_HEADER]
        h = C.c_void_p()
        _check(lib.nedf_trainer_create(int(model.device), C.byref(info), params.ctypes.data, self.n_params,
                                       int(max_batch), C.byref(h)))
        self.handle = h
        self.max_batch = int(max_batch)
        self.model = model
        self.set_lr(lr)

    def __del__(self):
        try:
            if getattr(self, "handle", None):
                _lib_trainer().nedf_trainer_destroy(self.handle)
                self.handle = None
        except Exception:
            pass

    def set_lr(self, lr: float):
        _check(_lib_trainer().nedf_trainer_set_lr(self.handle, float(lr)))

    def batch(self, oracle: AnalyticOracle, origins, dirs) -> np.ndarray:
        """GPU batch from host rays (model frame); returns the box-hit mask."""
        o = np.ascontiguousarray(origins, dtype=np.float64)
        d = np.ascontiguousarray(dirs, dtype=np.float64)
        nodes: list = []
        root = flatten(oracle, nodes, self.model.device)
        arr = (_lib.NedfField * len(nodes))(*nodes)
        hit = np.zeros(len(o), dtype=np.uint8)
        _check(_lib_trainer().nedf_trainer_batch(self.handle, arr, len(nodes), root, float(oracle.t_max),
                                                 o.ctypes.data, d.ctypes.data, len(o), hit.ctypes.data,
                                                 _lib.stream_handle()))
        return hit.astype(bool)

    def set_batch(self, feats, coarse, fine, alpha):
        """Explicit batch (tests): features (n, 1008), bin indices (-1 = no hit), alpha targets."""
        f = np.ascontiguousarray(feats, dtype=np.float32)
        c = np.ascontiguousarray(coarse, dtype=np.int32)
        fi = np.ascontiguousarray(fine, dtype=np.int32)
        a = np.ascontiguousarray(alpha, dtype=np.float32).reshape(-1)
        _check(_lib_trainer().nedf_trainer_set_batch(self.handle, f.ctypes.data, c.ctypes.data, fi.ctypes.data,
                                                     a.ctypes.data, len(f), _lib.stream_handle()))

    def loss_and_grads(self):
        """(total, (coarse, fine, alpha)) of the current batch; gradients stay on the GPU."""
        out = np.zeros(4, dtype=np.float64)
        _check(_lib_trainer().nedf_trainer_loss_and_grads(self.handle, out.ctypes.data, _lib.stream_handle()))
        return float(out[0]), (float(out[1]), float(out[2]), float(out[3]))

    def adam_step(self):
        _check(_lib_trainer().nedf_trainer_adam_step(self.handle, _lib.stream_handle()))

    def _read(self, what):
        out = np.empty(self.n_params, dtype=np.float32)
        _check(_lib_trainer().nedf_trainer_read(self.handle, what, out.ctypes.data, _lib.stream_handle()))
        return out

    def params(self) -> np.ndarray:
        return self._read(0)

    def grads(self) -> np.ndarray:
        return self._read(1)

    def nedm_bytes(self) -> bytes:
        return self._header + self.params().astype("<f4").tobytes() + self._trailer


@dataclass
class TrainingSampleBatch:
    """What build_training_batch produced (model.py:201-207); the arrays live on the GPU."""
    n: int
    origins: np.ndarray
    dirs: np.ndarray


def build_training_batch(oracle, sampler: RaySampler, trainer: Trainer, rng: np.random.Generator,
                         batch_size: int = 4096) -> TrainingSampleBatch:
    """model.py:210-235: draw rays, redraw box-missing stragglers, then encode,
    trace the oracle and quantise its depths into bin targets on the GPU."""
    origins, dirs = sampler.sample(rng, batch_size)
    hit = trainer.batch(oracle, origins, dirs)
    if not hit.all():
        retry = ~hit
        origins[retry], dirs[retry] = sampler.sample(rng, int(retry.sum()))
        hit = trainer.batch(oracle, origins, dirs)
        origins, dirs = origins[hit], dirs[hit]
        trainer.batch(oracle, origins, dirs)
    return TrainingSampleBatch(len(origins), origins, dirs)


def train(model, oracle, rng: np.random.Generator, iterations: int = 3000, batch_size: int = 1024,
          lr: float = 5e-4, sampler_mode: str = "direct", progress_every: int = 0) -> list[float]:
    """Distil the oracle into the model (model.py:251-274); returns the per-iteration loss."""
    ob = oracle.bounding_box
    box = model.relaxed_box
    if not (np.all(ob.min >= box.min - 1e-9) and np.all(ob.max <= box.max + 1e-9)):
        raise ValueError("oracle geometry escapes the model's relaxed box")
    sampler = RaySampler(box=box, mode=sampler_mode)
    trainer = Trainer(model, max_batch=batch_size, lr=lr)
    losses = []
    for it in range(iterations):
        build_training_batch(oracle, sampler, trainer, rng, batch_size)
        total, parts = trainer.loss_and_grads()
        if not np.isfinite(total):
            raise TrainingDiverged(f"non-finite loss at iteration {it}: coarse={parts[0]} fine={parts[1]} "
                                   f"alpha={parts[2]}")
        trainer.adam_step()
        losses.append(total)
        if progress_every and (it + 1) % progress_every == 0:
            print(f"iter {it + 1}/{iterations} loss {total:.4f}")
    model.reload(trainer.nedm_bytes())
    return losses
