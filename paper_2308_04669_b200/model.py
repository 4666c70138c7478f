"""NeDF models on the device: .nedm loading, random init, and the model-level
queries (reference model.py / nn.py).

`NedfModel` wraps a device handle (packed fp16 operand image for the tcgen05
kernel + fp32 copy for the guard path) plus the host metadata the pipeline
needs (classifier config, relaxed box, alpha threshold).
"""

from __future__ import annotations

import ctypes as C
import struct
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from . import _lib
from .errors import FormatError
from .geometry import Aabb, RigidTransform, relax_aabb

DEFAULT_RELAX_FACTOR = 1.5          # model.py:35
MODEL_MAGIC = b"NEDM"


@dataclass(frozen=True)
class TrainProfile:
    d_feat: int
    n_blocks: int
    batch_size: int = 4096
    iterations: int = 0
    lr: float = 5e-4


PROFILES = {                         # model.py:133-136
    "desk": TrainProfile(64, 4, 1024, 3000),
    "paper": TrainProfile(256, 16, 4096, 600_000),
}


@dataclass(frozen=True)
class ClassifierConfig:
    """mu quantisation grid: [-l, l], N_c coarse x N_f fine bins (model.py:38-65)."""
    half_range: float
    n_coarse: int = 64
    n_fine: int = 128

    def __post_init__(self):
        if not self.half_range > 0:
            raise ValueError("half_range must be positive")
        if self.n_coarse < 2 or self.n_fine < 2:
            raise ValueError("need at least 2 bins per level")

    @property
    def lambda1(self) -> float:
        return 2.0 * self.half_range

    @property
    def lambda2(self) -> float:
        return 2.0 * self.half_range / self.n_coarse

    @property
    def fine_width(self) -> float:
        return 2.0 * self.half_range / (self.n_coarse * self.n_fine)


def unsegment_batch(coarse, fine, cfg: ClassifierConfig):
    """Lower edge of the fine cell (model.py:89-92)."""
    return cfg.lambda1 * (np.asarray(coarse) / cfg.n_coarse) + cfg.lambda2 * (np.asarray(fine) / cfg.n_fine) \
        - cfg.half_range


class NedfModel:
    """A depth field resident on one GPU."""

    def __init__(self, raw: bytes, device: int | None = None):
        import torch
        dev = torch.cuda.current_device() if device is None else int(device)
        self._ctx = _lib.context(dev)
        lib = _lib.load_library()
        h = C.c_void_p()
        _lib.check(lib.nedf_model_load(self._ctx.handle, raw, len(raw), C.byref(h)))
        self.handle = h
        self.device = dev
        info = _lib.NedfModelInfo()
        _lib.check(lib.nedf_model_info(h, C.byref(info)))
        self.d_in, self.d_feat, self.n_blocks = info.d_in, info.d_feat, info.n_blocks
        self.config = ClassifierConfig(float(info.half_range), info.n_coarse, info.n_fine)
        self.relaxed_box = Aabb(np.array(info.box_min[:], dtype=np.float64),
                                np.array(info.box_max[:], dtype=np.float64))
        self.alpha_threshold = float(info.alpha_threshold)
        self.tensor_ok = bool(lib.nedf_model_tensor_ok(h))
        self._raw = bytes(raw)
        self._lib = lib

    @property
    def fine_width(self) -> float:
        return self.config.fine_width

    @property
    def n_coarse(self):
        return self.config.n_coarse

    @property
    def n_fine(self):
        return self.config.n_fine

    def nedm_bytes(self) -> bytes:
        return self._raw

    def reload(self, raw: bytes) -> None:
        """Replace the weights in place (after training) from a .nedm image of the
        same dimensions; scene tables built afterwards see the new handle."""
        h = C.c_void_p()
        _lib.check(self._lib.nedf_model_load(self._ctx.handle, raw, len(raw), C.byref(h)))
        info = _lib.NedfModelInfo()
        _lib.check(self._lib.nedf_model_info(h, C.byref(info)))
        if (info.d_in, info.d_feat, info.n_blocks) != (self.d_in, self.d_feat, self.n_blocks):
            self._lib.nedf_model_free(h)
            raise ValueError("reload: model dimensions differ")
        old, self.handle = self.handle, h
        self._raw = bytes(raw)
        self.tensor_ok = bool(self._lib.nedf_model_tensor_ok(h))
        if old:
            self._lib.nedf_model_free(old)

    def __del__(self):
        try:
            if getattr(self, "handle", None):
                self._lib.nedf_model_free(self.handle)
                self.handle = None
        except Exception:
            pass


# ---------------------------------------------------------------------------
# .nedm I/O (nn.py:235-281, model.py:354-369)
# ---------------------------------------------------------------------------

def layer_shapes(d_in, d_feat, n_blocks, n_coarse, n_fine):
    shapes = [(d_feat, d_in)] + [(d_feat, d_feat)] * (2 * n_blocks)
    return shapes + [(n_coarse + 1, d_feat), (n_fine, d_feat)]


def nedm_image(weights, half_range, box_min, box_max, alpha_threshold=0.5) -> bytes:
    """Serialise (W, b) pairs in file order into a .nedm image."""
    d_feat, d_in = weights[0][0].shape
    n_blocks = (len(weights) - 3) // 2
    n_coarse = weights[-2][0].shape[0] - 1
    n_fine = weights[-1][0].shape[0]
    out = [MODEL_MAGIC, struct.pack("<IIIIII", 1, d_in, d_feat, n_blocks, n_coarse, n_fine),
           struct.pack("<f", half_range)]
    for w, b in weights:
        out.append(np.asarray(w, dtype="<f4").tobytes())
        out.append(np.asarray(b, dtype="<f4").tobytes())
    out.append(struct.pack("<7f", *box_min, *box_max, alpha_threshold))
    return b"".join(out)


def loads_nedf(raw: bytes, device=None) -> NedfModel:
    return NedfModel(raw, device)


def load_nedf(path, device=None) -> NedfModel:
    return NedfModel(Path(path).read_bytes(), device)


def save_nedf(model: NedfModel, path) -> None:
    Path(path).write_bytes(model.nedm_bytes())


def random_weights(rng, d_in=1008, d_feat=256, n_blocks=16, n_coarse=64, n_fine=128):
    """Kaiming-uniform weights, zero biases, drawn layer by layer in file order
    (nn.py:31-35, 59-72)."""
    out = []
    for n_out, n_in in layer_shapes(d_in, d_feat, n_blocks, n_coarse, n_fine):
        bound = np.sqrt(6.0 / n_in)
        out.append((rng.uniform(-bound, bound, size=(n_out, n_in)), np.zeros(n_out)))
    return out


def new_model_bytes(bounding_box: Aabb, rng, profile: TrainProfile = PROFILES["paper"],
                    relax_factor: float = DEFAULT_RELAX_FACTOR, n_coarse=64, n_fine=128) -> bytes:
    """new_model (model.py:139-150) serialised: relaxed box, l = half diagonal."""
    box = relax_aabb(bounding_box, relax_factor)
    ws = random_weights(rng, 1008, profile.d_feat, profile.n_blocks, n_coarse, n_fine)
    return nedm_image(ws, box.half_diagonal, box.min, box.max, 0.5)


def new_model(oracle, rng, profile: TrainProfile = PROFILES["paper"], relax_factor=DEFAULT_RELAX_FACTOR,
              n_coarse=64, n_fine=128, device=None) -> NedfModel:
    if isinstance(rng, (int, np.integer)):
        rng = np.random.default_rng(int(rng))
    bb = oracle.bounding_box if hasattr(oracle, "bounding_box") else oracle
    if callable(bb):
        bb = bb()
    return NedfModel(new_model_bytes(bb, rng, profile, relax_factor, n_coarse, n_fine), device)


# ---------------------------------------------------------------------------
# model-level queries
# ---------------------------------------------------------------------------

def _as_dev_f64(x, device):
    import torch
    t = torch.as_tensor(x, dtype=torch.float64, device=f"cuda:{device}")
    return t.contiguous()


def query_rays(model: NedfModel, origins, dirs):
    """(mu, alpha) for local-space rays (model.py:277-293).  numpy in -> numpy
    out; CUDA tensors in -> CUDA tensors out."""
    import torch
    host = not (isinstance(origins, torch.Tensor) and origins.is_cuda)
    o = _as_dev_f64(origins, model.device)
    d = _as_dev_f64(dirs, model.device)
    if o.ndim != 2 or o.shape[1] != 3 or d.shape != o.shape:
        raise ValueError("origins/dirs must be (N, 3)")
    n = o.shape[0]
    mu = torch.empty(n, dtype=torch.float64, device=o.device)
    alpha = torch.empty(n, dtype=torch.uint8, device=o.device)
    ctx = model._ctx
    _lib.check(_lib.load_library().nedf_query_rays(ctx.handle, model.handle, _lib.ptr(o), _lib.ptr(d), n,
                                                   _lib.ptr(mu), _lib.ptr(alpha), _lib.stream_handle()))
    alpha = alpha.bool()
    if host:
        return mu.cpu().numpy(), alpha.cpu().numpy()
    return mu, alpha


def query_depth_world_batch(model: NedfModel, g: RigidTransform, origins, dirs):
    """World depth (model.py:301-319): |(o-T).d| - s mu, non-positive demoted."""
    import torch
    host = not (isinstance(origins, torch.Tensor) and origins.is_cuda)
    o = _as_dev_f64(origins, model.device)
    d = _as_dev_f64(dirs, model.device)
    if o.ndim != 2 or o.shape[1] != 3 or d.shape != o.shape:
        raise ValueError("origins/dirs must be (N, 3)")
    n = o.shape[0]
    depth = torch.empty(n, dtype=torch.float64, device=o.device)
    alpha = torch.empty(n, dtype=torch.uint8, device=o.device)
    R = (C.c_double * 9)(*np.asarray(g.rotation, dtype=np.float64).ravel())
    T = (C.c_double * 3)(*np.asarray(g.translation, dtype=np.float64))
    _lib.check(_lib.load_library().nedf_query_world(model._ctx.handle, model.handle, R, T, float(g.scale),
                                                    _lib.ptr(o), _lib.ptr(d), n, _lib.ptr(depth),
                                                    _lib.ptr(alpha), _lib.stream_handle()))
    alpha = alpha.bool()
    if host:
        return depth.cpu().numpy(), alpha.cpu().numpy()
    return depth, alpha


def forward(model: NedfModel, batch, precision: int = _lib.PREC_FP32):
    """nn.forward on a (B, 1008) batch -> (coarse (B,N_c), fine (B,N_f),
    alpha logit (B,1)) (nn.py:115-135)."""
    import torch
    host = not (isinstance(batch, torch.Tensor) and batch.is_cuda)
    x = torch.as_tensor(batch, dtype=torch.float32, device=f"cuda:{model.device}").contiguous()
    if x.ndim != 2 or x.shape[1] != model.d_in:
        raise ValueError(f"batch must be (B, {model.d_in}), got {tuple(x.shape)}")
    b = x.shape[0]
    lc = torch.empty(b, model.n_coarse, dtype=torch.float32, device=x.device)
    lf = torch.empty(b, model.n_fine, dtype=torch.float32, device=x.device)
    la = torch.empty(b, 1, dtype=torch.float32, device=x.device)
    _lib.check(_lib.load_library().nedf_mlp_forward(model._ctx.handle, model.handle, _lib.ptr(x), b,
                                                    _lib.ptr(lc), _lib.ptr(lf), _lib.ptr(la), int(precision),
                                                    _lib.stream_handle()))
    if host:
        return lc.cpu().numpy(), lf.cpu().numpy(), la.cpu().numpy()
    return lc, lf, la
