"""ctypes binding of the C-ABI library (include/nedf_b200.h).

The library is the only compute path: if it is missing or cannot initialise a
CUDA device this module raises -- there is no CPU fallback.
"""

from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

from .errors import FormatError

PKG = Path(__file__).resolve().parent
LIB_PATH = PKG / "libnedf_b200.so"

NEDF_OK = 0
NEDF_ERR_INVALID = -1
NEDF_ERR_FORMAT = -2
NEDF_ERR_CUDA = -3
NEDF_ERR_UNSUPPORTED = -4
NEDF_ERR_NOMEM = -5

PREC_AUTO, PREC_TENSOR, PREC_FP32 = 0, 1, 2
OPT_PRECISION, OPT_GUARD_PPM, OPT_TC_CTAS, OPT_PROFILE, OPT_TC_KERNEL, OPT_GUARD_CLUSTER = 1, 2, 3, 4, 5, 6
OPT_SETUP_EXACT, OPT_FUSE, OPT_GUARD_KERNEL, OPT_CULL, OPT_SHADOW_CERT = 7, 8, 9, 10, 11
GUARD_AUTO, GUARD_TCGEN05, GUARD_MMA_SYNC, GUARD_PRECISE = 0, 1, 2, 3
TC_AUTO, TC_SINGLE, TC_MCAST2, TC_MCAST4 = 0, 1, 3, 4

FIELD_SPHERE, FIELD_BOX, FIELD_TORUS, FIELD_PLANE, FIELD_UNION, FIELD_TRANSFORMED, FIELD_VOXEL = range(1, 8)
DEPTH_NEDF, DEPTH_ANALYTIC = 0, 1
LIGHT_POINT, LIGHT_DIRECTIONAL = 0, 1


class NedfModelInfo(C.Structure):
    _fields_ = [("d_in", C.c_int32), ("d_feat", C.c_int32), ("n_blocks", C.c_int32),
                ("n_coarse", C.c_int32), ("n_fine", C.c_int32), ("half_range", C.c_float),
                ("box_min", C.c_float * 3), ("box_max", C.c_float * 3), ("alpha_threshold", C.c_float)]


class NedfField(C.Structure):
    _fields_ = [("kind", C.c_int32), ("child", C.c_int32), ("count", C.c_int32), ("res", C.c_int32 * 3),
                ("p", C.c_double * 16), ("density_dev", C.c_void_p), ("color_dev", C.c_void_p)]


class NedfObject(C.Structure):
    _fields_ = [("R", C.c_double * 9), ("T", C.c_double * 3), ("s", C.c_double), ("id", C.c_int32),
                ("depth_kind", C.c_int32), ("model", C.c_void_p), ("depth_field", C.c_int32),
                ("radiance_field", C.c_int32)]


class NedfCamera(C.Structure):
    _fields_ = [("position", C.c_double * 3), ("orientation", C.c_double * 9), ("fov_y", C.c_double),
                ("width", C.c_int32), ("height", C.c_int32)]


class NedfLight(C.Structure):
    _fields_ = [("kind", C.c_int32), ("vec", C.c_double * 3), ("beta", C.c_double)]


class NedfRenderConfig(C.Structure):
    _fields_ = [("sigma_threshold", C.c_double), ("resample", C.c_int32), ("resample_samples", C.c_int32),
                ("shadow_epsilon", C.c_double), ("shadows", C.c_int32), ("clear_color", C.c_double * 3)]


class NedfFrameBuffers(C.Structure):
    _fields_ = [("depth_dev", C.c_void_p), ("id_dev", C.c_void_p), ("rgb_dev", C.c_void_p),
                ("shadow_dev", C.c_void_p), ("image_dev", C.c_void_p), ("planes_dev", C.c_void_p),
                ("rows_host", C.POINTER(C.c_int32)), ("n_rows", C.c_int32)]


class NedfStepStats(C.Structure):
    _fields_ = [("evals", C.c_int64), ("guarded", C.c_int64), ("covered", C.c_int64), ("resampled", C.c_int64),
                ("launches", C.c_int64), ("net_launches", C.c_int64), ("net_ms", C.c_double),
                ("guard_ms", C.c_double), ("h2d_bytes", C.c_int64), ("exact_clips", C.c_int64),
                ("culled", C.c_int64)]


P = C.c_void_p
I32, I64, F64 = C.c_int32, C.c_int64, C.c_double

# name -> (restype, argtypes); must list every function include/nedf_b200.h declares
PROTOTYPES = {
    "nedf_abi_version": (C.c_int, []),
    "nedf_last_error": (C.c_char_p, []),
    "nedf_context_create": (C.c_int, [C.c_int, C.POINTER(P)]),
    "nedf_context_destroy": (None, [P]),
    "nedf_set_option": (C.c_int, [P, C.c_int, I64]),
    "nedf_get_option": (C.c_int, [P, C.c_int, C.POINTER(I64)]),
    "nedf_read_stats": (C.c_int, [P, C.POINTER(NedfStepStats), P]),
    "nedf_model_load": (C.c_int, [P, C.c_char_p, C.c_size_t, C.POINTER(P)]),
    "nedf_model_create": (C.c_int, [P, C.POINTER(NedfModelInfo), P, C.c_size_t, C.POINTER(P)]),
    "nedf_model_free": (None, [P]),
    "nedf_model_info": (C.c_int, [P, C.POINTER(NedfModelInfo)]),
    "nedf_model_tensor_ok": (C.c_int, [P]),
    "nedf_mlp_forward": (C.c_int, [P, P, P, I64, P, P, P, C.c_int, P]),
    "nedf_query_rays": (C.c_int, [P, P, P, P, I64, P, P, P]),
    "nedf_query_world": (C.c_int, [P, P, C.POINTER(F64), C.POINTER(F64), F64, P, P, I64, P, P, P]),
    "nedf_generation_step": (C.c_int, [P, C.POINTER(NedfCamera), C.POINTER(NedfObject), C.c_int,
                                       C.POINTER(NedfField), C.c_int, C.POINTER(NedfFrameBuffers), P]),
    "nedf_reuse_step": (C.c_int, [P, C.POINTER(NedfCamera), C.POINTER(NedfObject), C.c_int,
                                  C.POINTER(NedfField), C.c_int, C.POINTER(C.c_int32), C.c_int,
                                  C.POINTER(NedfFrameBuffers), P]),
    "nedf_shading_step": (C.c_int, [P, C.POINTER(NedfCamera), C.POINTER(NedfObject), C.c_int,
                                    C.POINTER(NedfField), C.c_int, C.POINTER(NedfRenderConfig),
                                    C.POINTER(NedfFrameBuffers), P]),
    "nedf_shadow_step": (C.c_int, [P, C.POINTER(NedfCamera), C.POINTER(NedfObject), C.c_int,
                                   C.POINTER(NedfField), C.c_int, C.POINTER(NedfLight),
                                   C.POINTER(NedfRenderConfig), C.POINTER(NedfFrameBuffers), P]),
    "nedf_composite": (C.c_int, [P, C.POINTER(NedfFrameBuffers), C.c_int, P]),
    "nedf_stats_snapshot": (C.c_int, [P, C.c_int, C.POINTER(NedfStepStats), P]),
    "nedf_stats_slot": (C.c_int, [P, C.c_int, C.POINTER(NedfStepStats)]),
    "nedf_to_u8": (C.c_int, [P, I64, P, P]),
    "nedf_depth_to_f32": (C.c_int, [P, I64, P, P]),
    "nedf_depth_to_gray": (C.c_int, [P, I64, P, P, P]),
    "nedf_id_to_u16": (C.c_int, [P, I64, P, P]),
    "nedf_trainer_last_error": (C.c_char_p, []),
    "nedf_trainer_create": (C.c_int, [C.c_int, C.POINTER(NedfModelInfo), P, I64, C.c_int, C.POINTER(P)]),
    "nedf_trainer_destroy": (None, [P]),
    "nedf_trainer_set_lr": (C.c_int, [P, C.c_float]),
    "nedf_trainer_batch": (C.c_int, [P, P, C.c_int, C.c_int, C.c_double, P, P, C.c_int, P, P]),
    "nedf_trainer_set_batch": (C.c_int, [P, P, P, P, P, C.c_int, P]),
    "nedf_trainer_loss_and_grads": (C.c_int, [P, P, P]),
    "nedf_trainer_adam_step": (C.c_int, [P, P]),
    "nedf_trainer_read": (C.c_int, [P, C.c_int, P, P]),
    "nedf_render_frame": (C.c_int, [P, C.POINTER(NedfCamera), C.POINTER(NedfObject), C.c_int,
                                    C.POINTER(NedfField), C.c_int, C.POINTER(NedfLight), C.c_int,
                                    C.POINTER(NedfRenderConfig), C.POINTER(NedfFrameBuffers), P]),
    "nedf_render_frame_timed": (C.c_int, [P, C.POINTER(NedfCamera), C.POINTER(NedfObject), C.c_int,
                                          C.POINTER(NedfField), C.c_int, C.POINTER(NedfLight), C.c_int,
                                          C.POINTER(NedfRenderConfig), C.POINTER(NedfFrameBuffers),
                                          C.POINTER(P), P]),
}

_lib = None
_lock = threading.Lock()


def load_library(path: Path | str | None = None):
    """Load (once) the built library; raises if it is missing."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        # NEDF_LIB: load an alternative build (timing experiments); still the native library, no fallback
        p = Path(path) if path else Path(os.environ.get("NEDF_LIB", LIB_PATH))
        if not p.exists():
            raise RuntimeError(f"{p} not built: run `python -m paper_2308_04669_b200.build` "
                               "(there is no CPU fallback)")
        lib = C.CDLL(str(p))
        for name, (res, args) in PROTOTYPES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if lib.nedf_abi_version() != 1:
            raise RuntimeError("libnedf_b200 ABI version mismatch")
        _lib = lib
        return lib


def check(rc: int):
    if rc == NEDF_OK:
        return
    msg = (load_library().nedf_last_error() or b"").decode(errors="replace")
    if rc == NEDF_ERR_FORMAT:
        raise FormatError(msg)
    if rc == NEDF_ERR_INVALID:
        raise ValueError(msg)
    if rc == NEDF_ERR_UNSUPPORTED:
        raise TypeError(msg)
    raise RuntimeError(f"nedf_b200 error {rc}: {msg}")


class Context:
    """Owns a NedfContext (per device)."""

    def __init__(self, device: int = 0):
        lib = load_library()
        h = C.c_void_p()
        check(lib.nedf_context_create(int(device), C.byref(h)))
        self.handle = h
        self.device = int(device)
        self._lib = lib

    def set_option(self, key: int, value: int):
        check(self._lib.nedf_set_option(self.handle, key, int(value)))

    def get_option(self, key: int) -> int:
        v = C.c_int64()
        check(self._lib.nedf_get_option(self.handle, key, C.byref(v)))
        return int(v.value)

    def read_stats(self, stream) -> dict:
        s = NedfStepStats()
        check(self._lib.nedf_read_stats(self.handle, C.byref(s), stream))
        return {"evals": s.evals, "guarded": s.guarded, "covered": s.covered, "resampled": s.resampled,
                "launches": s.launches, "net_launches": s.net_launches, "net_ms": s.net_ms,
                "guard_ms": s.guard_ms, "h2d_bytes": s.h2d_bytes, "exact_clips": s.exact_clips,
                "culled": s.culled}

    _RESET_SLOT = 63                     # mapped slot 63 only absorbs resets; 0-62 rotate

    def reset_stats(self, stream) -> None:
        """Non-blocking: zero the device counters (their old values land in the reset slot)."""
        s = NedfStepStats()
        check(self._lib.nedf_stats_snapshot(self.handle, self._RESET_SLOT, C.byref(s), stream))

    def snapshot_stats(self, stream) -> tuple[tuple[int, int], dict]:
        """Non-blocking: enqueue this step's counters into the next mapped slot; returns
        (ticket, host-side counters).  Resolve with `slot_stats(ticket)` after the stream
        passes this point; 63 slots rotate, and a ticket whose slot has been reused since
        raises instead of returning another step's counters."""
        seq = getattr(self, "_seq", 0)
        self._seq = seq + 1
        slot = seq % self._RESET_SLOT
        if not hasattr(self, "_slot_owner"):
            self._slot_owner = {}
        self._slot_owner[slot] = seq
        s = NedfStepStats()
        check(self._lib.nedf_stats_snapshot(self.handle, slot, C.byref(s), stream))
        return (slot, seq), {"launches": s.launches, "h2d_bytes": s.h2d_bytes}

    def slot_stats(self, ticket) -> dict:
        slot, seq = ticket
        if self._slot_owner.get(slot) != seq:
            raise RuntimeError(f"stats of step {seq} were overwritten: read them within "
                               f"{self._RESET_SLOT} steps")
        s = NedfStepStats()
        check(self._lib.nedf_stats_slot(self.handle, slot, C.byref(s)))
        return {"evals": s.evals, "guarded": s.guarded, "covered": s.covered, "resampled": s.resampled,
                "exact_clips": s.exact_clips, "culled": s.culled}

    def __del__(self):
        try:
            if getattr(self, "handle", None):
                self._lib.nedf_context_destroy(self.handle)
                self.handle = None
        except Exception:
            pass


_contexts: dict = {}


def context(device: int | None = None) -> Context:
    import torch
    if device is None:
        device = torch.cuda.current_device()
    with _lock:
        ctx = _contexts.get(device)
    if ctx is None:
        ctx = Context(device)
        with _lock:
            _contexts[device] = ctx
    return ctx


def stream_handle(stream=None):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def ptr(t) -> C.c_void_p:
    return C.c_void_p(t.data_ptr()) if t is not None else C.c_void_p(0)
