"""Buffer export / import formats (the reference's imgio.py).

Colour goes out as binary PPM (P6) or PNG; depth as a raw little-endian f32
plane with a 16-byte header (NDPT) plus a normalised grayscale PNG; object ids
as 16-bit grayscale PNG (id + 1, zero = no hit).  The per-pixel conversions
(`to_u8`, the f32 depth plane, `depth_to_gray`, the id shift) run on the GPU
through the C ABI (`nedf_to_u8`, `nedf_depth_to_f32`, `nedf_depth_to_gray`,
`nedf_id_to_u16`, csrc/imgio.cu), so only 8/16-bit planes cross to the host;
PNG compression and file I/O stay on the host (Pillow, as in the reference).

Inputs may be CUDA tensors (converted where they are) or numpy arrays (uploaded
first -- there is no CPU conversion path).  Results are numpy arrays / bytes,
bit-identical to the reference's functions on the same values.
"""

from __future__ import annotations

import io
import struct

import numpy as np

from . import _lib
from .errors import FormatError

DEPTH_MAGIC = b"NDPT"                          # imgio.py:19
BUFFER_KINDS = {"color": 0, "depth": 1, "id": 2, "shadow": 3}   # service.py:33
ENCODING_PNG = 0
HEADER_FMT = "<IBBHII"                         # revision, buffer kind, encoding, reserved, W, H


def _dev(x, dtype):
    import torch
    if isinstance(x, torch.Tensor) and x.is_cuda:
        return x.to(dtype).contiguous()
    return torch.as_tensor(np.ascontiguousarray(x), dtype=dtype).cuda()


def _run(fn, *args):
    import torch
    _lib.check(fn(*args, _lib.stream_handle()))
    torch.cuda.current_stream().synchronize()


def to_u8(rgb) -> np.ndarray:
    """(clip(x, 0, 1) * 255 + 0.5) -> uint8 (imgio.py:23-24), on the GPU."""
    import torch
    src = _dev(rgb, torch.float32)
    out = torch.empty(src.shape, dtype=torch.uint8, device=src.device)
    _run(_lib.load_library().nedf_to_u8, _lib.ptr(src), src.numel(), _lib.ptr(out))
    return out.cpu().numpy()


def depth_plane_f32(depth) -> np.ndarray:
    """float64 depth -> float32 plane, misses stay +inf (imgio.py:63-71), on the GPU."""
    import torch
    src = _dev(depth, torch.float64)
    out = torch.empty(src.shape, dtype=torch.float32, device=src.device)
    _run(_lib.load_library().nedf_depth_to_f32, _lib.ptr(src), src.numel(), _lib.ptr(out))
    return out.cpu().numpy()


def depth_to_gray(depth) -> np.ndarray:
    """Nearest surface bright, farthest dark, misses black (imgio.py:88-97), on the GPU."""
    import torch
    src = _dev(depth, torch.float64)
    out = torch.empty(src.shape, dtype=torch.uint8, device=src.device)
    scratch = torch.empty(2, dtype=torch.int64, device=src.device)
    _run(_lib.load_library().nedf_depth_to_gray, _lib.ptr(src), src.numel(), _lib.ptr(out), _lib.ptr(scratch))
    return out.cpu().numpy()


def id_to_u16(id_plane) -> np.ndarray:
    """(id + 1).clip(0, 65535) as uint16 (imgio.py:106-111), on the GPU."""
    import torch
    src = _dev(id_plane, torch.int32)
    out = torch.empty(src.shape, dtype=torch.int16, device=src.device)     # bit pattern of uint16
    _run(_lib.load_library().nedf_id_to_u16, _lib.ptr(src), src.numel(), _lib.ptr(out))
    return out.cpu().numpy().view(np.uint16)


# ---- host-side encoders (same byte formats as the reference) ----------------------------

def write_ppm(path, rgb) -> None:
    """Binary PPM (P6) of an (H, W, 3) image in [0, 1] (imgio.py:27-32)."""
    u8 = to_u8(rgb)
    h, w, _ = u8.shape
    with open(path, "wb") as f:
        f.write(f"P6\n{w} {h}\n255\n".encode())
        f.write(u8.tobytes())


def read_ppm(path) -> np.ndarray:
    """imgio.py:35-45."""
    with open(path, "rb") as f:
        if f.readline().strip() != b"P6":
            raise FormatError(f"{path}: not a binary PPM")
        dims = f.readline().split()
        w, h = int(dims[0]), int(dims[1])
        maxval = int(f.readline())
        if maxval != 255:
            raise FormatError(f"{path}: only 8-bit PPM supported")
        data = np.frombuffer(f.read(w * h * 3), dtype=np.uint8)
    return data.reshape(h, w, 3).astype(np.float64) / 255.0


def _png(arr, mode=None) -> bytes:
    from PIL import Image
    buf = io.BytesIO()
    (Image.fromarray(arr, mode=mode) if mode else Image.fromarray(arr)).save(buf, format="PNG")
    return buf.getvalue()


def encode_color_png(rgb) -> bytes:
    return _png(to_u8(rgb), "RGB")


def write_color_png(path, rgb) -> None:
    with open(path, "wb") as f:
        f.write(encode_color_png(rgb))


def read_color_png(path) -> np.ndarray:
    from PIL import Image
    return np.asarray(Image.open(path).convert("RGB"), dtype=np.float64) / 255.0


def depth_raw_bytes(depth, scale: float = 1.0) -> bytes:
    """16-byte header (magic, u32 W, u32 H, f32 scale) + row-major f32 plane (imgio.py:63-71)."""
    plane = depth_plane_f32(depth)
    h, w = plane.shape
    return DEPTH_MAGIC + struct.pack("<IIf", w, h, scale) + plane.astype("<f4").tobytes(order="C")


def write_depth_raw(path, depth, scale: float = 1.0) -> None:
    with open(path, "wb") as f:
        f.write(depth_raw_bytes(depth, scale))


def read_depth_raw(path) -> tuple[np.ndarray, float]:
    """imgio.py:74-85 (same FormatError cases)."""
    with open(path, "rb") as f:
        raw = f.read()
    if raw[:4] != DEPTH_MAGIC:
        raise FormatError(f"{path}: not a raw depth plane")
    if len(raw) < 16:
        raise FormatError(f"{path}: truncated header")
    w, h, scale = struct.unpack_from("<IIf", raw, 4)
    if len(raw) != 16 + 4 * w * h:
        raise FormatError(f"{path}: expected {16 + 4 * w * h} bytes, found {len(raw)}")
    plane = np.frombuffer(raw, dtype="<f4", count=w * h, offset=16)
    return plane.reshape(h, w).astype(np.float64), float(scale)


def encode_depth_png(depth) -> bytes:
    return _png(depth_to_gray(depth), "L")


def encode_id_png(id_plane) -> bytes:
    return _png(id_to_u16(id_plane))


def encode_gray_png(plane01) -> bytes:
    """imgio.py:114-118: the same u8 mapping as colour."""
    return _png(to_u8(plane01), "L")


def encode_plane(kind: str, plane) -> bytes:
    """service.py:203-212."""
    if kind == "color":
        return encode_color_png(plane)
    if kind == "depth":
        return encode_depth_png(plane)
    if kind == "id":
        return encode_id_png(plane)
    if kind == "shadow":
        return encode_gray_png(plane)
    raise ValueError(f"unknown buffer kind {kind!r}")


def frame_message(revision: int, kind: str, plane) -> bytes:
    """Stream frame: 16-byte header + PNG payload (service.py:215-219)."""
    payload = encode_plane(kind, plane)
    h, w = tuple(plane.shape[:2])
    return struct.pack(HEADER_FMT, revision, BUFFER_KINDS[kind], ENCODING_PNG, 0, w, h) + payload
