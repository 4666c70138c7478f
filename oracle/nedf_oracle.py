"""CPU oracle for the NeDF per-frame hot path -- TEST INFRASTRUCTURE ONLY.

This module is a float64 numpy restatement of the reference algorithm
(`/root/reference/pkg/src/nedf/*`, cited below as file:line).  It exists so
that the B200 product path can be checked for parity without the reference
being present (the GPU box has no /root/reference).  Only `tests/`,
`__graft_entry__.smoke()` and `bench.py`'s CPU-baseline leg may import it,
and only as the checker / the timed CPU baseline -- never as a fallback of the
product path (`paper_2308_04669_b200` never imports this package).

Parity pinning: `tests/golden/make_golden.py` runs the real reference in the
build container and stores its outputs under `tests/golden/`;
`tests/test_oracle_golden.py` checks this restatement against them.

Layout conventions follow the reference: rays are (N, 3) float64, images are
row-major with row 0 at the top, misses are depth=+inf / id=-1.
"""

from __future__ import annotations

import math
import os
import struct
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field

import numpy as np

# geometry.py:21-24 -- 16 samples x 3 coords x (1 + 2*10) = 1008 features
N_POINTS = 16
N_LEVELS = 10
PER_POINT = 3 * (1 + 2 * N_LEVELS)
D_ENC = N_POINTS * PER_POINT

RELAX = 1.5                     # model.py:35
QUERY_CHUNK = 16384             # pipeline.py:33
SIGMA_SURFACE = 50.0            # fields.py:31
SURFACE_BAND = 0.02             # fields.py:32
INTERIOR_STEEPNESS = 1000.0     # fields.py:33
SURFACE_EPS = 1e-5              # fields.py:25
MAX_TRACE_STEPS = 512           # fields.py:26


# ---------------------------------------------------------------------------
# camera / primary rays  (pipeline.py:53-109)
# ---------------------------------------------------------------------------

def look_at(position, target, up=(0.0, 1.0, 0.0)) -> np.ndarray:
    """Camera-to-world rotation with columns [right, up, -forward]
    (pipeline.py:80-94)."""
    p = np.asarray(position, dtype=np.float64)
    f = np.asarray(target, dtype=np.float64) - p
    f = f / np.linalg.norm(f)
    r = np.cross(f, np.asarray(up, dtype=np.float64))
    r = r / np.linalg.norm(r)
    u = np.cross(r, f)
    return np.stack([r, u, -f], axis=1)


@dataclass
class Cam:
    position: np.ndarray
    orientation: np.ndarray
    fov_y: float
    width: int
    height: int


def primary_rays(cam: Cam, pixels: np.ndarray | None = None):
    """Pixel-centre pinhole rays (pipeline.py:97-109).  `pixels` optionally
    restricts to flat row-major pixel indices (results per pixel are
    independent of the others, so a subset is exact)."""
    w, h = cam.width, cam.height
    if pixels is None:
        pixels = np.arange(w * h)
    col = pixels % w
    row = pixels // w
    th = np.tan(cam.fov_y / 2.0)
    gx = (((col + 0.5) / w) * 2.0 - 1.0) * th * (w / h)
    gy = (1.0 - ((row + 0.5) / h) * 2.0) * th
    dc = np.stack([gx, gy, -np.ones_like(gx)], axis=1)
    d = dc @ np.asarray(cam.orientation, dtype=np.float64).T
    d = d / np.linalg.norm(d, axis=1, keepdims=True)
    o = np.broadcast_to(np.asarray(cam.position, dtype=np.float64), d.shape).copy()
    return o, d


# ---------------------------------------------------------------------------
# slab clip, sampling, sinusoidal encoding  (geometry.py:258-342)
# ---------------------------------------------------------------------------

def slab_clip(o, d, bmin, bmax):
    """(t_enter, t_exit, hit); NaN slab bounds (0*inf) widen to +-inf and a
    grazing t_exit == t_enter counts as a hit (geometry.py:258-280)."""
    with np.errstate(divide="ignore", invalid="ignore"):
        inv = 1.0 / d
        ta = (np.asarray(bmin)[None, :] - o) * inv
        tb = (np.asarray(bmax)[None, :] - o) * inv
    lo = np.minimum(ta, tb)
    hi = np.maximum(ta, tb)
    lo[np.isnan(lo)] = -np.inf
    hi[np.isnan(hi)] = np.inf
    t0 = np.maximum(lo.max(axis=1), 0.0)
    t1 = hi.min(axis=1)
    return t0, t1, t1 >= t0


def sample_points(o, d, t0, t1, bmin, bmax):
    """16 endpoint-inclusive samples over [t0, t1], mapped to the box's
    [-1, 1]^3 frame (geometry.py:336-340)."""
    bmin = np.asarray(bmin, dtype=np.float64)
    bmax = np.asarray(bmax, dtype=np.float64)
    frac = np.linspace(0.0, 1.0, N_POINTS)
    t = t0[:, None] + (t1 - t0)[:, None] * frac[None, :]
    pts = o[:, None, :] + t[:, :, None] * d[:, None, :]
    c = 0.5 * (bmin + bmax)
    h = 0.5 * (bmax - bmin)
    h = np.where(h > 0, h, 1.0)
    return (pts - c[None, None, :]) / h[None, None, :]


def encode_points(pts):
    """(N, 16, 3) -> (N, 1008); per coordinate [p, sin(2^k pi p), cos(2^k pi p)]
    for k = 0..9, coordinates then points in order (geometry.py:312-321)."""
    n = pts.shape[0]
    w = np.pi * (2.0 ** np.arange(N_LEVELS))
    ang = pts[..., None] * w
    out = np.empty(pts.shape + (1 + 2 * N_LEVELS,), dtype=np.float64)
    out[..., 0] = pts
    out[..., 1::2] = np.sin(ang)
    out[..., 2::2] = np.cos(ang)
    return out.reshape(n, D_ENC)


def encode_rays(o, d, bmin, bmax):
    """(features (N, 1008) zero on misses, hit) -- geometry.py:324-342."""
    t0, t1, hit = slab_clip(o, d, bmin, bmax)
    feats = np.zeros((o.shape[0], D_ENC))
    if hit.any():
        feats[hit] = encode_points(sample_points(o[hit], d[hit], t0[hit], t1[hit], bmin, bmax))
    return feats, hit


# ---------------------------------------------------------------------------
# network, model file, random init  (nn.py, model.py)
# ---------------------------------------------------------------------------

@dataclass
class OracleModel:
    """Parameters in the reference traversal order (nn.py:98-112):
    head, blocks (fc1, fc2) ..., tail_a (N_c + 1, alpha last), tail_b (N_f)."""
    weights: list            # list of (W (out,in) f64, b (out,) f64)
    half_range: float
    box_min: np.ndarray
    box_max: np.ndarray
    alpha_threshold: float = 0.5

    @property
    def d_in(self):
        return self.weights[0][0].shape[1]

    @property
    def d_feat(self):
        return self.weights[0][0].shape[0]

    @property
    def n_blocks(self):
        return (len(self.weights) - 3) // 2

    @property
    def n_coarse(self):
        return self.weights[-2][0].shape[0] - 1

    @property
    def n_fine(self):
        return self.weights[-1][0].shape[0]

    @property
    def fine_width(self):
        return 2.0 * self.half_range / (self.n_coarse * self.n_fine)


def layer_shapes(d_in, d_feat, n_blocks, n_coarse, n_fine):
    """(out, in) per linear layer in file order (nn.py:59-72, 98-104)."""
    shapes = [(d_feat, d_in)]
    shapes += [(d_feat, d_feat)] * (2 * n_blocks)
    shapes += [(n_coarse + 1, d_feat), (n_fine, d_feat)]
    return shapes


def random_init(seed, d_feat=256, n_blocks=16, n_coarse=64, n_fine=128, d_in=1008):
    """Kaiming-uniform weights with zero biases, drawn layer by layer from
    default_rng(seed) in file order (nn.py:31-35, 59-72)."""
    rng = np.random.default_rng(seed)
    out = []
    for n_out, n_in in layer_shapes(d_in, d_feat, n_blocks, n_coarse, n_fine):
        bound = np.sqrt(6.0 / n_in)
        out.append((rng.uniform(-bound, bound, size=(n_out, n_in)), np.zeros(n_out)))
    return out


def canonical_prim_box(kind):
    """Bounding boxes of the canonical CLI geometries (cli.py:25-29,
    fields.py:77-126)."""
    if kind == "sphere":
        h = np.array([1.0, 1.0, 1.0])
    elif kind == "box":
        h = np.array([0.8, 0.5, 0.6])
    elif kind == "torus":
        h = np.array([0.95, 0.25, 0.95])
    else:
        raise ValueError(kind)
    return -h, h


def new_paper_model(seed, kind="sphere", d_feat=256, n_blocks=16):
    """new_model(AnalyticOracle(prim), default_rng(seed), PROFILES[...]) as it
    is after save_nedf -> load_nedf, i.e. f32-exact parameters, f32 l and box
    (model.py:139-150, 354-369)."""
    lo, hi = canonical_prim_box(kind)
    c, h = 0.5 * (lo + hi), 0.5 * (hi - lo)
    bmin, bmax = c - RELAX * h, c + RELAX * h
    l = float(np.linalg.norm(0.5 * (bmax - bmin)))
    m = OracleModel(random_init(seed, d_feat, n_blocks), l, bmin, bmax, 0.5)
    return parse_nedm(nedm_bytes(m))


def nedm_bytes(m: OracleModel) -> bytes:
    """`.nedm` = b"NEDM", <6I version/dims, <f l, f32 params, <7f trailer
    (box min, box max, alpha threshold) -- nn.py:235-246, model.py:354-361."""
    parts = [b"NEDM", struct.pack("<IIIIII", 1, m.d_in, m.d_feat, m.n_blocks,
                                  m.n_coarse, m.n_fine), struct.pack("<f", m.half_range)]
    for w, b in m.weights:
        parts.append(np.asarray(w, dtype="<f4").tobytes())
        parts.append(np.asarray(b, dtype="<f4").tobytes())
    parts.append(struct.pack("<7f", *m.box_min, *m.box_max, m.alpha_threshold))
    return b"".join(parts)


def parse_nedm(raw: bytes) -> OracleModel:
    """Inverse of nedm_bytes with the reference's size checks (nn.py:249-281,
    model.py:364-369).  Raises ValueError on malformed input."""
    if raw[:4] != b"NEDM":
        raise ValueError("not a model file")
    if len(raw) < 32:
        raise ValueError("truncated header")
    ver, d_in, d_feat, nb, nc, nf = struct.unpack_from("<IIIIII", raw, 4)
    if ver != 1:
        raise ValueError(f"unsupported version {ver}")
    (l,) = struct.unpack_from("<f", raw, 28)
    shapes = layer_shapes(d_in, d_feat, nb, nc, nf)
    n_par = sum(o * i + o for o, i in shapes)
    if len(raw) != 32 + 4 * n_par + 28:
        raise ValueError("size does not match declared dimensions")
    flat = np.frombuffer(raw, dtype="<f4", count=n_par, offset=32).astype(np.float64)
    ws, off = [], 0
    for o, i in shapes:
        w = flat[off:off + o * i].reshape(o, i)
        off += o * i
        b = flat[off:off + o]
        off += o
        ws.append((w, b))
    tr = struct.unpack_from("<7f", raw, 32 + 4 * n_par)
    return OracleModel(ws, float(l), np.array(tr[0:3], dtype=np.float64),
                       np.array(tr[3:6], dtype=np.float64), float(tr[6]))


def mlp_forward(m: OracleModel, feats):
    """(coarse (B,N_c), fine (B,N_f), alpha logit (B,)) -- no activation on
    the head, ReLU before the residual add, y = x W^T + b (nn.py:45-46,
    115-135)."""
    (wh, bh) = m.weights[0]
    x = feats @ wh.T + bh
    for k in range(m.n_blocks):
        w1, b1 = m.weights[1 + 2 * k]
        w2, b2 = m.weights[2 + 2 * k]
        h = np.maximum(x @ w1.T + b1, 0.0)
        x = x + np.maximum(h @ w2.T + b2, 0.0)
    wa, ba = m.weights[-2]
    wb, bb = m.weights[-1]
    a = x @ wa.T + ba
    return a[:, :-1], x @ wb.T + bb, a[:, -1]


def decode_mu(m: OracleModel, coarse_idx, fine_idx):
    """Lower edge of the fine cell: 2l*c/N_c + (2l/N_c)*f/N_f - l
    (model.py:89-92)."""
    l = m.half_range
    return (2.0 * l) * (coarse_idx / m.n_coarse) + (2.0 * l / m.n_coarse) * (fine_idx / m.n_fine) - l


def query_local(m: OracleModel, o, d, return_logits=False):
    """(mu, alpha) for local rays; box misses skip the network with mu=NaN,
    alpha=False; argmax ties take the lowest bin (model.py:277-293).  The
    alpha test sigma(z) > thr is evaluated as in nn.py:169-175."""
    feats, hit = encode_rays(o, d, m.box_min, m.box_max)
    mu = np.full(o.shape[0], np.nan)
    alpha = np.zeros(o.shape[0], dtype=bool)
    logits = None
    if hit.any():
        lc, lf, la = mlp_forward(m, feats[hit])
        mu[hit] = decode_mu(m, lc.argmax(axis=1), lf.argmax(axis=1))
        alpha[hit] = _sigmoid(la) > m.alpha_threshold
        logits = (lc, lf, la)
    if return_logits:
        return mu, alpha, hit, logits
    return mu, alpha


def _sigmoid(z):
    out = np.empty_like(z)
    pos = z >= 0
    out[pos] = 1.0 / (1.0 + np.exp(-z[pos]))
    ez = np.exp(z[~pos])
    out[~pos] = ez / (1.0 + ez)
    return out


def world_depth(m: OracleModel, R, T, s, o, d):
    """query_depth_world_batch (model.py:301-319): local ray
    ((o-T) R / s, d R), depth = |(o-T).d| - s*mu, non-positive depth demoted."""
    R = np.asarray(R, dtype=np.float64)
    T = np.asarray(T, dtype=np.float64)
    lo = ((o - T) @ R) / s
    ld = d @ R
    mu, alpha = query_local(m, lo, ld)
    dist = np.abs(np.einsum("ij,ij->i", o - T, d))
    depth = dist - s * mu
    alpha = alpha & (depth > 0)
    return depth, alpha


# ---------------------------------------------------------------------------
# analytic fields: SDFs, sphere tracing, radiance  (fields.py)
# ---------------------------------------------------------------------------
# prim specs: ("sphere", c, r) ("box", c, h) ("torus", c, R, r)
#             ("plane", n, off) ("union", [children]) ("transformed", child, R, T, s)
#             ("voxel", res, bmin, bmax, density (nx,ny,nz), color (nx,ny,nz,3))

def sdf(prim, p):
    kind = prim[0]
    if kind == "sphere":
        return np.linalg.norm(p - np.asarray(prim[1]), axis=-1) - prim[2]
    if kind == "box":
        q = np.abs(p - np.asarray(prim[1])) - np.asarray(prim[2])
        return np.linalg.norm(np.maximum(q, 0.0), axis=-1) + np.minimum(q.max(axis=-1), 0.0)
    if kind == "torus":
        q = p - np.asarray(prim[1])
        return np.hypot(np.hypot(q[..., 0], q[..., 2]) - prim[2], q[..., 1]) - prim[3]
    if kind == "plane":
        return p @ np.asarray(prim[1]) - prim[2]
    if kind == "union":
        return np.minimum.reduce([sdf(ch, p) for ch in prim[1]])
    if kind == "transformed":
        _, ch, R, T, s = prim
        return s * sdf(ch, ((p - np.asarray(T)) @ np.asarray(R)) / s)
    raise ValueError(kind)


def prim_bounds(prim):
    kind = prim[0]
    if kind == "sphere":
        c = np.asarray(prim[1], dtype=np.float64)
        return c - prim[2], c + prim[2]
    if kind == "box":
        c = np.asarray(prim[1], dtype=np.float64)
        return c - np.asarray(prim[2]), c + np.asarray(prim[2])
    if kind == "torus":
        c = np.asarray(prim[1], dtype=np.float64)
        e = np.array([prim[2] + prim[3], prim[3], prim[2] + prim[3]])
        return c - e, c + e
    if kind == "union":
        bs = [prim_bounds(ch) for ch in prim[1]]
        return np.minimum.reduce([b[0] for b in bs]), np.maximum.reduce([b[1] for b in bs])
    if kind == "transformed":
        _, ch, R, T, s = prim
        lo, hi = prim_bounds(ch)
        corners = np.array([[x, y, z] for x in (lo[0], hi[0]) for y in (lo[1], hi[1])
                            for z in (lo[2], hi[2])])
        wc = s * (corners @ np.asarray(R).T) + np.asarray(T)
        return wc.min(axis=0), wc.max(axis=0)
    if kind == "voxel":
        return np.asarray(prim[2], dtype=np.float64), np.asarray(prim[3], dtype=np.float64)
    raise ValueError(f"{kind} has no finite bounds")


def sphere_trace(prim, o, d, t_max=100.0):
    """Sphere tracing + 6 secant iterations (fields.py:194-238)."""
    n = o.shape[0]
    t = np.zeros(n)
    hit = np.zeros(n, dtype=bool)
    inside = sdf(prim, o) <= -SURFACE_EPS
    hit[inside] = True
    act = ~inside
    for _ in range(MAX_TRACE_STEPS):
        if not act.any():
            break
        idx = np.flatnonzero(act)
        dist = sdf(prim, o[idx] + t[idx, None] * d[idx])
        conv = np.abs(dist) < SURFACE_EPS
        hit[idx[conv]] = True
        t[idx] += np.where(conv, 0.0, dist)
        act[idx] = ~conv & (t[idx] <= t_max)
    ref = hit & ~inside
    if ref.any():
        oo, dd = o[ref], d[ref]
        ta, tb = t[ref] - SURFACE_EPS, t[ref] + SURFACE_EPS
        fa = sdf(prim, oo + ta[:, None] * dd)
        fb = sdf(prim, oo + tb[:, None] * dd)
        for _ in range(6):
            den = fb - fa
            ok = np.abs(den) > 1e-300
            tn = np.where(ok, tb - fb * (tb - ta) / np.where(ok, den, 1.0), tb)
            ta, fa, tb = tb, fb, tn
            fb = sdf(prim, oo + tb[:, None] * dd)
        t[ref] = np.maximum(tb, 0.0)
    return t, hit


def voxel_sample(prim, p):
    """Trilinear over cell centres, clamped, zero outside the bounds
    (fields.py:294-319)."""
    _, res, bmin, bmax, dens, col = prim
    res = np.asarray(res)
    resf = res.astype(np.float64)
    bmin = np.asarray(bmin, dtype=np.float64)
    bmax = np.asarray(bmax, dtype=np.float64)
    u = (p - bmin) / (bmax - bmin) * resf - 0.5
    inside = np.all((p >= bmin) & (p <= bmax), axis=-1)
    u = np.clip(u, 0.0, resf - 1.0)
    i0 = np.clip(np.floor(u).astype(int), 0, res - 1)
    fr = u - i0
    sig = np.zeros(p.shape[0])
    rgb = np.zeros((p.shape[0], 3))
    for corner in range(8):
        bits = ((corner >> 2) & 1, (corner >> 1) & 1, corner & 1)
        ix = [np.minimum(i0[:, a] + bits[a], res[a] - 1) for a in range(3)]
        wgt = np.ones(p.shape[0])
        for a in range(3):
            wgt = wgt * (fr[:, a] if bits[a] else 1.0 - fr[:, a])
        sig += wgt * dens[ix[0], ix[1], ix[2]]
        rgb += wgt[:, None] * col[ix[0], ix[1], ix[2]]
    sig[~inside] = 0.0
    rgb[~inside] = 0.0
    return rgb, sig


def radiance(prim, p):
    """(rgb, sigma) at local points: procedural colour clip((p+1)/2) with the
    SDF-derived density, or the voxel lookup (fields.py:249-259, 468-469,
    502-504)."""
    if prim[0] == "voxel":
        return voxel_sample(prim, p)
    dist = sdf(prim, p)
    sig = INTERIOR_STEEPNESS * np.maximum(0.0, -dist)
    sig = np.where(np.abs(dist) < SURFACE_BAND, np.maximum(sig, SIGMA_SURFACE), sig)
    return np.clip((p + 1.0) / 2.0, 0.0, 1.0), sig


def volume_color(prim, o, d, t_n, t_f, n_samples):
    """Emission-absorption quadrature at interval midpoints
    (fields.py:364-370, 406-420)."""
    n = o.shape[0]
    delta = (t_f - t_n) / n_samples
    ts = t_n[:, None] + (np.arange(n_samples)[None, :] + 0.5) * delta[:, None]
    pts = o[:, None, :] + ts[:, :, None] * d[:, None, :]
    rgb, sig = radiance(prim, pts.reshape(-1, 3))
    sig = sig.reshape(n, n_samples)
    rgb = rgb.reshape(n, n_samples, 3)
    tau = sig * delta[:, None]
    trans = np.exp(-np.concatenate([np.zeros((n, 1)), np.cumsum(tau[:, :-1], axis=1)], axis=1))
    w = trans * (1.0 - np.exp(-tau))
    return (w[:, :, None] * rgb).sum(axis=1), w.sum(axis=1)


# ---------------------------------------------------------------------------
# frame composition  (pipeline.py:116-468)
# ---------------------------------------------------------------------------

@dataclass
class Obj:
    """Scene instance (pipeline.py:139-152): user id, placement
    v_world = s R v_local + T, depth backend (NeDF model or analytic prim),
    radiance field (prim spec)."""
    id: int
    R: np.ndarray
    T: np.ndarray
    s: float
    radiance: tuple
    model: OracleModel | None = None      # None -> analytic sphere-trace backend
    depth_prim: tuple | None = None       # analytic backend geometry (default: radiance)


@dataclass
class Light:
    kind: str                 # "point" | "directional"
    vec: np.ndarray           # position or unit travel direction
    beta: float = 0.4


@dataclass
class Config:
    sigma_threshold: float | None = None
    resample: bool = False
    resample_samples: int = 128
    shadow_epsilon: float | None = None
    shadows: bool = True
    clear_color: tuple = (0.0, 0.0, 0.0)


def _query_world(obj: Obj, o, d):
    """Depth backend query_world (pipeline.py:116-136)."""
    if obj.model is not None:
        return world_depth(obj.model, obj.R, obj.T, obj.s, o, d)
    prim = obj.depth_prim if obj.depth_prim is not None else obj.radiance
    lo = ((o - obj.T) @ obj.R) / obj.s
    ld = d @ obj.R
    t, hit = sphere_trace(prim, lo, ld)
    return obj.s * t, hit


def object_plane(obj: Obj, o, d, threads=1):
    """Alpha-folded depth (+inf on miss / non-finite / non-positive), chunked
    like _query_instance_chunked (pipeline.py:235-256)."""
    n = o.shape[0]
    plane = np.full(n, np.inf)
    sl = [slice(a, min(a + QUERY_CHUNK, n)) for a in range(0, n, QUERY_CHUNK)]

    def fill(s):
        dep, al = _query_world(obj, o[s], d[s])
        ok = al & np.isfinite(dep) & (dep > 0)
        chunk = np.full(s.stop - s.start, np.inf)
        chunk[ok] = dep[ok]
        plane[s] = chunk

    if threads > 1 and len(sl) > 1:
        with ThreadPoolExecutor(max_workers=threads) as ex:
            list(ex.map(fill, sl))
    else:
        for s in sl:
            fill(s)
    return plane


def default_eps(scene):
    """max(1e-4, 2 s * fine_width) over NeDF objects (pipeline.py:202-208)."""
    e = 1e-4
    for ob in scene:
        if ob.model is not None:
            e = max(e, 2.0 * ob.s * ob.model.fine_width)
    return e


def _bbox_for_resample(obj):
    return prim_bounds(obj.radiance)


@dataclass
class FrameOut:
    depth: np.ndarray
    id: np.ndarray
    rgb: np.ndarray
    shadow: np.ndarray
    image: np.ndarray
    planes: dict = field(default_factory=dict)
    evals_step1: int = 0
    evals_step3: int = 0
    resampled: int = 0


def render(scene, cam: Cam, lights, cfg: Config | None = None, pixels=None, threads=1):
    """compose_frame restated (pipeline.py:430-468): STEP 1 z-buffer over
    objects in scene order with strict < (ties to the earliest object,
    pipeline.py:259-268), STEP 2 single-sample shading (315-352), STEP 3 one
    shadow ray per covered pixel per light (371-403), image = rgb * shadow.
    With `pixels`, only those flat pixel indices are rendered (1-D outputs)."""
    cfg = cfg or Config()
    o, d = primary_rays(cam, pixels)
    n = o.shape[0]
    depth = np.full(n, np.inf)
    ids = np.full(n, -1, dtype=np.int32)
    out = FrameOut(depth, ids, np.zeros((n, 3)), np.ones(n), None)
    for ob in scene:
        plane = object_plane(ob, o, d, threads)
        out.planes[ob.id] = plane
        if ob.model is not None:
            lo = ((o - ob.T) @ ob.R) / ob.s
            out.evals_step1 += int(slab_clip(lo, d @ ob.R, ob.model.box_min, ob.model.box_max)[2].sum())
    for ob in scene:
        plane = out.planes[ob.id]
        closer = plane < depth
        depth[closer] = plane[closer]
        ids[closer] = ob.id
    # STEP 2
    rgb = out.rgb
    rgb[ids < 0] = np.asarray(cfg.clear_color, dtype=np.float64)
    for ob in scene:
        mask = ids == ob.id
        if not mask.any():
            continue
        x = o[mask] + depth[mask, None] * d[mask]
        lp = ((x - ob.T) @ ob.R) / ob.s
        ld = d[mask] @ ob.R
        color, sig = radiance(ob.radiance, lp)
        thr = cfg.sigma_threshold
        if thr is None:
            thr = 1.0 if ob.radiance[0] == "voxel" else SIGMA_SURFACE / 2.0
        outl = sig < thr
        if cfg.resample and outl.any():
            lo_ = ((o[mask][outl] - ob.T) @ ob.R) / ob.s
            ldo = ld[outl]
            bmin, bmax = _bbox_for_resample(ob)
            t0, t1, cr = slab_clip(lo_, ldo, bmin, bmax)
            if cr.any():
                vc, _ = volume_color(ob.radiance, lo_[cr], ldo[cr], t0[cr], t1[cr],
                                     cfg.resample_samples)
                sub = np.flatnonzero(outl)[cr]
                color[sub] = vc
            out.resampled += int(outl.sum())
        rgb[mask] = color
    # STEP 3
    shadow = out.shadow
    if cfg.shadows:
        eps = cfg.shadow_epsilon if cfg.shadow_epsilon is not None else default_eps(scene)
        for L in lights:
            valid = (ids >= 0) & np.isfinite(depth)
            if not valid.any():
                continue
            x = o[valid] + depth[valid, None] * d[valid]
            if L.kind == "point":
                to_x = x - np.asarray(L.vec)[None, :]
                dist = np.linalg.norm(to_x, axis=1)
                rd = to_x / np.maximum(dist, 1e-300)[:, None]
                ro = np.broadcast_to(np.asarray(L.vec, dtype=np.float64), x.shape).copy()
                ds = np.full(x.shape[0], np.inf)
                for ob in scene:
                    ds = np.minimum(ds, object_plane(ob, ro, rd, threads))
                    if ob.model is not None:
                        lo = ((ro - ob.T) @ ob.R) / ob.s
                        out.evals_step3 += int(slab_clip(lo, rd @ ob.R, ob.model.box_min,
                                                         ob.model.box_max)[2].sum())
                shadowed = ds + eps < dist
            elif L.kind == "directional":
                rd = np.broadcast_to(-np.asarray(L.vec, dtype=np.float64), x.shape).copy()
                ro = x + eps * rd
                ds = np.full(x.shape[0], np.inf)
                for ob in scene:
                    dep, al = _query_world(ob, ro, rd)
                    ok = al & np.isfinite(dep) & (dep >= 0)
                    ds = np.minimum(ds, np.where(ok, dep, np.inf))
                shadowed = np.isfinite(ds)
            else:
                raise TypeError(L.kind)
            shadow[valid] *= np.where(shadowed, L.beta, 1.0)
    out.image = rgb * shadow[:, None]
    if pixels is None:
        h, w = cam.height, cam.width
        out.depth = depth.reshape(h, w)
        out.id = ids.reshape(h, w)
        out.rgb = rgb.reshape(h, w, 3)
        out.shadow = shadow.reshape(h, w)
        out.image = out.image.reshape(h, w, 3)
        out.planes = {k: v.reshape(h, w) for k, v in out.planes.items()}
    return out


def host_threads():
    """Threads used by the timed CPU baseline (OPENBLAS + chunk threads)."""
    return max(1, os.cpu_count() or 1)


def rotation_y(angle):
    c, s = math.cos(angle), math.sin(angle)
    return np.array([[c, 0.0, s], [0.0, 1.0, 0.0], [-s, 0.0, c]])


def quat_to_matrix(q):
    """Unit quaternion [w, x, y, z] -> rotation (scene.py:51-57)."""
    w, x, y, z = q
    return np.array([
        [1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
        [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
        [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)],
    ])


# ---------------------------------------------------------------------------
# output formats (imgio.py)
# ---------------------------------------------------------------------------

def to_u8(rgb):
    """imgio.py:23-24."""
    return (np.clip(np.asarray(rgb, dtype=np.float64), 0.0, 1.0) * 255.0 + 0.5).astype(np.uint8)


def depth_to_gray(depth):
    """imgio.py:88-97: nearest surface bright, farthest dark, misses black."""
    depth = np.asarray(depth, dtype=np.float64)
    finite = np.isfinite(depth)
    out = np.zeros(depth.shape, dtype=np.uint8)
    if finite.any():
        lo, hi = depth[finite].min(), depth[finite].max()
        span = hi - lo if hi > lo else 1.0
        out[finite] = np.round((hi - depth[finite]) / span * 255.0).astype(np.uint8)
    return out


def id_to_u16(ids):
    """imgio.py:106-111 (the values the 16-bit PNG stores)."""
    return (np.asarray(ids).astype(np.int32) + 1).clip(0, 65535).astype(np.uint16)


def depth_raw_bytes(depth, scale=1.0):
    """imgio.py:63-71: NDPT header + little-endian f32 plane."""
    import struct
    depth = np.asarray(depth)
    h, w = depth.shape
    return b"NDPT" + struct.pack("<IIf", w, h, scale) + depth.astype("<f4").tobytes(order="C")


# ---------------------------------------------------------------------------
# distillation (model.py:74-81, 189-248; nn.py:115-232) -- float64
# ---------------------------------------------------------------------------

def segment_batch(mu, half_range, n_coarse=64, n_fine=128):
    """model.py:74-81."""
    l = half_range
    u = (np.clip(mu, -l, l) + l) / (2.0 * l)
    scaled = u * n_coarse
    coarse = np.minimum(scaled.astype(int), n_coarse - 1)
    fine = np.minimum(((scaled - coarse) * n_fine).astype(int), n_fine - 1)
    return coarse, fine


def flat_params(model: "OracleModel"):
    return [a for w, b in model.weights for a in (w, b)]


def forward_cached(model: "OracleModel", feats):
    """nn.py:115-135 with the activation cache."""
    W = model.weights
    x = feats @ W[0][0].T + W[0][1]
    cache = []
    nb = (len(W) - 3) // 2
    for i in range(nb):
        (w1, b1), (w2, b2) = W[1 + 2 * i], W[2 + 2 * i]
        a1 = x @ w1.T + b1
        h1 = np.maximum(a1, 0.0)
        a2 = h1 @ w2.T + b2
        cache.append((x, a1, h1, a2))
        x = x + np.maximum(a2, 0.0)
    la = x @ W[-2][0].T + W[-2][1]
    lf = x @ W[-1][0].T + W[-1][1]
    return la[:, :-1], lf, la[:, -1:], (feats, cache, x)


def _sigmoid(z):
    out = np.empty_like(z)
    pos = z >= 0
    out[pos] = 1.0 / (1.0 + np.exp(-z[pos]))
    ez = np.exp(z[~pos])
    out[~pos] = ez / (1.0 + ez)
    return out


def bce_loss(logits, targets, row_mask=None):
    """nn.py:178-196."""
    per = np.maximum(logits, 0.0) - logits * targets + np.log1p(np.exp(-np.abs(logits)))
    grad = _sigmoid(logits) - targets
    if row_mask is not None:
        per = per * row_mask[:, None]
        grad = grad * row_mask[:, None]
        count = int(row_mask.sum()) * logits.shape[1]
    else:
        count = logits.size
    if count == 0:
        return 0.0, np.zeros_like(logits)
    return float(per.sum() / count), grad / count


def backward(model: "OracleModel", cache, g_c, g_f, g_a):
    """nn.py:138-167; gradients parallel to flat_params."""
    feats, blocks, feat = cache
    W = model.weights
    gA = np.concatenate([g_c, g_a], axis=1)
    out_tail_a = (gA.T @ feat, gA.sum(axis=0))
    out_tail_b = (g_f.T @ feat, g_f.sum(axis=0))
    g_x = gA @ W[-2][0] + g_f @ W[-1][0]
    nb = len(blocks)
    per_block = []
    for i in reversed(range(nb)):
        x, a1, h1, a2 = blocks[i]
        (w1, _), (w2, _) = W[1 + 2 * i], W[2 + 2 * i]
        g_a2 = np.where(a2 > 0, g_x, 0.0)
        g_fc2 = (g_a2.T @ h1, g_a2.sum(axis=0))
        g_h1 = g_a2 @ w2
        g_a1 = np.where(a1 > 0, g_h1, 0.0)
        g_fc1 = (g_a1.T @ x, g_a1.sum(axis=0))
        per_block.append((g_fc1, g_fc2))
        g_x = g_x + g_a1 @ w1
    out = [g_x.T @ feats, g_x.sum(axis=0)]
    for g_fc1, g_fc2 in reversed(per_block):
        out.extend((g_fc1[0], g_fc1[1], g_fc2[0], g_fc2[1]))
    out.extend((out_tail_a[0], out_tail_a[1], out_tail_b[0], out_tail_b[1]))
    return out


def loss_and_grads(model: "OracleModel", feats, coarse, fine, hit, n_coarse=64, n_fine=128):
    """model.py:238-248 with bin indices (coarse / fine valid where hit) as targets."""
    lc, lf, la, cache = forward_cached(model, feats)
    n = feats.shape[0]
    tc = np.zeros((n, n_coarse))
    tf = np.zeros((n, n_fine))
    rows = np.flatnonzero(hit)
    tc[rows, coarse[rows]] = 1.0
    tf[rows, fine[rows]] = 1.0
    mask = hit.astype(np.float64)
    loss_c, g_c = bce_loss(lc, tc, row_mask=mask)
    loss_f, g_f = bce_loss(lf, tf, row_mask=mask)
    loss_a, g_a = bce_loss(la, hit.astype(np.float64)[:, None])
    total = loss_c + loss_f + 0.1 * loss_a
    return total, (loss_c, loss_f, loss_a), backward(model, cache, g_c, g_f, 0.1 * g_a)


def adam_step(params, grads, m, v, t, lr=5e-4, b1=0.9, b2=0.999, eps=1e-8):
    """nn.py:218-232 (t = the step count after incrementing)."""
    bc1 = 1.0 - b1 ** t
    bc2 = 1.0 - b2 ** t
    for p, g, mm, vv in zip(params, grads, m, v):
        mm *= b1
        mm += (1.0 - b1) * g
        vv *= b2
        vv += (1.0 - b2) * g * g
        p -= lr * (mm / bc1) / (np.sqrt(vv / bc2) + eps)
