"""Output formats: the oracle against the reference's imgio
outputs (CPU), and the GPU conversions + host encoders against both (GPU)."""

import io

import numpy as np
import pytest

from oracle import nedf_oracle as O


def test_oracle_matches_reference_imgio(golden):
    z = golden("imgio.npz")
    np.testing.assert_array_equal(O.to_u8(z["rgb"]), z["u8"])
    np.testing.assert_array_equal(O.depth_to_gray(z["depth"]), z["gray"])
    np.testing.assert_array_equal(O.id_to_u16(z["ids"]), z["id_u16"])
    assert O.depth_raw_bytes(z["depth"], 2.5) == z["depth_raw"].tobytes()


@pytest.mark.gpu
def test_gpu_conversions_bit_exact(golden):
    from paper_2308_04669_b200 import imgio
    z = golden("imgio.npz")
    np.testing.assert_array_equal(imgio.to_u8(z["rgb"].astype(np.float32)), z["u8"])
    np.testing.assert_array_equal(imgio.depth_to_gray(z["depth"]), z["gray"])
    np.testing.assert_array_equal(imgio.id_to_u16(z["ids"]), z["id_u16"])
    assert imgio.depth_raw_bytes(z["depth"], 2.5) == z["depth_raw"].tobytes()


@pytest.mark.gpu
def test_gpu_conversions_random_and_edge_planes():
    import torch
    from paper_2308_04669_b200 import imgio
    rng = np.random.default_rng(5)
    rgb = rng.uniform(-1, 2, size=(333, 77, 3)).astype(np.float32)
    rgb[0, 0] = [np.nan, 0.0, 1.0]
    got = imgio.to_u8(torch.from_numpy(rgb).cuda())
    ref = O.to_u8(rgb)
    ok = ~np.isnan(rgb)
    np.testing.assert_array_equal(got[ok], ref[ok])
    for depth in (np.full((5, 7), np.inf), np.full((5, 7), 3.0), rng.uniform(-5, 5, size=(257, 31))):
        np.testing.assert_array_equal(imgio.depth_to_gray(depth), O.depth_to_gray(depth))
    ids = rng.integers(-5, 70000, size=(100, 9)).astype(np.int32)
    np.testing.assert_array_equal(imgio.id_to_u16(ids), O.id_to_u16(ids))


@pytest.mark.gpu
def test_frame_buffers_encode_and_decode(tmp_path):
    """A rendered frame through the reference's file formats and the stream header."""
    import struct
    from PIL import Image
    from paper_2308_04669_b200 import configs as CF, imgio, pipeline, scenes
    scene, cam, lights, cfg = scenes.build(CF.config4(96, 40))
    res = pipeline.compose_frame(scene, cam, lights, cfg)
    b = res.buffers
    png = imgio.encode_color_png(res.image)
    back = np.asarray(Image.open(io.BytesIO(png)).convert("RGB"))
    np.testing.assert_array_equal(back, O.to_u8(res.image.cpu().numpy()))
    imgio.write_ppm(tmp_path / "f.ppm", res.image)
    np.testing.assert_allclose(imgio.read_ppm(tmp_path / "f.ppm"), O.to_u8(res.image.cpu().numpy()) / 255.0)
    imgio.write_depth_raw(tmp_path / "d.ndpt", b.depth, 1.0)
    plane, scale = imgio.read_depth_raw(tmp_path / "d.ndpt")
    np.testing.assert_array_equal(plane, b.depth.cpu().numpy().astype(np.float32).astype(np.float64))
    assert scale == 1.0
    ids = np.asarray(Image.open(io.BytesIO(imgio.encode_id_png(b.id))))
    np.testing.assert_array_equal(ids, O.id_to_u16(b.id.cpu().numpy()))
    msg = imgio.frame_message(7, "depth", b.depth)
    rev, kind, enc, _, w, h = struct.unpack_from("<IBBHII", msg)
    assert (rev, kind, enc, w, h) == (7, 1, 0, cam.width, cam.height)
    gray = np.asarray(Image.open(io.BytesIO(msg[16:])))
    np.testing.assert_array_equal(gray, O.depth_to_gray(b.depth.cpu().numpy()))
    with pytest.raises(ValueError):
        imgio.encode_plane("normals", b.depth)
