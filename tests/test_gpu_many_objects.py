"""Scenes with more objects than the setup kernels stage (kSetupStage = 64): the
work-list builders then visit every object per pixel (no warp cone culling) and
STEP 1 front-first culling is off (its per-pixel hit mask is 64 bits).  The frame
must still match the reference restatement (pipeline.py:430-468) and be the same
under every arrangement of the per-pixel passes."""

import numpy as np
import pytest

from paper_2308_04669_b200 import configs as CF

pytestmark = pytest.mark.gpu


def _grid_spec(n_obj, width=96, height=72):
    rng = np.random.default_rng(7)
    objs = []
    cols = 10
    for k in range(n_obj):
        r, c = divmod(k, cols)
        T = np.array([-2.25 + 0.5 * c, 1.5 - 0.5 * r, 0.3 * ((k * 7) % 5)])
        kind = ("sphere", "box", "torus")[k % 3]
        objs.append(CF.ObjSpec(100 + k, kind, (0, 1, 5)[k % 3], CF.random_rotation(rng), T, 0.17))
    cam = CF.CameraSpec((0.0, 0.0, -7.0), (0.0, 0.0, 0.0), np.deg2rad(45.0), width, height)
    return CF.SceneSpec(f"grid{n_obj}", objs, cam, [CF.LightSpec("point", (1.0, 4.0, -5.0), 0.4)])


def _render(spec, fuse=1, cull=1):
    import torch
    from paper_2308_04669_b200 import _lib, pipeline, scenes
    scene, cam, lights, cfg = scenes.build(spec)
    ctx = _lib.context()
    ctx.set_option(_lib.OPT_FUSE, fuse)
    ctx.set_option(_lib.OPT_CULL, cull)
    try:
        buf = pipeline.FrameBuffers(cam.width, cam.height)
        ctx.read_stats(_lib.stream_handle())
        pipeline.FrameRenderer(scene, cam, lights, cfg, buffers=buf).render()
        torch.cuda.synchronize()
        st = ctx.read_stats(_lib.stream_handle())
    finally:
        ctx.set_option(_lib.OPT_FUSE, 1)
        ctx.set_option(_lib.OPT_CULL, 1)
    b = buf.numpy()
    b["image"] = buf.image.cpu().numpy()
    return b, st


@pytest.mark.parametrize("n_obj", [64, 70])
def test_many_objects_match_oracle_and_arrangements(n_obj):
    from oracle import nedf_oracle as O
    from tests.helpers import oracle_scene
    from tests.parity import frame_parity
    spec = _grid_spec(n_obj)
    ref_b, st = _render(spec)
    assert st["evals"] > 0
    if n_obj > 64:
        assert st["culled"] == 0              # front-first culling needs a 64-bit hit mask
    for fuse, cull in ((0, 1), (1, 0)):
        b, _ = _render(spec, fuse, cull)
        for k in ("depth", "id", "rgb", "shadow", "image"):
            np.testing.assert_array_equal(b[k], ref_b[k], err_msg=f"fuse={fuse} cull={cull} {k}")
    objs, ocam, olights, ocfg = oracle_scene(spec)
    ref = O.render(objs, ocam, olights, ocfg, threads=8)
    rep, bad = frame_parity(ref_b["depth"], ref_b["id"], ref_b["image"], ref.depth, ref.id, ref.image,
                            np.stack([ref.planes[o.id] for o in objs]), [o.id for o in objs])
    print(n_obj, rep)
    assert not bad, bad
    assert (ref_b["id"] >= 0).mean() > 0.1   # the grid covers a good share of the frame


def test_camera_inside_a_box_and_objects_behind():
    """The camera sits inside object 0's relaxed box (rays start inside it: clipped
    entry t0 = 0), object 1 is behind the camera (|(o - T).d| makes its depth formula
    positive), objects 2-3 overlap in front: culling bounds, the z-buffer and shadows
    must still match the reference restatement."""
    from oracle import nedf_oracle as O
    from tests.helpers import oracle_scene
    from tests.parity import frame_parity
    rng = np.random.default_rng(3)
    objs = [CF.ObjSpec(1, "sphere", 0, CF.random_rotation(rng), np.array([0.1, 0.0, -5.9]), 0.8),
            CF.ObjSpec(2, "box", 1, CF.random_rotation(rng), np.array([0.0, 0.2, -8.5]), 0.9),
            CF.ObjSpec(3, "torus", 5, CF.random_rotation(rng), np.array([0.3, -0.2, 0.0]), 1.0),
            CF.ObjSpec(4, "sphere", 1, CF.random_rotation(rng), np.array([-0.2, 0.1, 0.4]), 1.1)]
    cam = CF.CameraSpec((0.0, 0.0, -6.0), (0.0, 0.0, 0.0), np.deg2rad(50.0), 120, 90)
    spec = CF.SceneSpec("inside", objs, cam, [CF.LightSpec("point", (2.0, 3.0, -4.0), 0.4)])
    ref_b, st = _render(spec)
    b0, _ = _render(spec, 1, 0)
    for k in ("depth", "id", "image"):
        np.testing.assert_array_equal(b0[k], ref_b[k], err_msg=k)
    o_objs, ocam, olights, ocfg = oracle_scene(spec)
    ref = O.render(o_objs, ocam, olights, ocfg, threads=8)
    rep, bad = frame_parity(ref_b["depth"], ref_b["id"], ref_b["image"], ref.depth, ref.id, ref.image,
                            np.stack([ref.planes[o.id] for o in o_objs]), [o.id for o in o_objs])
    print(rep, st["culled"])
    assert not bad, bad
