#!/usr/bin/env python3
"""The other SURVEY.md §8d workloads on one GPU, one JSON line each:

  config1  128x128, one object, STEP 1 only
  config2  800x800, one object, STEP 1 + STEP 2 (no lights), resample off and on
  config3  2000x800, four objects, no lights
  config4  2000x800, eight objects, point-light shadows (the bench.py headline)
  config5  60-frame dynamic run of config 4 (objects spin, the light orbits):
           per-frame transforms and light pushed through FrameRenderer, and the
           same through the public compose_frame (host scene marshalling included)
  sweep    MLP-only query_rays throughput at B in {64K, 256K, 1M, 4M, 16M}
           sweep rays (RaySampler-style, seed 0), device-resident inputs

Frame times are CUDA-event times with inputs resident on the GPU and L2 flushed
before each timed frame; NeDF evaluations per frame are reported beside them.

    python scripts/bench_configs.py [--only config1,sweep] [--out profiles/r1_configs.jsonl]
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_2308_04669_b200 import _lib, configs as CF, geometry, model, pipeline, scenes  # noqa: E402

FLOP_PER_EVAL = 4_809_216
PEAK = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["bf16_tflops"] if (ROOT / "MEASURED_PEAKS.json").exists() else 2250.0


def _flush_buf():
    return torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")


def time_frames(rnd, n, flush, per_frame=None):
    ctx = _lib.context()
    st = _lib.stream_handle()
    for _ in range(3):
        rnd.render()
    torch.cuda.synchronize()
    ctx.read_stats(st)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
    for i, (a, b) in enumerate(evs):
        if per_frame is not None:
            per_frame(i)
        flush.zero_()
        a.record()
        rnd.render()
        b.record()
    torch.cuda.synchronize()
    stats = ctx.read_stats(st)
    ms = [a.elapsed_time(b) for a, b in evs]
    return ms, stats


def frame_line(name, spec, lights_on, flush, steps=10, resample=False):
    scene, cam, lights, cfg = scenes.build(spec)
    if resample:
        cfg.resample = True
    if not lights_on:
        lights = []
    rnd = pipeline.FrameRenderer(scene, cam, lights, cfg)
    ms, st = time_frames(rnd, steps, flush)
    evals = st["evals"] / steps
    t = float(np.mean(ms))
    return {"workload": name, "width": cam.width, "height": cam.height, "objects": len(scene),
            "lights": len(lights), "resample": bool(resample), "ms_per_frame": t, "ms_min": float(np.min(ms)),
            "nedf_evals_per_frame": evals, "nedf_rays_per_s": evals / (t * 1e-3),
            "tflops": evals * FLOP_PER_EVAL / (t * 1e-3) / 1e12,
            "network_ms_per_frame": st["net_ms"] / steps, "guard_ms_per_frame": st["guard_ms"] / steps,
            "guarded_per_frame": st["guarded"] / steps}


def config1(flush):
    """STEP 1 only (nedf_generation_step) at 128x128."""
    scene, cam, lights, cfg = scenes.build(CF.config1())
    buf = pipeline.FrameBuffers(cam.width, cam.height)
    ctx = _lib.context()
    st = _lib.stream_handle()
    for _ in range(3):
        pipeline.nedf_generation_step(scene, cam, buf)
    torch.cuda.synchronize()
    ctx.read_stats(st)
    n = 20
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
    for a, b in evs:
        flush.zero_()
        a.record()
        pipeline.nedf_generation_step(scene, cam, buf)
        b.record()
    torch.cuda.synchronize()
    s = ctx.read_stats(st)
    t = float(np.mean([a.elapsed_time(b) for a, b in evs]))
    ev = s["evals"] / n
    return {"workload": "config1 (STEP 1 only, nedf_generation_step incl. host marshalling)", "width": cam.width,
            "height": cam.height, "objects": 1, "ms_per_frame": t, "nedf_evals_per_frame": ev,
            "nedf_rays_per_s": ev / (t * 1e-3)}


def config5(flush, n_frames=60):
    """Dynamic 60-frame run.  (a) FrameRenderer with per-frame transforms /
    light (device-resident scene, the serving loop); (b) compose_frame with a
    fresh scene list per frame (the reference's API, host marshalling included)."""
    specs = [CF.config5_frame(f, n_frames) for f in range(n_frames)]
    built = [scenes.build(s) for s in specs]
    scene0, cam, lights0, cfg = built[0]
    rnd = pipeline.FrameRenderer(scene0, cam, lights0, cfg)

    def per_frame(i):
        sc, _, li, _ = built[i]
        rnd.update_transforms([o.transform for o in sc])
        rnd.update_lights(li)

    ms, st = time_frames(rnd, n_frames, flush, per_frame)
    evals = st["evals"] / n_frames
    t = float(np.mean(ms))
    # (b) public API, wall clock per frame incl. host work, result synchronised
    buf = pipeline.FrameBuffers(cam.width, cam.height)
    for i in range(2):
        sc, _, li, cf = built[i]
        pipeline.compose_frame(sc, cam, li, cf, buffers=buf)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(n_frames):
        sc, _, li, cf = built[i]
        pipeline.compose_frame(sc, cam, li, cf, buffers=buf)
    torch.cuda.synchronize()
    api_ms = (time.perf_counter() - t0) * 1e3 / n_frames
    return {"workload": "config5 dynamic (60 frames, objects spin, light orbits)", "frames": n_frames,
            "width": cam.width, "height": cam.height, "objects": len(scene0),
            "ms_per_frame": t, "ms_max": float(np.max(ms)), "ms_total": float(np.sum(ms)),
            "nedf_evals_per_frame": evals, "nedf_rays_per_s": evals / (t * 1e-3),
            "tflops": evals * FLOP_PER_EVAL / (t * 1e-3) / 1e12,
            "compose_frame_wall_ms_per_frame": api_ms}


def trained(flush, steps=5):
    """The config-4 placements with the GPU-distilled models (scenes/config4_trained.json,
    2000x800, point light): trained networks populate many fine bins, so the near-tie
    guard carries a large share of the evaluations."""
    from paper_2308_04669_b200 import scene as S
    desc = S.load_scene(ROOT / "scenes" / "config4_trained.json")
    inst = desc.instantiate()
    cam = desc.camera()
    rnd = pipeline.FrameRenderer(inst, cam, desc.build_lights(), desc.render_config())
    _lib.context().set_option(_lib.OPT_PROFILE, 1)
    ms, st = time_frames(rnd, steps, flush)
    _lib.context().set_option(_lib.OPT_PROFILE, 0)
    evals = st["evals"] / steps
    t = float(np.mean(ms))
    return {"workload": "config4 placements, GPU-distilled models (scenes/config4_trained.json)",
            "width": cam.width, "height": cam.height, "objects": len(inst), "ms_per_frame": t,
            "nedf_evals_per_frame": evals, "guarded_per_frame": st["guarded"] / steps,
            "network_ms_per_frame": st["net_ms"] / steps, "guard_ms_per_frame": st["guard_ms"] / steps}


def sweep(flush, sizes=(1 << 16, 1 << 18, 1 << 20, 1 << 22, 1 << 24)):
    m = scenes.paper_model(0, "sphere")
    out = []
    for n in sizes:
        o, d = CF.sweep_rays(n, m.relaxed_box.min, m.relaxed_box.max, seed=0)
        od = torch.from_numpy(o).cuda()
        dd = torch.from_numpy(d).cuda()
        model.query_rays(m, od, dd)
        torch.cuda.synchronize()
        reps = max(3, min(20, (1 << 22) // n))
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
        for a, b in evs:
            flush.zero_()
            a.record()
            model.query_rays(m, od, dd)
            b.record()
        torch.cuda.synchronize()
        t = float(np.mean([a.elapsed_time(b) for a, b in evs]))
        tf = n * FLOP_PER_EVAL / (t * 1e-3) / 1e12
        out.append({"workload": f"sweep query_rays B={n}", "rays": n, "ms": t, "rays_per_s": n / (t * 1e-3),
                    "tflops": tf, "frac_of_peak": tf / PEAK})
        del od, dd
    return out


def training(flush):
    """GPU distillation iterations/s (the reference's train loop, model.py:251-274) for the
    desk and paper profiles on the unit sphere; batch 1024 / 4096 like TrainProfile.  Steady
    state: one Trainer, 3 warm-up iterations, then 20 timed iterations of batch construction
    (host ray sampling + GPU encode / oracle trace / targets), loss + gradients and Adam; the
    one-off Trainer set-up and the final .nedm reload are excluded."""
    from paper_2308_04669_b200 import fields, train
    out = []
    for name, bs in (("desk", 1024), ("paper", 4096)):
        oracle = fields.AnalyticOracle(fields.Sphere(geometry.vec3(0, 0, 0), 1.0))
        m = model.new_model(oracle, np.random.default_rng(0), model.PROFILES[name])
        trainer = train.Trainer(m, max_batch=bs)
        sampler = train.RaySampler(box=m.relaxed_box, mode="direct")
        rng = np.random.default_rng(1)

        def step():
            train.build_training_batch(oracle, sampler, trainer, rng, bs)
            total, _ = trainer.loss_and_grads()
            trainer.adam_step()
            return total

        for _ in range(3):
            step()
        torch.cuda.synchronize()
        n = 20
        t0 = time.perf_counter()
        losses = [step() for _ in range(n)]
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / n
        out.append({"workload": f"train {name} profile (batch {bs}), steady state incl. host ray sampling",
                    "ms_per_iteration": dt * 1e3, "iterations_per_s": 1.0 / dt, "rays_per_s": bs / dt,
                    "final_loss": float(losses[-1])})
        del trainer
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="config1,config2,config3,config4,config5,trained,sweep,train")
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    which = set(args.only.split(","))
    flush = _flush_buf()
    lines = []

    class _Out(list):
        def append(self, ln):
            ln["gpu"] = torch.cuda.get_device_name(0)
            print(json.dumps(ln), flush=True)
            super().append(ln)

        def extend(self, lns):
            for ln in lns:
                self.append(ln)

    lines = _Out()
    if "config1" in which:
        lines.append(config1(flush))
    if "config2" in which:
        lines.append(frame_line("config2 (STEP 1 + STEP 2, no lights)", CF.config2(), False, flush))
        lines.append(frame_line("config2 resample (STEP 1 + STEP 2 rs, no lights)", CF.config2(), False, flush,
                                resample=True))
    if "config3" in which:
        lines.append(frame_line("config3 (4 objects, no lights)", CF.config3(), False, flush))
    if "config4" in which:
        lines.append(frame_line("config4 (8 objects, point-light shadows)", CF.config4(), True, flush))
    if "config5" in which:
        lines.append(config5(flush))
    if "sweep" in which:
        lines.extend(sweep(flush))
    if "trained" in which:
        lines.append(trained(flush))
    if "train" in which:
        lines.extend(training(flush))
    if args.out:
        Path(args.out).write_text("".join(json.dumps(x) + "\n" for x in lines))


if __name__ == "__main__":
    main()
