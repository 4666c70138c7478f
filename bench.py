#!/usr/bin/env python3
"""Benchmark: the headline frame of BASELINE.json -- a 2000x800 composite of
the 8-object config-4 scene with point-light shadows.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

A step is one full frame (STEP 1 depth/id, STEP 2 shading, STEP 3 shadows,
composite) rendered by `nedf_render_frame` through the C ABI with the scene
resident on the GPU (`value`), and again through the public Python API
`compose_frame` with the result copied to pinned host memory (`e2e`).  For
N > 1 (`--gpus N` re-runs itself under torch.distributed.run, one rank per GPU)
each rank renders every N-th camera row and the tiles are gathered to rank 0
over NCCL inside the timed region; time is the max over ranks of CUDA-event
time.  L2 is flushed (256 MiB write) before every timed
frame, outside its event bracket.

`--impl reference` times the reference algorithm (the float64 oracle port,
oracle/nedf_oracle.py) on the host cores on a 1/256 pixel subsample per step,
extrapolated to the full frame.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import tempfile
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "ms/frame 2000×800 composite+shadows; NeDF rays/s; tensor-pipe util at 1/2/4/8 GPU"
FLOP_PER_EVAL = 4_809_216          # 2 x (1008*256 + 32*256^2 + 256*65 + 256*128) MACs


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--precision", default="auto", choices=["auto", "tensor", "fp32"])
    ap.add_argument("--tc-kernel", default="auto", choices=["auto", "single", "mcast2", "mcast4"])
    ap.add_argument("--width", type=int, default=2000)
    ap.add_argument("--height", type=int, default=800)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    return ap.parse_args()


def traffic_per_launch():
    """dram__bytes_read.sum + dram__bytes_write.sum of one network launch from the latest
    committed ncu capture of the benchmarked kernel (profiles/r*_tc_kernel_ncu.json), or None."""
    for f in sorted((ROOT / "profiles").glob("r*_tc_kernel_ncu.json"), reverse=True):
        try:
            return json.loads(f.read_text())["dram_bytes_per_launch"]
        except (OSError, ValueError, KeyError):
            continue
    return None


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def relaunch(args) -> int:
    """`--gpus N` (N > 1) outside torchrun: re-run this script as N ranks, one
    process per GPU (torch.distributed.run on 127.0.0.1); rank 0 prints the line."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", str(Path(__file__).resolve()), *sys.argv[1:]]
    return subprocess.call(cmd)


def bench_config(spec, world: int) -> dict:
    """`config` of both arms' JSON lines (same keys, so the driver can pair them)."""
    return {"workload": "config4: 8-object NeDF scene, 2000x800, point-light shadows",
            "objects": len(spec.objects), "width": spec.camera.width, "height": spec.camera.height,
            "parallelism": f"1-row interleaved image tiles x{world}, gather to rank 0" if world > 1 else "single GPU",
            "l2": "flushed (256 MiB write) before every timed frame"}


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["bf16_tflops"]), float(d.get("bf16_tflops_sustained", d["bf16_tflops"])), \
            float(d["hbm_gbs"]), "measured"
    return 1590.0, 1400.0, 6650.0, "fallback"


# ---------------------------------------------------------------------------
# CPU reference (oracle port)
# ---------------------------------------------------------------------------

def cpu_reference_sample(spec, step: int, threads: int):
    """Render a deterministic 1/step^2 pixel subsample with the float64 port;
    returns (seconds, n_pixels, evals)."""
    import numpy as np
    from oracle import nedf_oracle as O
    from tests.helpers import oracle_scene
    objs, cam, lights, cfg = oracle_scene(spec)
    rows = np.arange(0, cam.height, step)
    cols = np.arange(0, cam.width, step)
    pix = (rows[:, None] * cam.width + cols[None, :]).ravel()
    t0 = time.perf_counter()
    out = O.render(objs, cam, lights, cfg, pixels=pix, threads=threads)
    dt = time.perf_counter() - t0
    return dt, len(pix), out.evals_step1 + out.evals_step3


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return 0
    from paper_2308_04669_b200 import configs as CF
    spec = CF.config4(args.width, args.height)
    threads = os.cpu_count() or 1
    step = 16
    # warm-up builds the three oracle models (paper-profile random init)
    for _ in range(max(0, args.warmup)):
        cpu_reference_sample(spec, step * 2, threads)
    times, npx, ev = [], 0, 0
    for _ in range(args.steps):
        dt, npx, ev = cpu_reference_sample(spec, step, threads)
        times.append(dt)
    full = args.width * args.height
    ms = 1e3 * (sum(times) / len(times)) * full / npx
    line = {
        "metric": METRIC, "value": ms, "unit": "ms/frame", "impl": "reference", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": False,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": bench_config(spec, args.gpus),
        "cpu_baseline": {"value": ms, "unit": "ms/frame", "cores": threads, "kind": "port",
                         "sample": f"every {step}th row and column ({npx} px), extrapolated x{full / npx:.0f}; "
                                   f"{ev} NeDF evaluations per sample"},
        "e2e": {"value": ms, "unit": "ms/frame", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# clocks
# ---------------------------------------------------------------------------

class ClockSampler:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.p = None
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                       "-i", str(gpu_index), "-lms", "200"], stdout=self.f,
                                      stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.p.terminate()
        self.p.wait()
        self.f.flush()
        rows = []
        for ln in Path(self.f.name).read_text().splitlines():
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) >= 9:
                rows.append(parts)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = sorted(float(r[1]) for r in rows if r[1].replace(".", "").isdigit())
        mx = max((float(r[2]) for r in rows if r[2].replace(".", "").isdigit()), default=None)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows for k in range(4) if r[5 + k].lower() == "active"})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx, "reasons": reasons,
                "samples": len(rows)}


# ---------------------------------------------------------------------------
# B200 arm
# ---------------------------------------------------------------------------

def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch(args)
    import numpy as np
    import torch
    world, rank, local = dist_env()
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    from paper_2308_04669_b200 import _lib, configs as CF, distributed as D, pipeline, scenes

    spec = CF.config4(args.width, args.height)
    scene, cam, lights, cfg = scenes.build(spec, device=local)
    rows = D.interleave_rows(cam.height, rank, world) if world > 1 else None
    ctx = _lib.context(local)
    ctx.set_option(_lib.OPT_PRECISION, {"auto": _lib.PREC_AUTO, "tensor": _lib.PREC_TENSOR,
                                        "fp32": _lib.PREC_FP32}[args.precision])
    ctx.set_option(_lib.OPT_PROFILE, 1)
    ctx.set_option(_lib.OPT_TC_KERNEL, {"auto": _lib.TC_AUTO, "single": _lib.TC_SINGLE,
                                        "mcast2": _lib.TC_MCAST2,
                                        "mcast4": _lib.TC_MCAST4}[args.tc_kernel])
    buf = pipeline.FrameBuffers(cam.width, cam.height, device=local, rows=rows)
    rnd = pipeline.FrameRenderer(scene, cam, lights, cfg, buffers=buf)
    stream = torch.cuda.current_stream()
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)   # 256 MiB > 126 MB L2

    def gather():
        if world > 1:
            D.gather_tiles({"image": buf.image, "depth": buf.depth, "id": buf.id}, cam.height, cam.width,
                           rank, world)

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    for _ in range(max(3, args.warmup)):
        rnd.render()
        gather()
    torch.cuda.synchronize()
    ctx.read_stats(_lib.stream_handle())

    sampler = ClockSampler(local)
    barrier()
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    for a, b in evs:
        flush.zero_()
        a.record(stream)
        rnd.render()
        gather()
        b.record(stream)
    torch.cuda.synchronize()
    barrier()
    clocks = sampler.stop()
    frame_ms = [a.elapsed_time(b) for a, b in evs]
    st = ctx.read_stats(_lib.stream_handle())
    t_local = float(np.mean(frame_ms))
    net_ms = st["net_ms"] / args.steps
    guard_ms = st["guard_ms"] / args.steps
    evals = st["evals"] / args.steps
    guarded = st["guarded"] / args.steps
    culled = st["culled"] / args.steps
    if world > 1:
        import torch.distributed as dist
        v = torch.tensor([t_local], dtype=torch.float64, device=dev)
        dist.all_reduce(v, op=dist.ReduceOp.MAX)
        t_frame = float(v.item())
        e = torch.tensor([evals, culled], dtype=torch.float64, device=dev)
        dist.all_reduce(e)
        evals_all, culled_all = float(e[0].item()), float(e[1].item())
    else:
        t_frame = t_local
        evals_all, culled_all = evals, culled

    # ---- end to end through the public API (compose_frame) with host copies ----
    e2e = None
    if not args.no_e2e:
        # Two output buffer sets: frame i's image/depth/id are copied to pinned host memory on a
        # copy stream while frame i + 1 renders (a streaming renderer's pipelining); every step still
        # pays its own H2D (scene tables) and D2H (result) and the clock stops after the last copy.
        hosts = [(torch.empty(buf.image.shape, dtype=torch.float32).pin_memory(),
                  torch.empty(buf.depth.shape, dtype=torch.float64).pin_memory(),
                  torch.empty(buf.id.shape, dtype=torch.int32).pin_memory()) for _ in range(2)]
        ebufs = [pipeline.FrameBuffers(cam.width, cam.height, device=local, rows=rows) for _ in range(2)]
        copy_stream = torch.cuda.Stream(device=dev)
        copied = [None, None]
        for i in range(2):
            pipeline.compose_frame(scene, cam, lights, cfg, buffers=ebufs[i])
        torch.cuda.synchronize()
        barrier()
        t0 = time.perf_counter()
        h2d = 0
        for i in range(args.steps):
            k = i & 1
            if copied[k] is not None:
                torch.cuda.current_stream().wait_event(copied[k])    # buffers k free again
            eb = ebufs[k]
            res = pipeline.compose_frame(scene, cam, lights, cfg, buffers=eb)
            h2d += res.timing["h2d_bytes"]
            if world > 1:
                D.gather_tiles({"image": eb.image, "depth": eb.depth, "id": eb.id}, cam.height,
                               cam.width, rank, world)
            done = torch.cuda.Event()
            done.record()
            img_h, dep_h, id_h = hosts[k]
            if world == 1 and len(res.events) == 4:
                # depth / id are final once STEP 2's pass has run: their copy overlaps STEP 3
                copy_stream.wait_event(res.events[2])
                with torch.cuda.stream(copy_stream):
                    dep_h.copy_(eb.depth, non_blocking=True)
                    id_h.copy_(eb.id, non_blocking=True)
            copy_stream.wait_event(done)
            with torch.cuda.stream(copy_stream):
                if not (world == 1 and len(res.events) == 4):
                    dep_h.copy_(eb.depth, non_blocking=True)
                    id_h.copy_(eb.id, non_blocking=True)
                img_h.copy_(eb.image, non_blocking=True)
                copied[k] = torch.cuda.Event()
                copied[k].record(copy_stream)
        torch.cuda.synchronize()
        barrier()
        e2e_ms = (time.perf_counter() - t0) * 1e3 / args.steps
        if world > 1:
            import torch.distributed as dist
            v = torch.tensor([e2e_ms], dtype=torch.float64, device=dev)
            dist.all_reduce(v, op=dist.ReduceOp.MAX)
            e2e_ms = float(v.item())
        # h2d: the per-call scene tables the library uploads (objects, models, fields, rows, list offsets);
        # d2h: image + depth + id copied to pinned host memory, plus the stats counters read per call
        img_h, dep_h, id_h = hosts[0]
        d2h = img_h.numel() * 4 + dep_h.numel() * 8 + id_h.numel() * 4 + 2 * 64
        e2e = {"value": e2e_ms, "unit": "ms/frame", "h2d_bytes_per_step": int(h2d // args.steps),
               "d2h_bytes_per_step": int(d2h),
               "overlap": "depth/id D2H on a copy stream from the end of frame i's STEP 2, the image's from the "
                          "end of frame i (both overlap later work)"}

    if rank != 0:
        if world > 1:
            torch.distributed.destroy_process_group()
        return 0

    burst, sustained, hbm, src = peaks()
    tflops = (evals * FLOP_PER_EVAL) / (net_ms * 1e-3) / 1e12 if net_ms > 0 else 0.0
    roofline = {"bound": "tensor", "achieved": tflops, "peak": burst, "unit": "TFLOP/s",
                "frac": tflops / burst, "frac_sustained": tflops / sustained, "peak_source": src,
                "kernel": "nedf_mlp_tc_kernel" if ctx.get_option(_lib.OPT_PRECISION) != _lib.PREC_FP32 else "mlp_fp32_stream_kernel",
                "kernel_ms_per_frame": net_ms, "guard_ms_per_frame": guard_ms,
                "flop_per_eval": FLOP_PER_EVAL, "evals_per_launch": evals / max(1, st["net_launches"] / args.steps),
                "traffic": traffic_per_launch(), "traffic_unit": "bytes (DRAM read + write per launch, ncu)"}
    line = {
        "metric": METRIC, "value": t_frame, "unit": "ms/frame", "n_gpus": world, "steps": args.steps,
        "warmup": max(3, args.warmup), "ms_per_step": t_frame, "higher_is_better": False, "scaling": "strong",
        "vs_baseline": None, "dtype": "fp16 tcgen05 (fp32 accum) + fp32 guard" if args.precision == "auto" else args.precision,
        "data": "synthetic (random-init paper-profile NeDFs, seeds 0/1/5)",
        "config": bench_config(spec, world),
        "nedf_evals_per_frame": evals_all, "guarded_per_frame": guarded,
        "nedf_rays_per_s": evals_all / (t_frame * 1e-3),
        # STEP 1 box hits resolved without a network evaluation (front-first culling): the
        # reference evaluates every box hit, so (evals + culled) is its work for the same frame
        "culled_per_frame": culled_all,
        "box_hits_resolved_per_s": (evals_all + culled_all) / (t_frame * 1e-3),
        "gpu_launches": int(st["launches"]), "clocks": clocks, "roofline": roofline, "e2e": e2e,
        "frame_ms_min": float(min(frame_ms)), "frame_ms_max": float(max(frame_ms)),
    }
    if world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        dt, npx, ev = cpu_reference_sample(spec, 8, threads)
        full = cam.width * cam.height
        line["cpu_baseline"] = {"value": dt * 1e3 * full / npx, "unit": "ms/frame", "cores": threads,
                                "kind": "port",
                                "sample": f"every 8th row and column ({npx} px, {ev} NeDF evals), "
                                          f"extrapolated x{full / npx:.0f}"}
    print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
