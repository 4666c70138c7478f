# Where compose_frame's end-to-end time goes on top of the device frame time.
import sys, time, cProfile, pstats
sys.path.insert(0, '.')
import torch
from paper_2308_04669_b200 import configs as CF, pipeline, scenes
scene, cam, lights, cfg = scenes.build(CF.config4())
buf = pipeline.FrameBuffers(cam.width, cam.height)
rnd = pipeline.FrameRenderer(scene, cam, lights, cfg, buffers=buf)
for _ in range(3):
    pipeline.compose_frame(scene, cam, lights, cfg, buffers=buf); rnd.render()
torch.cuda.synchronize()
n = 20
t0 = time.perf_counter()
for _ in range(n):
    rnd.render()
torch.cuda.synchronize()
print("FrameRenderer.render wall ms/frame", (time.perf_counter() - t0) * 1e3 / n)
t0 = time.perf_counter()
for _ in range(n):
    pipeline.compose_frame(scene, cam, lights, cfg, buffers=buf)
torch.cuda.synchronize()
print("compose_frame wall ms/frame", (time.perf_counter() - t0) * 1e3 / n)
t0 = time.perf_counter()
for _ in range(n):
    pipeline._SceneTables(scene, buf.device)
print("_SceneTables ms", (time.perf_counter() - t0) * 1e3 / n)
pr = cProfile.Profile()
pr.enable()
for _ in range(n):
    pipeline.compose_frame(scene, cam, lights, cfg, buffers=buf)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(12)
