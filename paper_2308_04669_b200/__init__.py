"""B200-native NeDF per-frame render path (arXiv 2308.04669).

Drop-in for the reference package's hot path (`nedf.pipeline.compose_frame`
and its steps, the `query_world` depth-backend seam, `query_rays`,
`nn.forward`, `.nedm` loading).  All computation runs in the sm_100a CUDA
library `libnedf_b200.so` through its C ABI (include/nedf_b200.h); importing
the compute entry points fails loudly if the library is not built.
"""

__version__ = "0.1.0"

_LAZY = {
    "compose_frame": "pipeline", "nedf_generation_step": "pipeline", "deferred_shading_step": "pipeline",
    "shadow_step": "pipeline", "step_timing_report": "pipeline", "Camera": "pipeline", "look_at": "pipeline",
    "FrameBuffers": "pipeline", "RenderConfig": "pipeline", "RenderResult": "pipeline",
    "SceneInstance": "pipeline", "PointLight": "pipeline", "DirectionalLight": "pipeline",
    "NedfDepthBackend": "pipeline", "OracleDepthBackend": "pipeline", "FrameRenderer": "pipeline",
    "generate_primary_rays": "pipeline", "import_external_gbuffer": "pipeline", "reuse_buffers": "pipeline",
    "NedfModel": "model", "load_nedf": "model", "loads_nedf": "model", "save_nedf": "model",
    "new_model": "model", "query_rays": "model", "query_depth_world_batch": "model",
    "RigidTransform": "geometry", "Aabb": "geometry",
    "FormatError": "errors", "SceneValidationError": "errors",
}


def __getattr__(name):
    mod = _LAZY.get(name)
    if mod is None:
        raise AttributeError(name)
    import importlib
    return getattr(importlib.import_module(f"{__name__}.{mod}"), name)
