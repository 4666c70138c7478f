/*
 * nedf_b200.h -- C ABI of the B200-native NeDF per-frame render path.
 *
 * Drop-in boundary for the reference package's hot path
 * (/root/reference/pkg/src/nedf, cited as file:line):
 *
 *   frame level   compose_frame / nedf_generation_step / deferred_shading_step /
 *                 shadow_step                              pipeline.py:271-468
 *   backend level NedfDepthBackend.query_world            pipeline.py:116-123
 *                 -> query_depth_world_batch               model.py:301-319
 *   model level   query_rays (local rays -> mu, alpha)     model.py:277-293
 *                 nn.forward (features -> logits)          nn.py:115-135
 *   weights       load_nedf / nn.load_model (.nedm bytes)  model.py:364-369, nn.py:249-281
 *
 * Conventions
 *  - Plain C types only.  Pointers named *_dev are CUDA device pointers owned
 *    by the caller; the library never frees them.  Host pointers are read
 *    synchronously during the call.
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *    All work is enqueued on it; no call synchronises the device unless its
 *    comment says so.
 *  - Return value 0 = success, negative = error; nedf_last_error() returns a
 *    thread-local message.  Codes map to the reference's exceptions:
 *    NEDF_ERR_INVALID -> ValueError, NEDF_ERR_FORMAT -> FormatError
 *    (errors.py:4-6), NEDF_ERR_UNSUPPORTED -> TypeError / NotImplementedError,
 *    NEDF_ERR_CUDA -> RuntimeError.
 *  - Geometry is float64 on the way in (as in the reference); depth buffers are
 *    float64, colour buffers float32.
 *  - There is no CPU fallback: every entry point that computes runs CUDA
 *    kernels compiled for sm_100a.
 */
#ifndef NEDF_B200_H
#define NEDF_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NEDF_ABI_VERSION 1

enum {
  NEDF_OK = 0,
  NEDF_ERR_INVALID = -1,
  NEDF_ERR_FORMAT = -2,
  NEDF_ERR_CUDA = -3,
  NEDF_ERR_UNSUPPORTED = -4,
  NEDF_ERR_NOMEM = -5
};

/* Arithmetic used for the intersection network. */
enum {
  NEDF_PREC_AUTO = 0,   /* tcgen05 fp16 x fp16 -> fp32 chain + near-tie guard, fp32 re-evaluation of guarded rays */
  NEDF_PREC_TENSOR = 1, /* tcgen05 chain only, no guard (benchmark / diagnostics) */
  NEDF_PREC_FP32 = 2    /* fp32 CUDA-core chain for every ray */
};

/* Context options (nedf_set_option). */
enum {
  NEDF_OPT_PRECISION = 1,       /* one of NEDF_PREC_* */
  NEDF_OPT_GUARD_PPM = 2,       /* near-tie guard threshold tau, parts per million of max|logit| */
  NEDF_OPT_TC_CTAS = 3,         /* persistent CTAs for the tensor-core kernel (0 = one per SM) */
  NEDF_OPT_PROFILE = 4,         /* 1 = time every network launch with CUDA events (read back by nedf_read_stats) */
  NEDF_OPT_TC_KERNEL = 5,       /* one of NEDF_TC_*: which tensor-core network kernel runs */
  NEDF_OPT_GUARD_CLUSTER = 6,   /* near-tie guard kernel's cluster size: 4, 8, or 0 = by frame size */
  NEDF_OPT_SETUP_EXACT = 7,     /* 1 = every work-list box test in float64 (default 0: certified fp32 test,
                                   float64 only where its error bound cannot decide; same lists either way) */
  NEDF_OPT_FUSE = 8,            /* 1 (default) = nedf_render_frame fuses the per-pixel passes (STEP 1 resolve,
                                   STEP 2, shadow fill, first light's STEP 3 setup; last light's resolve +
                                   composite); 0 = one kernel per step, as the step entry points run */
  NEDF_OPT_GUARD_KERNEL = 9,    /* one of NEDF_GUARD_*: which kernel re-evaluates the near-tie rays */
  NEDF_OPT_CULL = 10,           /* 1 (default) = STEP 1 front-first culling: a pixel's pair with the nearest
                                   depth bound is evaluated first, the others only if their bound
                                   |(o - T).d| - s mu_max can still beat its result (same z-buffer, fewer
                                   evaluations); off with a plane cache.  0 = every box hit evaluated */
  NEDF_OPT_SHADOW_CERT = 11     /* 1 (default) = STEP 3: a near-tie shadow ray whose pair decision (shadows or
                                   not) is the same for every bin within the guard margin of the fast maxima
                                   and either alpha is finished by the fast kernel; 0 = all go to the guard */
};
/* Near-tie guard kernels (NEDF_OPT_GUARD_KERNEL); all fp32-accurate. */
enum {
  NEDF_GUARD_AUTO = 0,      /* by batch size (decided on the device): TCGEN05 when it fits one round, else PRECISE */
  NEDF_GUARD_TCGEN05 = 1,   /* latency form: tcgen05 tf32 + fp16 split products, 16 rays per 4-CTA cluster (guard_tc.cu) */
  NEDF_GUARD_MMA_SYNC = 2,  /* warp-level mma.sync 3xTF32, 4- or 8-CTA clusters (mlp_fp32c.cu) */
  NEDF_GUARD_PRECISE = 3    /* throughput form: 3-product fp16 split, 128-ray tiles, one CTA per SM (mlp_precise.cu) */
};

/* Tensor-core network kernels (NEDF_OPT_TC_KERNEL). */
enum {
  NEDF_TC_AUTO = 0,    /* the fastest measured one (currently NEDF_TC_MCAST2) */
  NEDF_TC_SINGLE = 1,  /* one CTA per 128-ray tile, M = 128, own weight stream */
  /* 2 is retired: the cta_group::2 variant (round 1) measured slower and was removed */
  NEDF_TC_MCAST2 = 3,  /* clusters of 2 CTAs (M = 128 each) sharing one multicast weight stream */
  NEDF_TC_MCAST4 = 4   /* clusters of 4 CTAs sharing one multicast weight stream */
};

typedef struct NedfContext NedfContext; /* one per device: streams' scratch, counters */
typedef struct NedfModel NedfModel;     /* one per .nedm: packed device weights */

/* Model dimensions and decode constants (nn.py:59-72, model.py:38-65, 102-117). */
typedef struct {
  int32_t d_in, d_feat, n_blocks, n_coarse, n_fine;
  float half_range;       /* l */
  float box_min[3], box_max[3];  /* relaxed sampling box */
  float alpha_threshold;
} NedfModelInfo;

/* Analytic / voxel field node (fields.py:64-186, 270-319).  A field is a tree
 * flattened into an array; children of a UNION are contiguous. */
enum {
  NEDF_FIELD_SPHERE = 1,      /* p: c[3], r */
  NEDF_FIELD_BOX = 2,         /* p: c[3], h[3] */
  NEDF_FIELD_TORUS = 3,       /* p: c[3], major_r, minor_r */
  NEDF_FIELD_PLANE = 4,       /* p: n[3], offset */
  NEDF_FIELD_UNION = 5,       /* child = first, count */
  NEDF_FIELD_TRANSFORMED = 6, /* child; p: R[9] row-major, T[3], s */
  NEDF_FIELD_VOXEL = 7        /* res[3]; p: bmin[3], bmax[3]; density[nx*ny*nz], color[nx*ny*nz*3] (C order, f32, device) */
};

typedef struct {
  int32_t kind;
  int32_t child;
  int32_t count;
  int32_t res[3];
  double p[16];
  const float* density_dev;
  const float* color_dev;
} NedfField;

/* Depth backend of a scene instance (pipeline.py:116-136). */
enum {
  NEDF_DEPTH_NEDF = 0,      /* NedfDepthBackend: the intersection network */
  NEDF_DEPTH_ANALYTIC = 1   /* OracleDepthBackend over an analytic field: sphere tracing */
};

/* Scene instance (pipeline.py:139-152): v_world = s * R v_local + T. */
typedef struct {
  double R[9];              /* row-major */
  double T[3];
  double s;
  int32_t id;               /* user id written to the id buffer */
  int32_t depth_kind;       /* NEDF_DEPTH_* */
  const NedfModel* model;   /* NEDF_DEPTH_NEDF */
  int32_t depth_field;      /* NEDF_DEPTH_ANALYTIC: root node index */
  int32_t radiance_field;   /* root node index of the appearance field (Step 2) */
} NedfObject;

/* Pinhole camera (pipeline.py:53-77); orientation is camera-to-world, row-major. */
typedef struct {
  double position[3];
  double orientation[9];
  double fov_y;
  int32_t width, height;
} NedfCamera;

enum { NEDF_LIGHT_POINT = 0, NEDF_LIGHT_DIRECTIONAL = 1 };

typedef struct {
  int32_t kind;
  double vec[3];            /* position, or unit travel direction */
  double beta;
} NedfLight;

/* RenderConfig (pipeline.py:180-193); negative = "None" (per-field / scene default). */
typedef struct {
  double sigma_threshold;
  int32_t resample;
  int32_t resample_samples;
  double shadow_epsilon;
  int32_t shadows;
  double clear_color[3];
} NedfRenderConfig;

/* Frame buffers (pipeline.py:211-232), device pointers, row-major over the
 * rendered rows.  `rows_host` selects which camera rows are rendered (image
 * tiles for multi-GPU); NULL = all rows.  Buffers hold n_rows * width pixels. */
typedef struct {
  double* depth_dev;        /* +inf = miss */
  int32_t* id_dev;          /* -1 = none */
  float* rgb_dev;           /* [n][3] */
  float* shadow_dev;        /* [n] */
  float* image_dev;         /* [n][3], may be NULL (composite skipped) */
  double* planes_dev;       /* optional per-object alpha-folded depth planes [n_objs][n] (reuse cache), or NULL */
  const int32_t* rows_host;
  int32_t n_rows;
} NedfFrameBuffers;

typedef struct {
  int64_t evals;            /* network evaluations (box hits) */
  int64_t guarded;          /* rays re-evaluated in fp32 by the near-tie guard */
  int64_t covered;          /* pixels with id >= 0 (Step 2) */
  int64_t resampled;        /* outlier pixels (Step 2) */
  int64_t launches;         /* kernels this library launched since the last read */
  int64_t net_launches;     /* network-kernel launches timed (NEDF_OPT_PROFILE) */
  double net_ms;            /* summed device time of the main network kernel (tensor-core or fp32) */
  double guard_ms;          /* summed device time of the fp32 re-evaluation of guarded rays */
  int64_t h2d_bytes;        /* host->device bytes this library copied (per-call scene tables) */
  int64_t exact_clips;      /* (ray, object) box tests the certified fp32 test left to float64 */
  int64_t culled;           /* STEP 1 box hits skipped by front-first culling (NEDF_OPT_CULL) */
} NedfStepStats;

/* ---- library / context ---------------------------------------------------- */
int nedf_abi_version(void);
const char* nedf_last_error(void);
int nedf_context_create(int device, NedfContext** out);
void nedf_context_destroy(NedfContext* ctx);
int nedf_set_option(NedfContext* ctx, int key, int64_t value);
int nedf_get_option(NedfContext* ctx, int key, int64_t* value);
/* Device-side counters of the last step (evals, guarded, ...); synchronises `stream`. */
int nedf_read_stats(NedfContext* ctx, NedfStepStats* out, void* stream);
/* Non-blocking counterpart of nedf_read_stats: enqueue a copy of this step's device
 * counters into mapped slot `slot` (0..63) and reset them; out receives the host-side
 * counters (launches, h2d_bytes) now.  After the stream reaches this point (event or
 * synchronize), nedf_stats_slot fills evals / guarded / covered / resampled from the slot. */
int nedf_stats_snapshot(NedfContext* ctx, int slot, NedfStepStats* out, void* stream);
int nedf_stats_slot(NedfContext* ctx, int slot, NedfStepStats* out);

/* ---- weights (model.py:354-369, nn.py:235-281) ------------------------------ */
/* Parse a .nedm image (header, f32 parameters, 7-f32 trailer) and upload the
 * packed weights.  NEDF_ERR_FORMAT on bad magic / version / size. */
int nedf_model_load(NedfContext* ctx, const void* nedm_bytes, size_t n_bytes, NedfModel** out);
/* Same from a flat f32 parameter array in file order. */
int nedf_model_create(NedfContext* ctx, const NedfModelInfo* info, const float* params_host,
                      size_t n_params, NedfModel** out);
void nedf_model_free(NedfModel* m);
int nedf_model_info(const NedfModel* m, NedfModelInfo* out);
/* 1 if the tcgen05 kernel supports this model's shape (else fp32 path is used). */
int nedf_model_tensor_ok(const NedfModel* m);

/* ---- model level ---------------------------------------------------------- */
/* nn.forward on caller-provided features [B][d_in] f32 -> logits (nn.py:115-135). */
int nedf_mlp_forward(NedfContext* ctx, const NedfModel* m, const float* feats_dev, int64_t batch,
                     float* coarse_dev, float* fine_dev, float* alpha_logit_dev, int precision,
                     void* stream);
/* query_rays: local-space rays -> (mu, alpha); box misses give mu=NaN, alpha=0
 * (model.py:277-293). */
int nedf_query_rays(NedfContext* ctx, const NedfModel* m, const double* origins_dev,
                    const double* dirs_dev, int64_t n, double* mu_dev, uint8_t* alpha_dev,
                    void* stream);

/* ---- backend level -------------------------------------------------------- */
/* NedfDepthBackend.query_world -> query_depth_world_batch (model.py:301-319):
 * world rays + placement -> (depth, alpha), non-positive depths demoted. */
int nedf_query_world(NedfContext* ctx, const NedfModel* m, const double R[9], const double T[3],
                     double s, const double* origins_dev, const double* dirs_dev, int64_t n,
                     double* depth_dev, uint8_t* alpha_dev, void* stream);

/* ---- frame level (pipeline.py:271-468) ------------------------------------- */
/* STEP 1: depth + id z-buffer over all objects (strict <, earliest scene index wins). */
int nedf_generation_step(NedfContext* ctx, const NedfCamera* cam, const NedfObject* objs, int n_objs,
                         const NedfField* fields, int n_fields, NedfFrameBuffers* fb, void* stream);
/* STEP 1 with the per-object plane cache (reuse_buffers, pipeline.py:281-305):
 * re-evaluate only the objects at scene indices changed_idx[0..n_changed), keep
 * the other planes in fb->planes_dev (required), then recombine all planes in
 * scene order with strict < -- bit-identical to a cold STEP 1 with planes. */
int nedf_reuse_step(NedfContext* ctx, const NedfCamera* cam, const NedfObject* objs, int n_objs,
                    const NedfField* fields, int n_fields, const int32_t* changed_idx, int n_changed,
                    NedfFrameBuffers* fb, void* stream);
/* STEP 2: deferred shading of covered pixels (clear colour elsewhere). */
int nedf_shading_step(NedfContext* ctx, const NedfCamera* cam, const NedfObject* objs, int n_objs,
                      const NedfField* fields, int n_fields, const NedfRenderConfig* cfg,
                      NedfFrameBuffers* fb, void* stream);
/* STEP 3 for one light: multiply the shadow buffer by beta where occluded. */
int nedf_shadow_step(NedfContext* ctx, const NedfCamera* cam, const NedfObject* objs, int n_objs,
                     const NedfField* fields, int n_fields, const NedfLight* light,
                     const NedfRenderConfig* cfg, NedfFrameBuffers* fb, void* stream);
/* image = rgb * shadow; also resets nothing. */
int nedf_composite(NedfContext* ctx, NedfFrameBuffers* fb, int width, void* stream);
/* The whole frame: STEP 1, STEP 2, shadow buffer := 1, STEP 3 per light, composite
 * (compose_frame, pipeline.py:430-468). */
int nedf_render_frame(NedfContext* ctx, const NedfCamera* cam, const NedfObject* objs, int n_objs,
                      const NedfField* fields, int n_fields, const NedfLight* lights, int n_lights,
                      const NedfRenderConfig* cfg, NedfFrameBuffers* fb, void* stream);

/* nedf_render_frame that also records events[0..3] (cudaEvent_t, may be NULL) on the
 * stream at frame start, end of STEP 1's network, end of STEP 2 and frame end, for
 * compose_frame's per-step timing.  With NEDF_OPT_FUSE the STEP 1 resolve and the first
 * light's STEP 3 ray setup run inside the STEP 2 interval. */
int nedf_render_frame_timed(NedfContext* ctx, const NedfCamera* cam, const NedfObject* objs, int n_objs,
                            const NedfField* fields, int n_fields, const NedfLight* lights, int n_lights,
                            const NedfRenderConfig* cfg, NedfFrameBuffers* fb, void* const* events, void* stream);
/* ---- output formats (imgio.py): per-pixel conversions on the GPU, so
 * only 8/16-bit planes or the f32 depth plane are copied to the host for encoding ---- */
/* (clip(x, 0, 1) * 255 + 0.5) -> uint8, truncating like numpy astype (imgio.py:23-24);
 * n = element count (3 per pixel for RGB). */
int nedf_to_u8(const float* src_dev, int64_t n, uint8_t* dst_dev, void* stream);
/* float64 depth -> float32 NDPT plane, misses stay +inf (imgio.py:63-71). */
int nedf_depth_to_f32(const double* depth_dev, int64_t n, float* dst_dev, void* stream);
/* depth_to_gray (imgio.py:88-97): nearest finite surface 255, farthest 0, misses 0;
 * round half to even like np.round.  scratch_dev: 16 bytes of device memory. */
int nedf_depth_to_gray(const double* depth_dev, int64_t n, uint8_t* dst_dev, uint64_t* scratch_dev, void* stream);
/* id plane -> 16-bit grayscale (id + 1, clipped to [0, 65535]; imgio.py:106-111). */
int nedf_id_to_u16(const int32_t* id_dev, int64_t n, uint16_t* dst_dev, void* stream);

/* ---- GPU distillation (model.py:238-274, nn.py:115-232) ----
 * A trainer owns fp32 parameters (the .nedm order: head W, b; per block fc1 W, b,
 * fc2 W, b; tail_a W, b; tail_b W, b), Adam moments and the activation cache for
 * batches of up to max_batch rays.  Errors: nedf_trainer_last_error(). */
typedef struct NedfTrainer NedfTrainer;
const char* nedf_trainer_last_error(void);
int nedf_trainer_create(int device, const NedfModelInfo* info, const float* params_host, int64_t n_params,
                        int max_batch, NedfTrainer** out);
void nedf_trainer_destroy(NedfTrainer* t);
int nedf_trainer_set_lr(NedfTrainer* t, float lr);
/* Training batch from host rays in the model frame (build_training_batch, model.py:189-235):
 * slab clip + encoding, sphere tracing of the analytic oracle field `root`, mu and bin
 * targets, all on the GPU; hit_host[n] receives the box-hit mask (misses are redrawn
 * by the caller, as the reference does). */
int nedf_trainer_batch(NedfTrainer* t, const NedfField* fields, int n_fields, int root, double t_max,
                       const double* origins_host, const double* dirs_host, int n, uint8_t* hit_host, void* stream);
/* Explicit batch: features [n][1008], coarse / fine bin targets (-1 = no hit), alpha targets. */
int nedf_trainer_set_batch(NedfTrainer* t, const float* feats_host, const int32_t* coarse_host,
                           const int32_t* fine_host, const float* alpha_host, int n, void* stream);
/* Forward, BCE losses, exact backward into the gradient buffer (loss_and_grads,
 * model.py:238-248); losses_host[4] = total, coarse, fine, alpha. */
int nedf_trainer_loss_and_grads(NedfTrainer* t, double* losses_host, void* stream);
/* Adam with bias correction (nn.py:218-232). */
int nedf_trainer_adam_step(NedfTrainer* t, void* stream);
/* Copy the parameters (what = 0) or the last gradients (what = 1) to the host. */
int nedf_trainer_read(NedfTrainer* t, int what, float* host, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* NEDF_B200_H */
