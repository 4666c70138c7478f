// Shared device-side types and float64 ray geometry for the NeDF frame path.
//
// Ray setup is float64 end to end, as in the reference (geometry.py, pipeline.py),
// so sample points agree with the numpy path to ~1 ulp; only the network runs
// in reduced precision.  This file must be compiled WITHOUT fast-math: the slab
// clip relies on IEEE inf/NaN (geometry.py:258-273).
#pragma once

#include <cuda_runtime.h>
#include <cuda_fp16.h>
#include <stdint.h>

#include "../../include/nedf_b200.h"

namespace nedf {

constexpr int kPoints = 16;          // geometry.py:21
constexpr int kLevels = 10;          // geometry.py:22
constexpr int kPerPoint = 63;        // 3 * (1 + 2 * 10)
constexpr int kDin = 1008;           // 16 * 63
constexpr int kMaxObjs = 65535;      // scene index packs into 16 bits of the z-key
constexpr unsigned long long kEmptyKey = 0xFFFFFFFFFFFFFFFFull;  // (bits(+inf) << 32) | 0xFFFFFFFF is above any hit

// ---------------------------------------------------------------------------
// device descriptors (built by the host in capi.cu)
// ---------------------------------------------------------------------------
struct DevModel {
  int d_in, d_feat, n_blocks, n_coarse, n_fine;
  int tensor_ok;                 // packed fp16 weights valid for the tcgen05 kernel
  double l;                      // half range
  double bmin[3], bmax[3];       // relaxed sampling box
  double c[3], h[3];             // box centre and half extents (h==0 -> 1)
  double alpha_threshold;
  float alpha_zthr;              // logit where sigmoid(z) > alpha_threshold flips (+-inf: never flips)
  int pad_;
  const float* wT;               // fp32 [in][out] per layer (head padded to 1024 rows)
  const float* bias;             // fp32 per layer, concatenated
  const __half* wpack;           // tcgen05 operand image (see mlp_tc.cu)
  const __half* wpack_lo;        // its low halves 4096 (w - fp16(w)) for mlp_precise.cu
  const float* bias_pack;        // tcgen05 bias image (fp32, padded to 256 per layer)
  const float* wstream;          // fp32 stream image for mlp_fp32s.cu (paper-shaped models)
  const float* wcluster;         // fp32 cluster-split images for mlp_fp32c.cu (paper-shaped models):
  const float* wcluster8;        //   4-CTA and 8-CTA clusters
  const void* wguard;            // tcgen05 guard image (guard_tc.cu, paper-shaped models)
  int64_t wT_off[40];            // layer offsets into wT  (n_layers <= 35 for the paper profile; general cap 40)
  int64_t b_off[40];
  int n_layers;
};

struct DevObj {
  double R[9];                   // row-major, v_world = s R v_local + T
  double T[3];
  double s;
  int id;
  int depth_kind;                // NEDF_DEPTH_*
  int group;                     // model group for NeDF objects
  int depth_field;
  int radiance_field;
  int pad;
  double rbox_min[3], rbox_max[3];   // appearance bounding box (SceneInstance.sampling_box)
  double sigma_default;             // default_sigma_threshold (pipeline.py:196-199)
  int recompute;                    // STEP 1 with a plane cache: 1 = evaluate this object's plane
  int pad2;
  float bs_c[3], bs_r;              // NeDF objects: world-space bounding sphere of the relaxed box (fp32 pre-test)
  // NeDF objects, fp32 copies for the setup kernels' certified fp32 slab clip (clip_hit_f32)
  float Rf[9], Tf[3], inv_sf;       // R, T, 1/s
  float bminf[3], bmaxf[3];         // the model's relaxed box
  float smu_f;                      // s * mu_max (rounded up): depth >= |(o - T).d| - smu_f (front-first culling)
  int pad3;
};

// Conservative fp32 rejection before the float64 slab clip: true only when the
// ray (o + t d, t >= 0) certainly misses the sphere (centre c, radius r)
// -- the margin covers fp32 rounding of coordinates up to ~1e4 with room to spare,
// so the exact clip still decides every pair that could hit.
// (c, r1 = 1.001 r) as staged by the setup kernel; o, d already rounded to fp32.
// Division-free: for t >= 0 the line misses iff (|w|^2 - r^2) |d|^2 > (w.d)^2.
__device__ __forceinline__ bool sphere_miss_f(float4 cr, float ox, float oy, float oz, float dx, float dy, float dz) {
  const float wx = cr.x - ox, wy = cr.y - oy, wz = cr.z - oz;
  const float w2 = wx * wx + wy * wy + wz * wz;
  const float tca = wx * dx + wy * dy + wz * dz;
  const float r = cr.w + 1e-3f * (1.0f + sqrtf(w2));
  const float e = w2 - r * r;
  if (e <= 0.f) return false;                // origin inside (or near) the sphere: no decision
  if (tca < 0.f) return true;                // sphere behind the origin
  const float dd = dx * dx + dy * dy + dz * dz;
  return e * dd > tca * tca;                 // the line passes outside
}
__device__ __forceinline__ bool sphere_miss(const DevObj& ob, const double o[3], const double d[3]) {
  return sphere_miss_f(make_float4(ob.bs_c[0], ob.bs_c[1], ob.bs_c[2], ob.bs_r * 1.001f), (float)o[0], (float)o[1],
                       (float)o[2], (float)d[0], (float)d[1], (float)d[2]);
}

struct DevCam {
  double pos[3];
  double rot[9];                 // camera-to-world, row-major
  double tan_half, aspect;
  int width, height;
};

enum RayMode : int {
  RAY_PRIMARY = 0,               // camera ray of pixel
  RAY_POINT_SHADOW = 1,          // from the point light toward the pixel's surface point
  RAY_DIR_SHADOW = 2,            // from surface point + eps toward a directional light
  RAY_WORLD = 3,                 // explicit world rays + object placement (query_world)
  RAY_LOCAL = 4                  // explicit local rays (query_rays)
};

struct RayJob {
  int mode;
  DevCam cam;
  const int* rows;               // local row -> camera row (device)
  const double* depth64;         // step-1 depth per local pixel (shadow modes)
  double light[3];               // point light position / directional travel direction
  double eps;
  const double* ex_o;            // explicit rays [n][3]
  const double* ex_d;
  const DevObj* objs;            // device array (scene order)
};

// output of one network evaluation
enum OutMode : int {
  OUT_ZBUF = 0,                  // atomicMin packed (depth f32, scene index, coarse, fine) key per local pixel
  OUT_QUERY_WORLD = 1,           // depth f64 + alpha per explicit ray
  OUT_QUERY_LOCAL = 2,           // mu f64 + alpha per explicit ray
  OUT_LOGITS = 3                 // raw logits per row (nn.forward)
};

struct OutSpec {
  int mode;
  unsigned long long* key;
  double* depth;
  double* mu;
  uint8_t* alpha;
  float* lc;
  float* lf;
  float* la;
  double* planes;                // optional per-object planes (OUT_ZBUF, primary rays)
  int64_t plane_stride;
  const float* feats;            // OUT_LOGITS input features [n][d_in]
};

// per-group work lists (group = one model)
struct ListSet {
  uint32_t* pix;                 // local pixel / ray index
  uint32_t* obj;                 // scene index
  int* count;                    // [n_groups]
  const int64_t* offset;         // [n_groups] start of each group's region
  int n_groups;
};

// guarded-ray list for fp32 re-evaluation
struct RedoList {
  uint32_t* pix;
  uint32_t* obj;
  int* count;                    // per group
  const int64_t* offset;
};

struct GroupTable {
  const DevModel* models;        // [n_groups] (device)
  int n_groups;
};

// ---------------------------------------------------------------------------
// float64 geometry (pipeline.py:97-109, model.py:310-311, geometry.py:258-342)
// ---------------------------------------------------------------------------
__device__ __forceinline__ void cam_ray(const DevCam& c, int row, int col, double o[3], double d[3]) {
  // xs = (i + 0.5) / w * 2 - 1 ; ys = 1 - (j + 0.5) / h * 2 ; gx = xs*tan*aspect ; gy = ys*tan
  double xs = ((col + 0.5) / c.width) * 2.0 - 1.0;
  double ys = 1.0 - ((row + 0.5) / c.height) * 2.0;
  double gx = xs * c.tan_half * c.aspect;
  double gy = ys * c.tan_half;
  double v[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) v[i] = gx * c.rot[3 * i + 0] + gy * c.rot[3 * i + 1] + (-1.0) * c.rot[3 * i + 2];
  double n = sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]);
#pragma unroll
  for (int i = 0; i < 3; ++i) { d[i] = v[i] / n; o[i] = c.pos[i]; }
}

__device__ __forceinline__ void to_local(const DevObj& ob, const double o[3], const double d[3],
                                         double lo[3], double ld[3]) {
  double q[3] = {o[0] - ob.T[0], o[1] - ob.T[1], o[2] - ob.T[2]};
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    lo[j] = (q[0] * ob.R[j] + q[1] * ob.R[3 + j] + q[2] * ob.R[6 + j]) / ob.s;
    ld[j] = d[0] * ob.R[j] + d[1] * ob.R[3 + j] + d[2] * ob.R[6 + j];
  }
}

// slab clip with the reference's NaN handling (NaN bounds widen the slab)
__device__ __forceinline__ bool slab_clip(const double o[3], const double d[3], const double bmin[3],
                                          const double bmax[3], double& t0, double& t1) {
  double lo_max = -INFINITY, hi_min = INFINITY;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    double inv = 1.0 / d[a];
    double ta = (bmin[a] - o[a]) * inv;
    double tb = (bmax[a] - o[a]) * inv;
    double lo, hi;
    if (isnan(ta) || isnan(tb)) { lo = -INFINITY; hi = INFINITY; }
    else { lo = ta < tb ? ta : tb; hi = ta < tb ? tb : ta; }
    lo_max = lo > lo_max ? lo : lo_max;
    hi_min = hi < hi_min ? hi : hi_min;
  }
  t0 = lo_max > 0.0 ? lo_max : 0.0;
  t1 = hi_min;
  return t1 >= t0;
}

// linspace(0, 1, 16)[i] exactly as numpy builds it: i * (1/15), last = 1
__device__ __forceinline__ double lin16(int i) { return i == kPoints - 1 ? 1.0 : i * (1.0 / 15.0); }

// sample point i, normalised to the box frame (geometry.py:336-340)
__device__ __forceinline__ void sample_point(const DevModel& m, const double lo[3], const double ld[3],
                                             double t0, double t1, int i, double p[3]) {
  double t = t0 + (t1 - t0) * lin16(i);
#pragma unroll
  for (int a = 0; a < 3; ++a) p[a] = ((lo[a] + t * ld[a]) - m.c[a]) / m.h[a];
}

// Shadow ray of a receiver x = co + D cd (camera ray, STEP-1 depth) for the job's light.
__device__ __forceinline__ void shadow_ray(const RayJob& job, const double co[3], const double cd[3], double D,
                                           double o[3], double d[3]) {
  double x[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) x[a] = co[a] + D * cd[a];
  if (job.mode == RAY_POINT_SHADOW) {
    // pipeline.py:385-388: dir = (x - L) / max(|x - L|, 1e-300), origin = L
    double v[3] = {x[0] - job.light[0], x[1] - job.light[1], x[2] - job.light[2]};
    double dist = sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]);
    double dn = dist > 1e-300 ? dist : 1e-300;
#pragma unroll
    for (int a = 0; a < 3; ++a) { o[a] = job.light[a]; d[a] = v[a] / dn; }
  } else {
    // pipeline.py:395-396: dir = -light_dir, origin = x + eps * dir
#pragma unroll
    for (int a = 0; a < 3; ++a) { d[a] = -job.light[a]; o[a] = x[a] + job.eps * d[a]; }
  }
}

// World ray of a work item for the given mode.
__device__ __forceinline__ void item_world_ray(const RayJob& job, uint32_t pix, double o[3], double d[3]) {
  if (job.mode == RAY_WORLD || job.mode == RAY_LOCAL) {
#pragma unroll
    for (int a = 0; a < 3; ++a) { o[a] = job.ex_o[3 * (size_t)pix + a]; d[a] = job.ex_d[3 * (size_t)pix + a]; }
    return;
  }
  int w = job.cam.width;
  int row = job.rows[pix / w];
  int col = pix % w;
  double co[3], cd[3];
  cam_ray(job.cam, row, col, co, cd);
  if (job.mode == RAY_PRIMARY) {
#pragma unroll
    for (int a = 0; a < 3; ++a) { o[a] = co[a]; d[a] = cd[a]; }
    return;
  }
  shadow_ray(job, co, cd, job.depth64[pix], o, d);
}

// Local-space ray of an item against its object (model.py:310-311).
__device__ __forceinline__ void item_local_ray(const RayJob& job, uint32_t pix, uint32_t sidx,
                                               double wo[3], double wd[3], double lo[3], double ld[3]) {
  item_world_ray(job, pix, wo, wd);
  if (job.mode == RAY_LOCAL) {
#pragma unroll
    for (int a = 0; a < 3; ++a) { lo[a] = wo[a]; ld[a] = wd[a]; }
    return;
  }
  to_local(job.objs[sidx], wo, wd, lo, ld);
}

// unsegment (model.py:89-92): lower edge of the fine cell
__device__ __forceinline__ double decode_mu(const DevModel& m, int c, int f) {
  return (2.0 * m.l) * ((double)c / m.n_coarse) + (2.0 * m.l / m.n_coarse) * ((double)f / m.n_fine) - m.l;
}

// stabilised sigmoid (nn.py:169-175) compared against the threshold
__device__ __forceinline__ bool alpha_of(double z, double thr) {
  double s;
  if (z >= 0) s = 1.0 / (1.0 + exp(-z));
  else { double e = exp(z); s = e / (1.0 + e); }
  return s > thr;
}

// |(o - T) . d| (geometry.py:203-205 applied as in model.py:313)
__device__ __forceinline__ double tangency_dist(const double o[3], const double T[3], const double d[3]) {
  return fabs((o[0] - T[0]) * d[0] + (o[1] - T[1]) * d[1] + (o[2] - T[2]) * d[2]);
}

__device__ __forceinline__ unsigned long long pack_key(double depth, uint32_t sidx, int c, int f) {
  float df = (float)depth;
  unsigned int bits = __float_as_uint(df);
  return ((unsigned long long)bits << 32) | ((unsigned long long)(sidx & 0xFFFF) << 16) |
         ((unsigned long long)(c & 0xFF) << 8) | (unsigned long long)(f & 0xFF);
}

// STEP 3 (pipeline.py:381-403): is a shadow pair's contribution certain when the
// exact network's bins are only known to lie in [cmin, cmax] x [fmin, fmax]
// (every bin whose fast logit is within the guard margin of the fast maximum)
// and alpha may be either value when alpha_amb?  The pair shadows iff alpha and
// 0 < ds (finite) and, for a point light, ds + eps < |x - light|; ds = |(o - T).d|
// - s mu is monotone in mu and mu in (c, f), so the box's two corners bound every
// candidate.  1 / 0: shadows / does not for every candidate; -1: undecided.
__device__ __forceinline__ int shadow_pair_certain(const DevModel& m, const RayJob& job, uint32_t pix,
                                                   uint32_t sidx, int cmin, int cmax, int fmin, int fmax,
                                                   bool alpha_fast, bool alpha_amb) {
  if (!alpha_fast && !alpha_amb) return 0;
  double wo[3], wd[3], lo[3], ld[3];
  item_local_ray(job, pix, sidx, wo, wd, lo, ld);
  const DevObj& ob = job.objs[sidx];
  const double tang = tangency_dist(wo, ob.T, wd);
  const double ds_lo = tang - ob.s * decode_mu(m, cmax, fmax);
  const double ds_hi = tang - ob.s * decode_mu(m, cmin, fmin);
  if (!isfinite(ds_lo) || !isfinite(ds_hi)) return -1;
  bool all_true, all_false;
  if (job.mode == RAY_POINT_SHADOW) {
    // |x - light| as the shadow resolve computes it
    const int w = job.cam.width;
    double co[3], cd[3], v[3];
    cam_ray(job.cam, job.rows[pix / w], pix % w, co, cd);
    const double D = job.depth64[pix];
#pragma unroll
    for (int a = 0; a < 3; ++a) v[a] = (co[a] + D * cd[a]) - job.light[a];
    const double dist = sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]);
    all_true = ds_lo > 0.0 && ds_hi + job.eps < dist;
    all_false = ds_hi <= 0.0 || !(ds_lo + job.eps < dist);
  } else {
    all_true = ds_lo > 0.0;
    all_false = ds_hi <= 0.0;
  }
  if (alpha_amb || !alpha_fast) return all_false ? 0 : -1;
  return all_true ? 1 : (all_false ? 0 : -1);
}

// Final per-ray bookkeeping shared by the fp32 and tensor-core kernels:
// decode bins -> mu -> world depth -> demotion -> output (model.py:288-318,
// pipeline.py:244-248).
__device__ __forceinline__ void finish_ray(const DevModel& m, const RayJob& job, const OutSpec& out,
                                           uint32_t pix, uint32_t sidx, int c, int f, double zlogit,
                                           const double wo[3], const double wd[3]) {
  bool alpha = alpha_of(zlogit, m.alpha_threshold);
  double mu = decode_mu(m, c, f);
  if (out.mode == OUT_QUERY_LOCAL) {
    out.mu[pix] = mu;
    out.alpha[pix] = alpha ? 1 : 0;
    return;
  }
  const DevObj& ob = job.objs[sidx];
  double depth = tangency_dist(wo, ob.T, wd) - ob.s * mu;
  alpha = alpha && (depth > 0.0);
  if (out.mode == OUT_QUERY_WORLD) {
    out.depth[pix] = depth;
    out.alpha[pix] = alpha ? 1 : 0;
    return;
  }
  bool ok = alpha && isfinite(depth) && depth > 0.0;
  if (out.planes != nullptr) out.planes[(size_t)sidx * out.plane_stride + pix] = ok ? depth : INFINITY;
  if (ok) atomicMin(out.key + pix, pack_key(depth, sidx, c, f));
}

}  // namespace nedf
