// Per-pixel frame kernels around the network: work-list generation (box-hit
// compaction), z-buffer resolve, deferred shading, shadow resolve, composite.
//
// All are HBM/latency-bound; each touches a pixel's state once.  Work lists
// are grouped by model so a tensor-core tile never mixes weights.
#include "common.cuh"
#include "fields.cuh"
#include "frame.cuh"

namespace nedf {

// Append (pix, sidx) to a group list with one atomic per warp (all 32 lanes
// must call; `hit` selects the contributing lanes).
__device__ __forceinline__ void warp_append(const ListSet& ls, int group, bool hit, uint32_t pix, uint32_t sidx) {
  unsigned mask = __ballot_sync(0xffffffffu, hit);
  if (mask == 0u) return;
  int lane = threadIdx.x & 31;
  int leader = __ffs(mask) - 1;
  int base = 0;
  if (lane == leader) base = atomicAdd(ls.count + group, __popc(mask));
  base = __shfl_sync(0xffffffffu, base, leader);
  if (hit) {
    int rank = __popc(mask & ((1u << lane) - 1u));
    int64_t at = ls.offset[group] + base + rank;
    ls.pix[at] = pix;
    ls.obj[at] = sidx;
  }
}

__device__ __noinline__ bool analytic_depth(const FrameJob& fj, const DevObj& ob, const double o[3],
                                               const double d[3], double& depth) {
  double lo[3], ld[3], t;
  to_local(ob, o, d, lo, ld);
  bool hit = sphere_trace(fj.fields, ob.depth_field, lo, ld, 100.0, t);
  depth = ob.s * t;
  return hit;
}

// ---------------------------------------------------------------------------
// Work-list generation.  Every (pixel ray, NeDF object) pair whose local ray
// crosses the model's relaxed box (geometry.py:258-280, model.py:284-288) is
// appended to the model's list.  The box test runs in fp32 with a certified
// error bound (clip_hit_f32); only pairs whose float64 outcome the bound cannot
// decide -- grazing rays, slabs nearly parallel to the ray -- run the exact
// float64 clip, so the lists are the reference's exactly.
// ---------------------------------------------------------------------------

// fp32 world ray with absolute error bounds on its origin (eo) and unit direction (ed).
struct RayF {
  float o[3], d[3];
  float eo, ed;
};

// Per-object setup data, staged in shared memory by the setup kernels.
struct SetupObj {
  float4 sph;                    // world bounding sphere (c, 1.001 r) of the relaxed box
  float R[9], T[3], inv_s;
  float bmin[3], bmax[3];
  float smu;                     // s * mu_max (rounded up)
  int flags;                     // bit 0: NeDF, bit 1: plane kept from the cache (skip)
};

__device__ __forceinline__ SetupObj make_setup_obj(const DevObj& ob, bool cached) {
  SetupObj so;
  so.sph = make_float4(ob.bs_c[0], ob.bs_c[1], ob.bs_c[2], ob.bs_r * 1.001f);
#pragma unroll
  for (int i = 0; i < 9; ++i) so.R[i] = ob.Rf[i];
#pragma unroll
  for (int i = 0; i < 3; ++i) { so.T[i] = ob.Tf[i]; so.bmin[i] = ob.bminf[i]; so.bmax[i] = ob.bmaxf[i]; }
  so.inv_s = ob.inv_sf;
  so.smu = ob.smu_f;
  so.flags = (ob.depth_kind == NEDF_DEPTH_NEDF ? 1 : 0) | (cached && !ob.recompute ? 2 : 0);
  return so;
}

__device__ __forceinline__ float amax3(float a, float b, float c) { return fmaxf(fabsf(a), fmaxf(fabsf(b), fabsf(c))); }

// fp32 slab clip of a world ray against a NeDF object's relaxed box with a
// bound on the rounding of every step (fp32 ray, transform, reciprocal, slab
// distances; each ~1e-7 relative, bounded here by >= 1e-6 per step and a
// safety factor of 8 on the total).  Returns 1 / 0 when the float64 decision
// t_exit >= t_enter is certainly hit / miss, -1 when |t_exit - t_enter| is
// within the bound or a slab is nearly parallel to the ray (|d_l| < 1e-3,
// where the reference's inf/NaN slab rules apply): the caller then runs the
// exact float64 clip.
__device__ __forceinline__ int clip_hit_f32(const SetupObj& so, const RayF& r) {
  float q[3], lo[3], ld[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) q[a] = r.o[a] - so.T[a];
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    lo[j] = (q[0] * so.R[j] + q[1] * so.R[3 + j] + q[2] * so.R[6 + j]) * so.inv_s;
    ld[j] = r.d[0] * so.R[j] + r.d[1] * so.R[3 + j] + r.d[2] * so.R[6 + j];
  }
  const float ldmin = fminf(fabsf(ld[0]), fminf(fabsf(ld[1]), fabsf(ld[2])));
  if (!(ldmin >= 1e-3f)) return -1;
  const float bn = fmaxf(amax3(so.bmin[0], so.bmin[1], so.bmin[2]), amax3(so.bmax[0], so.bmax[1], so.bmax[2]));
  const float e_lo = (2.f * r.eo + 1e-6f * (amax3(r.o[0], r.o[1], r.o[2]) + amax3(so.T[0], so.T[1], so.T[2]))) * so.inv_s +
                     1e-6f * (amax3(lo[0], lo[1], lo[2]) + bn);
  const float e_ld = 2.f * r.ed + 1e-6f;
  float lo_max = -INFINITY, hi_min = INFINITY;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const float inv = __fdividef(1.f, ld[a]);        // rcp.approx: <= 1 ulp, inside the 1e-6 per-step bound
    const float ta = (so.bmin[a] - lo[a]) * inv, tb = (so.bmax[a] - lo[a]) * inv;
    lo_max = fmaxf(lo_max, fminf(ta, tb));
    hi_min = fminf(hi_min, fmaxf(ta, tb));
  }
  const float t0 = fmaxf(lo_max, 0.f), t1 = hi_min;
  const float tm = fmaxf(fabsf(t0), fabsf(t1));
  const float margin = 8.f * ((e_lo + tm * e_ld) * __fdividef(1.f, ldmin) + 1e-6f * tm) + 1e-6f;
  const float g = t1 - t0;
  if (!(fabsf(g) <= 1e30f) || !(margin <= 1e30f)) return -1;
  return g > margin ? 1 : (g < -margin ? 0 : -1);
}

struct CamF {
  float pos[3], rot[9];
  float gx_scale, gy_scale, two_over_w, two_over_h;
};

__device__ __forceinline__ CamF make_cam_f(const DevCam& c) {
  CamF f;
#pragma unroll
  for (int i = 0; i < 3; ++i) f.pos[i] = (float)c.pos[i];
#pragma unroll
  for (int i = 0; i < 9; ++i) f.rot[i] = (float)c.rot[i];
  f.gx_scale = (float)(c.tan_half * c.aspect);
  f.gy_scale = (float)c.tan_half;
  f.two_over_w = 2.0f / (float)c.width;
  f.two_over_h = 2.0f / (float)c.height;
  return f;
}

// fp32 camera ray (pipeline.py:97-109): direction error <= ~1e-6, bounded by 4e-6
__device__ __forceinline__ void cam_ray_f(const CamF& c, int row, int col, float o[3], float d[3]) {
  const float gx = fmaf((float)col + 0.5f, c.two_over_w, -1.f) * c.gx_scale;
  const float gy = fmaf(-((float)row + 0.5f), c.two_over_h, 1.f) * c.gy_scale;
  float v[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) v[i] = gx * c.rot[3 * i] + gy * c.rot[3 * i + 1] - c.rot[3 * i + 2];
  const float rn = rsqrtf(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]);
#pragma unroll
  for (int i = 0; i < 3; ++i) { d[i] = v[i] * rn; o[i] = c.pos[i]; }
}

// fp32 ray of a frame pixel for the setup kernel's mode, with error bounds.
// (row = local row, col = column, p = row * width + col)
__device__ __forceinline__ void pixel_ray_f(const FrameJob& fj, const CamF& cf, int row, int col, int p, RayF& r) {
  float co[3], cd[3];
  cam_ray_f(cf, fj.ray.rows[row], col, co, cd);
  const float e_cd = 4e-6f;
  if (fj.ray.mode == RAY_PRIMARY) {
#pragma unroll
    for (int a = 0; a < 3; ++a) { r.o[a] = co[a]; r.d[a] = cd[a]; }
    r.eo = 2e-7f * amax3(co[0], co[1], co[2]);
    r.ed = e_cd;
    return;
  }
  const float D = (float)fj.ray.depth64[p];
  float x[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) x[a] = fmaf(D, cd[a], co[a]);
  const float ex = fabsf(D) * e_cd + 4e-7f * (amax3(co[0], co[1], co[2]) + fabsf(D));
  if (fj.ray.mode == RAY_POINT_SHADOW) {
    const float L[3] = {(float)fj.ray.light[0], (float)fj.ray.light[1], (float)fj.ray.light[2]};
    float v[3] = {x[0] - L[0], x[1] - L[1], x[2] - L[2]};
    const float d2 = v[0] * v[0] + v[1] * v[1] + v[2] * v[2];
    const float inv = rsqrtf(d2), dist = d2 * inv;
#pragma unroll
    for (int a = 0; a < 3; ++a) { r.o[a] = L[a]; r.d[a] = v[a] * inv; }
    r.eo = 2e-7f * amax3(L[0], L[1], L[2]);
    r.ed = dist > 1e-3f ? 2.f * (ex + 2e-7f * amax3(x[0], x[1], x[2])) * inv + 1e-6f : INFINITY;
  } else {
    const float eps = (float)fj.ray.eps;
#pragma unroll
    for (int a = 0; a < 3; ++a) { r.d[a] = -(float)fj.ray.light[a]; r.o[a] = fmaf(eps, r.d[a], x[a]); }
    r.ed = 2e-7f;
    r.eo = ex + 4e-7f * amax3(r.o[0], r.o[1], r.o[2]) + 1e-7f;
  }
}

// fp32 copy of a float64 ray (rounding only)
__device__ __forceinline__ void round_ray_f(const double o[3], const double d[3], RayF& r) {
#pragma unroll
  for (int a = 0; a < 3; ++a) { r.o[a] = (float)o[a]; r.d[a] = (float)d[a]; }
  r.eo = 2e-7f * amax3(r.o[0], r.o[1], r.o[2]);
  r.ed = 2e-7f;
}

constexpr int kSetupStage = 64;

__device__ __forceinline__ void stage_setup_objs(const FrameJob& fj, bool cached, SetupObj* s_obj) {
  for (int s = threadIdx.x; s < fj.n_objs && s < kSetupStage; s += blockDim.x)
    s_obj[s] = make_setup_obj(fj.ray.objs[s], cached);
}

// Warp culling (all 32 lanes call it; no block synchronisation): the objects
// whose bounding sphere can meet any live ray of this warp, as a bit mask over
// scene indices.  With a common ray origin o (camera rays, point-light shadow
// rays; `cone`), the warp's unit directions lie in a cone (axis a = normalised
// mean, half-angle h = max angle to a), and a ray within h of a reaches a sphere
// seen from o at angle w only if angle(w, a) <= h + asin(r / |w|) (triangle
// inequality on the sphere of directions); the radius carries the same margins
// as sphere_miss_f, so no object the per-ray tests could accept is dropped.
// Without a common origin (directional light), with a plane cache, or for a cone
// wider than 90 degrees every object is a candidate.  Needs n_objs <= kSetupStage.
__device__ __forceinline__ unsigned long long cull_warp(const FrameJob& fj, const SetupObj* s_obj, bool cone,
                                                        bool live, const RayF& rf) {
  const int lane = threadIdx.x & 31;
  const int n = fj.n_objs;
  const unsigned live_mask = __ballot_sync(0xffffffffu, live);
  if (live_mask == 0u) return 0ull;
  const unsigned long long all = n >= 64 ? ~0ull : ((1ull << n) - 1ull);
  if (!cone) return all;
  float ax = live ? rf.d[0] : 0.f, ay = live ? rf.d[1] : 0.f, az = live ? rf.d[2] : 0.f;
  for (int off = 16; off > 0; off >>= 1) {
    ax += __shfl_xor_sync(0xffffffffu, ax, off);
    ay += __shfl_xor_sync(0xffffffffu, ay, off);
    az += __shfl_xor_sync(0xffffffffu, az, off);
  }
  const float n2 = ax * ax + ay * ay + az * az;
  const float inn = rsqrtf(n2);
  if (!(n2 * inn > 1e-3f * (float)__popc(live_mask))) return all;  // directions spread over a half-space
  ax *= inn; ay *= inn; az *= inn;
  float cos_h = live ? rf.d[0] * ax + rf.d[1] * ay + rf.d[2] * az : 1.f;
  for (int off = 16; off > 0; off >>= 1) cos_h = fminf(cos_h, __shfl_xor_sync(0xffffffffu, cos_h, off));
  cos_h = fminf(cos_h, 1.f);
  if (!(cos_h > 0.f)) return all;
  const float sin_h = sqrtf(fmaxf(0.f, 1.f - cos_h * cos_h));
  float o[3];
  if (fj.ray.mode == RAY_PRIMARY) {
    for (int a = 0; a < 3; ++a) o[a] = (float)fj.ray.cam.pos[a];
  } else {
    for (int a = 0; a < 3; ++a) o[a] = (float)fj.ray.light[a];
  }
  unsigned long long mask = 0ull;
  for (int s0 = 0; s0 < n; s0 += 32) {
    const int s = s0 + lane;
    bool keep = false;
    if (s < n) {
      const SetupObj& so = s_obj[s];
      keep = true;
      if ((so.flags & 1) && !(so.flags & 2)) {
        const float wx = so.sph.x - o[0], wy = so.sph.y - o[1], wz = so.sph.z - o[2];
        const float w2 = wx * wx + wy * wy + wz * wz;
        const float ilw = rsqrtf(w2), lw = w2 * ilw;
        const float r = so.sph.w + 1e-3f * (1.f + lw);
        if (lw > r) {
          const float sin_s = r * ilw, cos_s = sqrtf(fmaxf(0.f, 1.f - sin_s * sin_s));
          const float cos_hs = cos_h * cos_s - sin_h * sin_s;          // cos(h + s), h + s < 180 degrees
          const float cw = (wx * ax + wy * ay + wz * az) * ilw;
          keep = cos_hs < -0.999f || cw >= cos_hs - 1e-4f;
        }
      }
    }
    mask |= (unsigned long long)__ballot_sync(0xffffffffu, keep) << s0;
  }
  return mask;
}

// One pixel's pass over its warp's candidate objects `cand` (warp-uniform; all 32
// lanes call it: the list appends are warp-aggregated).  `live` = the pixel has a
// ray; rf is its fp32 ray; ray64(o, d) produces its float64 ray, called at most
// once, when an exact clip or an analytic object needs it.  Returns the analytic
// objects' z-key (NeDF objects reach the key through the network).  all_objs:
// visit every object (plane cache, or more than kSetupStage objects).
// The reference's float64 box test (geometry.py:258-280 after model.py:310-311);
// out of line: the certified fp32 test leaves it a small share of the pairs.
__device__ __noinline__ int exact_box_hit(const DevObj& ob, const GroupTable& gt, const double o[3], const double d[3]) {
  const DevModel& m = gt.models[ob.group];
  double lo[3], ld[3], t0, t1;
  to_local(ob, o, d, lo, ld);
  return slab_clip(lo, ld, m.bmin, m.bmax, t0, t1) ? 1 : 0;
}

// Lower bound of a NeDF pair's world depth |(o - T).d| - s mu (model.py:301-319,
// finish_ray) over every bin pair the network can pick (mu <= mu_max), from the
// fp32 ray: the margin covers the ray's error bounds (eo per origin component,
// ed per direction component), T's fp32 rounding and the fp32 arithmetic.
__device__ __forceinline__ float depth_lower_f(const SetupObj& so, const RayF& r) {
  const float q0 = r.o[0] - so.T[0], q1 = r.o[1] - so.T[1], q2 = r.o[2] - so.T[2];
  const float ad = fabsf(q0 * r.d[0] + q1 * r.d[1] + q2 * r.d[2]);
  const float qn = sqrtf(q0 * q0 + q1 * q1 + q2 * q2);
  const float margin = 2.f * (qn * (r.ed + 1e-6f) + r.eo) + 2e-6f * (ad + so.smu + amax3(so.T[0], so.T[1], so.T[2])) + 1e-6f;
  return ad - so.smu - margin;
}

__device__ __forceinline__ void defer_append(const DeferList& df, bool take, uint32_t pix, uint32_t sidx, float low) {
  const unsigned mask = __ballot_sync(0xffffffffu, take);
  if (mask == 0u) return;
  const int lane = threadIdx.x & 31, leader = __ffs(mask) - 1;
  int base = 0;
  if (lane == leader) base = atomicAdd(df.count, __popc(mask));
  base = __shfl_sync(0xffffffffu, base, leader);
  if (take) {
    const int at = base + __popc(mask & ((1u << lane) - 1u));
    df.pix[at] = pix;
    df.obj[at] = sidx;
    df.low[at] = low;
  }
}

template <class Ray64>
__device__ __forceinline__ unsigned long long setup_pixel(const FrameJob& fj, const GroupTable& gt, const ListSet& ls,
                                                          const SetupObj* s_obj, unsigned long long cand, bool all_objs,
                                                          int mode, bool cached, bool live, uint32_t p, const RayF& rf,
                                                          bool exact, Ray64 ray64, unsigned& n_exact) {
  unsigned long long key = kEmptyKey;
  double o[3], d[3];
  bool have64 = false;
  int k = 0;
  // front-first culling (STEP 1): only the pair with the smallest depth bound goes to the
  // lists now; the rest wait in fj.defer for the front pair's result (defer_filter_kernel)
  const bool defer_on = fj.defer.pix != nullptr && mode == RAY_PRIMARY && !cached && !all_objs;
  unsigned long long hitmask = 0ull;
  int front = -1;
  float front_low = INFINITY;
  while (all_objs ? k < fj.n_objs : cand != 0ull) {
    int s;
    if (all_objs) {
      s = k++;
    } else {
      s = __ffsll((long long)cand) - 1;
      cand &= cand - 1ull;
    }
    const bool staged = s < kSetupStage;
    SetupObj tmp;
    if (!staged) tmp = make_setup_obj(fj.ray.objs[s], cached);
    const SetupObj& so = staged ? s_obj[s] : tmp;
    const int flags = so.flags;
    if (flags & 2) continue;                                                      // cached plane kept
    if (flags & 1) {
      bool hit = false;
      if (live && !sphere_miss_f(so.sph, rf.o[0], rf.o[1], rf.o[2], rf.d[0], rf.d[1], rf.d[2])) {
        int h = exact ? -1 : clip_hit_f32(so, rf);
        if (h < 0) {
          if (!have64) { ray64(o, d); have64 = true; }
          h = exact_box_hit(fj.ray.objs[s], gt, o, d);
          ++n_exact;
        }
        hit = h > 0;
      }
      if (defer_on) {
        if (hit) {
          hitmask |= 1ull << s;
          const float lw = depth_lower_f(so, rf);
          if (lw < front_low) { front_low = lw; front = s; }
        }
      } else if (__any_sync(0xffffffffu, hit)) {
        warp_append(ls, fj.ray.objs[s].group, hit, p, (uint32_t)s);
      }
      if (cached && live) fj.planes[(size_t)s * fj.n_pix + p] = INFINITY;
    } else if (live) {
      if (!have64) { ray64(o, d); have64 = true; }
      const DevObj& ob = fj.ray.objs[s];
      double dep;
      bool hit = analytic_depth(fj, ob, o, d, dep);
      // directional shadows accept depth-0 hits (pipeline.py:362-364)
      bool ok = hit && isfinite(dep) && (mode == RAY_DIR_SHADOW ? dep >= 0.0 : dep > 0.0);
      if (ok) {
        unsigned long long kk = pack_key(dep, (uint32_t)s, 0, 0);
        key = kk < key ? kk : key;
      }
      if (cached) fj.planes[(size_t)s * fj.n_pix + p] = ok ? dep : INFINITY;
    }
  }
  if (defer_on) {
    unsigned long long any = (unsigned long long)__reduce_or_sync(0xffffffffu, (unsigned)hitmask) |
                             ((unsigned long long)__reduce_or_sync(0xffffffffu, (unsigned)(hitmask >> 32)) << 32);
    while (any != 0ull) {
      const int s = __ffsll((long long)any) - 1;
      any &= any - 1ull;
      const bool h = (hitmask >> s) & 1ull;
      warp_append(ls, fj.ray.objs[s].group, h && s == front, p, (uint32_t)s);
      const bool later = h && s != front;
      if (__any_sync(0xffffffffu, later))
        defer_append(fj.defer, later, p, (uint32_t)s, later ? depth_lower_f(s_obj[s], rf) : 0.f);
    }
  }
  return key;
}

__device__ __forceinline__ void add_stat(unsigned long long* stats, int slot, unsigned v) {
  if (stats == nullptr) return;
  for (int off = 16; off > 0; off >>= 1) v += __shfl_down_sync(0xffffffffu, v, off);
  if ((threadIdx.x & 31) == 0 && v) atomicAdd(stats + slot, (unsigned long long)v);
}

// The setup kernels walk the frame in 32-pixel row segments, one per warp (a
// segment never straddles two rows, so its rays form a narrow cone), grid-
// striding over segments with the (row, segment column) position advanced
// incrementally (no integer division per pixel).
struct SegWalk {
  int per_row, row, col, step_r, step_c;
  __device__ __forceinline__ SegWalk(int width) {
    per_row = (width + 31) >> 5;
    const int seg = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int step = gridDim.x * (blockDim.x >> 5);
    row = seg / per_row;
    col = seg - row * per_row;
    step_r = step / per_row;
    step_c = step - step_r * per_row;
  }
  __device__ __forceinline__ void next() {
    col += step_c;
    row += step_r;
    if (col >= per_row) { col -= per_row; ++row; }
  }
};

// float64 world ray of frame pixel (row, x), p = row * width + x (item_world_ray without the division)
__device__ __forceinline__ void pixel_world_ray(const RayJob& job, int row, int x, int p, double o[3], double d[3]) {
  double co[3], cd[3];
  cam_ray(job.cam, job.rows[row], x, co, cd);
  if (job.mode == RAY_PRIMARY) {
#pragma unroll
    for (int a = 0; a < 3; ++a) { o[a] = co[a]; d[a] = cd[a]; }
    return;
  }
  shadow_ray(job, co, cd, job.depth64[p], o, d);
}

// Work lists for STEP 1 (mode RAY_PRIMARY) or one light of STEP 3 (a shadow
// mode; receivers are pixels with id >= 0 and finite depth, pipeline.py:376),
// the pixel's z-key initialised with its analytic objects' nearest hit.
// exact = 1: every box test in float64 (the pre-certified-clip behaviour).
__global__ void __launch_bounds__(256, 3) setup_kernel(FrameJob fj, GroupTable gt, ListSet ls, int mode, int exact) {
  __shared__ SetupObj s_obj[kSetupStage];
  __shared__ CamF s_cam;
  const bool cached = mode == RAY_PRIMARY && fj.planes != nullptr;
  stage_setup_objs(fj, cached, s_obj);
  if (threadIdx.x == 0) s_cam = make_cam_f(fj.ray.cam);
  __syncthreads();
  unsigned n_exact = 0;
  const int W = fj.ray.cam.width, n_rows = fj.n_pix / W;
  const bool all_objs = cached || fj.n_objs > kSetupStage;
  const bool cone = mode == RAY_PRIMARY || mode == RAY_POINT_SHADOW;
  for (SegWalk sw(W); sw.row < n_rows; sw.next()) {
    const int x = sw.col * 32 + (threadIdx.x & 31);
    const int p = x < W ? sw.row * W + x : -1;
    bool live = p >= 0;
    if (live && mode != RAY_PRIMARY) live = fj.id[p] >= 0 && isfinite(fj.depth[p]);
    RayF rf;
    if (live) {
      if (exact) {
        double o[3], d[3];
        pixel_world_ray(fj.ray, sw.row, x, p, o, d);
        round_ray_f(o, d, rf);
      } else {
        pixel_ray_f(fj, s_cam, sw.row, x, p, rf);
      }
    }
    const unsigned long long cand = all_objs ? 0ull : cull_warp(fj, s_obj, cone, live, rf);
    const int row = sw.row;
    auto ray64 = [&](double* o, double* d) { pixel_world_ray(fj.ray, row, x, p, o, d); };
    unsigned long long key = setup_pixel(fj, gt, ls, s_obj, cand, all_objs, mode, cached, live, (uint32_t)p, rf,
                                         exact != 0, ray64, n_exact);
    if (p >= 0) fj.key[p] = key;
  }
  add_stat(fj.stats, 4, n_exact);
}

// Exact float64 depth of the winning (object, bins) of a z-key along the ray.
__device__ __forceinline__ double key_depth(const FrameJob& fj, const GroupTable& gt, unsigned long long key,
                                            const double o[3], const double d[3], bool dir_shadow) {
  uint32_t sidx = (uint32_t)(key >> 16) & 0xFFFFu;
  const DevObj& ob = fj.ray.objs[sidx];
  if (ob.depth_kind == NEDF_DEPTH_NEDF) {
    int c = (int)((key >> 8) & 0xFF), f = (int)(key & 0xFF);
    const DevModel& m = gt.models[ob.group];
    return tangency_dist(o, ob.T, d) - ob.s * decode_mu(m, c, f);
  }
  double dep;
  analytic_depth(fj, ob, o, d, dep);
  return dep;
}

// Front-first culling, second half: a deferred pair is evaluated only if its depth
// lower bound does not exceed the pixel's z-key depth after the front pairs (and
// any analytic objects).  A skipped pair has fp32(depth) >= low > the key's fp32
// depth, so its key could not have won the atomicMin: the z-buffer is unchanged.
__global__ void defer_filter_kernel(FrameJob fj, ListSet ls) {
  const int n = *fj.defer.count;
  const int lane = threadIdx.x & 31;
  const int stride = gridDim.x * blockDim.x;
  unsigned n_cut = 0;
  for (int i0 = blockIdx.x * blockDim.x + (threadIdx.x & ~31); i0 < n; i0 += stride) {
    const int i = i0 + lane;
    bool take = false;
    uint32_t p = 0, s = 0;
    int g = -1;
    if (i < n) {
      p = fj.defer.pix[i];
      s = fj.defer.obj[i];
      const unsigned long long key = fj.key[p];
      const float best = __uint_as_float((uint32_t)(key >> 32));   // kEmptyKey: NaN -> taken
      take = !(fj.defer.low[i] > best);
      g = fj.ray.objs[s].group;
      n_cut += take ? 0u : 1u;
    }
    unsigned pend = __ballot_sync(0xffffffffu, take);
    while (pend != 0u) {
      const int g0 = __shfl_sync(0xffffffffu, g, __ffs(pend) - 1);
      const bool mine = take && g == g0;
      warp_append(ls, g0, mine, p, s);
      take = take && !mine;
      pend = __ballot_sync(0xffffffffu, take);
    }
  }
  add_stat(fj.stats, 5, n_cut);
}

// STEP 1 resolve: z-key -> depth (f64) and user id (pipeline.py:259-268).
__global__ void step1_resolve_kernel(FrameJob fj, GroupTable gt) {
  const int stride = gridDim.x * blockDim.x;
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < fj.n_pix; p += stride) {
    unsigned long long key = fj.key[p];
    if (key == kEmptyKey) {
      fj.depth[p] = INFINITY;
      fj.id[p] = -1;
      continue;
    }
    double o[3], d[3];
    item_world_ray(fj.ray, (uint32_t)p, o, d);
    uint32_t sidx = (uint32_t)(key >> 16) & 0xFFFFu;
    fj.depth[p] = key_depth(fj, gt, key, o, d, false);
    fj.id[p] = fj.ray.objs[sidx].id;
  }
}

// STEP 1 from per-object planes (_recombine, pipeline.py:259-268): scene order,
// strict <, so ties go to the earliest object and the result is a pure
// function of the planes (cached and cold renders are bit-identical).
__global__ void recombine_kernel(FrameJob fj) {
  const int stride = gridDim.x * blockDim.x;
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < fj.n_pix; p += stride) {
    double best = INFINITY;
    int bs = -1;
    for (int s = 0; s < fj.n_objs; ++s) {
      const double v = fj.planes[(size_t)s * fj.n_pix + p];
      if (v < best) { best = v; bs = s; }
    }
    fj.depth[p] = best;
    fj.id[p] = bs >= 0 ? fj.ray.objs[bs].id : -1;
    fj.key[p] = bs >= 0 ? pack_key(best, (uint32_t)bs, 0, 0) : kEmptyKey;
  }
}

cudaError_t launch_recombine(const FrameJob& fj, int n_sms, cudaStream_t st);

// emission-absorption colour over [t_n, t_f] (fields.py:364-370, 406-420)
__device__ void volume_color(const NedfField* fields, int root, const double o[3], const double d[3],
                             double t_n, double t_f, int n, double rgb[3]) {
  double delta = (t_f - t_n) / n;
  double acc_tau = 0.0;
  rgb[0] = rgb[1] = rgb[2] = 0.0;
  for (int i = 0; i < n; ++i) {
    double t = t_n + (i + 0.5) * delta;
    double p[3] = {o[0] + t * d[0], o[1] + t * d[1], o[2] + t * d[2]};
    double c[3], sig;
    field_radiance(fields, root, p, c, sig);
    double tau = sig * delta;
    double w = exp(-acc_tau) * (1.0 - exp(-tau));
    for (int a = 0; a < 3; ++a) rgb[a] += w * c[a];
    acc_tau += tau;
  }
}

// Colour of a covered pixel: object `ob` at depth D along the camera ray (o, d)
// (pipeline.py:326-350).  Returns true when the pixel was an outlier that got
// resampled (counted only when resampling is on, pipeline.py:340-350).
__device__ __forceinline__ bool shade_pixel(const FrameJob& fj, const DevObj& ob, const double o[3], const double d[3],
                                            double D, float out[3]) {
  double x[3] = {o[0] + D * d[0], o[1] + D * d[1], o[2] + D * d[2]};
  double lp[3], ld[3];
  to_local(ob, x, d, lp, ld);
  double rgb[3], sig;
  field_radiance(fj.fields, ob.radiance_field, lp, rgb, sig);
  double thr = fj.sigma_threshold >= 0.0 ? fj.sigma_threshold : ob.sigma_default;
  bool outlier = false;
  if (sig < thr && fj.resample) {
    outlier = true;
    double lo[3], ld2[3], t0, t1;
    to_local(ob, o, d, lo, ld2);
    if (slab_clip(lo, ld2, ob.rbox_min, ob.rbox_max, t0, t1))
      volume_color(fj.fields, ob.radiance_field, lo, ld2, t0, t1, fj.resample_samples, rgb);
  }
#pragma unroll
  for (int a = 0; a < 3; ++a) out[a] = (float)rgb[a];
  return outlier;
}

__device__ __forceinline__ void store_rgb(const FrameJob& fj, int p, const float c[3]) {
#pragma unroll
  for (int a = 0; a < 3; ++a) fj.rgb[3 * (size_t)p + a] = c[a];
}

// STEP 2: deferred shading (pipeline.py:315-352).
__global__ void shade_kernel(FrameJob fj, GroupTable gt) {
  const int stride = gridDim.x * blockDim.x;
  unsigned n_cov = 0, n_out = 0;
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < fj.n_pix; p += stride) {
    unsigned long long key = fj.key[p];
    const int idp = fj.id[p];
    if (idp < 0) {
      const float clear[3] = {(float)fj.clear[0], (float)fj.clear[1], (float)fj.clear[2]};
      store_rgb(fj, p, clear);
      continue;
    }
    ++n_cov;
    if (key == kEmptyKey) continue;
    const DevObj& ob = fj.ray.objs[(key >> 16) & 0xFFFFu];
    // a pixel taken over by an external layer keeps its imported colour (pipeline.py:406-420)
    if (ob.id != idp) continue;
    double o[3], d[3];
    item_world_ray(fj.ray, (uint32_t)p, o, d);
    float c[3];
    n_out += shade_pixel(fj, ob, o, d, fj.depth[p], c) ? 1u : 0u;
    store_rgb(fj, p, c);
  }
  add_stat(fj.stats, 0, n_cov);
  add_stat(fj.stats, 1, n_out);
}

// STEP 1 resolve + STEP 2 shading + shadow := 1 + the first light's STEP 3 work
// lists, in one pass over the pixels (nedf_render_frame without a plane cache):
// the same arithmetic as step1_resolve_kernel, shade_kernel, the shadow fill and
// setup_kernel(smode), which each re-read the pixel's state.  smode < 0: no
// shadow pass follows.  sj = the STEP 3 job (its key = the shadow z-keys).
#ifndef NEDF_RS_MINB
#define NEDF_RS_MINB 2
#endif
__global__ void __launch_bounds__(256, NEDF_RS_MINB) resolve_shade_kernel(FrameJob fj, GroupTable gt, ListSet ls, FrameJob sj,
                                                               int smode, int exact) {
  __shared__ SetupObj s_obj[kSetupStage];
  if (smode >= 0) {
    stage_setup_objs(fj, false, s_obj);
    __syncthreads();
  }
  unsigned n_cov = 0, n_out = 0, n_exact = 0;
  const float clear[3] = {(float)fj.clear[0], (float)fj.clear[1], (float)fj.clear[2]};
  const int W = fj.ray.cam.width, n_rows = fj.n_pix / W;
  const bool all_objs = fj.n_objs > kSetupStage;
  SegWalk sw(W);
  // the z-key of the warp's next segment is loaded one iteration ahead (its L2/HBM latency
  // overlaps this segment's work)
  auto seg_key = [&](const SegWalk& w) {
    const int xx = w.col * 32 + (threadIdx.x & 31);
    return (w.row < n_rows && xx < W) ? fj.key[w.row * W + xx] : kEmptyKey;
  };
  unsigned long long key_next = seg_key(sw);
  for (; sw.row < n_rows; sw.next()) {
    const int x = sw.col * 32 + (threadIdx.x & 31);
    const int p = x < W ? sw.row * W + x : -1;
    const bool live = p >= 0;
    const unsigned long long key = key_next;
    {
      SegWalk nx = sw;
      nx.next();
      key_next = seg_key(nx);
    }
    double co[3], cd[3], D = INFINITY;
    int idp = -1;
    if (key != kEmptyKey) {
      cam_ray(fj.ray.cam, fj.ray.rows[sw.row], x, co, cd);
      const DevObj& ob = fj.ray.objs[(key >> 16) & 0xFFFFu];
      D = key_depth(fj, gt, key, co, cd, false);
      idp = ob.id;
      if (idp >= 0) {
        float c[3];
        n_out += shade_pixel(fj, ob, co, cd, D, c) ? 1u : 0u;
        store_rgb(fj, p, c);
      }
    }
    if (live) {
      fj.depth[p] = D;
      fj.id[p] = idp;
      fj.shadow[p] = 1.0f;
      if (idp < 0) store_rgb(fj, p, clear);
      else ++n_cov;
    }
    if (smode >= 0) {
      const bool recv = live && idp >= 0 && isfinite(D);      // pipeline.py:376
      RayF rf;
      double so[3], sd[3];
      if (recv) {
        shadow_ray(sj.ray, co, cd, D, so, sd);
        round_ray_f(so, sd, rf);
      }
      const unsigned long long cand =
          all_objs ? 0ull : cull_warp(sj, s_obj, smode == RAY_POINT_SHADOW, recv, rf);
      auto ray64 = [&](double* o, double* d) {
#pragma unroll
        for (int a = 0; a < 3; ++a) { o[a] = so[a]; d[a] = sd[a]; }
      };
      unsigned long long sk = setup_pixel(sj, gt, ls, s_obj, cand, all_objs, smode, false, recv, (uint32_t)p, rf,
                                          exact != 0, ray64, n_exact);
      if (live) sj.key[p] = sk;
    }
  }
  add_stat(fj.stats, 0, n_cov);
  add_stat(fj.stats, 1, n_out);
  add_stat(fj.stats, 4, n_exact);
}

// STEP 3 resolve for one light (pipeline.py:381-403); with `image`, also the
// composite image = rgb * shadow (pipeline.py:467) of the frame's last light.
__global__ void shadow_resolve_kernel(FrameJob fj, GroupTable gt, int mode, float* image) {
  const int stride = gridDim.x * blockDim.x;
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < fj.n_pix; p += stride) {
    float sh = fj.shadow[p];
    const unsigned long long key = fj.key[p];
    if (fj.id[p] >= 0 && isfinite(fj.depth[p]) && (key != kEmptyKey || mode == RAY_DIR_SHADOW)) {
      bool shadowed;
      if (mode == RAY_DIR_SHADOW) {
        shadowed = key != kEmptyKey;
      } else {
        double co[3], cd[3], o[3], d[3];
        const int w = fj.ray.cam.width;
        cam_ray(fj.ray.cam, fj.ray.rows[p / w], p % w, co, cd);
        const double D = fj.depth[p];
        shadow_ray(fj.ray, co, cd, D, o, d);           // o = light, d = unit toward x
        double v[3];
        for (int a = 0; a < 3; ++a) v[a] = (co[a] + D * cd[a]) - fj.ray.light[a];
        double dist = sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]);
        double ds = key_depth(fj, gt, key, o, d, false);
        shadowed = ds + fj.eps < dist;
      }
      if (shadowed) {
        sh = (float)((double)sh * fj.beta);
        fj.shadow[p] = sh;
      }
    }
    if (image != nullptr) {
#pragma unroll
      for (int a = 0; a < 3; ++a) image[3 * (size_t)p + a] = fj.rgb[3 * (size_t)p + a] * sh;
    }
  }
}

__global__ void fill_kernel(float* buf, int64_t n, float v) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    buf[i] = v;
}

__global__ void composite_kernel(const float* rgb, const float* shadow, float* image, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    float s = shadow[i];
    image[3 * i + 0] = rgb[3 * i + 0] * s;
    image[3 * i + 1] = rgb[3 * i + 1] * s;
    image[3 * i + 2] = rgb[3 * i + 2] * s;
  }
}

// Explicit rays (query_world / query_rays): clip against the model box,
// enqueue hits, write the box-miss result (mu = NaN, alpha = 0) directly.
__global__ void explicit_setup_kernel(RayJob job, GroupTable gt, ListSet ls, OutSpec out, int64_t n) {
  const DevModel& m = gt.models[0];
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < n; base += stride) {
    int64_t i = base + threadIdx.x;
    bool live = i < n, hit = false;
    if (live) {
      double wo[3], wd[3], lo[3], ld[3], t0, t1;
      item_local_ray(job, (uint32_t)i, 0u, wo, wd, lo, ld);
      hit = slab_clip(lo, ld, m.bmin, m.bmax, t0, t1);
      if (!hit && out.mode != OUT_LOGITS) {
        if (out.mode == OUT_QUERY_LOCAL) out.mu[i] = NAN;
        else out.depth[i] = NAN;   // dist - s * NaN
        out.alpha[i] = 0;
      }
    }
    warp_append(ls, 0, hit, (uint32_t)i, 0u);
  }
}

// OUT_LOGITS: every row is evaluated (nn.forward has no box test).
__global__ void iota_setup_kernel(ListSet ls, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    ls.pix[i] = (uint32_t)i;
    ls.obj[i] = 0u;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) ls.count[0] = (int)n;
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
static int grid_for(int64_t n, int n_sms) {
  int64_t g = (n + 255) / 256;
  int64_t cap = (int64_t)n_sms * 8;
  return (int)(g < 1 ? 1 : (g > cap ? cap : g));
}

// blocks of 8 warps over the frame's 32-pixel row segments, at most per_sm resident blocks per SM
static int seg_grid(const FrameJob& fj, int n_sms, int per_sm) {
  const int w = fj.ray.cam.width > 0 ? fj.ray.cam.width : 1;
  const int64_t blocks = ((int64_t)((w + 31) / 32) * (fj.n_pix / w) + 7) / 8;
  const int64_t cap = (int64_t)n_sms * per_sm;
  return (int)(blocks < 1 ? 1 : (blocks > cap ? cap : blocks));
}

cudaError_t launch_setup(const FrameJob& fj, const GroupTable& gt, const ListSet& ls, int mode, int exact, int n_sms,
                         cudaStream_t st) {
  setup_kernel<<<seg_grid(fj, n_sms, 3), 256, 0, st>>>(fj, gt, ls, mode, exact);
  return cudaGetLastError();
}
cudaError_t launch_defer_filter(const FrameJob& fj, const ListSet& ls, int n_sms, cudaStream_t st) {
  defer_filter_kernel<<<4 * n_sms, 256, 0, st>>>(fj, ls);
  return cudaGetLastError();
}

cudaError_t launch_step1_resolve(const FrameJob& fj, const GroupTable& gt, int n_sms, cudaStream_t st) {
  step1_resolve_kernel<<<grid_for(fj.n_pix, n_sms), 256, 0, st>>>(fj, gt);
  return cudaGetLastError();
}
cudaError_t launch_recombine(const FrameJob& fj, int n_sms, cudaStream_t st) {
  recombine_kernel<<<grid_for(fj.n_pix, n_sms), 256, 0, st>>>(fj);
  return cudaGetLastError();
}
cudaError_t launch_shade(const FrameJob& fj, const GroupTable& gt, int n_sms, cudaStream_t st) {
  shade_kernel<<<grid_for(fj.n_pix, n_sms), 256, 0, st>>>(fj, gt);
  return cudaGetLastError();
}
cudaError_t launch_shadow_resolve(const FrameJob& fj, const GroupTable& gt, int mode, float* image, int n_sms,
                                  cudaStream_t st) {
  shadow_resolve_kernel<<<grid_for(fj.n_pix, n_sms), 256, 0, st>>>(fj, gt, mode, image);
  return cudaGetLastError();
}
cudaError_t launch_resolve_shade(const FrameJob& fj, const GroupTable& gt, const ListSet& ls, const FrameJob& sj,
                                 int smode, int exact, int n_sms, cudaStream_t st) {
  resolve_shade_kernel<<<seg_grid(fj, n_sms, NEDF_RS_MINB), 256, 0, st>>>(fj, gt, ls, sj, smode, exact);
  return cudaGetLastError();
}
cudaError_t launch_fill(float* buf, int64_t n, float v, int n_sms, cudaStream_t st) {
  fill_kernel<<<grid_for(n, n_sms), 256, 0, st>>>(buf, n, v);
  return cudaGetLastError();
}
cudaError_t launch_composite(const float* rgb, const float* shadow, float* image, int64_t n, int n_sms,
                             cudaStream_t st) {
  composite_kernel<<<grid_for(n, n_sms), 256, 0, st>>>(rgb, shadow, image, n);
  return cudaGetLastError();
}
cudaError_t launch_explicit_setup(const RayJob& job, const GroupTable& gt, const ListSet& ls, const OutSpec& out,
                                  int64_t n, int n_sms, cudaStream_t st) {
  explicit_setup_kernel<<<grid_for(n, n_sms), 256, 0, st>>>(job, gt, ls, out, n);
  return cudaGetLastError();
}
__global__ void stats_export_kernel(unsigned long long* stats, unsigned long long* host_mapped) {
  const int i = threadIdx.x;
  if (i < 8) {
    host_mapped[i] = stats[i];
    stats[i] = 0;
  }
}
cudaError_t launch_stats_export(unsigned long long* stats, unsigned long long* host_mapped, cudaStream_t st) {
  stats_export_kernel<<<1, 32, 0, st>>>(stats, host_mapped);
  return cudaGetLastError();
}
cudaError_t launch_iota_setup(const ListSet& ls, int64_t n, int n_sms, cudaStream_t st) {
  iota_setup_kernel<<<grid_for(n, n_sms), 256, 0, st>>>(ls, n);
  return cudaGetLastError();
}

}  // namespace nedf
