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

__device__ __forceinline__ bool analytic_depth(const FrameJob& fj, const DevObj& ob, const double o[3],
                                               const double d[3], double& depth) {
  double lo[3], ld[3], t;
  to_local(ob, o, d, lo, ld);
  bool hit = sphere_trace(fj.fields, ob.depth_field, lo, ld, 100.0, t);
  depth = ob.s * t;
  return hit;
}

// Enqueue the (ray, object) pairs that reach the network and trace analytic
// objects.  mode: RAY_PRIMARY (STEP 1) or a shadow mode (STEP 3).  The first
// kSetupStage objects' prefilter data (bounding sphere, kind, flags) is staged
// in shared memory once per block; the pixel loop then touches an object's
// full descriptor only when its fp32 sphere test passes.
constexpr int kSetupStage = 64;
__global__ void __launch_bounds__(256, 4) setup_kernel(FrameJob fj, GroupTable gt, ListSet ls, int mode) {
  __shared__ float4 s_sph[kSetupStage];
  __shared__ int s_flags[kSetupStage];      // bit 0: NeDF, bit 1: plane kept from the cache (skip)
  const bool cached = mode == RAY_PRIMARY && fj.planes != nullptr;
  for (int s = threadIdx.x; s < fj.n_objs && s < kSetupStage; s += blockDim.x) {
    const DevObj& ob = fj.ray.objs[s];
    s_sph[s] = make_float4(ob.bs_c[0], ob.bs_c[1], ob.bs_c[2], ob.bs_r * 1.001f);
    s_flags[s] = (ob.depth_kind == NEDF_DEPTH_NEDF ? 1 : 0) | (cached && !ob.recompute ? 2 : 0);
  }
  __syncthreads();
  const int stride = gridDim.x * blockDim.x;
  for (int base = blockIdx.x * blockDim.x; base < fj.n_pix; base += stride) {
    const int p = base + threadIdx.x;
    bool live = p < fj.n_pix;
    if (live && mode != RAY_PRIMARY) {
      // valid receivers only (pipeline.py:376): id >= 0 and finite depth
      live = fj.id[p] >= 0 && isfinite(fj.depth[p]);
    }
    double o[3] = {0, 0, 0}, d[3] = {0, 0, 1};
    if (live) item_world_ray(fj.ray, (uint32_t)p, o, d);
    const float ox = (float)o[0], oy = (float)o[1], oz = (float)o[2];
    const float dx = (float)d[0], dy = (float)d[1], dz = (float)d[2];
    unsigned long long key = kEmptyKey;
    for (int s = 0; s < fj.n_objs; ++s) {
      int flags;
      float4 sph;
      if (s < kSetupStage) {
        flags = s_flags[s];
        sph = s_sph[s];
      } else {
        const DevObj& ob = fj.ray.objs[s];
        flags = (ob.depth_kind == NEDF_DEPTH_NEDF ? 1 : 0) | (cached && !ob.recompute ? 2 : 0);
        sph = make_float4(ob.bs_c[0], ob.bs_c[1], ob.bs_c[2], ob.bs_r * 1.001f);
      }
      if (flags & 2) continue;                                                       // cached plane kept
      if (flags & 1) {
        bool hit = false;
        if (live && !sphere_miss_f(sph, ox, oy, oz, dx, dy, dz)) {
          const DevObj& ob = fj.ray.objs[s];
          const DevModel& m = gt.models[ob.group];
          double lo[3], ld[3], t0, t1;
          to_local(ob, o, d, lo, ld);
          hit = slab_clip(lo, ld, m.bmin, m.bmax, t0, t1);
        }
        if (__any_sync(0xffffffffu, hit)) warp_append(ls, fj.ray.objs[s].group, hit, (uint32_t)p, (uint32_t)s);
        if (cached && p < fj.n_pix) fj.planes[(size_t)s * fj.n_pix + p] = INFINITY;
      } else if (live) {
        const DevObj& ob = fj.ray.objs[s];
        double dep;
        bool hit = analytic_depth(fj, ob, o, d, dep);
        // directional shadows accept depth-0 hits (pipeline.py:362-364)
        bool ok = hit && isfinite(dep) && (mode == RAY_DIR_SHADOW ? dep >= 0.0 : dep > 0.0);
        if (ok) {
          unsigned long long k = pack_key(dep, (uint32_t)s, 0, 0);
          key = k < key ? k : key;
        }
        if (cached) fj.planes[(size_t)s * fj.n_pix + p] = ok ? dep : INFINITY;
      } else if (cached && p < fj.n_pix) {
        fj.planes[(size_t)s * fj.n_pix + p] = INFINITY;
      }
    }
    if (p < fj.n_pix) fj.key[p] = key;
  }
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

// STEP 2: deferred shading (pipeline.py:315-352).
__global__ void shade_kernel(FrameJob fj, GroupTable gt) {
  const int stride = gridDim.x * blockDim.x;
  unsigned long long n_cov = 0, n_out = 0;
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < fj.n_pix; p += stride) {
    unsigned long long key = fj.key[p];
    const int idp = fj.id[p];
    if (idp < 0) {
      for (int a = 0; a < 3; ++a) fj.rgb[3 * (size_t)p + a] = (float)fj.clear[a];
      continue;
    }
    ++n_cov;
    if (key == kEmptyKey) continue;
    const DevObj& ob = fj.ray.objs[(key >> 16) & 0xFFFFu];
    // a pixel taken over by an external layer keeps its imported colour (pipeline.py:406-420)
    if (ob.id != idp) continue;
    double o[3], d[3];
    item_world_ray(fj.ray, (uint32_t)p, o, d);
    double D = fj.depth[p];
    double x[3] = {o[0] + D * d[0], o[1] + D * d[1], o[2] + D * d[2]};
    double lp[3], ld[3];
    to_local(ob, x, d, lp, ld);
    double rgb[3], sig;
    field_radiance(fj.fields, ob.radiance_field, lp, rgb, sig);
    double thr = fj.sigma_threshold >= 0.0 ? fj.sigma_threshold : ob.sigma_default;
    if (sig < thr) {
      if (fj.resample) {
        ++n_out;   // counted only when resampling is on (pipeline.py:340-350)
        double lo[3], ld2[3], t0, t1;
        to_local(ob, o, d, lo, ld2);
        if (slab_clip(lo, ld2, ob.rbox_min, ob.rbox_max, t0, t1))
          volume_color(fj.fields, ob.radiance_field, lo, ld2, t0, t1, fj.resample_samples, rgb);
      }
    }
    for (int a = 0; a < 3; ++a) fj.rgb[3 * (size_t)p + a] = (float)rgb[a];
  }
  if (fj.stats != nullptr) {
    for (int off = 16; off > 0; off >>= 1) {
      n_cov += __shfl_down_sync(0xffffffffu, n_cov, off);
      n_out += __shfl_down_sync(0xffffffffu, n_out, off);
    }
    if ((threadIdx.x & 31) == 0) {
      if (n_cov) atomicAdd(fj.stats + 0, n_cov);
      if (n_out) atomicAdd(fj.stats + 1, n_out);
    }
  }
}

// STEP 3 resolve for one light (pipeline.py:381-403).
__global__ void shadow_resolve_kernel(FrameJob fj, GroupTable gt, int mode) {
  const int stride = gridDim.x * blockDim.x;
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < fj.n_pix; p += stride) {
    if (!(fj.id[p] >= 0 && isfinite(fj.depth[p]))) continue;
    unsigned long long key = fj.key[p];
    bool shadowed;
    if (mode == RAY_DIR_SHADOW) {
      shadowed = key != kEmptyKey;
    } else {
      if (key == kEmptyKey) continue;
      double o[3], d[3];
      item_world_ray(fj.ray, (uint32_t)p, o, d);     // o = light, d = unit toward x
      double co[3], cd[3];
      int w = fj.ray.cam.width;
      cam_ray(fj.ray.cam, fj.ray.rows[p / w], p % w, co, cd);
      double D = fj.depth[p];
      double v[3];
      for (int a = 0; a < 3; ++a) v[a] = (co[a] + D * cd[a]) - fj.ray.light[a];
      double dist = sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]);
      double ds = key_depth(fj, gt, key, o, d, false);
      shadowed = ds + fj.eps < dist;
    }
    if (shadowed) fj.shadow[p] = (float)((double)fj.shadow[p] * fj.beta);
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

cudaError_t launch_setup(const FrameJob& fj, const GroupTable& gt, const ListSet& ls, int mode, int n_sms,
                         cudaStream_t st) {
  setup_kernel<<<grid_for(fj.n_pix, n_sms), 256, 0, st>>>(fj, gt, ls, mode);
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
cudaError_t launch_shadow_resolve(const FrameJob& fj, const GroupTable& gt, int mode, int n_sms, cudaStream_t st) {
  shadow_resolve_kernel<<<grid_for(fj.n_pix, n_sms), 256, 0, st>>>(fj, gt, mode);
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
