// C ABI of the NeDF frame path (include/nedf_b200.h): contexts, weights,
// per-call scene tables, and the step drivers that sequence the kernels.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>
#include <algorithm>

#include "common.cuh"
#include "frame.cuh"
#include "../../include/nedf_b200_diag.h"

using namespace nedf;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define CUDA_TRY(expr)                                                                       \
  do {                                                                                       \
    cudaError_t _e = (expr);                                                                 \
    if (_e != cudaSuccess)                                                                   \
      return fail(NEDF_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e));        \
  } while (0)

// grow-only device buffer
struct DevBuf {
  void* ptr = nullptr;
  size_t bytes = 0;
  cudaError_t ensure(size_t need) {
    if (need <= bytes) return cudaSuccess;
    if (ptr) cudaFree(ptr);
    ptr = nullptr;
    bytes = 0;
    size_t n = std::max<size_t>(need, 256);
    cudaError_t e = cudaMalloc(&ptr, n);
    if (e == cudaSuccess) e = cudaMemset(ptr, 0, n);     // counters (stats, list counts) start at zero
    if (e == cudaSuccess) bytes = n;
    return e;
  }
  template <class T> T* as() const { return reinterpret_cast<T*>(ptr); }
  void release() { if (ptr) cudaFree(ptr); ptr = nullptr; bytes = 0; }
};

}  // namespace

struct NedfModel {
  NedfModelInfo info;
  DevModel host;          // with device pointers
  DevModel* dev = nullptr;
  float* wT = nullptr;
  float* bias = nullptr;
  __half* wpack = nullptr;
  __half* wpack_lo = nullptr;
  float* bias_pack = nullptr;
  float* wstream = nullptr;
  float* wcluster = nullptr;
  float* wcluster8 = nullptr;
  void* wguard = nullptr;
  int device = 0;
};

constexpr int kStatSlots = 64;   // mapped snapshot slots (nedf_stats_snapshot)

struct NedfContext {
  int device = 0;
  int n_sms = 148;
  int precision = NEDF_PREC_AUTO;
  int guard_ppm = 3000;
  int tc_ctas = 0;
  int tc_kernel = NEDF_TC_AUTO;
  int guard_cluster = 0;
  int guard_kernel = NEDF_GUARD_AUTO;
  int setup_exact = 0;
  int fuse = 1;
  int cull = 1;
  int shadow_cert = 1;
  int guard_direct = 0;      // diagnostics: run only the guard kernel NEDF_GUARD_* on every list entry
  int profile = 0;
  int64_t launches = 0;
  // event pairs around network launches (NEDF_OPT_PROFILE); kind 0 = main, 1 = guard
  std::vector<cudaEvent_t> ev_pool;
  std::vector<std::pair<int, int>> ev_pairs;   // (start index, kind)
  size_t ev_used = 0;
  DevBuf models, objs, fields, rows, offsets, counts, redo_counts, lists_pix, lists_obj, redo_pix, redo_obj,
      key, skey, stats, tile_counter, defer_pix, defer_obj, defer_low, defer_count;
  int64_t h2d_bytes = 0;
  // mapped pinned mirror of the 8 stats counters: read back by a one-warp kernel, so reading stats
  // never queues behind a caller's large device-to-host copy on the copy engine
  unsigned long long* stats_host = nullptr;
  unsigned long long* stats_host_dev = nullptr;
};

namespace {

// host -> device copy of per-call tables, counted for the e2e byte report
cudaError_t h2d_async(NedfContext* ctx, void* dst, const void* src, size_t n, cudaStream_t st) {
  ctx->h2d_bytes += (int64_t)n;
  return cudaMemcpyAsync(dst, src, n, cudaMemcpyHostToDevice, st);
}

const int64_t kNoStats = -1;

int layer_count(int n_blocks) { return 3 + 2 * n_blocks; }

int validate_dims(const NedfModelInfo& in) {
  if (in.d_in != kDin) return fail(NEDF_ERR_FORMAT, "d_in must be 1008 (16 points x 63 features)");
  if (in.d_feat < 4 || in.d_feat > 256 || in.d_feat % 4)
    return fail(NEDF_ERR_UNSUPPORTED, "d_feat must be a multiple of 4 in [4, 256]");
  if (in.n_blocks < 0 || layer_count(in.n_blocks) > 40) return fail(NEDF_ERR_UNSUPPORTED, "n_blocks must be <= 18");
  if (in.n_coarse < 2 || in.n_fine < 2) return fail(NEDF_ERR_FORMAT, "need at least 2 bins per level");
  if (in.n_coarse + 1 > 128 || in.n_fine > 128) return fail(NEDF_ERR_UNSUPPORTED, "n_coarse + 1 and n_fine must be <= 128");
  if (!(in.half_range > 0)) return fail(NEDF_ERR_INVALID, "half_range must be positive");
  for (int a = 0; a < 3; ++a)
    if (!(in.box_min[a] <= in.box_max[a])) return fail(NEDF_ERR_INVALID, "box min must not exceed max");
  return NEDF_OK;
}

size_t param_count(const NedfModelInfo& in) {
  size_t n = (size_t)in.d_feat * in.d_in + in.d_feat;
  n += (size_t)2 * in.n_blocks * ((size_t)in.d_feat * in.d_feat + in.d_feat);
  n += (size_t)(in.n_coarse + 1) * in.d_feat + (in.n_coarse + 1);
  n += (size_t)in.n_fine * in.d_feat + in.n_fine;
  return n;
}

// Per-call scene tables.
struct Scene {
  std::vector<DevObj> objs;
  std::vector<const NedfModel*> group_models;
  std::vector<int> objs_per_group;
  int n_objs = 0;
  bool all_tc = true;
};

int build_scene(NedfContext* ctx, const NedfObject* objs, int n_objs, const NedfField* fields, int n_fields,
                Scene& sc, cudaStream_t st) {
  if (n_objs < 0 || n_objs > kMaxObjs) return fail(NEDF_ERR_INVALID, "too many objects (max 65535)");
  if (n_objs > 0 && objs == nullptr) return fail(NEDF_ERR_INVALID, "objects pointer is NULL");
  sc.n_objs = n_objs;
  sc.objs.resize(std::max(n_objs, 1));
  for (int s = 0; s < n_objs; ++s) {
    const NedfObject& o = objs[s];
    DevObj& d = sc.objs[s];
    memset(&d, 0, sizeof(d));
    for (int i = 0; i < 9; ++i) d.R[i] = o.R[i];
    for (int i = 0; i < 3; ++i) d.T[i] = o.T[i];
    if (!(o.s > 0) || !std::isfinite(o.s)) return fail(NEDF_ERR_INVALID, "scale must be a positive real");
    d.s = o.s;
    d.id = o.id;
    d.depth_kind = o.depth_kind;
    d.depth_field = o.depth_field;
    d.radiance_field = o.radiance_field;
    if (o.radiance_field < 0 || o.radiance_field >= n_fields)
      return fail(NEDF_ERR_INVALID, "radiance field index out of range");
    const NedfField& rf = fields[o.radiance_field];
    d.sigma_default = rf.kind == NEDF_FIELD_VOXEL ? 1.0 : 25.0;
    d.group = -1;
    if (o.depth_kind == NEDF_DEPTH_NEDF) {
      if (o.model == nullptr) return fail(NEDF_ERR_INVALID, "NeDF object without a model");
      int g = -1;
      for (size_t k = 0; k < sc.group_models.size(); ++k)
        if (sc.group_models[k] == o.model) g = (int)k;
      if (g < 0) {
        g = (int)sc.group_models.size();
        sc.group_models.push_back(o.model);
        sc.objs_per_group.push_back(0);
      }
      sc.objs_per_group[g] += 1;
      d.group = g;
      {   // world bounding sphere of the relaxed box: v_world = s R v_local + T
        const DevModel& hm = o.model->host;
        double cl[3], r2 = 0;
        for (int a = 0; a < 3; ++a) {
          cl[a] = 0.5 * (hm.bmin[a] + hm.bmax[a]);
          const double h = 0.5 * (hm.bmax[a] - hm.bmin[a]);
          r2 += h * h;
        }
        for (int i = 0; i < 3; ++i)
          d.bs_c[i] = (float)(o.T[i] + o.s * (o.R[3 * i] * cl[0] + o.R[3 * i + 1] * cl[1] + o.R[3 * i + 2] * cl[2]));
        d.bs_r = (float)(o.s * std::sqrt(r2));
        for (int i = 0; i < 9; ++i) d.Rf[i] = (float)o.R[i];
        for (int i = 0; i < 3; ++i) {
          d.Tf[i] = (float)o.T[i];
          d.bminf[i] = (float)hm.bmin[i];
          d.bmaxf[i] = (float)hm.bmax[i];
        }
        d.inv_sf = (float)(1.0 / o.s);
        // s * mu_max, mu_max = decode_mu(N_c - 1, N_f - 1) (model.py:89-92), rounded up
        const double mu_max = 2.0 * hm.l * ((double)(hm.n_coarse - 1) / hm.n_coarse) +
                              (2.0 * hm.l / hm.n_coarse) * ((double)(hm.n_fine - 1) / hm.n_fine) - hm.l;
        d.smu_f = std::nextafter((float)(o.s * mu_max), INFINITY);
      }
      if (!o.model->host.tensor_ok) sc.all_tc = false;
    } else if (o.depth_kind == NEDF_DEPTH_ANALYTIC) {
      if (o.depth_field < 0 || o.depth_field >= n_fields)
        return fail(NEDF_ERR_INVALID, "depth field index out of range");
    } else {
      return fail(NEDF_ERR_UNSUPPORTED, "unsupported depth backend");
    }
  }
  if (sc.group_models.size() > 64) return fail(NEDF_ERR_UNSUPPORTED, "at most 64 distinct models per frame");
  // device tables
  std::vector<DevModel> gm(std::max<size_t>(sc.group_models.size(), 1));
  for (size_t g = 0; g < sc.group_models.size(); ++g) gm[g] = sc.group_models[g]->host;
  CUDA_TRY(ctx->models.ensure(gm.size() * sizeof(DevModel)));
  CUDA_TRY(h2d_async(ctx, ctx->models.ptr, gm.data(), gm.size() * sizeof(DevModel), st));
  CUDA_TRY(ctx->objs.ensure(sc.objs.size() * sizeof(DevObj)));   // uploaded by prepare_frame
  if (n_fields > 0) {
    CUDA_TRY(ctx->fields.ensure(n_fields * sizeof(NedfField)));
    CUDA_TRY(h2d_async(ctx, ctx->fields.ptr, fields, n_fields * sizeof(NedfField), st));
  }
  return NEDF_OK;
}

// field bounding boxes for resample bounds (fields.py:77-186)
void field_bounds(const NedfField* f, int root, double lo[3], double hi[3]) {
  const NedfField& n = f[root];
  switch (n.kind) {
    case NEDF_FIELD_SPHERE:
      for (int a = 0; a < 3; ++a) { lo[a] = n.p[a] - n.p[3]; hi[a] = n.p[a] + n.p[3]; }
      return;
    case NEDF_FIELD_BOX:
      for (int a = 0; a < 3; ++a) { lo[a] = n.p[a] - n.p[3 + a]; hi[a] = n.p[a] + n.p[3 + a]; }
      return;
    case NEDF_FIELD_TORUS: {
      double e[3] = {n.p[3] + n.p[4], n.p[4], n.p[3] + n.p[4]};
      for (int a = 0; a < 3; ++a) { lo[a] = n.p[a] - e[a]; hi[a] = n.p[a] + e[a]; }
      return;
    }
    case NEDF_FIELD_VOXEL:
      for (int a = 0; a < 3; ++a) { lo[a] = n.p[a]; hi[a] = n.p[3 + a]; }
      return;
    case NEDF_FIELD_UNION: {
      for (int a = 0; a < 3; ++a) { lo[a] = INFINITY; hi[a] = -INFINITY; }
      for (int k = 0; k < n.count; ++k) {
        double l2[3], h2[3];
        field_bounds(f, n.child + k, l2, h2);
        for (int a = 0; a < 3; ++a) { lo[a] = std::min(lo[a], l2[a]); hi[a] = std::max(hi[a], h2[a]); }
      }
      return;
    }
    case NEDF_FIELD_TRANSFORMED: {
      double l2[3], h2[3];
      field_bounds(f, n.child, l2, h2);
      const double* R = n.p; const double* T = n.p + 9; double s = n.p[12];
      for (int a = 0; a < 3; ++a) { lo[a] = INFINITY; hi[a] = -INFINITY; }
      for (int c = 0; c < 8; ++c) {
        double q[3] = {(c & 4) ? h2[0] : l2[0], (c & 2) ? h2[1] : l2[1], (c & 1) ? h2[2] : l2[2]};
        for (int a = 0; a < 3; ++a) {
          double v = s * (R[3 * a] * q[0] + R[3 * a + 1] * q[1] + R[3 * a + 2] * q[2]) + T[a];
          lo[a] = std::min(lo[a], v); hi[a] = std::max(hi[a], v);
        }
      }
      return;
    }
    default:
      for (int a = 0; a < 3; ++a) { lo[a] = -INFINITY; hi[a] = INFINITY; }
  }
}

DevCam make_cam(const NedfCamera* c) {
  DevCam d;
  for (int i = 0; i < 3; ++i) d.pos[i] = c->position[i];
  for (int i = 0; i < 9; ++i) d.rot[i] = c->orientation[i];
  d.tan_half = std::tan(c->fov_y / 2.0);
  d.aspect = (double)c->width / (double)c->height;
  d.width = c->width;
  d.height = c->height;
  return d;
}

int check_camera(const NedfCamera* c) {
  if (!c) return fail(NEDF_ERR_INVALID, "camera is NULL");
  if (!(c->fov_y > 0.0 && c->fov_y < M_PI)) return fail(NEDF_ERR_INVALID, "vertical field of view must be in (0, pi)");
  if (c->width < 1 || c->height < 1) return fail(NEDF_ERR_INVALID, "image size must be at least 1x1");
  return NEDF_OK;
}

// Per-frame context: tables + lists for n_pix pixels.
struct Frame {
  Scene sc;
  FrameJob fj;
  GroupTable gt;
  ListSet ls, redo;
  int64_t n_pix = 0;
};

int prepare_frame(NedfContext* ctx, const NedfCamera* cam, const NedfObject* objs, int n_objs,
                  const NedfField* fields, int n_fields, NedfFrameBuffers* fb, Frame& F, cudaStream_t st,
                  const int32_t* recompute_idx = nullptr, int n_recompute = -1) {
  int rc = check_camera(cam);
  if (rc) return rc;
  if (!fb) return fail(NEDF_ERR_INVALID, "frame buffers are NULL");
  CUDA_TRY(cudaSetDevice(ctx->device));
  rc = build_scene(ctx, objs, n_objs, fields, n_fields, F.sc, st);
  if (rc) return rc;
  for (int s = 0; s < n_objs; ++s) {
    double lo[3], hi[3];
    field_bounds(fields, objs[s].radiance_field, lo, hi);
    for (int a = 0; a < 3; ++a) { F.sc.objs[s].rbox_min[a] = lo[a]; F.sc.objs[s].rbox_max[a] = hi[a]; }
    F.sc.objs[s].recompute = recompute_idx ? 0 : 1;
  }
  if (recompute_idx) {
    for (int k = 0; k < n_recompute; ++k) {
      if (recompute_idx[k] < 0 || recompute_idx[k] >= n_objs) return fail(NEDF_ERR_INVALID, "recompute index out of range");
      F.sc.objs[recompute_idx[k]].recompute = 1;
    }
  }
  if (n_objs > 0)
    CUDA_TRY(h2d_async(ctx, ctx->objs.ptr, F.sc.objs.data(), n_objs * sizeof(DevObj), st));
  // rows
  std::vector<int> rows;
  if (fb->rows_host) {
    if (fb->n_rows < 0) return fail(NEDF_ERR_INVALID, "n_rows must be >= 0");
    rows.assign(fb->rows_host, fb->rows_host + fb->n_rows);
    for (int r : rows)
      if (r < 0 || r >= cam->height) return fail(NEDF_ERR_INVALID, "row index out of range");
  } else {
    rows.resize(cam->height);
    for (int r = 0; r < cam->height; ++r) rows[r] = r;
  }
  int n_rows = (int)rows.size();
  F.n_pix = (int64_t)n_rows * cam->width;
  if (F.n_pix > 0xFFFFFFFFll) return fail(NEDF_ERR_INVALID, "frame too large");
  CUDA_TRY(ctx->rows.ensure(std::max<size_t>(rows.size(), 1) * sizeof(int)));
  if (n_rows) CUDA_TRY(h2d_async(ctx, ctx->rows.ptr, rows.data(), rows.size() * sizeof(int), st));
  // lists: per group capacity = n_pix * objects of that group
  int ng = (int)F.sc.group_models.size();
  std::vector<int64_t> off(std::max(ng, 1), 0);
  int64_t cap = 0;
  for (int g = 0; g < ng; ++g) { off[g] = cap; cap += F.n_pix * F.sc.objs_per_group[g]; }
  CUDA_TRY(ctx->offsets.ensure(off.size() * sizeof(int64_t)));
  CUDA_TRY(h2d_async(ctx, ctx->offsets.ptr, off.data(), off.size() * sizeof(int64_t), st));
  CUDA_TRY(ctx->counts.ensure(64 * sizeof(int)));
  CUDA_TRY(ctx->redo_counts.ensure(64 * sizeof(int)));
  CUDA_TRY(ctx->lists_pix.ensure(std::max<int64_t>(cap, 1) * sizeof(uint32_t)));
  CUDA_TRY(ctx->lists_obj.ensure(std::max<int64_t>(cap, 1) * sizeof(uint32_t)));
  CUDA_TRY(ctx->redo_pix.ensure(std::max<int64_t>(cap, 1) * sizeof(uint32_t)));
  CUDA_TRY(ctx->redo_obj.ensure(std::max<int64_t>(cap, 1) * sizeof(uint32_t)));
  CUDA_TRY(ctx->key.ensure(std::max<int64_t>(F.n_pix, 1) * sizeof(unsigned long long)));
  CUDA_TRY(ctx->skey.ensure(std::max<int64_t>(F.n_pix, 1) * sizeof(unsigned long long)));
  CUDA_TRY(ctx->stats.ensure(8 * sizeof(unsigned long long)));
  CUDA_TRY(ctx->tile_counter.ensure(64 * sizeof(int)));
  CUDA_TRY(ctx->defer_count.ensure(sizeof(int)));

  F.gt.models = ctx->models.as<DevModel>();
  F.gt.n_groups = ng;
  F.ls.pix = ctx->lists_pix.as<uint32_t>();
  F.ls.obj = ctx->lists_obj.as<uint32_t>();
  F.ls.count = ctx->counts.as<int>();
  F.ls.offset = ctx->offsets.as<int64_t>();
  F.ls.n_groups = ng;
  F.redo = F.ls;
  F.redo.pix = ctx->redo_pix.as<uint32_t>();
  F.redo.obj = ctx->redo_obj.as<uint32_t>();
  F.redo.count = ctx->redo_counts.as<int>();

  FrameJob& fj = F.fj;
  memset(&fj, 0, sizeof(fj));
  fj.ray.mode = RAY_PRIMARY;
  fj.ray.cam = make_cam(cam);
  fj.ray.rows = ctx->rows.as<int>();
  fj.ray.objs = ctx->objs.as<DevObj>();
  fj.fields = ctx->fields.as<NedfField>();
  fj.n_objs = n_objs;
  fj.n_pix = (int)F.n_pix;
  fj.key = ctx->key.as<unsigned long long>();
  fj.depth = fb->depth_dev;
  fj.id = fb->id_dev;
  fj.rgb = fb->rgb_dev;
  fj.shadow = fb->shadow_dev;
  fj.image = fb->image_dev;
  fj.planes = fb->planes_dev;
  fj.stats = ctx->stats.as<unsigned long long>();
  fj.sigma_threshold = -1.0;
  return NEDF_OK;
}

__global__ void add_counts_kernel(const int* counts, const int* redo, int ng, unsigned long long* stats, int use_redo) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    unsigned long long a = 0, b = 0;
    for (int g = 0; g < ng; ++g) { a += counts[g]; if (use_redo) b += redo[g]; }
    stats[2] += a;
    stats[3] += b;
  }
}

// CUDA-event bracket around a network launch when profiling is on.
int prof_mark(NedfContext* ctx, cudaStream_t st, int kind, bool start) {
  if (!ctx->profile) return NEDF_OK;
  if (ctx->ev_used + 1 > ctx->ev_pool.size()) {
    cudaEvent_t e;
    CUDA_TRY(cudaEventCreate(&e));
    ctx->ev_pool.push_back(e);
  }
  int idx = (int)ctx->ev_used++;
  if (start) ctx->ev_pairs.push_back({idx, kind});
  CUDA_TRY(cudaEventRecord(ctx->ev_pool[idx], st));
  return NEDF_OK;
}

#define LAUNCH(ctx, expr)       \
  do {                          \
    CUDA_TRY(expr);             \
    (ctx)->launches += 1;       \
  } while (0)

// Evaluate the network on every list entry with the context's precision.
// two_pass: F.fj.defer holds STEP 1's deferred pairs (front-first culling) -- the
// network runs on the front pairs, then on the deferred ones that can still win.
int run_network(NedfContext* ctx, Frame& F, const RayJob& job, const OutSpec& out, cudaStream_t st) {
  if (F.gt.n_groups == 0) return NEDF_OK;
  const bool two_pass = job.mode == RAY_PRIMARY && F.fj.defer.pix != nullptr && out.mode == OUT_ZBUF;
  if (ctx->guard_direct) {
    if (ctx->guard_direct == NEDF_GUARD_TCGEN05) LAUNCH(ctx, launch_guard_tc(F.gt, F.ls, job, out, ctx->n_sms, st));
    else if (ctx->guard_direct == NEDF_GUARD_PRECISE) LAUNCH(ctx, launch_mlp_precise(F.gt, F.ls, job, out, ctx->n_sms, -1, st));
    else LAUNCH(ctx, launch_mlp_fp32_cluster(F.gt, F.ls, job, out, ctx->n_sms, ctx->guard_cluster ? ctx->guard_cluster : 4, st));
    return NEDF_OK;
  }
  bool use_tc = ctx->precision != NEDF_PREC_FP32 && F.sc.all_tc && tc_available();
  int rc;
  if (use_tc) {
    TcArgs a;
    a.gt = F.gt; a.ls = F.ls; a.redo = F.redo; a.job = job; a.out = out;
    a.use_guard = ctx->precision == NEDF_PREC_AUTO;
    a.shadow_cert = ctx->shadow_cert;
    a.guard = (float)(ctx->guard_ppm * 1e-6);
    a.tile_counter = ctx->tile_counter.as<int>();
    CUDA_TRY(cudaMemsetAsync(F.redo.count, 0, 64 * sizeof(int), st));
    CUDA_TRY(cudaMemsetAsync(a.tile_counter, 0, 64 * sizeof(int), st));
    int ctas = ctx->tc_ctas > 0 ? ctx->tc_ctas : ctx->n_sms;
    if ((rc = prof_mark(ctx, st, 0, true))) return rc;
    const int mc = ctx->tc_kernel == NEDF_TC_SINGLE ? 1 : ctx->tc_kernel == NEDF_TC_MCAST4 ? 4 : 2;
    LAUNCH(ctx, launch_mlp_tc(a, ctas, mc, st));
    if ((rc = prof_mark(ctx, st, 0, false))) return rc;
    if (two_pass) {
      // front-first culling: the deferred pairs that can still win, then one guard for both passes
      add_counts_kernel<<<1, 32, 0, st>>>(F.ls.count, F.redo.count, F.gt.n_groups, F.fj.stats, 0);
      ctx->launches += 1;
      CUDA_TRY(cudaMemsetAsync(F.ls.count, 0, 64 * sizeof(int), st));
      LAUNCH(ctx, launch_defer_filter(F.fj, F.ls, ctx->n_sms, st));
      CUDA_TRY(cudaMemsetAsync(a.tile_counter, 0, 64 * sizeof(int), st));
      if ((rc = prof_mark(ctx, st, 0, true))) return rc;
      LAUNCH(ctx, launch_mlp_tc(a, ctas, mc, st));
      if ((rc = prof_mark(ctx, st, 0, false))) return rc;
    }
    if (a.use_guard) {
      if ((rc = prof_mark(ctx, st, 1, true))) return rc;
      // 8-CTA clusters halve the MMA work per layer on a CTA's critical path but only ~18 fit at
      // once (vs ~33 of 4): by default they take frames with at most half a 2000 x 800 x 8-object
      // frame's (pixel, object) pairs, whose guard batch then still fits one round
      if (ctx->guard_kernel != NEDF_GUARD_MMA_SYNC && guard_tc_available()) {
        // the batch size is only known on the device: both kernels are launched and the one that
        // does not fit returns at once -- guard_tc (latency) for batches that fit its clusters in
        // one round, mlp_precise (throughput: 128-ray tiles, one CTA per SM) beyond
        const int cap = ctx->guard_kernel == NEDF_GUARD_TCGEN05 ? 1 << 30 : guard_tc_capacity(ctx->n_sms);
        LAUNCH(ctx, launch_guard_tc(F.gt, F.redo, job, out, ctx->n_sms, st, cap));
        if (ctx->guard_kernel == NEDF_GUARD_AUTO) LAUNCH(ctx, launch_mlp_precise(F.gt, F.redo, job, out, ctx->n_sms, cap, st));
      } else if (ctx->guard_kernel == NEDF_GUARD_PRECISE) {
        LAUNCH(ctx, launch_mlp_precise(F.gt, F.redo, job, out, ctx->n_sms, -1, st));
      } else {
        int cl = ctx->guard_cluster;
        if (cl == 0) cl = (int64_t)F.n_pix * F.sc.n_objs <= 6400000 ? 8 : 4;
        LAUNCH(ctx, launch_mlp_fp32_cluster(F.gt, F.redo, job, out, ctx->n_sms, cl, st));
      }
      if ((rc = prof_mark(ctx, st, 1, false))) return rc;
    }
    add_counts_kernel<<<1, 32, 0, st>>>(F.ls.count, F.redo.count, F.gt.n_groups, F.fj.stats, a.use_guard);
    ctx->launches += 1;
  } else {
    if ((rc = prof_mark(ctx, st, 0, true))) return rc;
    for (int pass = 0; pass < (two_pass ? 2 : 1); ++pass) {
      if (pass == 1) {
        add_counts_kernel<<<1, 32, 0, st>>>(F.ls.count, F.redo.count, F.gt.n_groups, F.fj.stats, 0);
        ctx->launches += 1;
        CUDA_TRY(cudaMemsetAsync(F.ls.count, 0, 64 * sizeof(int), st));
        LAUNCH(ctx, launch_defer_filter(F.fj, F.ls, ctx->n_sms, st));
        if ((rc = prof_mark(ctx, st, 0, true))) return rc;
      }
      if (F.sc.all_tc && tc_available() && out.feats == nullptr)
        LAUNCH(ctx, launch_mlp_fp32_stream(F.gt, F.ls, job, out, ctx->n_sms, 32, st));
      else
        LAUNCH(ctx, launch_mlp_fp32(F.gt, F.ls, job, out, ctx->n_sms, st));
      if ((rc = prof_mark(ctx, st, 0, false))) return rc;
    }
    add_counts_kernel<<<1, 32, 0, st>>>(F.ls.count, F.redo.count, F.gt.n_groups, F.fj.stats, 0);
    ctx->launches += 1;
  }
  CUDA_TRY(cudaGetLastError());
  return NEDF_OK;
}

// resolve = false: leave the z-keys for the fused resolve_shade_kernel
int do_step1(NedfContext* ctx, Frame& F, cudaStream_t st, bool resolve = true) {
  FrameJob& fj = F.fj;
  fj.ray.mode = RAY_PRIMARY;
  CUDA_TRY(cudaMemsetAsync(F.ls.count, 0, 64 * sizeof(int), st));
  if (F.n_pix == 0) return NEDF_OK;
  // front-first culling: worth it with two or more NeDF objects; not with a plane cache (every
  // plane is an output) or a direct guard run (diagnostics evaluate the lists as built)
  int n_nedf = 0;
  for (const DevObj& o : F.sc.objs) n_nedf += o.depth_kind == NEDF_DEPTH_NEDF ? 1 : 0;
  memset(&fj.defer, 0, sizeof(fj.defer));
  if (ctx->cull && n_nedf >= 2 && fj.planes == nullptr && !ctx->guard_direct && F.sc.n_objs <= 64 &&
      F.n_pix * (n_nedf - 1) <= INT32_MAX) {         // the deferred list is indexed by an int counter
    const int64_t cap = F.n_pix * (n_nedf - 1);
    CUDA_TRY(ctx->defer_pix.ensure(cap * sizeof(uint32_t)));
    CUDA_TRY(ctx->defer_obj.ensure(cap * sizeof(uint32_t)));
    CUDA_TRY(ctx->defer_low.ensure(cap * sizeof(float)));
    fj.defer.pix = ctx->defer_pix.as<uint32_t>();
    fj.defer.obj = ctx->defer_obj.as<uint32_t>();
    fj.defer.low = ctx->defer_low.as<float>();
    fj.defer.count = ctx->defer_count.as<int>();
    CUDA_TRY(cudaMemsetAsync(fj.defer.count, 0, sizeof(int), st));
  }
  LAUNCH(ctx, launch_setup(fj, F.gt, F.ls, RAY_PRIMARY, ctx->setup_exact, ctx->n_sms, st));
  OutSpec out;
  memset(&out, 0, sizeof(out));
  out.mode = OUT_ZBUF;
  out.key = fj.key;
  out.planes = fj.planes;
  out.plane_stride = F.n_pix;
  int rc = run_network(ctx, F, fj.ray, out, st);
  if (rc) return rc;
  if (fj.planes != nullptr) LAUNCH(ctx, launch_recombine(fj, ctx->n_sms, st));   // plane cache kept
  else if (resolve) LAUNCH(ctx, launch_step1_resolve(fj, F.gt, ctx->n_sms, st));
  return NEDF_OK;
}

void fill_config(FrameJob& fj, const NedfRenderConfig* cfg) {
  if (!cfg) {
    fj.sigma_threshold = -1.0;
    fj.resample = 0;
    fj.resample_samples = 128;
    fj.clear[0] = fj.clear[1] = fj.clear[2] = 0.0;
    return;
  }
  fj.sigma_threshold = cfg->sigma_threshold;
  fj.resample = cfg->resample;
  fj.resample_samples = cfg->resample_samples > 0 ? cfg->resample_samples : 128;
  for (int a = 0; a < 3; ++a) fj.clear[a] = cfg->clear_color[a];
}

int do_step2(NedfContext* ctx, Frame& F, const NedfRenderConfig* cfg, cudaStream_t st) {
  fill_config(F.fj, cfg);
  F.fj.ray.mode = RAY_PRIMARY;
  if (F.n_pix == 0) return NEDF_OK;
  LAUNCH(ctx, launch_shade(F.fj, F.gt, ctx->n_sms, st));
  return NEDF_OK;
}

double default_eps(const Frame& F, const NedfObject* objs) {
  // pipeline.py:202-208: max(1e-4, 2 * s * fine_width) over NeDF objects
  double e = 1e-4;
  for (int s = 0; s < F.sc.n_objs; ++s) {
    if (objs[s].depth_kind != NEDF_DEPTH_NEDF) continue;
    const NedfModelInfo& in = objs[s].model->info;
    double fw = 2.0 * (double)in.half_range / ((double)in.n_coarse * in.n_fine);
    e = std::max(e, 2.0 * objs[s].s * fw);
  }
  return e;
}

// STEP 3 job of one light: the frame job with the light's ray mode, epsilon
// (pipeline.py:202-208 default) and beta; z-keys in the context's shadow keys.
int make_shadow_job(NedfContext* ctx, const Frame& F, const NedfObject* objs, const NedfLight* L,
                    const NedfRenderConfig* cfg, FrameJob& sj, int& mode) {
  if (!L) return fail(NEDF_ERR_INVALID, "light is NULL");
  if (!(L->beta > 0.0 && L->beta < 1.0)) return fail(NEDF_ERR_INVALID, "shadow intensity beta must be in (0, 1)");
  if (L->kind == NEDF_LIGHT_POINT) mode = RAY_POINT_SHADOW;
  else if (L->kind == NEDF_LIGHT_DIRECTIONAL) mode = RAY_DIR_SHADOW;
  else return fail(NEDF_ERR_UNSUPPORTED, "unsupported light type");
  sj = F.fj;
  fill_config(sj, cfg);
  double eps = (cfg && cfg->shadow_epsilon > 0.0) ? cfg->shadow_epsilon : default_eps(F, objs);
  sj.eps = eps;
  sj.beta = L->beta;
  sj.ray.mode = mode;
  sj.ray.eps = eps;
  sj.ray.depth64 = F.fj.depth;
  for (int a = 0; a < 3; ++a) sj.ray.light[a] = L->vec[a];
  sj.planes = nullptr;
  memset(&sj.defer, 0, sizeof(sj.defer));
  sj.key = ctx->skey.as<unsigned long long>();
  return NEDF_OK;
}

// STEP 3 for one light.  lists_ready: the light's work lists and z-keys were
// built by resolve_shade_kernel.  image != NULL: the resolve also composites.
int do_step3(NedfContext* ctx, Frame& F, const NedfObject* objs, const NedfLight* L, const NedfRenderConfig* cfg,
             cudaStream_t st, float* image = nullptr, bool lists_ready = false) {
  FrameJob sj;
  int mode = 0;
  int rc = make_shadow_job(ctx, F, objs, L, cfg, sj, mode);
  if (rc) return rc;
  if (!lists_ready) {
    CUDA_TRY(cudaMemsetAsync(F.ls.count, 0, 64 * sizeof(int), st));
    if (F.n_pix == 0) return NEDF_OK;
    LAUNCH(ctx, launch_setup(sj, F.gt, F.ls, mode, ctx->setup_exact, ctx->n_sms, st));
  }
  if (F.n_pix == 0) return NEDF_OK;
  OutSpec out;
  memset(&out, 0, sizeof(out));
  out.mode = OUT_ZBUF;
  out.key = sj.key;
  rc = run_network(ctx, F, sj.ray, out, st);
  if (rc) return rc;
  LAUNCH(ctx, launch_shadow_resolve(sj, F.gt, mode, image, ctx->n_sms, st));
  return NEDF_OK;
}

int record(void* const* events, int i, cudaStream_t st) {
  if (events && events[i]) CUDA_TRY(cudaEventRecord((cudaEvent_t)events[i], st));
  return NEDF_OK;
}

// compose_frame (pipeline.py:430-468) on the device.  Fused (ctx->fuse, no plane
// cache): setup -> network -> [resolve + shade + shadow fill + light 0 setup] ->
// per light: network -> resolve (+ composite for the last light).
int render_frame(NedfContext* ctx, const NedfCamera* cam, const NedfObject* objs, int n_objs,
                 const NedfField* fields, int n_fields, const NedfLight* lights, int n_lights,
                 const NedfRenderConfig* cfg, NedfFrameBuffers* fb, void* const* events, cudaStream_t st) {
  if (!ctx) return fail(NEDF_ERR_INVALID, "context is NULL");
  if (n_lights < 0 || (n_lights > 0 && !lights)) return fail(NEDF_ERR_INVALID, "bad light list");
  Frame F;
  int rc = prepare_frame(ctx, cam, objs, n_objs, fields, n_fields, fb, F, st);
  if (rc) return rc;
  if ((rc = record(events, 0, st))) return rc;
  const bool fuse = ctx->fuse && fb->planes_dev == nullptr;
  rc = do_step1(ctx, F, st, !fuse);
  if (rc) return rc;
  if ((rc = record(events, 1, st))) return rc;
  const bool shadows = cfg ? cfg->shadows != 0 : true;
  const int nl = shadows ? n_lights : 0;
  if (fuse) {
    fill_config(F.fj, cfg);
    F.fj.ray.mode = RAY_PRIMARY;
    FrameJob sj = F.fj;
    int smode = -1;
    if (nl > 0 && (rc = make_shadow_job(ctx, F, objs, lights, cfg, sj, smode))) return rc;
    CUDA_TRY(cudaMemsetAsync(F.ls.count, 0, 64 * sizeof(int), st));
    if (F.n_pix > 0)
      LAUNCH(ctx, launch_resolve_shade(F.fj, F.gt, F.ls, sj, smode, ctx->setup_exact, ctx->n_sms, st));
    if ((rc = record(events, 2, st))) return rc;
    for (int i = 0; i < nl; ++i) {
      rc = do_step3(ctx, F, objs, lights + i, cfg, st, i == nl - 1 ? fb->image_dev : nullptr, i == 0);
      if (rc) return rc;
    }
    if (nl == 0 && fb->image_dev && F.n_pix > 0)
      LAUNCH(ctx, launch_composite(fb->rgb_dev, fb->shadow_dev, fb->image_dev, F.n_pix, ctx->n_sms, st));
  } else {
    rc = do_step2(ctx, F, cfg, st);
    if (rc) return rc;
    if ((rc = record(events, 2, st))) return rc;
    if (F.n_pix > 0) LAUNCH(ctx, launch_fill(fb->shadow_dev, F.n_pix, 1.0f, ctx->n_sms, st));
    for (int i = 0; i < nl; ++i) {
      rc = do_step3(ctx, F, objs, lights + i, cfg, st);
      if (rc) return rc;
    }
    if (fb->image_dev && F.n_pix > 0)
      LAUNCH(ctx, launch_composite(fb->rgb_dev, fb->shadow_dev, fb->image_dev, F.n_pix, ctx->n_sms, st));
  }
  return record(events, 3, st);
}

}  // namespace

// ===========================================================================
// exported C ABI
// ===========================================================================
extern "C" {

int nedf_abi_version(void) { return NEDF_ABI_VERSION; }

const char* nedf_last_error(void) { return g_err.c_str(); }

int nedf_context_create(int device, NedfContext** out) {
  if (!out) return fail(NEDF_ERR_INVALID, "out is NULL");
  int n = 0;
  CUDA_TRY(cudaGetDeviceCount(&n));
  if (device < 0 || device >= n) return fail(NEDF_ERR_INVALID, "no such CUDA device");
  CUDA_TRY(cudaSetDevice(device));
  cudaDeviceProp prop;
  CUDA_TRY(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10) return fail(NEDF_ERR_UNSUPPORTED, "this build targets sm_100a (B200)");
  NedfContext* c = new NedfContext();
  c->device = device;
  c->n_sms = prop.multiProcessorCount;
  // slot kStatSlots: nedf_read_stats; slots [0, kStatSlots): nedf_stats_snapshot
  if (cudaHostAlloc(&c->stats_host, 8 * (kStatSlots + 1) * sizeof(unsigned long long), cudaHostAllocMapped) !=
          cudaSuccess ||
      cudaHostGetDevicePointer(&c->stats_host_dev, c->stats_host, 0) != cudaSuccess) {
    if (c->stats_host) cudaFreeHost(c->stats_host);
    delete c;
    return fail(NEDF_ERR_CUDA, "mapped host allocation failed");
  }
  *out = c;
  return NEDF_OK;
}

void nedf_context_destroy(NedfContext* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  DevBuf* bufs[] = {&c->models, &c->objs, &c->fields, &c->rows, &c->offsets, &c->counts, &c->redo_counts,
                    &c->lists_pix, &c->lists_obj, &c->redo_pix, &c->redo_obj, &c->key, &c->skey, &c->stats,
                    &c->tile_counter, &c->defer_pix, &c->defer_obj, &c->defer_low, &c->defer_count};
  for (DevBuf* b : bufs) b->release();
  if (c->stats_host) cudaFreeHost(c->stats_host);
  delete c;
}

int nedf_set_option(NedfContext* c, int key, int64_t v) {
  if (!c) return fail(NEDF_ERR_INVALID, "context is NULL");
  switch (key) {
    case NEDF_OPT_PRECISION:
      if (v < NEDF_PREC_AUTO || v > NEDF_PREC_FP32) return fail(NEDF_ERR_INVALID, "bad precision");
      c->precision = (int)v;
      return NEDF_OK;
    case NEDF_OPT_GUARD_PPM:
      if (v < 0 || v > 1000000) return fail(NEDF_ERR_INVALID, "bad guard");
      c->guard_ppm = (int)v;
      return NEDF_OK;
    case NEDF_OPT_TC_CTAS:
      if (v < 0) return fail(NEDF_ERR_INVALID, "bad CTA count");
      c->tc_ctas = (int)v;
      return NEDF_OK;
    case NEDF_OPT_PROFILE:
      c->profile = v != 0;
      return NEDF_OK;
    case NEDF_OPT_TC_KERNEL:
      if (v < NEDF_TC_AUTO || v > NEDF_TC_MCAST4 || v == 2) return fail(NEDF_ERR_INVALID, "bad tensor-core kernel");
      c->tc_kernel = (int)v;
      return NEDF_OK;
    case NEDF_OPT_GUARD_CLUSTER:
      if (v != 0 && v != 4 && v != 8) return fail(NEDF_ERR_INVALID, "guard cluster size must be 0, 4 or 8");
      c->guard_cluster = (int)v;
      return NEDF_OK;
    case NEDF_OPT_SETUP_EXACT:
      c->setup_exact = v != 0;
      return NEDF_OK;
    case NEDF_OPT_GUARD_KERNEL:
      if (v != NEDF_GUARD_AUTO && v != NEDF_GUARD_TCGEN05 && v != NEDF_GUARD_MMA_SYNC && v != NEDF_GUARD_PRECISE)
        return fail(NEDF_ERR_INVALID, "bad guard kernel");
      c->guard_kernel = (int)v;
      return NEDF_OK;
    case NEDF_OPT_FUSE:
      c->fuse = v != 0;
      return NEDF_OK;
    case NEDF_OPT_CULL:
      c->cull = v != 0;
      return NEDF_OK;
    case NEDF_OPT_SHADOW_CERT:
      c->shadow_cert = v != 0;
      return NEDF_OK;
  }
  return fail(NEDF_ERR_INVALID, "unknown option");
}

int nedf_get_option(NedfContext* c, int key, int64_t* v) {
  if (!c || !v) return fail(NEDF_ERR_INVALID, "NULL argument");
  switch (key) {
    case NEDF_OPT_PRECISION: *v = c->precision; return NEDF_OK;
    case NEDF_OPT_GUARD_PPM: *v = c->guard_ppm; return NEDF_OK;
    case NEDF_OPT_TC_CTAS: *v = c->tc_ctas; return NEDF_OK;
    case NEDF_OPT_PROFILE: *v = c->profile; return NEDF_OK;
    case NEDF_OPT_TC_KERNEL: *v = c->tc_kernel; return NEDF_OK;
    case NEDF_OPT_GUARD_CLUSTER: *v = c->guard_cluster; return NEDF_OK;
    case NEDF_OPT_SETUP_EXACT: *v = c->setup_exact; return NEDF_OK;
    case NEDF_OPT_GUARD_KERNEL: *v = c->guard_kernel; return NEDF_OK;
    case NEDF_OPT_FUSE: *v = c->fuse; return NEDF_OK;
    case NEDF_OPT_CULL: *v = c->cull; return NEDF_OK;
    case NEDF_OPT_SHADOW_CERT: *v = c->shadow_cert; return NEDF_OK;
  }
  return fail(NEDF_ERR_INVALID, "unknown option");
}

int nedf_stats_snapshot(NedfContext* c, int slot, NedfStepStats* out, void* stream) {
  if (!c || !out) return fail(NEDF_ERR_INVALID, "NULL argument");
  if (slot < 0 || slot >= kStatSlots) return fail(NEDF_ERR_INVALID, "stats slot out of range");
  memset(out, 0, sizeof(*out));
  CUDA_TRY(cudaSetDevice(c->device));
  if (c->stats.ptr) {
    CUDA_TRY(launch_stats_export(c->stats.as<unsigned long long>(), c->stats_host_dev + 8 * slot,
                                 (cudaStream_t)stream));
  } else {
    for (int i = 0; i < 8; ++i) c->stats_host[8 * slot + i] = 0;
  }
  out->launches = c->launches;
  c->launches = 0;
  out->h2d_bytes = c->h2d_bytes;
  c->h2d_bytes = 0;
  return NEDF_OK;
}

int nedf_stats_slot(NedfContext* c, int slot, NedfStepStats* out) {
  if (!c || !out) return fail(NEDF_ERR_INVALID, "NULL argument");
  if (slot < 0 || slot >= kStatSlots) return fail(NEDF_ERR_INVALID, "stats slot out of range");
  const volatile unsigned long long* h = c->stats_host + 8 * slot;
  out->covered = (int64_t)h[0];
  out->resampled = (int64_t)h[1];
  out->evals = (int64_t)h[2];
  out->guarded = (int64_t)h[3];
  out->exact_clips = (int64_t)h[4];
  out->culled = (int64_t)h[5];
  return NEDF_OK;
}

int nedf_read_stats(NedfContext* c, NedfStepStats* out, void* stream) {
  if (!c || !out) return fail(NEDF_ERR_INVALID, "NULL argument");
  unsigned long long h[8] = {0};
  CUDA_TRY(cudaSetDevice(c->device));
  if (c->stats.ptr) {
    cudaStream_t st = (cudaStream_t)stream;
    CUDA_TRY(launch_stats_export(c->stats.as<unsigned long long>(), c->stats_host_dev + 8 * kStatSlots, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    for (int i = 0; i < 8; ++i)
      h[i] = reinterpret_cast<volatile unsigned long long*>(c->stats_host)[8 * kStatSlots + i];
  }
  out->covered = (int64_t)h[0];
  out->resampled = (int64_t)h[1];
  out->evals = (int64_t)h[2];
  out->guarded = (int64_t)h[3];
  out->exact_clips = (int64_t)h[4];
  out->culled = (int64_t)h[5];
  out->launches = c->launches;
  c->launches = 0;
  out->h2d_bytes = c->h2d_bytes;
  c->h2d_bytes = 0;
  out->net_launches = 0;
  out->net_ms = 0.0;
  out->guard_ms = 0.0;
  if (!c->ev_pairs.empty()) {
    CUDA_TRY(cudaStreamSynchronize((cudaStream_t)stream));
    for (auto& pr : c->ev_pairs) {
      float ms = 0.f;
      CUDA_TRY(cudaEventElapsedTime(&ms, c->ev_pool[pr.first], c->ev_pool[pr.first + 1]));
      if (pr.second == 0) { out->net_ms += ms; out->net_launches += 1; }
      else out->guard_ms += ms;
    }
  }
  c->ev_pairs.clear();
  c->ev_used = 0;
  return NEDF_OK;
}

// Logit z* at which the reference's alpha decision sigmoid(z) > thr (nn.py:169-175,
// model.py:292, float64) changes; the tensor-core kernel re-evaluates rays whose
// alpha logit lies within the fp16 error of z*.  thr = 0: sigmoid(z) is exactly 0 only
// once exp(z) underflows (z < -745.13); thr < 0, thr >= 1 or NaN: the decision is the
// same for every finite z, so there is nothing to guard (+inf never passes the test).
static float alpha_boundary_logit(double thr) {
  if (!(thr > 0.0)) return thr == 0.0 ? -745.1332f : INFINITY;
  if (thr >= 1.0) return INFINITY;
  return (float)(log(thr) - log1p(-thr));
}

int nedf_model_create(NedfContext* ctx, const NedfModelInfo* info, const float* params, size_t n_params,
                      NedfModel** out) {
  if (!ctx || !info || !params || !out) return fail(NEDF_ERR_INVALID, "NULL argument");
  int rc = validate_dims(*info);
  if (rc) return rc;
  if (n_params != param_count(*info)) return fail(NEDF_ERR_FORMAT, "parameter count does not match dimensions");
  CUDA_TRY(cudaSetDevice(ctx->device));
  const int F = info->d_feat, nl = layer_count(info->n_blocks);
  // fp32 transposed copies: WT[k][o] = W[o][k]; head padded to 1024 input rows
  std::vector<int> n_in(nl), n_out(nl);
  n_in[0] = info->d_in; n_out[0] = F;
  for (int l = 1; l < nl - 2; ++l) { n_in[l] = F; n_out[l] = F; }
  n_in[nl - 2] = F; n_out[nl - 2] = info->n_coarse + 1;
  n_in[nl - 1] = F; n_out[nl - 1] = info->n_fine;
  std::vector<int64_t> wt_off(nl), b_off(nl);
  int64_t wt_total = 0, b_total = 0;
  for (int l = 0; l < nl; ++l) {
    wt_off[l] = wt_total;
    int rows = l == 0 ? 1024 : n_in[l];
    wt_total += (int64_t)rows * n_out[l];
    b_off[l] = b_total;
    b_total += n_out[l];
  }
  std::vector<float> wT(wt_total, 0.f), bias(b_total, 0.f);
  size_t p = 0;
  for (int l = 0; l < nl; ++l) {
    for (int o = 0; o < n_out[l]; ++o)
      for (int k = 0; k < n_in[l]; ++k) wT[wt_off[l] + (int64_t)k * n_out[l] + o] = params[p++];
    for (int o = 0; o < n_out[l]; ++o) bias[b_off[l] + o] = params[p++];
  }
  NedfModel* m = new NedfModel();
  m->info = *info;
  m->device = ctx->device;
  DevModel& h = m->host;
  memset(&h, 0, sizeof(h));
  h.d_in = info->d_in; h.d_feat = F; h.n_blocks = info->n_blocks;
  h.n_coarse = info->n_coarse; h.n_fine = info->n_fine;
  h.l = (double)info->half_range;
  for (int a = 0; a < 3; ++a) {
    h.bmin[a] = (double)info->box_min[a];
    h.bmax[a] = (double)info->box_max[a];
    h.c[a] = 0.5 * (h.bmin[a] + h.bmax[a]);
    double hh = 0.5 * (h.bmax[a] - h.bmin[a]);
    h.h[a] = hh > 0.0 ? hh : 1.0;
  }
  h.alpha_threshold = (double)info->alpha_threshold;
  h.alpha_zthr = alpha_boundary_logit(h.alpha_threshold);
  h.n_layers = nl;
  for (int l = 0; l < nl; ++l) { h.wT_off[l] = wt_off[l]; h.b_off[l] = b_off[l]; }
  auto cleanup = [&]() {
    if (m->wT) cudaFree(m->wT);
    if (m->bias) cudaFree(m->bias);
    if (m->wpack) cudaFree(m->wpack);
    if (m->wpack_lo) cudaFree(m->wpack_lo);
    if (m->bias_pack) cudaFree(m->bias_pack);
    if (m->wstream) cudaFree(m->wstream);
    if (m->wcluster) cudaFree(m->wcluster);
    if (m->wcluster8) cudaFree(m->wcluster8);
    if (m->wguard) cudaFree(m->wguard);
    if (m->dev) cudaFree(m->dev);
    delete m;
  };
  cudaError_t e = cudaMalloc(&m->wT, wT.size() * sizeof(float));
  if (e == cudaSuccess) e = cudaMalloc(&m->bias, bias.size() * sizeof(float));
  if (e == cudaSuccess) e = cudaMemcpy(m->wT, wT.data(), wT.size() * sizeof(float), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(m->bias, bias.data(), bias.size() * sizeof(float), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) { cleanup(); return fail(NEDF_ERR_CUDA, std::string("weight upload: ") + cudaGetErrorString(e)); }
  h.wT = m->wT;
  h.bias = m->bias;
  // tensor-core operand image (paper-shaped models)
  h.tensor_ok = 0;
  // exactly the paper profile (nn.py:59-112 with PROFILES["paper"], model.py:35): the packers
  // below lay out 16 head points x 63 features, 32 body layers of 256 and a 128 + 65 tail;
  // any other shape runs on the fp32 path (mlp_simt.cu)
  if (tc_available() && F == 256 && info->d_in == kDin && info->n_blocks == 16 && info->n_coarse == 64 &&
      info->n_fine == 128) {
    size_t bytes = 0;
    e = tc_pack_weights(params, info->d_in, F, info->n_blocks, info->n_coarse, info->n_fine, &m->wpack,
                        &m->bias_pack, &bytes);
    if (e != cudaSuccess) { cleanup(); return fail(NEDF_ERR_CUDA, std::string("tc pack: ") + cudaGetErrorString(e)); }
    h.wpack = m->wpack;
    h.bias_pack = m->bias_pack;
    e = tc_pack_weights(params, info->d_in, F, info->n_blocks, info->n_coarse, info->n_fine, &m->wpack_lo, nullptr,
                        &bytes, 1);
    if (e != cudaSuccess) { cleanup(); return fail(NEDF_ERR_CUDA, std::string("tc pack (lo): ") + cudaGetErrorString(e)); }
    h.wpack_lo = m->wpack_lo;
    e = fp32_pack_stream(params, info->d_in, F, info->n_blocks, info->n_coarse, info->n_fine, &m->wstream);
    if (e != cudaSuccess) { cleanup(); return fail(NEDF_ERR_CUDA, std::string("fp32 pack: ") + cudaGetErrorString(e)); }
    h.wstream = m->wstream;
    e = fp32_pack_cluster(params, info->d_in, F, info->n_blocks, info->n_coarse, info->n_fine, 4, &m->wcluster);
    if (e == cudaSuccess)
      e = fp32_pack_cluster(params, info->d_in, F, info->n_blocks, info->n_coarse, info->n_fine, 8, &m->wcluster8);
    if (e != cudaSuccess) { cleanup(); return fail(NEDF_ERR_CUDA, std::string("fp32 pack: ") + cudaGetErrorString(e)); }
    h.wcluster = m->wcluster;
    h.wcluster8 = m->wcluster8;
    e = guard_tc_pack(params, info->d_in, F, info->n_blocks, info->n_coarse, info->n_fine, &m->wguard);
    if (e != cudaSuccess) { cleanup(); return fail(NEDF_ERR_CUDA, std::string("guard pack: ") + cudaGetErrorString(e)); }
    h.wguard = m->wguard;
    h.tensor_ok = 1;
  }
  e = cudaMalloc(&m->dev, sizeof(DevModel));
  if (e == cudaSuccess) e = cudaMemcpy(m->dev, &h, sizeof(DevModel), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) { cleanup(); return fail(NEDF_ERR_CUDA, std::string("model upload: ") + cudaGetErrorString(e)); }
  *out = m;
  return NEDF_OK;
}

int nedf_model_load(NedfContext* ctx, const void* bytes, size_t n, NedfModel** out) {
  // nn.py:249-281 + model.py:364-369
  if (!ctx || !bytes || !out) return fail(NEDF_ERR_INVALID, "NULL argument");
  const unsigned char* raw = (const unsigned char*)bytes;
  if (n < 4 || memcmp(raw, "NEDM", 4) != 0) return fail(NEDF_ERR_FORMAT, "not a model file");
  if (n < 32) return fail(NEDF_ERR_FORMAT, "truncated header");
  uint32_t hdr[6];
  memcpy(hdr, raw + 4, sizeof(hdr));
  if (hdr[0] != 1) return fail(NEDF_ERR_FORMAT, "unsupported version " + std::to_string(hdr[0]));
  NedfModelInfo info;
  memset(&info, 0, sizeof(info));
  info.d_in = (int)hdr[1]; info.d_feat = (int)hdr[2]; info.n_blocks = (int)hdr[3];
  info.n_coarse = (int)hdr[4]; info.n_fine = (int)hdr[5];
  memcpy(&info.half_range, raw + 28, 4);
  if (hdr[1] > (1u << 20) || hdr[2] > (1u << 16) || hdr[3] > (1u << 16) || hdr[4] > (1u << 16) || hdr[5] > (1u << 16))
    return fail(NEDF_ERR_FORMAT, "implausible dimensions");
  size_t np = param_count(info);
  if (n != 32 + 4 * np + 28)
    return fail(NEDF_ERR_FORMAT, "expected " + std::to_string(32 + 4 * np + 28) + " bytes for the declared dimensions, found " +
                                     std::to_string(n));
  float trailer[7];
  memcpy(trailer, raw + 32 + 4 * np, sizeof(trailer));
  for (int a = 0; a < 3; ++a) { info.box_min[a] = trailer[a]; info.box_max[a] = trailer[3 + a]; }
  info.alpha_threshold = trailer[6];
  std::vector<float> params(np);
  memcpy(params.data(), raw + 32, 4 * np);
  return nedf_model_create(ctx, &info, params.data(), np, out);
}

void nedf_model_free(NedfModel* m) {
  if (!m) return;
  cudaSetDevice(m->device);
  if (m->wT) cudaFree(m->wT);
  if (m->bias) cudaFree(m->bias);
  if (m->wpack) cudaFree(m->wpack);
  if (m->wpack_lo) cudaFree(m->wpack_lo);
  if (m->bias_pack) cudaFree(m->bias_pack);
  if (m->wstream) cudaFree(m->wstream);
  if (m->wcluster) cudaFree(m->wcluster);
  if (m->wcluster8) cudaFree(m->wcluster8);
  if (m->wguard) cudaFree(m->wguard);
  if (m->dev) cudaFree(m->dev);
  delete m;
}

int nedf_model_info(const NedfModel* m, NedfModelInfo* out) {
  if (!m || !out) return fail(NEDF_ERR_INVALID, "NULL argument");
  *out = m->info;
  return NEDF_OK;
}

int nedf_model_tensor_ok(const NedfModel* m) { return m && m->host.tensor_ok ? 1 : 0; }

static int single_model_frame(NedfContext* ctx, const NedfModel* m, int64_t n, Frame& F, cudaStream_t st) {
  if (!ctx || !m) return fail(NEDF_ERR_INVALID, "NULL argument");
  if (n < 0 || n > 0xFFFFFFFFll) return fail(NEDF_ERR_INVALID, "bad batch size");
  CUDA_TRY(cudaSetDevice(ctx->device));
  F.sc.group_models.assign(1, m);
  F.sc.objs_per_group.assign(1, 1);
  F.sc.all_tc = m->host.tensor_ok != 0;
  F.sc.n_objs = 1;
  CUDA_TRY(ctx->models.ensure(sizeof(DevModel)));
  CUDA_TRY(h2d_async(ctx, ctx->models.ptr, &m->host, sizeof(DevModel), st));
  int64_t off0 = 0;
  CUDA_TRY(ctx->offsets.ensure(sizeof(int64_t)));
  CUDA_TRY(h2d_async(ctx, ctx->offsets.ptr, &off0, sizeof(int64_t), st));
  CUDA_TRY(ctx->counts.ensure(64 * sizeof(int)));
  CUDA_TRY(ctx->redo_counts.ensure(64 * sizeof(int)));
  CUDA_TRY(ctx->lists_pix.ensure(std::max<int64_t>(n, 1) * 4));
  CUDA_TRY(ctx->lists_obj.ensure(std::max<int64_t>(n, 1) * 4));
  CUDA_TRY(ctx->redo_pix.ensure(std::max<int64_t>(n, 1) * 4));
  CUDA_TRY(ctx->redo_obj.ensure(std::max<int64_t>(n, 1) * 4));
  CUDA_TRY(ctx->stats.ensure(8 * sizeof(unsigned long long)));
  CUDA_TRY(ctx->tile_counter.ensure(64 * sizeof(int)));
  CUDA_TRY(cudaMemsetAsync(ctx->counts.ptr, 0, 64 * sizeof(int), st));
  F.gt.models = ctx->models.as<DevModel>();
  F.gt.n_groups = 1;
  F.ls.pix = ctx->lists_pix.as<uint32_t>();
  F.ls.obj = ctx->lists_obj.as<uint32_t>();
  F.ls.count = ctx->counts.as<int>();
  F.ls.offset = ctx->offsets.as<int64_t>();
  F.ls.n_groups = 1;
  F.redo = F.ls;
  F.redo.pix = ctx->redo_pix.as<uint32_t>();
  F.redo.obj = ctx->redo_obj.as<uint32_t>();
  F.redo.count = ctx->redo_counts.as<int>();
  memset(&F.fj, 0, sizeof(F.fj));
  F.fj.stats = ctx->stats.as<unsigned long long>();
  F.n_pix = n;
  return NEDF_OK;
}

int nedf_mlp_forward(NedfContext* ctx, const NedfModel* m, const float* feats, int64_t batch, float* lc, float* lf,
                     float* la, int precision, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (!feats || !lc || !lf || !la) return fail(NEDF_ERR_INVALID, "NULL buffer");
  if (m && m->info.d_in != kDin) return fail(NEDF_ERR_INVALID, "batch width does not match d_in");
  Frame F;
  int rc = single_model_frame(ctx, m, batch, F, st);
  if (rc) return rc;
  if (batch == 0) return NEDF_OK;
  LAUNCH(ctx, launch_iota_setup(F.ls, batch, ctx->n_sms, st));
  OutSpec out;
  memset(&out, 0, sizeof(out));
  out.mode = OUT_LOGITS;
  out.lc = lc; out.lf = lf; out.la = la; out.feats = feats;
  RayJob job;
  memset(&job, 0, sizeof(job));
  int saved = ctx->precision;
  // logits have no decode step to guard, so AUTO means fp32 here
  ctx->precision = precision == NEDF_PREC_TENSOR ? NEDF_PREC_TENSOR : NEDF_PREC_FP32;
  if (ctx->precision == NEDF_PREC_TENSOR) F.sc.all_tc = false;  // tc kernel encodes rays itself; logits mode is fp32-only
  rc = run_network(ctx, F, job, out, st);
  ctx->precision = saved;
  return rc;
}

static int query_common(NedfContext* ctx, const NedfModel* m, int mode, const double* R, const double* T, double s,
                        const double* o, const double* d, int64_t n, double* depth_or_mu, uint8_t* alpha,
                        cudaStream_t st, float* lc = nullptr, float* lf = nullptr, float* la = nullptr) {
  const bool logits = lc != nullptr;
  if (!o || !d || (!logits && (!depth_or_mu || !alpha)) || (logits && (!lf || !la)))
    return fail(NEDF_ERR_INVALID, "NULL buffer");
  Frame F;
  int rc = single_model_frame(ctx, m, n, F, st);
  if (rc) return rc;
  DevObj ob;
  memset(&ob, 0, sizeof(ob));
  if (mode == RAY_WORLD) {
    if (!(s > 0) || !std::isfinite(s)) return fail(NEDF_ERR_INVALID, "scale must be a positive real");
    for (int i = 0; i < 9; ++i) ob.R[i] = R[i];
    for (int i = 0; i < 3; ++i) ob.T[i] = T[i];
    ob.s = s;
  } else {
    for (int i = 0; i < 3; ++i) ob.R[4 * i] = 1.0;
    ob.s = 1.0;
  }
  CUDA_TRY(ctx->objs.ensure(sizeof(DevObj)));
  CUDA_TRY(h2d_async(ctx, ctx->objs.ptr, &ob, sizeof(DevObj), st));
  if (n == 0) return NEDF_OK;
  RayJob job;
  memset(&job, 0, sizeof(job));
  job.mode = mode;
  job.ex_o = o;
  job.ex_d = d;
  job.objs = ctx->objs.as<DevObj>();
  OutSpec out;
  memset(&out, 0, sizeof(out));
  out.mode = mode == RAY_WORLD ? OUT_QUERY_WORLD : OUT_QUERY_LOCAL;
  if (mode == RAY_WORLD) out.depth = depth_or_mu; else out.mu = depth_or_mu;
  out.alpha = alpha;
  if (logits) {
    out.mode = OUT_LOGITS;
    out.lc = lc; out.lf = lf; out.la = la;
  }
  LAUNCH(ctx, launch_explicit_setup(job, F.gt, F.ls, out, n, ctx->n_sms, st));
  return run_network(ctx, F, job, out, st);
}

extern "C" int nedf_diag_ray_logits(NedfContext* ctx, const NedfModel* m, const double* o, const double* d,
                                    int64_t n, float* lc, float* lf, float* la, int precision, void* stream) {
  if (!ctx || !m) return fail(NEDF_ERR_INVALID, "NULL argument");
  if (!lc) return fail(NEDF_ERR_INVALID, "NULL buffer");
  if (precision == NEDF_PREC_TENSOR && !m->host.tensor_ok) return fail(NEDF_ERR_UNSUPPORTED, "model not tensor-core shaped");
  int saved = ctx->precision;
  ctx->precision = precision == NEDF_PREC_TENSOR ? NEDF_PREC_TENSOR : NEDF_PREC_FP32;
  if (precision == 16 + NEDF_GUARD_TCGEN05 || precision == 16 + NEDF_GUARD_MMA_SYNC ||
      precision == 16 + NEDF_GUARD_PRECISE) {
    if (!m->host.tensor_ok) return fail(NEDF_ERR_UNSUPPORTED, "model not tensor-core shaped");
    ctx->guard_direct = precision - 16;
  }
  int rc = query_common(ctx, m, RAY_LOCAL, nullptr, nullptr, 1.0, o, d, n, nullptr, nullptr, (cudaStream_t)stream,
                        lc, lf, la);
  ctx->guard_direct = 0;
  ctx->precision = saved;
  return rc;
}

int nedf_query_rays(NedfContext* ctx, const NedfModel* m, const double* o, const double* d, int64_t n, double* mu,
                    uint8_t* alpha, void* stream) {
  return query_common(ctx, m, RAY_LOCAL, nullptr, nullptr, 1.0, o, d, n, mu, alpha, (cudaStream_t)stream);
}

int nedf_query_world(NedfContext* ctx, const NedfModel* m, const double R[9], const double T[3], double s,
                     const double* o, const double* d, int64_t n, double* depth, uint8_t* alpha, void* stream) {
  if (!R || !T) return fail(NEDF_ERR_INVALID, "NULL transform");
  return query_common(ctx, m, RAY_WORLD, R, T, s, o, d, n, depth, alpha, (cudaStream_t)stream);
}

int nedf_generation_step(NedfContext* ctx, const NedfCamera* cam, const NedfObject* objs, int n_objs,
                         const NedfField* fields, int n_fields, NedfFrameBuffers* fb, void* stream) {
  if (!ctx) return fail(NEDF_ERR_INVALID, "context is NULL");
  cudaStream_t st = (cudaStream_t)stream;
  Frame F;
  int rc = prepare_frame(ctx, cam, objs, n_objs, fields, n_fields, fb, F, st);
  if (rc) return rc;
  return do_step1(ctx, F, st);
}

int nedf_reuse_step(NedfContext* ctx, const NedfCamera* cam, const NedfObject* objs, int n_objs,
                    const NedfField* fields, int n_fields, const int32_t* changed_idx, int n_changed,
                    NedfFrameBuffers* fb, void* stream) {
  if (!ctx) return fail(NEDF_ERR_INVALID, "context is NULL");
  if (!fb || !fb->planes_dev) return fail(NEDF_ERR_INVALID, "reuse needs the per-object plane cache (planes_dev)");
  if (n_changed < 0 || (n_changed > 0 && !changed_idx)) return fail(NEDF_ERR_INVALID, "bad changed list");
  cudaStream_t st = (cudaStream_t)stream;
  Frame F;
  static const int32_t kNone = -1;
  int rc = prepare_frame(ctx, cam, objs, n_objs, fields, n_fields, fb, F, st, n_changed ? changed_idx : &kNone,
                         n_changed);
  if (rc) return rc;
  return do_step1(ctx, F, st);
}

int nedf_shading_step(NedfContext* ctx, const NedfCamera* cam, const NedfObject* objs, int n_objs,
                      const NedfField* fields, int n_fields, const NedfRenderConfig* cfg, NedfFrameBuffers* fb,
                      void* stream) {
  if (!ctx) return fail(NEDF_ERR_INVALID, "context is NULL");
  cudaStream_t st = (cudaStream_t)stream;
  Frame F;
  int rc = prepare_frame(ctx, cam, objs, n_objs, fields, n_fields, fb, F, st);
  if (rc) return rc;
  return do_step2(ctx, F, cfg, st);
}

int nedf_shadow_step(NedfContext* ctx, const NedfCamera* cam, const NedfObject* objs, int n_objs,
                     const NedfField* fields, int n_fields, const NedfLight* light, const NedfRenderConfig* cfg,
                     NedfFrameBuffers* fb, void* stream) {
  if (!ctx) return fail(NEDF_ERR_INVALID, "context is NULL");
  cudaStream_t st = (cudaStream_t)stream;
  Frame F;
  int rc = prepare_frame(ctx, cam, objs, n_objs, fields, n_fields, fb, F, st);
  if (rc) return rc;
  return do_step3(ctx, F, objs, light, cfg, st);
}

int nedf_composite(NedfContext* ctx, NedfFrameBuffers* fb, int width, void* stream) {
  if (!ctx || !fb) return fail(NEDF_ERR_INVALID, "NULL argument");
  int64_t n = (int64_t)fb->n_rows * width;
  if (n <= 0 || !fb->image_dev) return NEDF_OK;
  CUDA_TRY(cudaSetDevice(ctx->device));
  LAUNCH(ctx, launch_composite(fb->rgb_dev, fb->shadow_dev, fb->image_dev, n, ctx->n_sms, (cudaStream_t)stream));
  return NEDF_OK;
}

int nedf_render_frame(NedfContext* ctx, const NedfCamera* cam, const NedfObject* objs, int n_objs,
                      const NedfField* fields, int n_fields, const NedfLight* lights, int n_lights,
                      const NedfRenderConfig* cfg, NedfFrameBuffers* fb, void* stream) {
  return render_frame(ctx, cam, objs, n_objs, fields, n_fields, lights, n_lights, cfg, fb, nullptr,
                      (cudaStream_t)stream);
}

int nedf_render_frame_timed(NedfContext* ctx, const NedfCamera* cam, const NedfObject* objs, int n_objs,
                            const NedfField* fields, int n_fields, const NedfLight* lights, int n_lights,
                            const NedfRenderConfig* cfg, NedfFrameBuffers* fb, void* const* events, void* stream) {
  return render_frame(ctx, cam, objs, n_objs, fields, n_fields, lights, n_lights, cfg, fb, events,
                      (cudaStream_t)stream);
}

}  // extern "C"
