// Analytic / voxel appearance fields on the device (fields.py).
//
// Step 2 evaluates the object's radiance F_Theta once per covered pixel
// (pipeline.py:336): procedural colour clip((p+1)/2) with the SDF-derived
// density for analytic objects (fields.py:249-259), trilinear lookup for voxel
// objects (fields.py:294-319).  Sphere tracing (fields.py:194-238) backs the
// analytic depth backend (OracleDepthBackend, pipeline.py:126-136).
#pragma once

#include "common.cuh"

namespace nedf {

constexpr double kSigmaSurface = 50.0;         // fields.py:31
constexpr double kSurfaceBand = 0.02;          // fields.py:32
constexpr double kInteriorSteepness = 1000.0;  // fields.py:33
constexpr double kSurfaceEps = 1e-5;           // fields.py:25
constexpr int kMaxTraceSteps = 512;            // fields.py:26

__device__ __forceinline__ double leaf_sdf(const NedfField& f, const double p[3]) {
  switch (f.kind) {
    case NEDF_FIELD_SPHERE: {
      double a = p[0] - f.p[0], b = p[1] - f.p[1], c = p[2] - f.p[2];
      return sqrt(a * a + b * b + c * c) - f.p[3];
    }
    case NEDF_FIELD_BOX: {
      double q[3], mx = -INFINITY, o2 = 0.0;
      for (int i = 0; i < 3; ++i) {
        q[i] = fabs(p[i] - f.p[i]) - f.p[3 + i];
        mx = q[i] > mx ? q[i] : mx;
        double m = q[i] > 0.0 ? q[i] : 0.0;
        o2 += m * m;
      }
      return sqrt(o2) + (mx < 0.0 ? mx : 0.0);
    }
    case NEDF_FIELD_TORUS: {
      double x = p[0] - f.p[0], y = p[1] - f.p[1], z = p[2] - f.p[2];
      return hypot(hypot(x, z) - f.p[3], y) - f.p[4];
    }
    case NEDF_FIELD_PLANE:
      return p[0] * f.p[0] + p[1] * f.p[1] + p[2] * f.p[2] - f.p[3];
    default:
      return INFINITY;
  }
}

// Signed distance of a field tree (fields.py:57-186).  min distributes over
// positive scales, so a DFS with a running min handles unions and nested
// transforms without recursion.
__device__ inline double field_sdf(const NedfField* fields, int root, const double p0[3]) {
  const NedfField& r = fields[root];
  if (r.kind != NEDF_FIELD_UNION && r.kind != NEDF_FIELD_TRANSFORMED) {   // a single primitive: no DFS stack
    const double v = leaf_sdf(r, p0);
    return v < INFINITY ? v : INFINITY;
  }
  struct Frame { int node; double p[3]; double scale; };
  Frame st[12];
  int sp = 0;
  st[sp].node = root; st[sp].p[0] = p0[0]; st[sp].p[1] = p0[1]; st[sp].p[2] = p0[2]; st[sp].scale = 1.0; ++sp;
  double best = INFINITY;
  while (sp > 0) {
    Frame fr = st[--sp];
    const NedfField& f = fields[fr.node];
    if (f.kind == NEDF_FIELD_UNION) {
      for (int k = f.count - 1; k >= 0 && sp < 12; --k) {
        st[sp] = fr; st[sp].node = f.child + k; ++sp;
      }
    } else if (f.kind == NEDF_FIELD_TRANSFORMED) {
      // local = ((p - T) @ R) / s ; sdf = s * child(local)
      const double* R = f.p; const double* T = f.p + 9; double s = f.p[12];
      double q[3] = {fr.p[0] - T[0], fr.p[1] - T[1], fr.p[2] - T[2]};
      Frame ch;
      ch.node = f.child;
      for (int j = 0; j < 3; ++j) ch.p[j] = (q[0] * R[j] + q[1] * R[3 + j] + q[2] * R[6 + j]) / s;
      ch.scale = fr.scale * s;
      if (sp < 12) st[sp++] = ch;
    } else {
      double v = fr.scale * leaf_sdf(f, fr.p);
      best = v < best ? v : best;
    }
  }
  return best;
}

// VoxelField.sample (fields.py:294-319)
__device__ inline void voxel_sample(const NedfField& f, const double p[3], double rgb[3], double& sigma) {
  int res[3] = {f.res[0], f.res[1], f.res[2]};
  const double* bmin = f.p;
  const double* bmax = f.p + 3;
  double u[3], fr[3];
  int i0[3];
  bool inside = true;
  for (int a = 0; a < 3; ++a) {
    inside = inside && (p[a] >= bmin[a]) && (p[a] <= bmax[a]);
    double v = (p[a] - bmin[a]) / (bmax[a] - bmin[a]) * (double)res[a] - 0.5;
    double hi = (double)res[a] - 1.0;
    v = v < 0.0 ? 0.0 : (v > hi ? hi : v);
    u[a] = v;
    int k = (int)floor(v);
    k = k < 0 ? 0 : (k > res[a] - 1 ? res[a] - 1 : k);
    i0[a] = k;
    fr[a] = v - k;
  }
  sigma = 0.0;
  rgb[0] = rgb[1] = rgb[2] = 0.0;
  if (!inside) return;
  for (int corner = 0; corner < 8; ++corner) {
    int bits[3] = {(corner >> 2) & 1, (corner >> 1) & 1, corner & 1};
    int ix[3];
    double w = 1.0;
    for (int a = 0; a < 3; ++a) {
      int k = i0[a] + bits[a];
      ix[a] = k < res[a] - 1 ? k : res[a] - 1;
    }
    // weights multiply in axis order, as wx * wy * wz in the reference
    w = (bits[0] ? fr[0] : 1.0 - fr[0]) * (bits[1] ? fr[1] : 1.0 - fr[1]) * (bits[2] ? fr[2] : 1.0 - fr[2]);
    size_t lin = ((size_t)ix[0] * res[1] + ix[1]) * res[2] + ix[2];
    sigma += w * (double)f.density_dev[lin];
    for (int c = 0; c < 3; ++c) rgb[c] += w * (double)f.color_dev[3 * lin + c];
  }
}

// radiance(p, d) -> (rgb, sigma) of an appearance field (fields.py:249-259, 468-469, 502-504)
__device__ inline void field_radiance(const NedfField* fields, int root, const double p[3], double rgb[3],
                               double& sigma) {
  const NedfField& f = fields[root];
  if (f.kind == NEDF_FIELD_VOXEL) {
    voxel_sample(f, p, rgb, sigma);
    return;
  }
  double d = field_sdf(fields, root, p);
  double s = kInteriorSteepness * (-d > 0.0 ? -d : 0.0);
  if (fabs(d) < kSurfaceBand) s = s > kSigmaSurface ? s : kSigmaSurface;
  sigma = s;
  for (int a = 0; a < 3; ++a) {
    double c = (p[a] + 1.0) / 2.0;
    rgb[a] = c < 0.0 ? 0.0 : (c > 1.0 ? 1.0 : c);
  }
}

// sphere_trace_batch for one ray + secant polish (fields.py:194-238).
// Returns hit; t is the local depth.
__device__ inline bool sphere_trace(const NedfField* fields, int root, const double o[3], const double d[3],
                             double t_max, double& t_out) {
  double t = 0.0;
  if (field_sdf(fields, root, o) <= -kSurfaceEps) { t_out = 0.0; return true; }
  bool hit = false;
  for (int it = 0; it < kMaxTraceSteps; ++it) {
    double p[3] = {o[0] + t * d[0], o[1] + t * d[1], o[2] + t * d[2]};
    double dist = field_sdf(fields, root, p);
    if (fabs(dist) < kSurfaceEps) { hit = true; break; }
    t += dist;
    if (!(t <= t_max)) break;
  }
  if (!hit) { t_out = t; return false; }
  double ta = t - kSurfaceEps, tb = t + kSurfaceEps;
  double pa[3] = {o[0] + ta * d[0], o[1] + ta * d[1], o[2] + ta * d[2]};
  double pb[3] = {o[0] + tb * d[0], o[1] + tb * d[1], o[2] + tb * d[2]};
  double fa = field_sdf(fields, root, pa), fb = field_sdf(fields, root, pb);
  for (int k = 0; k < 6; ++k) {
    double den = fb - fa;
    double tn = fabs(den) > 1e-300 ? tb - fb * (tb - ta) / den : tb;
    ta = tb; fa = fb; tb = tn;
    double pn[3] = {o[0] + tb * d[0], o[1] + tb * d[1], o[2] + tb * d[2]};
    fb = field_sdf(fields, root, pn);
  }
  t_out = tb > 0.0 ? tb : 0.0;
  return true;
}

// bounding box of a field (fields.py:77-186, 270-292), for resample bounds
__device__ void field_bounds(const NedfField* fields, int root, double bmin[3], double bmax[3]);

}  // namespace nedf
