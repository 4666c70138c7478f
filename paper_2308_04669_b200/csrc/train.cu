// GPU distillation of a NeDF from an analytic oracle:
// the reference's training step (model.py:238-274, nn.py:115-232) in fp32.
//
//   batch     rays sampled on the host with the reference's RaySampler stream;
//             here: slab clip + 16-point float64 encoding (geometry.py:324-342),
//             oracle sphere tracing (fields.py:194-238), mu = |o . d| - depth and
//             the coarse / fine bin targets (model.py:74-81, 189-235)
//   forward   head, 16 residual blocks (activations cached), tails (nn.py:115-135)
//   loss      BCE_coarse + BCE_fine (rows with a hit) + 0.1 BCE_alpha (nn.py:178-196)
//   backward  exact reverse mode (nn.py:138-167)
//   update    Adam with bias correction (nn.py:218-232)
//
// The matrix products run on the tensor cores as fp32-accurate split tf32 GEMMs
// (train_gemm.cu: hi / lo operand split, three tcgen05 MMAs per k-step, so the
// gradients stay at fp32 accuracy for the parity tests); the encoding, tracing,
// targets, bias / activation epilogues, loss, column sums and the Adam update are
// the kernels below.

#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "common.cuh"
#include "encode.cuh"
#include "frame.cuh"
#include "fields.cuh"
#include "../../include/nedf_b200.h"

namespace nedf {
namespace {

constexpr int kNc = 64, kNf = 128, kNa = kNc + 1;

struct Box {                                   // relaxed sampling box (model.py:133-150)
  double bmin[3], bmax[3], c[3], h[3];
};
constexpr float kAlphaWeight = 0.1f;           // model.py:236

struct Dims {
  int F = 0, NB = 0;
  int64_t off_head_w, off_head_b, off_tail_a_w, off_tail_a_b, off_tail_b_w, off_tail_b_b, total;
  int64_t off_w1(int i) const { return off_head_b + F + (int64_t)i * (2LL * F * F + 2 * F); }
  int64_t off_b1(int i) const { return off_w1(i) + (int64_t)F * F; }
  int64_t off_w2(int i) const { return off_b1(i) + F; }
  int64_t off_b2(int i) const { return off_w2(i) + (int64_t)F * F; }
  void init(int f, int nb) {
    F = f; NB = nb;
    off_head_w = 0;
    off_head_b = (int64_t)F * kDin;
    off_tail_a_w = off_w1(NB);
    off_tail_a_b = off_tail_a_w + (int64_t)kNa * F;
    off_tail_b_w = off_tail_a_b + kNa;
    off_tail_b_b = off_tail_b_w + (int64_t)kNf * F;
    total = off_tail_b_b + kNf;
  }
};

template <class T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
  cudaError_t ensure(size_t need) {
    if (need <= n) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
    cudaError_t e = cudaMalloc(&p, need * sizeof(T));
    if (e == cudaSuccess) { n = need; e = cudaMemset(p, 0, need * sizeof(T)); }
    return e;
  }
  void release() { if (p) cudaFree(p); p = nullptr; n = 0; }
};

thread_local std::string g_train_err;
int tfail(int code, const std::string& msg) {
  g_train_err = msg;
  return code;
}
#define TTRY(expr)                                                                      \
  do {                                                                                  \
    cudaError_t e_ = (expr);                                                            \
    if (e_ != cudaSuccess) return tfail(NEDF_ERR_CUDA, std::string(#expr ": ") + cudaGetErrorString(e_)); \
  } while (0)
#define BTRY(expr) TTRY(expr)

int blocks(int64_t n, int per = 256) {
  const int64_t b = (n + per - 1) / per;
  return (int)(b < 8 * 148 ? (b > 0 ? b : 1) : 8 * 148);
}

// ---- batch: encoding (geometry.py:324-342) ----------------------------------------------
__global__ void encode_batch_kernel(const double* __restrict__ o, const double* __restrict__ d, int n, Box box,
                                    float* __restrict__ feats, uint8_t* __restrict__ hit_out) {
  const int r = blockIdx.x;
  if (r >= n) return;
  double lo[3] = {o[3 * r], o[3 * r + 1], o[3 * r + 2]}, ld[3] = {d[3 * r], d[3 * r + 1], d[3 * r + 2]};
  double t0, t1;
  const bool hit = slab_clip(lo, ld, box.bmin, box.bmax, t0, t1);
  if (threadIdx.x == 0) hit_out[r] = hit;
  // thread = (point, coordinate): 48 of them write 21 features each
  for (int e = threadIdx.x; e < kPoints * 3; e += blockDim.x) {
    const int pt = e / 3, a = e % 3;
    float* dst = feats + (size_t)r * kDin + pt * kPerPoint + 21 * a;
    if (!hit) {
      for (int j = 0; j < 21; ++j) dst[j] = 0.f;
      continue;
    }
    const double t = t0 + (t1 - t0) * lin16(pt);
    const double h = box.h[a];
    const double p = ((lo[a] + t * ld[a]) - box.c[a]) / h;
    double v[21];
    encode_coord_f64(p, v);
    for (int j = 0; j < 21; ++j) dst[j] = (float)v[j];
  }
}

// ---- batch: oracle trace + targets (fields.py:194-238, model.py:74-81, 222-235) ---------
__global__ void targets_kernel(const NedfField* fields, int root, double t_max, const double* __restrict__ o,
                               const double* __restrict__ d, int n, double l, int* __restrict__ tc,
                               int* __restrict__ tf, float* __restrict__ valid) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  double lo[3] = {o[3 * r], o[3 * r + 1], o[3 * r + 2]}, ld[3] = {d[3 * r], d[3 * r + 1], d[3 * r + 2]};
  double t;
  const bool hit = sphere_trace(fields, root, lo, ld, t_max, t);
  valid[r] = hit ? 1.f : 0.f;
  tc[r] = -1;
  tf[r] = -1;
  if (hit) {
    const double mu = fabs(lo[0] * ld[0] + lo[1] * ld[1] + lo[2] * ld[2]) - t;
    double u = (fmin(fmax(mu, -l), l) + l) / (2.0 * l);
    const double scaled = u * kNc;
    int c = (int)scaled;
    c = c < kNc - 1 ? c : kNc - 1;
    int f = (int)((scaled - c) * kNf);
    f = f < kNf - 1 ? f : kNf - 1;
    tc[r] = c;
    tf[r] = f;
  }
}

// ---- loss (nn.py:178-196): BCE and its logit gradient, rows masked for the bin heads ------
__device__ __forceinline__ float bce_elem(float z, float t) {
  return fmaxf(z, 0.f) - z * t + log1pf(expf(-fabsf(z)));
}
__device__ __forceinline__ float sigmoidf_(float z) {
  return z >= 0.f ? 1.f / (1.f + expf(-z)) : expf(z) / (1.f + expf(z));
}
// la65: [B][65] (coarse 0-63, alpha 64); lf: [B][128].  Writes g65 / gf in place of the logits.
__global__ void loss_kernel(float* __restrict__ la65, float* __restrict__ lf, const int* __restrict__ tc,
                            const int* __restrict__ tf, const float* __restrict__ valid, int n, float inv_cnt_c,
                            float inv_cnt_f, float inv_cnt_a, double* __restrict__ sums) {
  double sc = 0, sf = 0, sa = 0;
  const int64_t total = (int64_t)n * (kNa + kNf);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(i / (kNa + kNf)), c = (int)(i % (kNa + kNf));
    const float m = valid[r];
    if (c < kNc) {
      float& z = la65[(size_t)r * kNa + c];
      const float t = (tc[r] == c) ? 1.f : 0.f;
      sc += (double)(bce_elem(z, t) * m);
      z = (sigmoidf_(z) - t) * m * inv_cnt_c;
    } else if (c == kNc) {
      float& z = la65[(size_t)r * kNa + c];
      sa += (double)bce_elem(z, m);
      z = kAlphaWeight * (sigmoidf_(z) - m) * inv_cnt_a;
    } else {
      const int cf = c - kNa;
      float& z = lf[(size_t)r * kNf + cf];
      const float t = (tf[r] == cf) ? 1.f : 0.f;
      sf += (double)(bce_elem(z, t) * m);
      z = (sigmoidf_(z) - t) * m * inv_cnt_f;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    sc += __shfl_xor_sync(0xffffffffu, sc, o);
    sf += __shfl_xor_sync(0xffffffffu, sf, o);
    sa += __shfl_xor_sync(0xffffffffu, sa, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(&sums[0], sc);
    atomicAdd(&sums[1], sf);
    atomicAdd(&sums[2], sa);
  }
}

// ---- backward helpers --------------------------------------------------------------------
// db[c] = sum_r g[r][c] in two deterministic passes: block (column block, row slice) sums its
// slice into part[slice][c] (8 warps striding the slice's rows, then a fixed-order combine),
// then colsum_final adds the slices in order
constexpr int kColSlices = 64;
__global__ void colsum_partial_kernel(const float* __restrict__ g, int rows, int cols, int rows_per_slice,
                                      float* __restrict__ part) {
  __shared__ float acc[8][33];
  const int c = blockIdx.x * 32 + (threadIdx.x & 31), w = threadIdx.x >> 5;
  const int r0 = blockIdx.y * rows_per_slice, r1 = min(rows, r0 + rows_per_slice);
  float s = 0.f;
  if (c < cols)
    for (int r = r0 + w; r < r1; r += 8) s += g[(size_t)r * cols + c];
  acc[w][threadIdx.x & 31] = s;
  __syncthreads();
  if (w == 0 && c < cols) {
    float t = 0.f;
    for (int k = 0; k < 8; ++k) t += acc[k][threadIdx.x];
    part[(size_t)blockIdx.y * cols + c] = t;
  }
}
__global__ void colsum_final_kernel(const float* __restrict__ part, int slices, int cols, float* __restrict__ db) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= cols) return;
  float t = 0.f;
  for (int k = 0; k < slices; ++k) t += part[(size_t)k * cols + c];
  db[c] = t;
}
// Adam (nn.py:218-232)
__global__ void adam_kernel(float* __restrict__ p, const float* __restrict__ g, float* __restrict__ m,
                            float* __restrict__ v, int64_t n, float lr, float b1, float b2, float eps, float bc1,
                            float bc2) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float gi = g[i];
    const float mi = b1 * m[i] + (1.f - b1) * gi;
    const float vi = b2 * v[i] + (1.f - b2) * gi * gi;
    m[i] = mi;
    v[i] = vi;
    p[i] -= lr * (mi / bc1) / (sqrtf(vi / bc2) + eps);
  }
}

}  // namespace
}  // namespace nedf

using namespace nedf;

struct NedfTrainer {
  int device = 0;
  Dims dm;
  float lr = 5e-4f, beta1 = 0.9f, beta2 = 0.999f, eps = 1e-8f;
  int64_t step = 0;
  int cap = 0, n = 0, n_valid = 0;
  double l = 1.0;
  Box box;
  int n_sms = 148;
  DBuf<float> ws;                                // split-K workspace of the weight-gradient GEMMs
  DBuf<float> params, grads, m, v;
  DBuf<float> feats, xs, a1, h1, a2, la65, lf, gx, gtmp, g2;
  DBuf<double> o, d, sums;
  DBuf<uint8_t> hit;
  DBuf<int> tc, tf;
  DBuf<float> valid;
  DBuf<NedfField> fields;
};

namespace {

constexpr size_t kWsFloats = (size_t)1 << 22;   // 16 MB

cudaError_t colsum(NedfTrainer* t, const float* g, int rows, int cols, float* db, cudaStream_t st) {
  const int per = (rows + kColSlices - 1) / kColSlices;
  const int slices = (rows + per - 1) / per;
  colsum_partial_kernel<<<dim3((cols + 31) / 32, slices), 256, 0, st>>>(g, rows, cols, per, t->ws.p);
  colsum_final_kernel<<<(cols + 127) / 128, 128, 0, st>>>(t->ws.p, slices, cols, db);
  return cudaGetLastError();
}

// Y[rows][N] = X[rows][K] . W[N][K]^T  (row-major)
cudaError_t gemm_xwT(NedfTrainer* t, const float* X, const float* W, float* Y, int rows, int N, int K, cudaStream_t st,
                     const GemmEpi& epi) {
  return gemm_tf32x3(X, K, 0, W, K, 0, Y, N, rows, N, K, 0.f, nullptr, 0, t->n_sms, st, epi);
}
// dW[N][K] = G[rows][N]^T . X[rows][K]  (reduction over the batch: split K)
cudaError_t gemm_gTx(NedfTrainer* t, const float* G, const float* X, float* dW, int rows, int N, int K, cudaStream_t st) {
  return gemm_tf32x3(G, N, 1, X, K, 1, dW, K, N, K, rows, 0.f, t->ws.p, t->ws.n, t->n_sms, st);
}
// dX[rows][K] (+)= G[rows][N] . W[N][K]
cudaError_t gemm_gW(NedfTrainer* t, const float* G, const float* W, float* dX, int rows, int N, int K, float beta,
                    cudaStream_t st, const GemmEpi& epi = GemmEpi()) {
  return gemm_tf32x3(G, N, 0, W, K, 1, dX, K, rows, K, N, beta, nullptr, 0, t->n_sms, st, epi);
}
GemmEpi epi_of(int mode, const float* bias, const float* in = nullptr, float* aux = nullptr) {
  GemmEpi e;
  e.mode = mode;
  e.bias = bias;
  e.in = in;
  e.aux = aux;
  return e;
}

}  // namespace

extern "C" const char* nedf_trainer_last_error() { return g_train_err.c_str(); }

extern "C" int nedf_trainer_create(int device, const NedfModelInfo* info, const float* params_host, int64_t n_params,
                                   int max_batch, NedfTrainer** out) {
  if (!info || !params_host || !out || max_batch <= 0) return tfail(NEDF_ERR_INVALID, "NULL argument or batch <= 0");
  if (info->d_in != kDin || info->n_coarse != kNc || info->n_fine != kNf || info->d_feat <= 0 || info->n_blocks < 0)
    return tfail(NEDF_ERR_UNSUPPORTED, "training supports d_in 1008 with 64 coarse / 128 fine bins");
  TTRY(cudaSetDevice(device));
  auto* t = new NedfTrainer();
  t->device = device;
  t->dm.init(info->d_feat, info->n_blocks);
  if (n_params != t->dm.total) {
    delete t;
    return tfail(NEDF_ERR_INVALID, "parameter count does not match the model dimensions");
  }
  t->l = info->half_range;
  for (int a = 0; a < 3; ++a) {
    t->box.bmin[a] = info->box_min[a];
    t->box.bmax[a] = info->box_max[a];
    t->box.c[a] = 0.5 * ((double)info->box_min[a] + (double)info->box_max[a]);
    const double h = 0.5 * ((double)info->box_max[a] - (double)info->box_min[a]);
    t->box.h[a] = h > 0 ? h : 1.0;
  }
  const int64_t P = t->dm.total, B = max_batch, F = t->dm.F, NB = t->dm.NB;
  t->cap = max_batch;
  cudaError_t e = cudaSuccess;
  for (auto* b : {&t->params, &t->grads, &t->m, &t->v}) if (e == cudaSuccess) e = b->ensure(P);
  if (e == cudaSuccess) e = t->feats.ensure(B * kDin);
  if (e == cudaSuccess) e = t->xs.ensure((NB + 1) * B * F);          // block inputs x_0..x_NB (x_NB = feat)
  if (e == cudaSuccess) e = t->a1.ensure(std::max<int64_t>(NB, 1) * B * F);
  if (e == cudaSuccess) e = t->h1.ensure(std::max<int64_t>(NB, 1) * B * F);
  if (e == cudaSuccess) e = t->a2.ensure(std::max<int64_t>(NB, 1) * B * F);
  if (e == cudaSuccess) e = t->la65.ensure(B * kNa);
  if (e == cudaSuccess) e = t->lf.ensure(B * kNf);
  if (e == cudaSuccess) e = t->gx.ensure(B * F);
  if (e == cudaSuccess) e = t->gtmp.ensure(B * F);
  if (e == cudaSuccess) e = t->g2.ensure(B * F);
  if (e == cudaSuccess) e = t->o.ensure(B * 3);
  if (e == cudaSuccess) e = t->d.ensure(B * 3);
  if (e == cudaSuccess) e = t->sums.ensure(4);
  if (e == cudaSuccess) e = t->hit.ensure(B);
  if (e == cudaSuccess) e = t->tc.ensure(B);
  if (e == cudaSuccess) e = t->tf.ensure(B);
  if (e == cudaSuccess) e = t->valid.ensure(B);
  if (e == cudaSuccess) e = t->ws.ensure(kWsFloats);
  if (e == cudaSuccess) e = cudaMemcpy(t->params.p, params_host, P * sizeof(float), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&t->n_sms, cudaDevAttrMultiProcessorCount, device);
  if (e != cudaSuccess) {
    nedf_trainer_destroy(t);
    return tfail(NEDF_ERR_CUDA, std::string("trainer allocation: ") + cudaGetErrorString(e));
  }
  *out = t;
  return NEDF_OK;
}

extern "C" void nedf_trainer_destroy(NedfTrainer* t) {
  if (!t) return;
  cudaSetDevice(t->device);
  for (auto* b : {&t->ws, &t->params, &t->grads, &t->m, &t->v, &t->feats, &t->xs, &t->a1, &t->h1, &t->a2, &t->la65, &t->lf,
                  &t->gx, &t->gtmp, &t->g2, &t->valid})
    b->release();
  t->o.release(); t->d.release(); t->sums.release(); t->hit.release(); t->tc.release(); t->tf.release();
  t->fields.release();
  delete t;
}

extern "C" int nedf_trainer_set_lr(NedfTrainer* t, float lr) {
  if (!t || !(lr > 0)) return tfail(NEDF_ERR_INVALID, "bad learning rate");
  t->lr = lr;
  return NEDF_OK;
}

extern "C" int nedf_trainer_batch(NedfTrainer* t, const NedfField* fields, int n_fields, int root, double t_max,
                                  const double* origins_host, const double* dirs_host, int n, uint8_t* hit_host,
                                  void* stream) {
  if (!t || !origins_host || !dirs_host || !hit_host || n <= 0 || n > t->cap)
    return tfail(NEDF_ERR_INVALID, "bad batch");
  if (!fields || n_fields <= 0 || root < 0 || root >= n_fields) return tfail(NEDF_ERR_INVALID, "bad oracle field");
  cudaStream_t st = (cudaStream_t)stream;
  TTRY(t->fields.ensure(n_fields));
  TTRY(cudaMemcpyAsync(t->fields.p, fields, n_fields * sizeof(NedfField), cudaMemcpyHostToDevice, st));
  TTRY(cudaMemcpyAsync(t->o.p, origins_host, (size_t)n * 3 * sizeof(double), cudaMemcpyHostToDevice, st));
  TTRY(cudaMemcpyAsync(t->d.p, dirs_host, (size_t)n * 3 * sizeof(double), cudaMemcpyHostToDevice, st));
  encode_batch_kernel<<<n, 64, 0, st>>>(t->o.p, t->d.p, n, t->box, t->feats.p, t->hit.p);
  targets_kernel<<<(n + 127) / 128, 128, 0, st>>>(t->fields.p, root, t_max, t->o.p, t->d.p, n, t->l, t->tc.p, t->tf.p,
                                                  t->valid.p);
  TTRY(cudaGetLastError());
  TTRY(cudaMemcpyAsync(hit_host, t->hit.p, n, cudaMemcpyDeviceToHost, st));
  TTRY(cudaStreamSynchronize(st));
  t->n = n;
  return NEDF_OK;
}

// Explicit batch (tests): features [n][1008] f32, bin targets (-1 = none), alpha targets.
extern "C" int nedf_trainer_set_batch(NedfTrainer* t, const float* feats_host, const int32_t* tc_host,
                                      const int32_t* tf_host, const float* alpha_host, int n, void* stream) {
  if (!t || !feats_host || !tc_host || !tf_host || !alpha_host || n <= 0 || n > t->cap)
    return tfail(NEDF_ERR_INVALID, "bad batch");
  cudaStream_t st = (cudaStream_t)stream;
  TTRY(cudaMemcpyAsync(t->feats.p, feats_host, (size_t)n * kDin * sizeof(float), cudaMemcpyHostToDevice, st));
  TTRY(cudaMemcpyAsync(t->tc.p, tc_host, n * sizeof(int), cudaMemcpyHostToDevice, st));
  TTRY(cudaMemcpyAsync(t->tf.p, tf_host, n * sizeof(int), cudaMemcpyHostToDevice, st));
  TTRY(cudaMemcpyAsync(t->valid.p, alpha_host, n * sizeof(float), cudaMemcpyHostToDevice, st));
  TTRY(cudaStreamSynchronize(st));
  t->n = n;
  return NEDF_OK;
}

// Loss and gradients of the current batch (model.py:238-248); losses_host[0..3] =
// total, coarse, fine, alpha.
extern "C" int nedf_trainer_loss_and_grads(NedfTrainer* t, double* losses_host, void* stream) {
  if (!t || !losses_host || t->n <= 0) return tfail(NEDF_ERR_INVALID, "no batch");
  cudaStream_t st = (cudaStream_t)stream;
  TTRY(cudaSetDevice(t->device));
  const Dims& D = t->dm;
  const int B = t->n, F = D.F, NB = D.NB;
  float* P = t->params.p;
  float* G = t->grads.p;
  auto X = [&](int i) { return t->xs.p + (size_t)i * B * F; };
  auto A1 = [&](int i) { return t->a1.p + (size_t)i * B * F; };
  auto H1 = [&](int i) { return t->h1.p + (size_t)i * B * F; };
  auto A2 = [&](int i) { return t->a2.p + (size_t)i * B * F; };
  // ---- forward (nn.py:115-135)
  // (bias, ReLU and the residual add are the GEMMs' fused epilogues)
  BTRY(gemm_xwT(t, t->feats.p, P + D.off_head_w, X(0), B, F, kDin, st, epi_of(GEMM_EPI_BIAS, P + D.off_head_b)));
  for (int i = 0; i < NB; ++i) {
    BTRY(gemm_xwT(t, X(i), P + D.off_w1(i), A1(i), B, F, F, st,
                  epi_of(GEMM_EPI_BIAS_RELU, P + D.off_b1(i), nullptr, H1(i))));
    BTRY(gemm_xwT(t, H1(i), P + D.off_w2(i), A2(i), B, F, F, st,
                  epi_of(GEMM_EPI_RESIDUAL, P + D.off_b2(i), X(i), X(i + 1))));
  }
  float* feat = X(NB);
  BTRY(gemm_xwT(t, feat, P + D.off_tail_a_w, t->la65.p, B, kNa, F, st, epi_of(GEMM_EPI_BIAS, P + D.off_tail_a_b)));
  BTRY(gemm_xwT(t, feat, P + D.off_tail_b_w, t->lf.p, B, kNf, F, st, epi_of(GEMM_EPI_BIAS, P + D.off_tail_b_b)));
  // ---- loss (the row-mask count needs the number of rows with a hit)
  std::vector<float> valid_h(B);
  TTRY(cudaMemcpyAsync(valid_h.data(), t->valid.p, B * sizeof(float), cudaMemcpyDeviceToHost, st));
  TTRY(cudaStreamSynchronize(st));
  int nv = 0;
  for (float v : valid_h) nv += v > 0.5f;
  t->n_valid = nv;
  TTRY(cudaMemsetAsync(t->sums.p, 0, 4 * sizeof(double), st));
  const float inv_c = nv > 0 ? 1.f / ((float)nv * kNc) : 0.f, inv_f = nv > 0 ? 1.f / ((float)nv * kNf) : 0.f;
  const float inv_a = 1.f / (float)B;
  loss_kernel<<<blocks((int64_t)B * (kNa + kNf)), 256, 0, st>>>(t->la65.p, t->lf.p, t->tc.p, t->tf.p, t->valid.p, B,
                                                                inv_c, inv_f, inv_a, t->sums.p);
  TTRY(cudaGetLastError());
  // ---- backward (nn.py:138-167); la65 / lf now hold g_a (with 0.1 alpha) and g_f
  BTRY(gemm_gTx(t, t->la65.p, feat, G + D.off_tail_a_w, B, kNa, F, st));
  TTRY(colsum(t, t->la65.p, B, kNa, G + D.off_tail_a_b, st));
  BTRY(gemm_gTx(t, t->lf.p, feat, G + D.off_tail_b_w, B, kNf, F, st));
  TTRY(colsum(t, t->lf.p, B, kNf, G + D.off_tail_b_b, st));
  BTRY(gemm_gW(t, t->la65.p, P + D.off_tail_a_w, t->gx.p, B, kNa, F, 0.f, st));
  // g_x; with blocks, also g_a2 = (a2 > 0) g_x of the last block (fused epilogue)
  BTRY(gemm_gW(t, t->lf.p, P + D.off_tail_b_w, t->gx.p, B, kNf, F, 1.f, st,
               NB > 0 ? epi_of(GEMM_EPI_MASK_AUX, nullptr, A2(NB - 1), t->g2.p) : GemmEpi()));
  for (int i = NB - 1; i >= 0; --i) {
    BTRY(gemm_gTx(t, t->g2.p, H1(i), G + D.off_w2(i), B, F, F, st));
    TTRY(colsum(t, t->g2.p, B, F, G + D.off_b2(i), st));
    // g_a1 = (a1 > 0) g_h1, g_h1 = g_a2 W2
    BTRY(gemm_gW(t, t->g2.p, P + D.off_w2(i), t->gtmp.p, B, F, F, 0.f, st, epi_of(GEMM_EPI_MASK, nullptr, A1(i))));
    BTRY(gemm_gTx(t, t->gtmp.p, X(i), G + D.off_w1(i), B, F, F, st));
    TTRY(colsum(t, t->gtmp.p, B, F, G + D.off_b1(i), st));
    // g_x += g_a1 W1; g_a2 of block i - 1 = (a2 > 0) g_x
    BTRY(gemm_gW(t, t->gtmp.p, P + D.off_w1(i), t->gx.p, B, F, F, 1.f, st,
                 i > 0 ? epi_of(GEMM_EPI_MASK_AUX, nullptr, A2(i - 1), t->g2.p) : GemmEpi()));
  }
  BTRY(gemm_gTx(t, t->gx.p, t->feats.p, G + D.off_head_w, B, F, kDin, st));
  TTRY(colsum(t, t->gx.p, B, F, G + D.off_head_b, st));
  TTRY(cudaGetLastError());
  double s[4];
  TTRY(cudaMemcpyAsync(s, t->sums.p, 3 * sizeof(double), cudaMemcpyDeviceToHost, st));
  TTRY(cudaStreamSynchronize(st));
  const double lc = nv > 0 ? s[0] / ((double)nv * kNc) : 0.0, lf = nv > 0 ? s[1] / ((double)nv * kNf) : 0.0;
  const double la = s[2] / (double)B;
  losses_host[0] = lc + lf + kAlphaWeight * la;
  losses_host[1] = lc;
  losses_host[2] = lf;
  losses_host[3] = la;
  return NEDF_OK;
}

extern "C" int nedf_trainer_adam_step(NedfTrainer* t, void* stream) {
  if (!t) return tfail(NEDF_ERR_INVALID, "NULL trainer");
  t->step += 1;
  const float bc1 = 1.f - (float)std::pow((double)t->beta1, (double)t->step);
  const float bc2 = 1.f - (float)std::pow((double)t->beta2, (double)t->step);
  adam_kernel<<<blocks(t->dm.total), 256, 0, (cudaStream_t)stream>>>(t->params.p, t->grads.p, t->m.p, t->v.p,
                                                                     t->dm.total, t->lr, t->beta1, t->beta2, t->eps,
                                                                     bc1, bc2);
  TTRY(cudaGetLastError());
  return NEDF_OK;
}

extern "C" int nedf_trainer_read(NedfTrainer* t, int what, float* host, void* stream) {
  if (!t || !host || what < 0 || what > 1) return tfail(NEDF_ERR_INVALID, "bad read");
  cudaStream_t st = (cudaStream_t)stream;
  TTRY(cudaMemcpyAsync(host, what == 0 ? t->params.p : t->grads.p, t->dm.total * sizeof(float),
                       cudaMemcpyDeviceToHost, st));
  TTRY(cudaStreamSynchronize(st));
  return NEDF_OK;
}
