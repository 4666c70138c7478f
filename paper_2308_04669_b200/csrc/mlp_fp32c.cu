// fp32 network for small ray batches, split across a cluster of 8 CTAs.
//
// Role: the near-tie guard's re-evaluation (a few hundred rays per frame).
// Its cost is latency, not FLOPs: one ray still walks a 35-layer chain.  The
// streaming kernel (mlp_fp32s.cu) runs that chain inside one SM, streaming the
// whole 9.5 MB fp32 weight image through it.  Here the 8 CTAs of a cluster
// share each ray tile: CTA r owns output columns [32 r, 32 r + 32) of every
// layer, reads only its 1/8 of the weights (straight from L2, each thread a
// contiguous 128-byte run per layer), and scatters its outputs into every
// peer's activation buffer through distributed shared memory; one cluster
// barrier per layer publishes them.  Same arithmetic as mlp_fp32s.cu: float64
// features, float32 weights / accumulation (a different summation order).
//
// Thread (kp, c): K part kp = warp (K / 8 rows), output column c = lane.
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "common.cuh"
#include "encode.cuh"
#include "frame.cuh"
#include "tc_ptx.cuh"

namespace nedf {
namespace {

constexpr int kC = 8;                 // CTAs per cluster
constexpr int kThreads = 256;         // 8 K parts x 32 columns
constexpr int kR = 16;                // rays per cluster tile
constexpr int kHeadK = 1024;          // 16 points x (63 features + 1 zero)
constexpr int kHeadPer = kHeadK / 8;  // 128 weights per thread
constexpr int kBodyPer = 256 / 8;     // 32 weights per thread
constexpr int kLayers = 34;           // head, 32 block layers, fused tail
constexpr size_t kHeadFloats = (size_t)kC * kThreads * kHeadPer;   // 262144
constexpr size_t kLayerFloats = (size_t)kC * kThreads * kBodyPer;  // 65536

struct ClSmem {
  float f[kR][kHeadK];
  float x[kR][256];
  float h[kR][256];
  float part[8][kR][32];
  double ray[kR][8];
  uint32_t pix[kR], obj[kR];
  int valid[kR];
};

__device__ __forceinline__ void st_cluster_f32(uint32_t addr, float v) {
  asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(addr), "f"(v) : "memory");
}

}  // namespace

__global__ void __cluster_dims__(kC, 1, 1) __launch_bounds__(kThreads, 1)
mlp_fp32_cluster_kernel(GroupTable gt, ListSet ls, RayJob job, OutSpec out) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  ClSmem& S = *reinterpret_cast<ClSmem*>(smem_raw);
  __shared__ int s_tiles[65];
  const int tid = threadIdx.x;
  const int kp = tid >> 5, c = tid & 31;
  const uint32_t rank = tc::cluster_rank();
  const int cid = blockIdx.x / kC, n_cl = gridDim.x / kC;
  const int ng = ls.n_groups < 64 ? ls.n_groups : 64;
  const bool feats_in = out.feats != nullptr;
  // shared::cluster address of S in every CTA of the cluster
  uint32_t peer[kC];
#pragma unroll
  for (int q = 0; q < kC; ++q) peer[q] = tc::peer_addr(&S, q);
  const uint32_t self = tc::smem_u32(&S);
  auto remote = [&](int q, const void* p) { return peer[q] + (uint32_t)(tc::smem_u32(p) - self); };

  if (tid == 0) {
    int cum = 0;
    s_tiles[0] = 0;
    for (int g = 0; g < ng; ++g) {
      cum += (ls.count[g] + kR - 1) / kR;
      s_tiles[g + 1] = cum;
    }
  }
  __syncthreads();
  const int total = s_tiles[ng];
  for (int t = cid; t < total; t += n_cl) {
    int g = 0;
    while (g < ng - 1 && t >= s_tiles[g + 1]) ++g;
    const int lt = t - s_tiles[g];
    int n = ls.count[g] - lt * kR;
    n = n < kR ? n : kR;
    const int64_t base = ls.offset[g] + (int64_t)lt * kR;
    const DevModel& m = gt.models[g];
    if (tid < kR) {
      const int r = tid;
      const int v = r < n;
      S.valid[r] = v;
      S.pix[r] = v ? ls.pix[base + r] : 0u;
      S.obj[r] = v ? ls.obj[base + r] : 0u;
      if (v && !feats_in) {
        double wo[3], wd[3], lo[3], ld[3], t0 = 0, t1 = 0;
        item_local_ray(job, S.pix[r], S.obj[r], wo, wd, lo, ld);
        slab_clip(lo, ld, m.bmin, m.bmax, t0, t1);
        for (int a = 0; a < 3; ++a) {
          S.ray[r][a] = lo[a];
          S.ray[r][3 + a] = ld[a];
        }
        S.ray[r][6] = t0;
        S.ray[r][7] = t1;
      }
    }
    __syncthreads();
    // ---- head features: this CTA computes sample points 2 rank, 2 rank + 1 and broadcasts them
    // (float64, geometry.py:312-342); one (ray, point, coordinate, level) per thread
    for (int e = tid; e < kR * 2 * 33; e += kThreads) {
      const int r = e / 66, rem = e % 66, p2 = rem / 33, a = (rem / 11) % 3, lev = rem % 11;
      const int pt = 2 * (int)rank + p2;
      float v0 = 0.f, v1 = 0.f;       // lev < 10: sin, cos; lev 10: raw p, pad
      if (S.valid[r]) {
        if (feats_in) {
          const float* src = out.feats + (size_t)S.pix[r] * kDin + pt * kPerPoint + 21 * a;
          if (lev < 10) { v0 = src[1 + 2 * lev]; v1 = src[2 + 2 * lev]; }
          else v0 = src[0];
        } else {
          const double t0 = S.ray[r][6], t1 = S.ray[r][7];
          const double tt = t0 + (t1 - t0) * lin16(pt);
          const double p = ((S.ray[r][a] + tt * S.ray[r][3 + a]) - m.c[a]) / m.h[a];
          if (lev < 10) {
            double sn, cs;
            sincos(p * ldexp(3.141592653589793, lev), &sn, &cs);
            v0 = (float)sn;
            v1 = (float)cs;
          } else {
            v0 = (float)p;
          }
        }
      }
      float* dst = &S.f[r][64 * pt + 21 * a];
#pragma unroll
      for (int q = 0; q < kC; ++q) {
        if (lev < 10) {
          st_cluster_f32(remote(q, dst + 1 + 2 * lev), v0);
          st_cluster_f32(remote(q, dst + 2 + 2 * lev), v1);
        } else {
          st_cluster_f32(remote(q, dst), v0);
          if (a == 0) st_cluster_f32(remote(q, &S.f[r][64 * pt + 63]), 0.f);
        }
      }
    }
    tc::cluster_sync();
    // ---- 34 layers: head (K = 1024), 16 x (fc1, fc2), fused tail (nn.py:115-135)
    const float* wl = m.wcluster;
    for (int L = 0; L < kLayers; ++L) {
      const int per = L == 0 ? kHeadPer : kBodyPer;
      const float* in = L == 0 ? &S.f[0][0] : ((L & 1) ? &S.x[0][0] : &S.h[0][0]);
      const int ld_in = L == 0 ? kHeadK : 256;
      const float* w = wl + (L == 0 ? 0 : kHeadFloats + (size_t)(L - 1) * kLayerFloats) +
                       ((size_t)rank * kThreads + tid) * per;
      float acc[kR];
#pragma unroll
      for (int r = 0; r < kR; ++r) acc[r] = 0.f;
      const float* inp = in + kp * per;
#pragma unroll 2
      for (int k = 0; k < per; k += 4) {
        const float4 wv = __ldg(reinterpret_cast<const float4*>(w + k));
#pragma unroll
        for (int r = 0; r < kR; ++r) {
          const float4 a4 = *reinterpret_cast<const float4*>(inp + r * ld_in + k);
          acc[r] = fmaf(a4.x, wv.x, acc[r]);
          acc[r] = fmaf(a4.y, wv.y, acc[r]);
          acc[r] = fmaf(a4.z, wv.z, acc[r]);
          acc[r] = fmaf(a4.w, wv.w, acc[r]);
        }
      }
#pragma unroll
      for (int r = 0; r < kR; ++r) S.part[kp][r][c] = acc[r];
      __syncthreads();
      for (int o = tid; o < kR * 32; o += kThreads) {
        const int r = o >> 5, cc = o & 31, col = 32 * (int)rank + cc;
        float s = 0.f;
#pragma unroll
        for (int q = 0; q < 8; ++q) s += S.part[q][r][cc];
        const float b = __ldg(m.bias_pack + L * 256 + col);
        float v;
        float* dst;
        if (L == 0) { v = s + b; dst = &S.x[r][col]; }                          // head: no activation
        else if (L == kLayers - 1) { v = s + b; dst = &S.h[r][col]; }            // tail logits
        else if (L & 1) { v = fmaxf(s + b, 0.f); dst = &S.h[r][col]; }           // fc1
        else { v = S.x[r][col] + fmaxf(s + b, 0.f); dst = &S.x[r][col]; }        // fc2 + residual
#pragma unroll
        for (int q = 0; q < kC; ++q) st_cluster_f32(remote(q, dst), v);
      }
      tc::cluster_sync();
    }
    // ---- decode: fine = logits[0:128), coarse = [128:192), alpha = [192] (model.py:277-293)
    if (rank == 0 && tid < kR && S.valid[tid]) {
      const int r = tid;
      const float* lg = S.h[r];
      if (out.mode == OUT_LOGITS) {
        const size_t row = S.pix[r];
        for (int k = 0; k < 64; ++k) out.lc[row * 64 + k] = lg[128 + k];
        for (int k = 0; k < 128; ++k) out.lf[row * 128 + k] = lg[k];
        out.la[row] = lg[192];
      } else {
        int cb = 0, fb = 0;
        float best = lg[128];
        for (int k = 1; k < 64; ++k) if (lg[128 + k] > best) { best = lg[128 + k]; cb = k; }
        best = lg[0];
        for (int k = 1; k < 128; ++k) if (lg[k] > best) { best = lg[k]; fb = k; }
        double wo[3], wd[3], lo[3], ld[3];
        item_local_ray(job, S.pix[r], S.obj[r], wo, wd, lo, ld);
        finish_ray(m, job, out, S.pix[r], S.obj[r], cb, fb, (double)lg[192], wo, wd);
      }
    }
    __syncthreads();
  }
}

cudaError_t launch_mlp_fp32_cluster(const GroupTable& gt, const ListSet& ls, const RayJob& job, const OutSpec& out,
                                    int n_sms, cudaStream_t stream) {
  static int max_clusters = 0;
  const size_t smem = sizeof(ClSmem);
  if (max_clusters == 0) {
    cudaError_t e = cudaFuncSetAttribute(mlp_fp32_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(kC * (n_sms / kC), 1, 1);
    cfg.blockDim = dim3(kThreads, 1, 1);
    cfg.dynamicSmemBytes = smem;
    int n = 0;
    e = cudaOccupancyMaxActiveClusters(&n, mlp_fp32_cluster_kernel, &cfg);
    if (e != cudaSuccess) return e;
    max_clusters = n > 0 ? n : 1;
    if (getenv("NEDF_VERBOSE")) fprintf(stderr, "nedf: fp32 cluster kernel, %d co-resident clusters\n", n);
  }
  mlp_fp32_cluster_kernel<<<kC * max_clusters, kThreads, smem, stream>>>(gt, ls, job, out);
  return cudaGetLastError();
}

// Cluster image: layer L, CTA r, thread (kp, c) -> `per` consecutive floats
// W[out = 32 r + c][in = kp * per + k], k < per (head rows are the 16 points'
// 63 features + 1 zero; tail outputs: fine 0-127, coarse 128-191, alpha 192).
cudaError_t fp32_pack_cluster(const float* P, int d_in, int F, int n_blocks, int n_coarse, int n_fine, float** dev) {
  if (F != 256 || n_blocks != 16 || d_in != kDin || n_coarse != 64 || n_fine != 128) return cudaErrorInvalidValue;
  std::vector<float> img(kHeadFloats + 33 * kLayerFloats, 0.f);
  size_t p = 0;
  const float* Wh = P + p; p += (size_t)F * d_in + F;
  std::vector<const float*> Wl(32);
  for (int l = 0; l < 32; ++l) { Wl[l] = P + p; p += (size_t)F * F + F; }
  const float* Wa = P + p; p += (size_t)(n_coarse + 1) * F + n_coarse + 1;
  const float* Wb = P + p;
  auto w_of = [&](int L, int o, int k) -> float {     // W_L[o][k] in the kernel's row/column numbering
    if (L == 0) {
      const int pt = k / 64, j = k % 64;
      return j < 63 ? Wh[(size_t)o * d_in + 63 * pt + j] : 0.f;
    }
    if (L <= 32) return Wl[L - 1][(size_t)o * F + k];
    if (o < 128) return Wb[(size_t)o * F + k];
    if (o < 128 + n_coarse + 1) return Wa[(size_t)(o - 128) * F + k];
    return 0.f;
  };
  for (int L = 0; L < kLayers; ++L) {
    const int per = L == 0 ? kHeadPer : kBodyPer;
    float* dst = img.data() + (L == 0 ? 0 : kHeadFloats + (size_t)(L - 1) * kLayerFloats);
    for (int r = 0; r < kC; ++r)
      for (int t = 0; t < kThreads; ++t) {
        const int kp = t >> 5, cc = t & 31, o = 32 * r + cc;
        for (int k = 0; k < per; ++k) dst[((size_t)r * kThreads + t) * per + k] = w_of(L, o, kp * per + k);
      }
  }
  cudaError_t e = cudaMalloc(dev, img.size() * sizeof(float));
  if (e == cudaSuccess) e = cudaMemcpy(*dev, img.data(), img.size() * sizeof(float), cudaMemcpyHostToDevice);
  return e;
}

}  // namespace nedf
