// fp32 network for small ray batches, split across a cluster of kC = 4 CTAs.
//
// Role: the near-tie guard's re-evaluation (a few hundred rays per frame).
// Its cost is latency, not FLOPs: one ray still walks a 35-layer chain.  The
// streaming kernel (mlp_fp32s.cu) runs that chain inside one SM, streaming the
// whole 9.5 MB fp32 weight image through it.  Here the 4 CTAs of a cluster
// share each ray tile: CTA r owns output columns [64 r, 64 r + 64) of every
// layer, so it needs only its 1/4 of the weights, and scatters its outputs into
// every peer's activation buffer with st.async through distributed shared
// memory.  Each store completes transaction bytes on the receiving CTA's
// mbarrier, so a CTA starts layer L+1 as soon as all 16 KB of layer L have
// landed -- no cluster-wide barrier per layer.  Buffer reuse is safe without
// one: a CTA can only produce layer L+1 after receiving every peer's layer-L
// outputs, i.e. after every peer finished reading the buffer layer L+1
// overwrites.  Two layer barriers alternate so a peer one layer ahead never
// completes the current phase.  Same arithmetic as mlp_fp32s.cu: float64
// features, float32 weights and accumulation (a different summation order).
//
// Weights: a producer warp (warp 8) streams the CTA's slice of the image as
// 32 KB stages (one 8 K-row x 4-column chunk per compute thread; the head is 8
// stages, every later layer 2) through a 3-slot shared-memory ring with bulk
// copies, so the compute warps never wait on L2 latency; a compute warp copies
// its chunk into registers and releases the slot before its FMAs.  The FMAs are
// FFMA2 (fma.rn.f32x2: one x value times a pair of columns), the same fp32
// operations in the same order as scalar FMAs, at half the issue slots.
//
// Thread layout (256 compute threads): column quad cg = lane & 15 (columns 4 cg
// .. 4 cg + 3 of the CTA's 64), K part kp = 2 warp + (lane >> 4) of 16 (16 K rows
// per layer, 64 for the head), so every x value loaded from shared memory feeds
// 4 FMAs.  Cluster size: 4 CTAs lets ~35 clusters (140 SMs) co-reside, so a
// frame's guard batch is one round of 16-ray tiles.
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "common.cuh"
#include "encode.cuh"
#include "frame.cuh"
#include "tc_ptx.cuh"
#include "../../include/nedf_b200_diag.h"

namespace nedf {
namespace {

constexpr int kC = 4;                 // CTAs per cluster
constexpr int kCols = 256 / kC;       // output columns per CTA (64)
constexpr int kQuads = kCols / 4;     // column quads per CTA (one per lane group)
constexpr int kLanesK = 32 / kQuads;  // K parts per warp
constexpr int kThreads = 256;         // compute threads: kKP K parts x kQuads column quads
constexpr int kBlock = kThreads + 32; // + the weight producer warp
constexpr int kKP = 8 * kLanesK;      // K parts (8 warps)
constexpr int kRMax = 16;             // rays per cluster tile: 8, 12 or 16, the smallest that fits one round
constexpr int kHeadK = 1024;          // 16 points x (63 features + 1 zero)
constexpr int kChunk = 32;            // weights per thread per chunk: 8 K rows x 4 columns
constexpr int kHeadChunks = kHeadK / kKP / 8;   // 8-row chunks per thread: head (8)
constexpr int kBodyChunks = 256 / kKP / 8;      // body / tail (2)
constexpr int kLayers = 34;           // head, 32 block layers, fused tail
constexpr int kStagesPerTile = kHeadChunks + (kLayers - 1) * kBodyChunks;       // 74
constexpr uint32_t kStageBytes = kThreads * kChunk * 4;                         // 32 KB
constexpr int kRing = 3;
constexpr size_t kImageFloats = (size_t)kStagesPerTile * kC * kThreads * kChunk;

struct ClSmem {
  float4 ring[kRing][kStageBytes / 16];   // weight stage slots: float4 i of compute thread t at [256 i + t]
  float f[kRMax][kHeadK];
  float x[kRMax][256];
  float h[kRMax][256];
  float part[8][kRMax][kCols];   // per warp (its K parts pre-reduced by shuffle)
  double ray[kRMax][8];
  uint32_t pix[kRMax], obj[kRMax];
  int valid[kRMax];
  uint64_t full[kRing], empty[kRing];
  uint64_t feat_bar;             // features of the tile: 64 KB from the 4 CTAs
  uint64_t layer_bar[2];         // layer L outputs (16 KB from the 4 CTAs) on layer_bar[L & 1]
};

// remote store that completes its bytes on the receiving CTA's mbarrier
__device__ __forceinline__ void st_async_v2(uint32_t addr, float a, float b, uint32_t mbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f32 [%0], {%1, %2}, [%3];" ::"r"(addr),
               "f"(a), "f"(b), "r"(mbar)
               : "memory");
}
__device__ __forceinline__ void st_async_v4(uint32_t addr, float a, float b, float c, float d, uint32_t mbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.f32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(addr),
               "f"(a), "f"(b), "f"(c), "f"(d), "r"(mbar)
               : "memory");
}
__device__ __forceinline__ void st_async_f32(uint32_t addr, float v, uint32_t mbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f32 [%0], %1, [%2];" ::"r"(addr), "f"(v),
               "r"(mbar)
               : "memory");
}
// acc (two fp32 lanes) += x * (w0, w1), each lane one fma.rn.f32
__device__ __forceinline__ uint64_t ffma2(float x, uint64_t w, uint64_t acc) {
  uint64_t d;
  asm("{\n\t.reg .b64 xx;\n\tmov.b64 xx, {%1, %1};\n\tfma.rn.f32x2 %0, xx, %2, %3;\n\t}"
      : "=l"(d)
      : "f"(x), "l"(w), "l"(acc));
  return d;
}
__device__ __forceinline__ uint64_t f2_as_u64(float lo, float hi) {
  uint64_t d;
  asm("mov.b64 %0, {%1, %2};" : "=l"(d) : "f"(lo), "f"(hi));
  return d;
}
__device__ __forceinline__ float2 u64_as_f2(uint64_t v) {
  float2 r;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(v));
  return r;
}

}  // namespace

// optional timeline of cluster 0 / CTA 0 (diagnostics, nedf_diag_cl_trace): per tile i < 4,
// [64 i + 0] start, [+1] rays set up, [+2] features landed, [+3 + L] layer L landed, [+40] decoded
__device__ unsigned long long g_cl_trace[256];
__device__ int g_cl_trace_on;

// The compute warps' tile loop for R-ray tiles (R = 8, 12, 16).
template <int R>
__device__ __forceinline__ void guard_tiles(ClSmem& S, const int* s_tiles, int total, int ng, const GroupTable& gt,
                                            const ListSet& ls, const RayJob& job, const OutSpec& out, uint32_t rank,
                                            int cid, int n_cl) {
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const bool feats_in = out.feats != nullptr;
  // ------------------------------------------------------------------ compute warps
  const int cg = lane % kQuads, kp = kLanesK * warp + lane / kQuads;
  // shared::cluster address of S in every CTA of the cluster
  uint32_t peer[kC];
#pragma unroll
  for (int q = 0; q < kC; ++q) peer[q] = tc::peer_addr(&S, q);
  const uint32_t self = tc::smem_u32(&S);
  auto remote = [&](int q, const void* p) { return peer[q] + (uint32_t)(tc::smem_u32(p) - self); };
  uint32_t feat_phase = 0, layer_count = 0, gq = 0;
  int ti = 0;
  for (int t = cid; t < total; t += n_cl, ++ti) {
    const bool tr = g_cl_trace_on && cid == 0 && rank == 0 && tid == 0 && ti < 4;
    if (tr) g_cl_trace[64 * ti] = clock64();
    int g = 0;
    while (g < ng - 1 && t >= s_tiles[g + 1]) ++g;
    const int lt = t - s_tiles[g];
    int n = ls.count[g] - lt * R;
    n = n < R ? n : R;
    const int64_t base = ls.offset[g] + (int64_t)lt * R;
    const DevModel& m = gt.models[g];
    if (tid < R) {
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
    tc::named_bar(1, kThreads);
    if (tr) g_cl_trace[64 * ti + 1] = clock64();
    // ---- head features: this CTA computes sample points kPtsPerCta rank .. kPtsPerCta (rank + 1) - 1 and broadcasts them
    // (float64, geometry.py:312-342); one (ray, point, coordinate, level) per thread
    constexpr int kPtsPerCta = kPoints / kC;
    for (int e = tid; e < R * kPtsPerCta * 33; e += kThreads) {
      const int r = e / (kPtsPerCta * 33), rem = e % (kPtsPerCta * 33), p2 = rem / 33, a = (rem / 11) % 3,
                lev = rem % 11;
      const int pt = kPtsPerCta * (int)rank + p2;
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
            sincospi(ldexp(p, lev), &sn, &cs);     // sin/cos(2^lev pi p), exact argument scaling
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
        const uint32_t fb = remote(q, &S.feat_bar);
        if (lev < 10) {
          st_async_f32(remote(q, dst + 1 + 2 * lev), v0, fb);     // odd offsets for a = 0: no v2
          st_async_f32(remote(q, dst + 2 + 2 * lev), v1, fb);
        } else {
          st_async_f32(remote(q, dst), v0, fb);
          if (a == 0) st_async_f32(remote(q, &S.f[r][64 * pt + 63]), 0.f, fb);
        }
      }
    }
    if (tid == 0) tc::mbar_expect_tx(&S.feat_bar, (uint32_t)(R * kHeadK * 4));
    tc::mbar_wait(&S.feat_bar, feat_phase);
    feat_phase ^= 1;
    if (tr) g_cl_trace[64 * ti + 2] = clock64();
    // ---- 34 layers: head (K = 1024), 16 x (fc1, fc2), fused tail (nn.py:115-135)
    const float* bias_p = m.bias_pack;
    constexpr int kOut = kCols / 16;                 // outputs per thread in the reduce phase (4)
    const int rr = tid >> 4, cc2 = kOut * (tid & 15), col2 = kCols * (int)rank + cc2;   // reduce role
    float bnext[kOut];
#pragma unroll
    for (int u = 0; u < kOut; ++u) bnext[u] = __ldg(bias_p + col2 + u);
    for (int L = 0; L < kLayers; ++L) {
      const int nch = L == 0 ? kHeadChunks : kBodyChunks;
      const float* in = L == 0 ? &S.f[0][0] : ((L & 1) ? &S.x[0][0] : &S.h[0][0]);
      const int ld_in = L == 0 ? kHeadK : 256;
      float b[kOut];
#pragma unroll
      for (int u = 0; u < kOut; ++u) b[u] = bnext[u];
      if (L + 1 < kLayers) {
#pragma unroll
        for (int u = 0; u < kOut; ++u) bnext[u] = __ldg(bias_p + (L + 1) * 256 + col2 + u);
      }
      uint64_t acc[R][2];                           // columns (4 cg, 4 cg + 1), (4 cg + 2, 4 cg + 3)
#pragma unroll
      for (int r = 0; r < R; ++r) acc[r][0] = acc[r][1] = 0ull;
      for (int j = 0; j < nch; ++j) {
        // this chunk's weights: float4 i = W[c0 .. c0 + 3][k0 + i], copied out of the ring slot, which is
        // then released to the producer before the FMAs
        const int slot = gq % kRing;
        tc::mbar_wait(&S.full[slot], (gq / kRing) & 1);
        ++gq;
        uint64_t w[8][2];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const float4 v = S.ring[slot][kThreads * i + tid];
          w[i][0] = f2_as_u64(v.x, v.y);
          w[i][1] = f2_as_u64(v.z, v.w);
        }
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&S.empty[slot]);
        const float* inp = in + kp * (8 * nch) + 8 * j;
#pragma unroll
        for (int h2 = 0; h2 < 2; ++h2) {
#pragma unroll
          for (int r = 0; r < R; ++r) {
            const float4 x4 = *reinterpret_cast<const float4*>(inp + r * ld_in + 4 * h2);
            const float xs[4] = {x4.x, x4.y, x4.z, x4.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              acc[r][0] = ffma2(xs[e], w[4 * h2 + e][0], acc[r][0]);
              acc[r][1] = ffma2(xs[e], w[4 * h2 + e][1], acc[r][1]);
            }
          }
        }
      }
      if (tr && L == 5) g_cl_trace[64 * ti + 41] = clock64();
      if (g_cl_trace_on && cid == 0 && rank == 0 && lane == 0 && ti == 0 && L == 5) g_cl_trace[200 + warp] = clock64();
      // pre-reduce the warp's K parts (lanes l, l + kQuads, ...), then across the 8 warps
      float a[R][4];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const float2 lo = u64_as_f2(acc[r][0]), hi = u64_as_f2(acc[r][1]);
        a[r][0] = lo.x; a[r][1] = lo.y; a[r][2] = hi.x; a[r][3] = hi.y;
      }
#pragma unroll
      for (int r = 0; r < R; ++r)
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int off = kQuads; off < 32; off <<= 1) a[r][u] += __shfl_xor_sync(0xffffffffu, a[r][u], off);
      if (lane < kQuads) {
#pragma unroll
        for (int r = 0; r < R; ++r)
          *reinterpret_cast<float4*>(&S.part[warp][r][4 * cg]) = make_float4(a[r][0], a[r][1], a[r][2], a[r][3]);
      }
      tc::named_bar(1, kThreads);
      if (tr && L == 5) g_cl_trace[64 * ti + 42] = clock64();
      if (rr < R) {   // kOut adjacent outputs per thread: R rays x kCols columns
        float sv[kOut];
#pragma unroll
        for (int u = 0; u < kOut; ++u) sv[u] = 0.f;
#pragma unroll
        for (int w8 = 0; w8 < 8; ++w8)
#pragma unroll
          for (int u = 0; u < kOut; ++u) sv[u] += S.part[w8][rr][cc2 + u];
        float v[kOut];
        float* dst;
        if (L == 0 || L == kLayers - 1) {                         // head (no activation) / tail logits
#pragma unroll
          for (int u = 0; u < kOut; ++u) v[u] = sv[u] + b[u];
          dst = L == 0 ? &S.x[rr][col2] : &S.h[rr][col2];
        } else if (L & 1) {                                       // fc1
#pragma unroll
          for (int u = 0; u < kOut; ++u) v[u] = fmaxf(sv[u] + b[u], 0.f);
          dst = &S.h[rr][col2];
        } else {                                                  // fc2 + residual
#pragma unroll
          for (int u = 0; u < kOut; ++u) v[u] = S.x[rr][col2 + u] + fmaxf(sv[u] + b[u], 0.f);
          dst = &S.x[rr][col2];
        }
        const int lb = layer_count & 1;
#pragma unroll
        for (int qq = 0; qq < kC; ++qq) st_async_v4(remote(qq, dst), v[0], v[1], v[2], v[3], remote(qq, &S.layer_bar[lb]));
      }
      if (tr && L == 5) g_cl_trace[64 * ti + 43] = clock64();
      if (tid == 0) tc::mbar_expect_tx(&S.layer_bar[layer_count & 1], (uint32_t)(R * 256 * 4));
      tc::mbar_wait(&S.layer_bar[layer_count & 1], (layer_count >> 1) & 1);
      ++layer_count;
      if (tr) g_cl_trace[64 * ti + 3 + L] = clock64();
    }
    // ---- decode: fine = logits[0:128), coarse = [128:192), alpha = [192] (model.py:277-293)
    if (rank == 0 && tid < R && S.valid[tid]) {
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
    tc::named_bar(1, kThreads);
    if (tr) g_cl_trace[64 * ti + 40] = clock64();
  }
}

__global__ void __cluster_dims__(kC, 1, 1) __launch_bounds__(kBlock, 1)
mlp_fp32_cluster_kernel(GroupTable gt, ListSet ls, RayJob job, OutSpec out) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  ClSmem& S = *reinterpret_cast<ClSmem*>(smem_raw);
  __shared__ int s_tiles[65];
  __shared__ int s_R;
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const uint32_t rank = tc::cluster_rank();
  const int cid = blockIdx.x / kC, n_cl = gridDim.x / kC;
  const int ng = ls.n_groups < 64 ? ls.n_groups : 64;

  if (tid == 0) {
    // tile size: the smallest of 8, 12, 16 rays whose tiles all run in one round of clusters (the
    // per-layer FMA time scales with the rays per tile, the exchange latency does not)
    int R = 16;
    for (int cand = 8; cand < 16; cand += 4) {
      int tiles = 0;
      for (int g = 0; g < ng; ++g) tiles += (ls.count[g] + cand - 1) / cand;
      if (tiles <= n_cl) { R = cand; break; }
    }
    s_R = R;
    int cum = 0;
    s_tiles[0] = 0;
    for (int g = 0; g < ng; ++g) {
      cum += (ls.count[g] + R - 1) / R;
      s_tiles[g + 1] = cum;
    }
    for (int i = 0; i < kRing; ++i) { tc::mbar_init(&S.full[i], 1); tc::mbar_init(&S.empty[i], 8); }
    tc::mbar_init(&S.feat_bar, 1);
    tc::mbar_init(&S.layer_bar[0], 1);
    tc::mbar_init(&S.layer_bar[1], 1);
    tc::mbar_fence_init();
  }
  tc::cluster_sync();           // peers' barriers initialised before anyone stores into them
  const int total = s_tiles[ng];

  if (warp == 8) {
    // ---------------------------------------------------------------- weight producer
    // stage q of a tile = this CTA's 32 KB slice of (head chunk q | layer 1 + (q - 8) / 2, chunk (q - 8) % 2)
    if (lane == 0) {
      uint32_t gq = 0;
      for (int t = cid; t < total; t += n_cl) {
        int g = 0;
        while (g < ng - 1 && t >= s_tiles[g + 1]) ++g;
        const unsigned char* img = reinterpret_cast<const unsigned char*>(gt.models[g].wcluster);
        for (int q = 0; q < kStagesPerTile; ++q, ++gq) {
          const int slot = gq % kRing;
          tc::mbar_wait(&S.empty[slot], ((gq / kRing) & 1) ^ 1);
          tc::mbar_expect_tx(&S.full[slot], kStageBytes);
          tc::bulk_g2s(&S.ring[slot][0], img + ((size_t)q * kC + rank) * kStageBytes, kStageBytes, &S.full[slot]);
        }
      }
    }
    __syncwarp();
    tc::cluster_sync();
    return;
  }

  // ------------------------------------------------------------------ compute warps
  if (s_R == 8) guard_tiles<8>(S, s_tiles, total, ng, gt, ls, job, out, rank, cid, n_cl);
  else if (s_R == 12) guard_tiles<12>(S, s_tiles, total, ng, gt, ls, job, out, rank, cid, n_cl);
  else guard_tiles<16>(S, s_tiles, total, ng, gt, ls, job, out, rank, cid, n_cl);
  tc::cluster_sync();           // no CTA leaves while its stores to peers may be in flight
}

}  // namespace nedf

extern "C" int nedf_diag_cl_trace(int enable, unsigned long long* out, int n) {
  using namespace nedf;
  if (enable >= 0) {
    int v = enable;
    if (cudaMemcpyToSymbol(g_cl_trace_on, &v, sizeof(int)) != cudaSuccess) return NEDF_ERR_CUDA;
  }
  if (out && n > 0) {
    if (n > 256) n = 256;
    if (cudaMemcpyFromSymbol(out, g_cl_trace, n * sizeof(unsigned long long)) != cudaSuccess) return NEDF_ERR_CUDA;
  }
  return NEDF_OK;
}

namespace nedf {

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
    cfg.blockDim = dim3(kBlock, 1, 1);
    cfg.dynamicSmemBytes = smem;
    int n = 0;
    e = cudaOccupancyMaxActiveClusters(&n, mlp_fp32_cluster_kernel, &cfg);
    if (e != cudaSuccess) return e;
    max_clusters = n > 0 ? n : 1;
    if (getenv("NEDF_VERBOSE")) fprintf(stderr, "nedf: fp32 cluster kernel, %d co-resident clusters\n", n);
  }
  mlp_fp32_cluster_kernel<<<kC * max_clusters, kBlock, smem, stream>>>(gt, ls, job, out);
  return cudaGetLastError();
}

// Cluster image, streamed as 32 KB stages: stage q (head chunk q < 8, then layer
// L = 1 + (q - 8) / 2, chunk j = (q - 8) % 2), CTA r -> float4 [(q kC + r) 2048 +
// 256 i + t] = W[c0 .. c0 + 3][k] for compute thread t (column quad cg = t & 15,
// K part kp = 2 (t >> 5) + ((t >> 4) & 1)), K row k = kp * 8 n + 8 j + i (n =
// chunks of the layer: 8 for the head, 2 after) and c0 = 64 r + 4 cg (head rows
// are the 16 points' 63 features + 1 zero; tail outputs: fine 0-127, coarse
// 128-191, alpha 192).  Thread-minor float4s make each ring read conflict-free.
cudaError_t fp32_pack_cluster(const float* P, int d_in, int F, int n_blocks, int n_coarse, int n_fine, float** dev) {
  if (F != 256 || n_blocks != 16 || d_in != kDin || n_coarse != 64 || n_fine != 128) return cudaErrorInvalidValue;
  std::vector<float> img(kImageFloats, 0.f);
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
  for (int q = 0; q < kStagesPerTile; ++q) {
    const int L = q < kHeadChunks ? 0 : 1 + (q - kHeadChunks) / kBodyChunks;
    const int j = q < kHeadChunks ? q : (q - kHeadChunks) % kBodyChunks;
    const int nch = L == 0 ? kHeadChunks : kBodyChunks;
    for (int r = 0; r < kC; ++r)
      for (int t = 0; t < kThreads; ++t) {
        const int lane = t & 31, cg = lane % kQuads, kp = kLanesK * (t >> 5) + lane / kQuads;
        const int c0 = kCols * r + 4 * cg;
        for (int i = 0; i < 8; ++i) {
          float* dst = img.data() + 4 * (((size_t)q * kC + r) * (kStageBytes / 16) + (size_t)kThreads * i + t);
          const int k = kp * 8 * nch + 8 * j + i;
          for (int u = 0; u < 4; ++u) dst[u] = w_of(L, c0 + u, k);
        }
      }
  }
  cudaError_t e = cudaMalloc(dev, img.size() * sizeof(float));
  if (e == cudaSuccess) e = cudaMemcpy(*dev, img.data(), img.size() * sizeof(float), cudaMemcpyHostToDevice);
  return e;
}

}  // namespace nedf
