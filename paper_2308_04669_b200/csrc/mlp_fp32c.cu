// fp32-accurate network for small ray batches, split across a cluster of KC
// CTAs (4 or 8), on the warp-level tensor cores (mma.sync, 3xTF32).
//
// Role: the near-tie guard's re-evaluation (a few hundred rays per frame).
// Its cost is latency, not FLOPs: one ray still walks a 35-layer chain.  The
// KC CTAs of a cluster share a 16-ray tile: CTA r owns output columns
// [(256 / KC) r, (256 / KC) (r + 1)) of every layer, so it needs only its
// 1/KC of the weights, and sends its outputs into every peer's activation
// buffer with st.async through distributed shared memory.  Each store completes
// transaction bytes on the receiving CTA's mbarrier, so a CTA starts layer L+1
// as soon as all 16 KB of layer L have landed -- no cluster-wide barrier per
// layer.  Buffer reuse is safe without one: a warp sends its layer-L outputs
// only after its layer-L MMAs, so once every layer-L output has landed
// anywhere, every warp of the cluster is done reading the buffer layer L+1
// overwrites.  Two layer barriers alternate so a peer one layer ahead never
// completes the current phase.
//
// Arithmetic: a CTA's columns form 8-column groups (one m16n8 n-tile each):
// with KC = 4, warp w owns group w and the whole K range; with KC = 8, two warps
// share a group, taking alternate weight stages (K halves), and the second
// hands its partial fragment to the first through shared memory and a named
// barrier.  m16n8k8 TF32 MMAs with fp32 accumulation, each operand split into a
// TF32 high part and a TF32 remainder and three products accumulated (a_lo b_hi
// + a_hi b_lo + a_hi b_hi; the dropped a_lo b_lo term is ~2^-20 of a product),
// i.e. near-fp32 accuracy on the tensor pipe.  A 16 x 64 x 256 layer slice takes
// ~3.4k cycles of HMMA (ncu: "math" throttle on the MMA pipe;
// scripts/cl_trace.py) against ~4.2k for the same slice as FFMA2 (the previous
// version of this kernel); the split runs on LOP3/FADD, since cvt.rna.tf32
// issues at a quarter rate.  Float64 features (sincospi and double-angle
// steps), float32 weights and activations.
//
// Weights: a producer warp (warp 8) streams the CTA's slice of the image as
// stages of 128 K rows (32 KB for KC = 4, 16 KB for KC = 8; the head is 8
// stages, every later layer 2) through a 3-slot shared-memory ring with bulk
// copies; a compute warp copies its part of a stage into registers and
// releases the slot before its MMAs.
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

constexpr int kThreads = 256;         // compute threads (8 warps)
constexpr int kBlock = kThreads + 32; // + the weight producer warp
constexpr int kR = 16;                // rays per cluster tile (the MMA M dimension)
constexpr int kHeadK = 1024;          // 16 points x (63 features + 1 zero)
constexpr int kFStride = kHeadK + 4;  // padded rows: the A-fragment loads are bank-conflict free
constexpr int kXStride = 256 + 4;
constexpr int kKSteps = 16;           // k-steps of 8 rows per stage (128 K rows)
constexpr int kHeadStages = kHeadK / (8 * kKSteps);   // 8
constexpr int kBodyStages = 256 / (8 * kKSteps);      // 2
constexpr int kLayers = 34;           // head, 32 block layers, fused tail
constexpr int kStagesPerTile = kHeadStages + (kLayers - 1) * kBodyStages;       // 74
constexpr int kRing = 3;

// Cluster shapes: KC = 4 CTAs x 64 output columns (8 column groups of 8, one warp each, whole K),
// or KC = 8 CTAs x 32 columns (4 column groups, two warps each splitting K) -- half the MMA work
// per layer on a CTA's critical path for frames whose guard batch fits 8-CTA clusters in one round.
template <int KC>
struct Cfg {
  static constexpr int kC = KC;
  static constexpr int kCols = 256 / KC;              // output columns per CTA
  static constexpr int kNG = kCols / 8;               // column groups (one MMA n-tile each)
  static constexpr int kKP = 8 / kNG;                 // K parts per column group (warps)
  static constexpr uint32_t kStageBytes = kNG * kKSteps * 32 * 8;   // 32 KB / 16 KB
  static constexpr uint32_t kPeerBytes = (KC - 1) * kR * kCols * 4; // the peers' columns of one layer
  static constexpr size_t kImageFloats = (size_t)kStagesPerTile * KC * (kStageBytes / 4);
};

template <int KC>
struct ClSmem {
  float2 ring[kRing][Cfg<KC>::kStageBytes / 8];   // weight stage slots: [column group][k-step][lane] (W[n][k], W[n][k + 4])
  float f[kR][kFStride];
  float x[kR][kXStride];
  float h[kR][kXStride];
  double ray[kR][8];
  uint32_t pix[kR], obj[kR];
  int valid[kR];
  float4 part[8][32];            // KC = 8: the second K part's partial fragments, per column group and lane
  uint64_t full[kRing], empty[kRing];
  uint64_t layer_bar[2];         // layer L outputs on layer_bar[L & 1]: the peers' bytes + the local finishing warps' arrivals
};

// remote store that completes its bytes on the receiving CTA's mbarrier
__device__ __forceinline__ void st_async_v4(uint32_t addr, float a, float b, float c, float d, uint32_t mbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.f32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(addr),
               "f"(a), "f"(b), "f"(c), "f"(d), "r"(mbar)
               : "memory");
}
// TF32 split without conversions (cvt.rna.tf32 issues at a quarter rate): hi = x with the 13 low
// mantissa bits cleared, lo = x - hi (exact in fp32); the MMA reads the top 19 bits of each operand,
// so lo enters truncated to TF32 -- the split keeps ~2^-21 of |x|.
__device__ __forceinline__ void split_tf32(float x, uint32_t& hi, uint32_t& lo) {
  hi = __float_as_uint(x) & 0xFFFFE000u;
  lo = __float_as_uint(x - __uint_as_float(hi));
}
// C[16 x 8] += A[16 x 8] B[8 x 8], TF32 inputs, fp32 accumulation
__device__ __forceinline__ void mma_tf32(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
      "{%0, %1, %2, %3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

}  // namespace

// optional timeline of cluster 0 / CTA 0 (diagnostics, nedf_diag_cl_trace): per tile i < 4,
// [64 i + 0] start, [+1] rays set up, [+2] features landed, [+3 + L] layer L landed, [+40] decoded,
// layer 5: [+41] MMAs done (warp 0), [+42] outputs sent
__device__ unsigned long long g_cl_trace[256];
__device__ int g_cl_trace_on;

template <int KC>
__global__ void __cluster_dims__(KC, 1, 1) __launch_bounds__(kBlock, 1)
mlp_fp32_cluster_kernel(GroupTable gt, ListSet ls, RayJob job, OutSpec out) {
  using G = Cfg<KC>;
  constexpr int kC = KC, kCols = G::kCols, kNG = G::kNG, kKP = G::kKP;
  constexpr uint32_t kStageBytes = G::kStageBytes;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  ClSmem<KC>& S = *reinterpret_cast<ClSmem<KC>*>(smem_raw);
  __shared__ int s_tiles[65];
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const uint32_t rank = tc::cluster_rank();
  const int cid = blockIdx.x / kC, n_cl = gridDim.x / kC;
  const int ng = ls.n_groups < 64 ? ls.n_groups : 64;
  const bool feats_in = out.feats != nullptr;

  if (tid == 0) {
    int cum = 0;
    s_tiles[0] = 0;
    for (int g = 0; g < ng; ++g) {
      cum += (ls.count[g] + kR - 1) / kR;
      s_tiles[g + 1] = cum;
    }
    // a stage is consumed by the kNG warps of one K part; a layer is finished by kNG warps
    for (int i = 0; i < kRing; ++i) { tc::mbar_init(&S.full[i], 1); tc::mbar_init(&S.empty[i], kNG); }
    tc::mbar_init(&S.layer_bar[0], 1 + kNG);   // tid 0's expect_tx + one arrival per finishing warp
    tc::mbar_init(&S.layer_bar[1], 1 + kNG);
    tc::mbar_fence_init();
  }
  tc::cluster_sync();           // peers' barriers initialised before anyone stores into them
  const int total = s_tiles[ng];

  if (warp == 8) {
    // ---------------------------------------------------------------- weight producer
    // stage q of a tile = this CTA's 32 KB slice of (head K block q | layer 1 + (q - 8) / 2, K block (q - 8) % 2)
    // bulk copies issued by one thread serialise, so each stage goes out as kCopyLanes parallel pieces
    constexpr int kCopyLanes = 4;
    constexpr uint32_t kPiece = kStageBytes / kCopyLanes;
    uint32_t gq = 0;
    for (int t = cid; t < total; t += n_cl) {
      int g = 0;
      while (g < ng - 1 && t >= s_tiles[g + 1]) ++g;
      const unsigned char* img =
          reinterpret_cast<const unsigned char*>(KC == 8 ? gt.models[g].wcluster8 : gt.models[g].wcluster);
      for (int q = 0; q < kStagesPerTile; ++q, ++gq) {
        const int slot = gq % kRing;
        if (lane == 0) {
          tc::mbar_wait(&S.empty[slot], ((gq / kRing) & 1) ^ 1);
          tc::mbar_expect_tx(&S.full[slot], kStageBytes);
        }
        __syncwarp();
        if (lane < kCopyLanes)
          tc::bulk_g2s(reinterpret_cast<unsigned char*>(&S.ring[slot][0]) + lane * kPiece,
                       img + ((size_t)q * kC + rank) * kStageBytes + lane * kPiece, kPiece, &S.full[slot]);
      }
    }
    __syncwarp();
    tc::cluster_sync();
    return;
  }

  // ------------------------------------------------------------------ compute warps
  const int gid = lane >> 2, tig = lane & 3;          // MMA fragment coordinates
  const int ngw = warp % kNG, kpart = warp / kNG;    // column group, K part (stages alternate K parts)
  const int col = kCols * (int)rank + 8 * ngw + 2 * tig;    // this lane's two output columns: col, col + 1
  // shared::cluster address of S in every CTA of the cluster
  uint32_t peer[kC];
#pragma unroll
  for (int q = 0; q < kC; ++q) peer[q] = tc::peer_addr(&S, q);
  const uint32_t self = tc::smem_u32(&S);
  auto remote = [&](int q, const void* p) { return peer[q] + (uint32_t)(tc::smem_u32(p) - self); };
  uint32_t layer_count = 0, gq = 0;
  int ti = 0;
  for (int t = cid; t < total; t += n_cl, ++ti) {
    const bool tr = g_cl_trace_on && cid == 0 && rank == 0 && tid == 0 && ti < 4;
    if (tr) g_cl_trace[64 * ti] = clock64();
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
    tc::named_bar(1, kThreads);
    if (tr) g_cl_trace[64 * ti + 1] = clock64();
    // ---- head features (float64, geometry.py:312-342), computed by every CTA of the cluster for itself:
    // one (ray, point, coordinate) per thread, sin/cos at levels 0 and 5 with exact argument scaling,
    // the other levels by float64 double-angle steps (error ~1e-15, far below the float32 rounding)
    for (int e = tid; e < kR * kPoints * 3; e += kThreads) {
      const int r = e / (kPoints * 3), rem = e % (kPoints * 3), pt = rem / 3, a = rem % 3;
      float* dst = &S.f[r][64 * pt + 21 * a];
      if (!S.valid[r]) {
#pragma unroll
        for (int j = 0; j < 21; ++j) dst[j] = 0.f;
      } else if (feats_in) {
        const float* src = out.feats + (size_t)S.pix[r] * kDin + pt * kPerPoint + 21 * a;
#pragma unroll
        for (int j = 0; j < 21; ++j) dst[j] = src[j];
      } else {
        const double t0 = S.ray[r][6], t1 = S.ray[r][7];
        const double tt = t0 + (t1 - t0) * lin16(pt);
        const double p = ((S.ray[r][a] + tt * S.ray[r][3 + a]) - m.c[a]) / m.h[a];
        dst[0] = (float)p;
#pragma unroll
        for (int base = 0; base < kLevels; base += 5) {
          double sn, cs;
          sincospi(ldexp(p, base), &sn, &cs);
          dst[1 + 2 * base] = (float)sn;
          dst[2 + 2 * base] = (float)cs;
#pragma unroll
          for (int k = base + 1; k < base + 5; ++k) {
            const double s2 = 2.0 * sn * cs, c2 = (cs - sn) * (cs + sn);
            sn = s2;
            cs = c2;
            dst[1 + 2 * k] = (float)sn;
            dst[2 + 2 * k] = (float)cs;
          }
        }
      }
      if (a == 0) S.f[r][64 * pt + 63] = 0.f;
    }
    tc::named_bar(1, kThreads);
    if (tr) g_cl_trace[64 * ti + 2] = clock64();
    // ---- 34 layers: head (K = 1024), 16 x (fc1, fc2), fused tail (nn.py:115-135)
    const float* bias_p = m.bias_pack;
    float2 bnext = *reinterpret_cast<const float2*>(bias_p + col);
    for (int L = 0; L < kLayers; ++L) {
      const int nst = L == 0 ? kHeadStages : kBodyStages;
      const float* A = L == 0 ? &S.f[0][0] : ((L & 1) ? &S.x[0][0] : &S.h[0][0]);
      const int lda = L == 0 ? kFStride : kXStride;
      const float2 b = bnext;
      if (L + 1 < kLayers) bnext = *reinterpret_cast<const float2*>(bias_p + (L + 1) * 256 + col);
      // twelve independent accumulator chains (lo-hi, hi-lo, hi-hi products x k-step mod 4) so
      // consecutive MMAs of a warp do not wait on each other's results
      float acc[12][4];
#pragma unroll
      for (int i = 0; i < 12; ++i) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.f;
      const float* a_lo_row = A + gid * lda + tig;           // rows gid, gid + 8; columns k0 + tig, k0 + tig + 4
      const float* a_hi_row = A + (gid + 8) * lda + tig;
      for (int st = 0; st < nst; ++st, ++gq) {
        if (kKP > 1 && st % kKP != kpart) continue;
        // this warp's 16 k-steps of the stage, copied out of the ring slot, which is then released
        const int slot = gq % kRing;
        const long long tw0 = (tr && L == 5) ? clock64() : 0;
        tc::mbar_wait(&S.full[slot], (gq / kRing) & 1);
        if (tr && L == 5) g_cl_trace[64 * ti + 43] += clock64() - tw0;
        float2 wv[kKSteps];
#pragma unroll
        for (int ks = 0; ks < kKSteps; ++ks) wv[ks] = S.ring[slot][(ngw * kKSteps + ks) * 32 + lane];
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&S.empty[slot]);
#pragma unroll
        for (int ks = 0; ks < kKSteps; ++ks) {
          const int k0 = (st * kKSteps + ks) * 8;
          uint32_t ah[4], al[4], bh0, bl0, bh1, bl1;
          split_tf32(a_lo_row[k0], ah[0], al[0]);
          split_tf32(a_hi_row[k0], ah[1], al[1]);
          split_tf32(a_lo_row[k0 + 4], ah[2], al[2]);
          split_tf32(a_hi_row[k0 + 4], ah[3], al[3]);
          split_tf32(wv[ks].x, bh0, bl0);
          split_tf32(wv[ks].y, bh1, bl1);
          const int par = 3 * (ks & 3);
          mma_tf32(acc[par + 0], al, bh0, bh1);
          mma_tf32(acc[par + 1], ah, bl0, bl1);
          mma_tf32(acc[par + 2], ah, bh0, bh1);
        }
      }
      float c[4];
#pragma unroll
      for (int i = 0; i < 4; ++i)
        c[i] = (((acc[0][i] + acc[3][i]) + (acc[6][i] + acc[9][i])) + ((acc[1][i] + acc[4][i]) + (acc[7][i] + acc[10][i]))) +
               ((acc[2][i] + acc[5][i]) + (acc[8][i] + acc[11][i]));
      if (kKP > 1) {
        // the second K part hands its partial fragment to its column group's first (a named barrier
        // per pair), which finishes the layer; the buffer is rewritten only after this layer's exchange
        if (kpart == 1) {
          S.part[ngw][lane] = make_float4(c[0], c[1], c[2], c[3]);
          tc::named_bar_arrive(2 + ngw, 64);
          tc::mbar_wait(&S.layer_bar[layer_count & 1], (layer_count >> 1) & 1);
          ++layer_count;
          continue;
        }
        tc::named_bar(2 + ngw, 64);
        const float4 pp = S.part[ngw][lane];
        c[0] += pp.x; c[1] += pp.y; c[2] += pp.z; c[3] += pp.w;
      }
      if (tr && L == 5) g_cl_trace[64 * ti + 41] = clock64();
      // epilogue: rows gid / gid + 8, columns col / col + 1 (c0 c1 / c2 c3)
      float v[4];
      float* dst0;
      float* dst1;
      if (L == 0 || L == kLayers - 1) {                         // head (no activation) / tail logits
        v[0] = c[0] + b.x; v[1] = c[1] + b.y; v[2] = c[2] + b.x; v[3] = c[3] + b.y;
        float* base_buf = L == 0 ? &S.x[0][0] : &S.h[0][0];
        dst0 = base_buf + gid * kXStride + col;
        dst1 = base_buf + (gid + 8) * kXStride + col;
      } else if (L & 1) {                                       // fc1
        v[0] = fmaxf(c[0] + b.x, 0.f); v[1] = fmaxf(c[1] + b.y, 0.f);
        v[2] = fmaxf(c[2] + b.x, 0.f); v[3] = fmaxf(c[3] + b.y, 0.f);
        dst0 = &S.h[gid][col];
        dst1 = &S.h[gid + 8][col];
      } else {                                                  // fc2 + residual
        dst0 = &S.x[gid][col];
        dst1 = &S.x[gid + 8][col];
        v[0] = dst0[0] + fmaxf(c[0] + b.x, 0.f); v[1] = dst0[1] + fmaxf(c[1] + b.y, 0.f);
        v[2] = dst1[0] + fmaxf(c[2] + b.x, 0.f); v[3] = dst1[1] + fmaxf(c[3] + b.y, 0.f);
      }
      // lanes t, t ^ 1 of a quad swap halves so each sends one 16-byte run: the even lane row gid,
      // columns col .. col + 3; the odd lane row gid + 8, columns col - 2 .. col + 1 (half the remote stores)
      const bool odd = tig & 1;
      const float r0 = __shfl_xor_sync(0xffffffffu, odd ? v[0] : v[2], 1);
      const float r1 = __shfl_xor_sync(0xffffffffu, odd ? v[1] : v[3], 1);
      float* dst = odd ? dst1 - 2 : dst0;
      const float4 o4 = odd ? make_float4(r0, r1, v[2], v[3]) : make_float4(v[0], v[1], r0, r1);
      const int lb = layer_count & 1;
#pragma unroll
      for (int qq = 1; qq < kC; ++qq) {       // the peers, through distributed shared memory
        const int peer_rank = ((int)rank + qq) % kC;
        st_async_v4(remote(peer_rank, dst), o4.x, o4.y, o4.z, o4.w, remote(peer_rank, &S.layer_bar[lb]));
      }
      *reinterpret_cast<float4*>(dst) = o4;     // this CTA: a plain store, published by the warp's arrival
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&S.layer_bar[lb]);
      if (tr && L == 5) g_cl_trace[64 * ti + 42] = clock64();
      if (tid == 0) tc::mbar_expect_tx(&S.layer_bar[lb], G::kPeerBytes);
      tc::mbar_wait(&S.layer_bar[lb], (layer_count >> 1) & 1);
      ++layer_count;
      if (tr) g_cl_trace[64 * ti + 3 + L] = clock64();
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
    tc::named_bar(1, kThreads);
    if (tr) g_cl_trace[64 * ti + 40] = clock64();
  }
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

template <int KC>
cudaError_t launch_guard(const GroupTable& gt, const ListSet& ls, const RayJob& job, const OutSpec& out, int n_sms,
                         cudaStream_t stream) {
  static int max_clusters_dev[kMaxDevices] = {};
  int& max_clusters = max_clusters_dev[current_device()];
  const size_t smem = sizeof(ClSmem<KC>);
  if (max_clusters == 0) {
    cudaError_t e = cudaFuncSetAttribute(mlp_fp32_cluster_kernel<KC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(KC * (n_sms / KC), 1, 1);
    cfg.blockDim = dim3(kBlock, 1, 1);
    cfg.dynamicSmemBytes = smem;
    int n = 0;
    e = cudaOccupancyMaxActiveClusters(&n, mlp_fp32_cluster_kernel<KC>, &cfg);
    if (e != cudaSuccess) return e;
    max_clusters = n > 0 ? n : 1;
    if (getenv("NEDF_VERBOSE")) fprintf(stderr, "nedf: fp32 cluster kernel x%d, %d co-resident clusters\n", KC, n);
  }
  mlp_fp32_cluster_kernel<KC><<<KC * max_clusters, kBlock, smem, stream>>>(gt, ls, job, out);
  return cudaGetLastError();
}

cudaError_t launch_mlp_fp32_cluster(const GroupTable& gt, const ListSet& ls, const RayJob& job, const OutSpec& out,
                                    int n_sms, int cluster, cudaStream_t stream) {
  return cluster == 8 ? launch_guard<8>(gt, ls, job, out, n_sms, stream)
                      : launch_guard<4>(gt, ls, job, out, n_sms, stream);
}

// Cluster image for KC-CTA clusters, streamed as stages of 128 K rows: stage q
// (head K block q < 8, then layer L = 1 + (q - 8) / 2, K block j = (q - 8) % 2),
// CTA r -> float2 [(q KC + r) (kStageBytes / 8) + (16 w + s) 32 + lane] =
// (W[n][k], W[n][k + 4]) for column group w, k-step s, lane = 4 gid + tig:
// output column n = (256 / KC) r + 8 w + gid, K row k = 128 j + 8 s + tig (the B
// fragment of an m16n8k8 MMA).  Head rows are the 16 points' 63 features + 1
// zero; tail outputs: fine 0-127, coarse 128-191, alpha 192, zero padding.
template <int KC>
cudaError_t pack_guard(const float* P, int d_in, int F, int n_blocks, int n_coarse, int n_fine, float** dev) {
  using G = Cfg<KC>;
  if (F != 256 || n_blocks != 16 || d_in != kDin || n_coarse != 64 || n_fine != 128) return cudaErrorInvalidValue;
  std::vector<float> img(G::kImageFloats, 0.f);
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
    const int L = q < kHeadStages ? 0 : 1 + (q - kHeadStages) / kBodyStages;
    const int j = q < kHeadStages ? q : (q - kHeadStages) % kBodyStages;
    for (int r = 0; r < KC; ++r)
      for (int w = 0; w < G::kNG; ++w)
        for (int s = 0; s < kKSteps; ++s)
          for (int lane = 0; lane < 32; ++lane) {
            const int n = G::kCols * r + 8 * w + (lane >> 2);
            const int k = 8 * kKSteps * j + 8 * s + (lane & 3);
            float* dst = img.data() +
                         2 * (((size_t)q * KC + r) * (G::kStageBytes / 8) + (size_t)(w * kKSteps + s) * 32 + lane);
            dst[0] = w_of(L, n, k);
            dst[1] = w_of(L, n, k + 4);
          }
  }
  cudaError_t e = cudaMalloc(dev, img.size() * sizeof(float));
  if (e == cudaSuccess) e = cudaMemcpy(*dev, img.data(), img.size() * sizeof(float), cudaMemcpyHostToDevice);
  return e;
}

cudaError_t fp32_pack_cluster(const float* P, int d_in, int F, int n_blocks, int n_coarse, int n_fine, int cluster,
                              float** dev) {
  return cluster == 8 ? pack_guard<8>(P, d_in, F, n_blocks, n_coarse, n_fine, dev)
                      : pack_guard<4>(P, d_in, F, n_blocks, n_coarse, n_fine, dev);
}

}  // namespace nedf
