// Fused, persistent tcgen05 evaluation of the NeDF intersection network
// (nn.py:115-135) for 128-ray tiles, with the ray encoding produced on chip
// and the decode / world depth / z-buffer update in the epilogue.
//
// Per CTA (one per SM), 16 warps:
//   warp 0        bulk-copy producer: streams the model's pre-swizzled fp16
//                 operand image (592 x 8 KB stages per tile) into a 16-stage ring
//   warp 1        MMA issuer (one thread) + TMEM owner
//   warps 4-7     encoders: thread = ray; float64 ray setup, 16 sample points,
//                 sinusoidal features -> fp16 A tiles (128B swizzle) in a 4-stage ring
//   warps 8-15    epilogue: thread = (ray, 32-column half of each 64-column slice);
//                 fp32 residual stream x[256] lives in registers (128 per thread)
//
// TMEM (512 columns): [0,256) fp32 accumulator as four 64-column slices,
// [256,384) A_P = fp16 x (input of fc1 and the tails), [384,512) A_Q = fp16 h
// (input of fc2).  Layers after the head use the TS form (A from TMEM).
//
// Wavefront: layer L+1's MMA for output slice s, K-slice k waits only for the
// epilogue of layer L's slice k, so the epilogue of slice k overlaps the MMAs
// of later slices.
//
// Precision guard: fp16 operands / fp32 accumulation perturb the logits by
// ~1e-3 relative; rays whose top-2 coarse or fine margin, or |alpha logit|,
// is below guard * max|logit| are appended to `redo` and re-evaluated by the
// fp32 kernel instead of being written here.
#include <cstdio>
#include <vector>

#include "common.cuh"
#include "encode.cuh"
#include "frame.cuh"
#include "tc_ptx.cuh"

namespace nedf {
namespace {

constexpr int kThreads = 512;
constexpr int kStageBytes = 8192;          // [64 N x 64 K] fp16, 128B swizzle
constexpr int kStages = 16;
constexpr int kEncStages = 4;
constexpr int kEncBytes = 16384;           // [128 rows x 64 K] fp16
constexpr int kHeadStages = 64;            // 16 K chunks x 4 N blocks
constexpr int kLayerStages = 16;           // 4 N slices x 4 K chunks
constexpr int kBodyLayers = 32;
constexpr int kStagesPerTile = kHeadStages + (kBodyLayers + 1) * kLayerStages;   // 592
constexpr int kBiasLayers = kBodyLayers + 2;                                     // 34
constexpr uint32_t kAccCol = 0, kAPCol = 256, kAQCol = 384;

struct __align__(16) RowRed {
  float fbest, fsecond, cbest, csecond;
  float maxabs, alpha;
  int fidx, cidx;
};

struct TcShared {
  uint64_t full[kStages], empty[kStages];
  uint64_t enc_full[kEncStages], enc_empty[kEncStages];
  uint64_t acc_full[4], epi_done[4];
  uint32_t tmem_base;
  int tiles[65];
  RowRed red[128][2];
};

constexpr size_t kSmemBytes = 1024 /*align slack*/ + kStages * kStageBytes + kEncStages * kEncBytes + sizeof(TcShared);

__device__ __forceinline__ void tile_lookup(const int* tiles, int ng, int t, const ListSet& ls, int& g,
                                            int64_t& base, int& n) {
  g = 0;
  while (g < ng - 1 && t >= tiles[g + 1]) ++g;
  int lt = t - tiles[g];
  n = ls.count[g] - lt * 128;
  n = n < 128 ? n : 128;
  base = ls.offset[g] + (int64_t)lt * 128;
}

// argmax bookkeeping: first maximum wins, `second` is the runner-up value
__device__ __forceinline__ void top2_push(float v, int col, float& best, float& second, int& idx) {
  if (v > best) {
    second = best;
    best = v;
    idx = col;
  } else if (v > second) {
    second = v;
  }
}

}  // namespace

__global__ void __launch_bounds__(kThreads, 1) nedf_mlp_tc_kernel(TcArgs a) {
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem =
      reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  unsigned char* ring = smem;
  unsigned char* enc = ring + kStages * kStageBytes;
  TcShared& S = *reinterpret_cast<TcShared*>(enc + kEncStages * kEncBytes);

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const ListSet& ls = a.ls;
  const int ng = ls.n_groups < 64 ? ls.n_groups : 64;

  if (tid == 0) {
    int cum = 0;
    S.tiles[0] = 0;
    for (int g = 0; g < ng; ++g) {
      cum += (ls.count[g] + 127) / 128;
      S.tiles[g + 1] = cum;
    }
    for (int i = 0; i < kStages; ++i) { tc::mbar_init(&S.full[i], 1); tc::mbar_init(&S.empty[i], 1); }
    for (int i = 0; i < kEncStages; ++i) { tc::mbar_init(&S.enc_full[i], 4); tc::mbar_init(&S.enc_empty[i], 1); }
    for (int i = 0; i < 4; ++i) { tc::mbar_init(&S.acc_full[i], 1); tc::mbar_init(&S.epi_done[i], 8); }
    tc::mbar_fence_init();
  }
  if (warp == 1) tc::tmem_alloc<512>(&S.tmem_base);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tbase = S.tmem_base;
  const int total_tiles = S.tiles[ng];

  if (warp < 4) {
    tc::reg_dealloc<40>();
    if (warp == 0 && lane == 0) {
      // ------------------------------------------------------------------ producer
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < total_tiles; t += gridDim.x) {
        int g, n;
        int64_t base;
        tile_lookup(S.tiles, ng, t, ls, g, base, n);
        const unsigned char* w = reinterpret_cast<const unsigned char*>(a.gt.models[g].wpack);
        for (int i = 0; i < kStagesPerTile; ++i) {
          tc::mbar_wait(&S.empty[stage], phase ^ 1);
          tc::mbar_expect_tx(&S.full[stage], kStageBytes);
          tc::bulk_g2s(ring + stage * kStageBytes, w + (size_t)i * kStageBytes, kStageBytes, &S.full[stage]);
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
      }
    } else if (warp == 1 && lane == 0) {
      // ------------------------------------------------------------------ MMA issuer
      int stage = 0, es = 0;
      uint32_t phase = 0, ephase = 0;
      uint32_t layer_ctr = 0;
      const uint32_t id256 = tc::idesc_f16(128, 256), id64 = tc::idesc_f16(128, 64);
      for (int t = blockIdx.x; t < total_tiles; t += gridDim.x) {
        // head: A = encoded rays (smem), B = W_head chunk [256 x 64]
        if (layer_ctr > 0)
          for (int s = 0; s < 4; ++s) tc::mbar_wait(&S.epi_done[s], (layer_ctr - 1) & 1);
        for (int c = 0; c < 16; ++c) {
          tc::mbar_wait(&S.enc_full[es], ephase);
          for (int j = 0; j < 4; ++j) tc::mbar_wait(&S.full[stage + j], phase);
          tc::tc_fence_after();
          const uint32_t a0 = tc::smem_u32(enc + es * kEncBytes);
          const uint32_t b0 = tc::smem_u32(ring + stage * kStageBytes);
#pragma unroll
          for (int k = 0; k < 4; ++k)
            tc::mma_ss(tbase + kAccCol, tc::sw128_desc(a0 + k * 32), tc::sw128_desc(b0 + k * 32), id256,
                       (c | k) ? 1u : 0u);
          for (int j = 0; j < 4; ++j) tc::mma_commit(&S.empty[stage + j]);
          tc::mma_commit(&S.enc_empty[es]);
          stage += 4;
          if (stage == kStages) { stage = 0; phase ^= 1; }
          if (++es == kEncStages) { es = 0; ephase ^= 1; }
        }
        for (int s = 0; s < 4; ++s) tc::mma_commit(&S.acc_full[s]);
        ++layer_ctr;
        // 32 residual-block layers + the fused tail (TS form, 64-column output slices)
        for (int L = 1; L <= kBodyLayers + 1; ++L) {
          const uint32_t a_col = (L & 1) ? kAPCol : (L == kBodyLayers + 1 ? kAPCol : kAQCol);
          const uint32_t par = (layer_ctr - 1) & 1;
          uint32_t waited = 0;
          for (int s = 0; s < 4; ++s) {
            if (!(waited & (1u << s))) { tc::mbar_wait(&S.epi_done[s], par); waited |= 1u << s; }
            for (int kc = 0; kc < 4; ++kc) {
              if (!(waited & (1u << kc))) { tc::mbar_wait(&S.epi_done[kc], par); waited |= 1u << kc; }
              tc::mbar_wait(&S.full[stage], phase);
              tc::tc_fence_after();
              const uint32_t b0 = tc::smem_u32(ring + stage * kStageBytes);
#pragma unroll
              for (int k = 0; k < 4; ++k)
                tc::mma_ts(tbase + kAccCol + 64 * s, tbase + a_col + kc * 32 + k * 8, tc::sw128_desc(b0 + k * 32),
                           id64, (kc | k) ? 1u : 0u);
              tc::mma_commit(&S.empty[stage]);
              if (++stage == kStages) { stage = 0; phase ^= 1; }
            }
            tc::mma_commit(&S.acc_full[s]);
          }
          ++layer_ctr;
        }
      }
    }
  } else if (warp < 8) {
    tc::reg_dealloc<104>();
    // -------------------------------------------------------------------- encoders
    const int row = tid - 128;
    int es = 0;
    uint32_t ephase = 0;
    for (int t = blockIdx.x; t < total_tiles; t += gridDim.x) {
      int g, n;
      int64_t base;
      tile_lookup(S.tiles, ng, t, ls, g, base, n);
      const DevModel& m = a.gt.models[g];
      const bool valid = row < n;
      double lo[3] = {0, 0, 0}, ld[3] = {0, 0, 0}, t0 = 0, t1 = 0;
      if (valid) {
        double wo[3], wd[3];
        item_local_ray(a.job, ls.pix[base + row], ls.obj[base + row], wo, wd, lo, ld);
        slab_clip(lo, ld, m.bmin, m.bmax, t0, t1);
      }
      for (int pt = 0; pt < 16; ++pt) {
        uint32_t packed[32];
        if (valid) {
          double tt = t0 + (t1 - t0) * lin16(pt);
          float f[64];
#pragma unroll
          for (int ax = 0; ax < 3; ++ax) {
            double p = ((lo[ax] + tt * ld[ax]) - m.c[ax]) / m.h[ax];
            float e[21];
            encode_coord_fast(p, e);
#pragma unroll
            for (int j = 0; j < 21; ++j) f[21 * ax + j] = e[j];
          }
          f[63] = 0.f;
#pragma unroll
          for (int j = 0; j < 32; ++j) packed[j] = tc::pack_h2(f[2 * j], f[2 * j + 1]);
        } else {
#pragma unroll
          for (int j = 0; j < 32; ++j) packed[j] = 0u;
        }
        tc::mbar_wait(&S.enc_empty[es], ephase ^ 1);
        unsigned char* dst = enc + es * kEncBytes;
#pragma unroll
        for (int j = 0; j < 8; ++j)
          *reinterpret_cast<uint4*>(dst + tc::sw128_offset(row, j)) =
              make_uint4(packed[4 * j], packed[4 * j + 1], packed[4 * j + 2], packed[4 * j + 3]);
        tc::fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&S.enc_full[es]);
        if (++es == kEncStages) { es = 0; ephase ^= 1; }
      }
    }
  } else {
    tc::reg_alloc<184>();
    // -------------------------------------------------------------------- epilogue
    const int ew = warp - 8;
    const int q = warp & 3;                 // TMEM lane quadrant of this warp
    const int hc = ew >> 2;                 // column half within each 64-column slice
    const int row = 32 * q + lane;
    const uint32_t lane_addr = tbase + ((uint32_t)(32 * q) << 16);
    uint32_t layer_ctr = 0;
    float x[4][32];
    for (int t = blockIdx.x; t < total_tiles; t += gridDim.x) {
      int g, n;
      int64_t base;
      tile_lookup(S.tiles, ng, t, ls, g, base, n);
      const DevModel& m = a.gt.models[g];
      const float* bias = m.bias_pack;
      // ---- head: x = acc + b ----
#pragma unroll
      for (int s = 0; s < 4; ++s) {
        const float4* b4 = reinterpret_cast<const float4*>(bias + 64 * s + 32 * hc);
        tc::mbar_wait(&S.acc_full[s], layer_ctr & 1);
        tc::tc_fence_after();
        uint32_t v[32];
        tc::tmem_ld32(lane_addr + kAccCol + 64 * s + 32 * hc, v);
        tc::tmem_ld_wait();
        uint32_t pk[16];
#pragma unroll
        for (int j4 = 0; j4 < 8; ++j4) {
          float4 b = __ldg(b4 + j4);
          x[s][4 * j4 + 0] = __uint_as_float(v[4 * j4 + 0]) + b.x;
          x[s][4 * j4 + 1] = __uint_as_float(v[4 * j4 + 1]) + b.y;
          x[s][4 * j4 + 2] = __uint_as_float(v[4 * j4 + 2]) + b.z;
          x[s][4 * j4 + 3] = __uint_as_float(v[4 * j4 + 3]) + b.w;
        }
#pragma unroll
        for (int j = 0; j < 16; ++j) pk[j] = tc::pack_h2(x[s][2 * j], x[s][2 * j + 1]);
        tc::tmem_st16(lane_addr + kAPCol + 32 * s + 16 * hc, pk);
        tc::tmem_st_wait();
        tc::tc_fence_before();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&S.epi_done[s]);
      }
      ++layer_ctr;
      // ---- residual blocks ----
      for (int blk = 0; blk < kBodyLayers / 2; ++blk) {
        const float* b1 = bias + (size_t)(1 + 2 * blk) * 256;
        const float* b2 = b1 + 256;
#pragma unroll
        for (int s = 0; s < 4; ++s) {     // fc1: h = relu(acc + b1) -> A_Q
          const float4* b4 = reinterpret_cast<const float4*>(b1 + 64 * s + 32 * hc);
          tc::mbar_wait(&S.acc_full[s], layer_ctr & 1);
          tc::tc_fence_after();
          uint32_t v[32];
          tc::tmem_ld32(lane_addr + kAccCol + 64 * s + 32 * hc, v);
          tc::tmem_ld_wait();
          uint32_t pk[16];
#pragma unroll
          for (int j4 = 0; j4 < 8; ++j4) {
            float4 b = __ldg(b4 + j4);
            pk[2 * j4 + 0] = tc::pack_h2_relu(__uint_as_float(v[4 * j4 + 0]) + b.x, __uint_as_float(v[4 * j4 + 1]) + b.y);
            pk[2 * j4 + 1] = tc::pack_h2_relu(__uint_as_float(v[4 * j4 + 2]) + b.z, __uint_as_float(v[4 * j4 + 3]) + b.w);
          }
          tc::tmem_st16(lane_addr + kAQCol + 32 * s + 16 * hc, pk);
          tc::tmem_st_wait();
          tc::tc_fence_before();
          __syncwarp();
          if (lane == 0) tc::mbar_arrive(&S.epi_done[s]);
        }
        ++layer_ctr;
#pragma unroll
        for (int s = 0; s < 4; ++s) {     // fc2: x += relu(acc + b2) -> A_P = fp16(x)
          const float4* b4 = reinterpret_cast<const float4*>(b2 + 64 * s + 32 * hc);
          tc::mbar_wait(&S.acc_full[s], layer_ctr & 1);
          tc::tc_fence_after();
          uint32_t v[32];
          tc::tmem_ld32(lane_addr + kAccCol + 64 * s + 32 * hc, v);
          tc::tmem_ld_wait();
          uint32_t pk[16];
#pragma unroll
          for (int j4 = 0; j4 < 8; ++j4) {
            float4 b = __ldg(b4 + j4);
            x[s][4 * j4 + 0] += fmaxf(__uint_as_float(v[4 * j4 + 0]) + b.x, 0.f);
            x[s][4 * j4 + 1] += fmaxf(__uint_as_float(v[4 * j4 + 1]) + b.y, 0.f);
            x[s][4 * j4 + 2] += fmaxf(__uint_as_float(v[4 * j4 + 2]) + b.z, 0.f);
            x[s][4 * j4 + 3] += fmaxf(__uint_as_float(v[4 * j4 + 3]) + b.w, 0.f);
          }
#pragma unroll
          for (int j = 0; j < 16; ++j) pk[j] = tc::pack_h2(x[s][2 * j], x[s][2 * j + 1]);
          tc::tmem_st16(lane_addr + kAPCol + 32 * s + 16 * hc, pk);
          tc::tmem_st_wait();
          tc::tc_fence_before();
          __syncwarp();
          if (lane == 0) tc::mbar_arrive(&S.epi_done[s]);
        }
        ++layer_ctr;
      }
      // ---- tail: fine = slices 0,1; coarse = slice 2; alpha = slice 3 column 0 ----
      const float* bt = bias + (size_t)(kBiasLayers - 1) * 256;
      float fbest = -INFINITY, fsecond = -INFINITY, cbest = -INFINITY, csecond = -INFINITY, maxabs = 0.f,
            alpha = 0.f;
      int fidx = 0, cidx = 0;
      bool finite = true;
#pragma unroll
      for (int s = 0; s < 4; ++s) {
        const float4* b4 = reinterpret_cast<const float4*>(bt + 64 * s + 32 * hc);
        tc::mbar_wait(&S.acc_full[s], layer_ctr & 1);
        tc::tc_fence_after();
        uint32_t v[32];
        tc::tmem_ld32(lane_addr + kAccCol + 64 * s + 32 * hc, v);
        tc::tmem_ld_wait();
        tc::tc_fence_before();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&S.epi_done[s]);
        if (s < 3) {
#pragma unroll
          for (int j4 = 0; j4 < 8; ++j4) {
            float4 b = __ldg(b4 + j4);
            float vv[4] = {__uint_as_float(v[4 * j4]) + b.x, __uint_as_float(v[4 * j4 + 1]) + b.y,
                           __uint_as_float(v[4 * j4 + 2]) + b.z, __uint_as_float(v[4 * j4 + 3]) + b.w};
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int col = 64 * s + 32 * hc + 4 * j4 + u;
              finite = finite && isfinite(vv[u]);
              maxabs = fmaxf(maxabs, fabsf(vv[u]));
              if (s < 2) top2_push(vv[u], col, fbest, fsecond, fidx);
              else top2_push(vv[u], col - 128, cbest, csecond, cidx);
            }
            if (a.out.mode == OUT_LOGITS && row < n) {   // diagnostics: raw logits
              const size_t r = ls.pix[base + row];
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                const int col = 64 * s + 32 * hc + 4 * j4 + u;
                if (s < 2) a.out.lf[r * 128 + col] = vv[u];
                else a.out.lc[r * 64 + col - 128] = vv[u];
              }
            }
          }
        } else if (hc == 0) {
          alpha = __uint_as_float(v[0]) + __ldg(bt + 192);
          finite = finite && isfinite(alpha);
          maxabs = fmaxf(maxabs, fabsf(alpha));
          if (a.out.mode == OUT_LOGITS && row < n) a.out.la[ls.pix[base + row]] = alpha;
        }
      }
      ++layer_ctr;
      RowRed rr;
      rr.fbest = fbest; rr.fsecond = fsecond; rr.cbest = cbest; rr.csecond = csecond;
      rr.maxabs = finite ? maxabs : INFINITY; rr.alpha = alpha; rr.fidx = fidx; rr.cidx = cidx;
      S.red[row][hc] = rr;
      tc::named_bar(1, 256);
      if (hc == 0 && row < n) {
        const RowRed o = S.red[row][1];
        // merge: larger value wins, equal values keep the lower column (ours for fine slice 0 vs 1
        // interleave is handled by comparing indices)
        auto merge = [](float b1, float s1, int i1, float b2, float s2, int i2, float& b, float& sec, int& idx) {
          if (b2 > b1 || (b2 == b1 && i2 < i1)) { b = b2; idx = i2; sec = fmaxf(fmaxf(b1, s1), s2); }
          else { b = b1; idx = i1; sec = fmaxf(fmaxf(b2, s1), s2); }
        };
        float fb, fs, cb, cs;
        int fi, ci;
        merge(fbest, fsecond, fidx, o.fbest, o.fsecond, o.fidx, fb, fs, fi);
        merge(cbest, csecond, cidx, o.cbest, o.csecond, o.cidx, cb, cs, ci);
        const float S_ = fmaxf(rr.maxabs, o.maxabs);
        const float thr = a.guard * S_;
        const uint32_t pix = ls.pix[base + row], obj = ls.obj[base + row];
        const bool risky = a.use_guard &&
                           (!(S_ < INFINITY) || (fb - fs) < thr || (cb - cs) < thr || fabsf(alpha) < thr);
        if (a.out.mode == OUT_LOGITS) {
          // diagnostics: logits already written
        } else if (risky) {
          int at = atomicAdd(a.redo.count + g, 1);
          a.redo.pix[a.redo.offset[g] + at] = pix;
          a.redo.obj[a.redo.offset[g] + at] = obj;
        } else {
          double wo[3], wd[3], lo[3], ld[3];
          item_local_ray(a.job, pix, obj, wo, wd, lo, ld);
          finish_ray(m, a.job, a.out, pix, obj, ci, fi, (double)alpha, wo, wd);
        }
      }
      tc::named_bar(1, 256);
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc<512>(tbase);
}

bool tc_available() { return true; }

cudaError_t launch_mlp_tc(const TcArgs& a, int n_ctas, cudaStream_t stream) {
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(nedf_mlp_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)kSmemBytes);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  nedf_mlp_tc_kernel<<<n_ctas, kThreads, kSmemBytes, stream>>>(a);
  return cudaGetLastError();
}

// Pack a paper-shaped model (d_feat 256, 16 blocks) into the stage image the
// kernel streams: head [16 K chunks][4 N blocks], then per layer
// [4 N slices][4 K chunks], each stage a 128B-swizzled [64 x 64] fp16 tile;
// tail rows = fine (0-127), coarse (128-191), alpha (192), zero padding.
cudaError_t tc_pack_weights(const float* P, int d_in, int F, int n_blocks, int n_coarse, int n_fine,
                            __half** wpack_dev, float** bias_dev, size_t* bytes) {
  if (F != 256 || n_blocks != kBodyLayers / 2 || d_in != kDin || n_coarse != 64 || n_fine != 128)
    return cudaErrorInvalidValue;
  std::vector<__half> img((size_t)kStagesPerTile * kStageBytes / 2, __float2half(0.f));
  std::vector<float> bias((size_t)kBiasLayers * 256, 0.f);
  auto put = [&](int stage, int r, int k, float v) {
    size_t off = (size_t)stage * kStageBytes + tc::sw128_offset(r, k >> 3) + (k & 7) * 2;
    img[off / 2] = __float2half_rn(v);
  };
  // parameter offsets in file order
  size_t p = 0;
  const float* Wh = P + p; p += (size_t)F * d_in;
  const float* bh = P + p; p += F;
  std::vector<const float*> Wl(kBodyLayers), bl(kBodyLayers);
  for (int l = 0; l < kBodyLayers; ++l) { Wl[l] = P + p; p += (size_t)F * F; bl[l] = P + p; p += F; }
  const float* Wa = P + p; p += (size_t)(n_coarse + 1) * F;
  const float* ba = P + p; p += n_coarse + 1;
  const float* Wb = P + p; p += (size_t)n_fine * F;
  const float* bb = P + p; p += n_fine;
  // head
  for (int c = 0; c < 16; ++c)
    for (int nb = 0; nb < 4; ++nb)
      for (int r = 0; r < 64; ++r)
        for (int k = 0; k < 63; ++k) put(4 * c + nb, r, k, Wh[(size_t)(64 * nb + r) * d_in + 63 * c + k]);
  for (int o = 0; o < F; ++o) bias[o] = bh[o];
  // body
  for (int l = 0; l < kBodyLayers; ++l) {
    int st0 = kHeadStages + l * kLayerStages;
    for (int s = 0; s < 4; ++s)
      for (int kc = 0; kc < 4; ++kc)
        for (int r = 0; r < 64; ++r)
          for (int k = 0; k < 64; ++k) put(st0 + 4 * s + kc, r, k, Wl[l][(size_t)(64 * s + r) * F + 64 * kc + k]);
    for (int o = 0; o < F; ++o) bias[(size_t)(1 + l) * 256 + o] = bl[l][o];
  }
  // tail
  auto tail_row = [&](int n) -> const float* {
    if (n < 128) return Wb + (size_t)n * F;
    if (n < 128 + n_coarse + 1) return Wa + (size_t)(n - 128) * F;
    return nullptr;
  };
  int st0 = kHeadStages + kBodyLayers * kLayerStages;
  for (int s = 0; s < 4; ++s)
    for (int kc = 0; kc < 4; ++kc)
      for (int r = 0; r < 64; ++r) {
        const float* w = tail_row(64 * s + r);
        if (!w) continue;
        for (int k = 0; k < 64; ++k) put(st0 + 4 * s + kc, r, k, w[64 * kc + k]);
      }
  float* bt = bias.data() + (size_t)(kBiasLayers - 1) * 256;
  for (int o = 0; o < 128; ++o) bt[o] = bb[o];
  for (int o = 0; o < n_coarse + 1; ++o) bt[128 + o] = ba[o];
  *bytes = img.size() * sizeof(__half);
  cudaError_t e = cudaMalloc(wpack_dev, *bytes);
  if (e == cudaSuccess) e = cudaMalloc(bias_dev, bias.size() * sizeof(float));
  if (e == cudaSuccess) e = cudaMemcpy(*wpack_dev, img.data(), *bytes, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(*bias_dev, bias.data(), bias.size() * sizeof(float), cudaMemcpyHostToDevice);
  return e;
}

}  // namespace nedf
