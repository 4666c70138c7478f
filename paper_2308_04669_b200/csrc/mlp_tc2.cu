// CTA-pair (cta_group::2) version of the fused NeDF network kernel.
//
// Same roles and dataflow as mlp_tc.cu, but two SMs of a cluster cooperate on
// a 256-ray super-tile: CTA r owns rays [128r, 128r+128) (its TMEM holds their
// accumulators, fp16 activations and its registers their fp32 residuals), and
// each MMA instruction is M = 256.  The weight operand is split by output
// columns, so each SM ingests only half of every weight stage -- the per-SM
// bulk-copy stream that limited the single-CTA kernel (~55 of ~71 B/cycle)
// drops to ~28 B/cycle -- and the even CTA issues half as many MMA
// instructions per ray.
//
// Cross-CTA synchronisation:
//   weights   each CTA's producer lane j streams its half into slot j; the odd
//             CTA relays completion to the even CTA's peer_full[j]
//   encoding  the odd CTA's encoders arrive remotely on the even CTA's enc_full
//   epilogue  the odd CTA's epilogue warps arrive remotely on epi_done
//   MMA done  tcgen05.commit ... multicast::cluster releases both CTAs
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

constexpr int kThreads = 512;
constexpr int kUnitBytes = 8192;           // one ring slot: [64 weight rows x 64 K] fp16, SW128
constexpr int kRing = 16;
constexpr int kEncStages = 2;
constexpr int kEncBytes = 16384;           // [128 rows x 64 K] fp16
constexpr int kHeadUnits = 32;             // per CTA: 16 points x [128 x 64] = 2 units each
constexpr int kLayerUnits = 8;             // 2 N slices x 4 K chunks
constexpr int kBodyLayers = 32;
constexpr int kUnitsPerTile = kHeadUnits + (kBodyLayers + 1) * kLayerUnits;   // 296
constexpr int kImageStageBytes = 16384;    // image layout (mlp_tc.cu): 16 KB stages
constexpr int kImageHeadStages = 32;       // image layout (mlp_tc.cu): 16 KB stages
constexpr int kBiasLayers = kBodyLayers + 2;
constexpr int kBiasBytes = kBiasLayers * 256 * 4;
constexpr uint32_t kAccCol = 0, kAPCol = 256, kAQCol = 384;

struct __align__(16) RowRed {
  float fbest, fsecond, cbest, csecond;
  float maxabs, alpha;
  int fidx, cidx;
};

struct PairShared {
  uint64_t full[kRing], peer_full[kRing], empty[kRing];
  uint64_t enc_full[kEncStages], enc_empty[kEncStages];
  uint64_t acc_full[2], epi_done[2];
  uint32_t tmem_base;
  int tiles[65];
  RowRed red[128][2];
};

constexpr size_t kSmemBytes =
    1024 + kRing * kUnitBytes + kEncStages * kEncBytes + kBiasBytes + sizeof(PairShared);

// super-tile t of 256 rays -> this CTA's 128-row half
__device__ __forceinline__ void pair_tile(const int* tiles, int ng, int t, const ListSet& ls, uint32_t rank,
                                          int& g, int64_t& base, int& n) {
  g = 0;
  while (g < ng - 1 && t >= tiles[g + 1]) ++g;
  const int lt = t - tiles[g];
  const int first = lt * 256 + 128 * (int)rank;
  n = ls.count[g] - first;
  n = n < 0 ? 0 : (n < 128 ? n : 128);
  base = ls.offset[g] + first;
}

__device__ __forceinline__ void top2_push(float v, int col, float& best, float& second, int& idx) {
  if (v > best) {
    second = best;
    best = v;
    idx = col;
  } else if (v > second) {
    second = v;
  }
}

__device__ __forceinline__ void encode_coord_tc(double p, float out[21]) {
  const float ph = (float)p;
  const float pl = (float)(p - (double)ph);
  out[0] = ph;
#pragma unroll
  for (int base = 0; base < kLevels; base += 5) {
    float r;
    if (base == 0) {
      r = ph + pl;
    } else {
      const float t = ph * 32.0f;
      r = fmaf(-2.0f, rintf(0.5f * t), t) + 32.0f * pl;
    }
    float s, c;
    __sincosf(3.14159265358979f * r, &s, &c);
    out[1 + 2 * base] = s;
    out[2 + 2 * base] = c;
#pragma unroll
    for (int k = base + 1; k < base + 5; ++k) {
      const float s2 = 2.0f * s * c;
      const float c2 = (c - s) * (c + s);
      s = s2;
      c = c2;
      out[1 + 2 * k] = s;
      out[2 + 2 * k] = c;
    }
  }
}

}  // namespace

// optional wait accounting for cluster 0's second tile (diagnostics, nedf_diag_tc2_trace):
// [0..3] MMA cycles waiting on full / peer_full / epi_done / enc_full, [4] MMA tile cycles,
// [8+r] producer lane 0 of CTA r waiting on empty, [10] follower relay wait on full,
// [12+r] encoder warp 4 of CTA r waiting on enc_empty, [14+r] encoder tile cycles,
// [16+r] epilogue warp 8 of CTA r waiting on acc_full, [18+r] epilogue tile cycles
// timing experiments only (results invalid): 1 = skip the peer_full relay wait, 2 = leader ignores the odd
// CTA's epilogue
#ifndef NEDF_PAIR_EXP
#define NEDF_PAIR_EXP 0
#endif
__device__ unsigned long long g_tc2_trace[512];
__device__ int g_tc2_trace_on;

__device__ __forceinline__ void twait(uint64_t* bar, uint32_t ph, bool tr, unsigned long long& acc) {
  if (tr) {
    const long long t0 = clock64();
    tc::mbar_wait(bar, ph);
    acc += clock64() - t0;
  } else {
    tc::mbar_wait(bar, ph);
  }
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1) nedf_mlp_tc2_kernel(TcArgs a) {
  extern __shared__ unsigned char smem_raw[];
  // align by offsetting the shared array itself (not via an integer round trip), so the compiler
  // keeps the shared address space and emits LDS/STS instead of generic loads/stores
  unsigned char* smem = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);
  unsigned char* ring = smem;
  unsigned char* enc = ring + kRing * kUnitBytes;
  float* bias_s = reinterpret_cast<float*>(enc + kEncStages * kEncBytes);
  PairShared& S = *reinterpret_cast<PairShared*>(enc + kEncStages * kEncBytes + kBiasBytes);

  const int tid = threadIdx.x;
  const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);
  const int lane = tid & 31;
  const uint32_t rank = tc::cluster_rank();
  const int cluster = blockIdx.x >> 1, n_clusters = gridDim.x >> 1;
  const ListSet& ls = a.ls;
  const int ng = ls.n_groups < 64 ? ls.n_groups : 64;

  if (tid == 0) {
    int cum = 0;
    S.tiles[0] = 0;
    for (int g = 0; g < ng; ++g) {
      cum += (ls.count[g] + 255) / 256;
      S.tiles[g + 1] = cum;
    }
    for (int i = 0; i < kRing; ++i) {
      tc::mbar_init(&S.full[i], 1);
      tc::mbar_init(&S.peer_full[i], 1);
      tc::mbar_init(&S.empty[i], 1);
    }
    for (int i = 0; i < kEncStages; ++i) { tc::mbar_init(&S.enc_full[i], 8); tc::mbar_init(&S.enc_empty[i], 1); }
    for (int i = 0; i < 2; ++i) { tc::mbar_init(&S.acc_full[i], 1); tc::mbar_init(&S.epi_done[i], (NEDF_PAIR_EXP & 2) ? 8 : 16); }
    tc::mbar_fence_init();
  }
  if (warp == 1) tc::tmem_alloc2<512>(&S.tmem_base);
  tc::tc_fence_before();
  tc::cluster_sync();
  tc::tc_fence_after();
  const uint32_t tbase = S.tmem_base;
  const int total_tiles = S.tiles[ng];

  if (warp < 4) {
    tc::reg_dealloc<40>();
    if (warp == 0) {
      // ------------------------------------------------------------------ producer (both CTAs)
      if (lane < kRing) {
        // lane j owns ring slot j and streams every unit u of the global sequence with u = j (mod kRing)
        const int slot = lane;
        uint32_t phase = 0;
        const uint32_t peer_bar = tc::peer_addr(&S.peer_full[slot], 0);
        uint32_t gbase = 0;
        int ti = 0;
        for (int t = cluster; t < total_tiles; t += n_clusters, ++ti) {
          const bool tr = g_tc2_trace_on && cluster == 0 && ti == 1 && slot == 0;
          unsigned long long w_empty = 0, w_relay = 0;
          int g, n;
          int64_t base;
          pair_tile(S.tiles, ng, t, ls, rank, g, base, n);
          const unsigned char* w = reinterpret_cast<const unsigned char*>(a.gt.models[g].wpack);
          for (int i = (slot - (int)(gbase % kRing) + kRing) % kRing; i < kUnitsPerTile; i += kRing) {
            twait(&S.empty[slot], phase ^ 1, tr, w_empty);
            // head unit i: half (i & 1) of this CTA's 128 weight rows of point i >> 1 (image stage 2c + rank);
            // body unit: this CTA's 64 rows of the slice's [128 x 64] image stage
            const unsigned char* src =
                i < kHeadUnits
                    ? w + (size_t)(2 * (i >> 1) + rank) * kImageStageBytes + (i & 1) * kUnitBytes
                    : w + (size_t)(2 * 16 + (i - kHeadUnits)) * kImageStageBytes + rank * kUnitBytes;
            tc::mbar_expect_tx(&S.full[slot], kUnitBytes);
            tc::bulk_g2s(ring + slot * kUnitBytes, src, kUnitBytes, &S.full[slot]);
            if (rank == 1) {                // relay to the MMA issuer in the even CTA
              twait(&S.full[slot], phase, tr, w_relay);
              tc::mbar_arrive_remote(peer_bar);
            }
            phase ^= 1;
          }
          gbase += kUnitsPerTile;
          if (tr) {
            g_tc2_trace[8 + rank] = w_empty;
            if (rank == 1) g_tc2_trace[10] = w_relay;
          }
        }
      }
      __syncwarp();
    } else if (warp == 1 && rank == 0) {
      // ------------------------------------------------------------------ MMA issuer (even CTA)
      uint32_t gs = 0;
      uint32_t layer_ctr = 0, ephase = 0;
      int es = 0;
      const uint32_t id256 = tc::idesc_f16(256, 256), id128 = tc::idesc_f16(256, 128);
      const uint32_t ring_s = tc::smem_u32(ring), enc_s = tc::smem_u32(enc);
      int ti = 0;
      const long long t_kernel = clock64();
      unsigned long long ns0;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ns0));
      for (int t = cluster; t < total_tiles; t += n_clusters, ++ti) {
        const bool tr = g_tc2_trace_on && cluster == 0 && ti == 1;
        unsigned long long wf = 0, wp = 0, we = 0, wn = 0;
        const long long t_tile = clock64();
        if (tr && lane == 0) { g_tc2_trace[63] = t_tile; g_tc2_trace[64] = t_tile; }
        if (layer_ctr > 0) {
          twait(&S.epi_done[0], (layer_ctr - 1) & 1, tr, we);
          twait(&S.epi_done[1], (layer_ctr - 1) & 1, tr, we);
        }
        for (int c = 0; c < 16; ++c) {           // head (SS, N = 256: 128 weight rows per CTA)
          const uint32_t slot = gs % kRing, ph = (gs / kRing) & 1;   // gs even: units in slots slot, slot + 1
          twait(&S.enc_full[es], ephase, tr, wn);
          twait(&S.full[slot], ph, tr, wf);
          twait(&S.full[slot + 1], ph, tr, wf);
          if (!(NEDF_PAIR_EXP & 1)) {
            twait(&S.peer_full[slot], ph, tr, wp);
            twait(&S.peer_full[slot + 1], ph, tr, wp);
          }
          tc::tc_fence_after();
          const uint32_t a0 = enc_s + es * kEncBytes, b0 = ring_s + slot * kUnitBytes;
          if (tc::elect_one()) {
#pragma unroll
            for (int k = 0; k < 4; ++k)
              tc::mma2_ss(tbase + kAccCol, tc::sw128_desc(a0 + k * 32), tc::sw128_desc(b0 + k * 32), id256,
                          (c | k) ? 1u : 0u);
            tc::mma2_commit_both(&S.empty[slot]);
            tc::mma2_commit_both(&S.empty[slot + 1]);
            tc::mma2_commit_both(&S.enc_empty[es]);
          }
          __syncwarp();
          gs += 2;
          if (++es == kEncStages) { es = 0; ephase ^= 1; }
        }
        if (tc::elect_one()) {
          tc::mma2_commit_both(&S.acc_full[0]);
          tc::mma2_commit_both(&S.acc_full[1]);
        }
        __syncwarp();
        if (tr && lane == 0) g_tc2_trace[100] = clock64();
        ++layer_ctr;
        for (int L = 1; L <= kBodyLayers + 1; ++L) {     // body + tail (TS, N = 128 per slice: 64 rows per CTA)
          if (tr && lane == 0) g_tc2_trace[64 + L] = clock64();
          const uint32_t a_col = (L & 1) ? kAPCol : kAQCol;
          const uint32_t par = (layer_ctr - 1) & 1;
          twait(&S.epi_done[0], par, tr, we);
          bool have1 = false;
#pragma unroll 1
          for (int s = 0; s < 2; ++s) {
#pragma unroll 1
            for (int kc = 0; kc < 4; ++kc) {
              if (!have1 && (kc >= 2 || s == 1)) {
                twait(&S.epi_done[1], par, tr, we);
                have1 = true;
              }
              const uint32_t slot = gs % kRing, ph = (gs / kRing) & 1;
              twait(&S.full[slot], ph, tr, wf);
              if (!(NEDF_PAIR_EXP & 1)) twait(&S.peer_full[slot], ph, tr, wp);
              tc::tc_fence_after();
              const uint32_t b0 = ring_s + slot * kUnitBytes;
              const uint32_t ac = tbase + a_col + kc * 32;
              if (tc::elect_one()) {
#pragma unroll
                for (int k = 0; k < 4; ++k)
                  tc::mma2_ts(tbase + kAccCol + 128 * s, ac + k * 8, tc::sw128_desc(b0 + k * 32), id128,
                              (kc | k) ? 1u : 0u);
                tc::mma2_commit_both(&S.empty[slot]);
                if (kc == 3) tc::mma2_commit_both(&S.acc_full[s]);
              }
              __syncwarp();
              ++gs;
            }
          }
          if (tr && lane == 0) g_tc2_trace[100 + L] = clock64();
          ++layer_ctr;
        }
        if (tr && lane == 0) {
          g_tc2_trace[0] = wf; g_tc2_trace[1] = wp; g_tc2_trace[2] = we; g_tc2_trace[3] = wn;
          g_tc2_trace[4] = clock64() - t_tile;
        }
      }
      if (g_tc2_trace_on && cluster == 0 && lane == 0) {
        unsigned long long ns1;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ns1));
        g_tc2_trace[5] = clock64() - t_kernel;
        g_tc2_trace[6] = ti;
        g_tc2_trace[7] = ns1 - ns0;
      }
    }
  } else if (warp < 8) {
    tc::reg_dealloc<104>();
    // -------------------------------------------------------------------- encoders (both CTAs)
    const int row = tid - 128;
    int es = 0;
    uint32_t ephase = 0;
    const uint32_t leader_enc_full0 = tc::peer_addr(&S.enc_full[0], 0);
    int ti = 0;
    for (int t = cluster; t < total_tiles; t += n_clusters, ++ti) {
      const bool tr = g_tc2_trace_on && cluster == 0 && ti == 1 && tid == 128;
      unsigned long long wq = 0;
      const long long t_tile = clock64();
      int g, n;
      int64_t base;
      pair_tile(S.tiles, ng, t, ls, rank, g, base, n);
      const DevModel& m = a.gt.models[g];
      const bool valid = row < n;
      double pa[3] = {0, 0, 0}, pb[3] = {0, 0, 0}, t0 = 0, t1 = 0;
      if (valid) {
        double wo[3], wd[3], lo[3], ld[3];
        item_local_ray(a.job, ls.pix[base + row], ls.obj[base + row], wo, wd, lo, ld);
        slab_clip(lo, ld, m.bmin, m.bmax, t0, t1);
#pragma unroll
        for (int ax = 0; ax < 3; ++ax) {
          pa[ax] = (lo[ax] - m.c[ax]) / m.h[ax];
          pb[ax] = ld[ax] / m.h[ax];
        }
      }
      for (int pt = 0; pt < 16; ++pt) {
        uint32_t packed[32];
        if (valid) {
          const double tt = t0 + (t1 - t0) * lin16(pt);
          float f[64];
#pragma unroll
          for (int ax = 0; ax < 3; ++ax) {
            float e[21];
            encode_coord_tc(pa[ax] + tt * pb[ax], e);
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
        twait(&S.enc_empty[es], ephase ^ 1, tr, wq);
        unsigned char* dst = enc + es * kEncBytes;
#pragma unroll
        for (int j = 0; j < 8; ++j)
          *reinterpret_cast<uint4*>(dst + tc::sw128_offset(row, j)) =
              make_uint4(packed[4 * j], packed[4 * j + 1], packed[4 * j + 2], packed[4 * j + 3]);
        tc::fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive_remote(leader_enc_full0 + es * (uint32_t)sizeof(uint64_t));
        if (++es == kEncStages) { es = 0; ephase ^= 1; }
      }
      if (tr) {
        g_tc2_trace[12 + rank] = wq;
        g_tc2_trace[14 + rank] = clock64() - t_tile;
      }
    }
  } else {
    tc::reg_alloc<184>();
    // -------------------------------------------------------------------- epilogue (both CTAs)
    const int ew = warp - 8;
    const int q = warp & 3;
    const int hc = ew >> 2;
    const int row = 32 * q + lane;
    const uint32_t lane_addr = tbase + ((uint32_t)(32 * q) << 16);
    const uint32_t leader_epi0 = tc::peer_addr(&S.epi_done[0], 0);
    uint32_t layer_ctr = 0;
    const float* cached_bias = nullptr;
    float x[2][2][32];
    int ti = 0;
    for (int t = cluster; t < total_tiles; t += n_clusters, ++ti) {
      const bool tr = g_tc2_trace_on && cluster == 0 && ti == 1 && tid == 256;
      unsigned long long wa = 0;
      const long long t_tile = clock64();
      int g, n;
      int64_t base;
      pair_tile(S.tiles, ng, t, ls, rank, g, base, n);
      const DevModel& m = a.gt.models[g];
      if (m.bias_pack != cached_bias) {
        const float4* src = reinterpret_cast<const float4*>(m.bias_pack);
        float4* dst = reinterpret_cast<float4*>(bias_s);
        for (int i = tid - 256; i < kBiasLayers * 64; i += 256) dst[i] = __ldg(src + i);
        cached_bias = m.bias_pack;
        tc::named_bar(1, 256);
      }
      const uint32_t layer0 = layer_ctr;
      const bool tr0 = tr && rank == 0;
      auto release = [&](int s) {          // slice s of this CTA's accumulator / A operand is done
        tc::tc_fence_before();
        __syncwarp();
        if (lane == 0 && (!(NEDF_PAIR_EXP & 2) || rank == 0))
          tc::mbar_arrive_remote(leader_epi0 + s * (uint32_t)sizeof(uint64_t));
        if (tr0) g_tc2_trace[204 + 2 * (layer_ctr - layer0) + s] = clock64();
      };
      // ---- head: x = acc + b ----
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        twait(&S.acc_full[s], layer_ctr & 1, tr, wa);
        if (tr0) g_tc2_trace[136 + 2 * (layer_ctr - layer0) + s] = clock64();
        tc::tc_fence_after();
#pragma unroll
        for (int j2 = 0; j2 < 2; ++j2) {
          const int col = 128 * s + 64 * hc + 32 * j2;
          const float4* b4 = reinterpret_cast<const float4*>(bias_s + col);
          uint32_t v[32];
          tc::tmem_ld32(lane_addr + kAccCol + col, v);
          tc::tmem_ld_wait();
          uint32_t pk[16];
#pragma unroll
          for (int j4 = 0; j4 < 8; ++j4) {
            const float4 b = b4[j4];
            x[s][j2][4 * j4 + 0] = __uint_as_float(v[4 * j4 + 0]) + b.x;
            x[s][j2][4 * j4 + 1] = __uint_as_float(v[4 * j4 + 1]) + b.y;
            x[s][j2][4 * j4 + 2] = __uint_as_float(v[4 * j4 + 2]) + b.z;
            x[s][j2][4 * j4 + 3] = __uint_as_float(v[4 * j4 + 3]) + b.w;
          }
#pragma unroll
          for (int j = 0; j < 16; ++j) pk[j] = tc::pack_h2(x[s][j2][2 * j], x[s][j2][2 * j + 1]);
          tc::tmem_st16(lane_addr + kAPCol + col / 2, pk);
        }
        tc::tmem_st_wait();
        release(s);
      }
      ++layer_ctr;
      for (int blk = 0; blk < kBodyLayers / 2; ++blk) {
        const float* b1 = bias_s + (1 + 2 * blk) * 256;
        const float* b2 = b1 + 256;
#pragma unroll
        for (int s = 0; s < 2; ++s) {     // fc1: h = relu(acc + b1) -> A_Q
          twait(&S.acc_full[s], layer_ctr & 1, tr, wa);
        if (tr0) g_tc2_trace[136 + 2 * (layer_ctr - layer0) + s] = clock64();
          tc::tc_fence_after();
#pragma unroll
          for (int j2 = 0; j2 < 2; ++j2) {
            const int col = 128 * s + 64 * hc + 32 * j2;
            const float4* b4 = reinterpret_cast<const float4*>(b1 + col);
            uint32_t v[32];
            tc::tmem_ld32(lane_addr + kAccCol + col, v);
            tc::tmem_ld_wait();
            uint32_t pk[16];
#pragma unroll
            for (int j4 = 0; j4 < 8; ++j4) {
              const float4 b = b4[j4];
              pk[2 * j4 + 0] =
                  tc::pack_h2_relu(__uint_as_float(v[4 * j4 + 0]) + b.x, __uint_as_float(v[4 * j4 + 1]) + b.y);
              pk[2 * j4 + 1] =
                  tc::pack_h2_relu(__uint_as_float(v[4 * j4 + 2]) + b.z, __uint_as_float(v[4 * j4 + 3]) + b.w);
            }
            tc::tmem_st16(lane_addr + kAQCol + col / 2, pk);
          }
          tc::tmem_st_wait();
          release(s);
        }
        ++layer_ctr;
#pragma unroll
        for (int s = 0; s < 2; ++s) {     // fc2: x += relu(acc + b2) -> A_P = fp16(x)
          twait(&S.acc_full[s], layer_ctr & 1, tr, wa);
        if (tr0) g_tc2_trace[136 + 2 * (layer_ctr - layer0) + s] = clock64();
          tc::tc_fence_after();
#pragma unroll
          for (int j2 = 0; j2 < 2; ++j2) {
            const int col = 128 * s + 64 * hc + 32 * j2;
            const float4* b4 = reinterpret_cast<const float4*>(b2 + col);
            uint32_t v[32];
            tc::tmem_ld32(lane_addr + kAccCol + col, v);
            tc::tmem_ld_wait();
            uint32_t pk[16];
#pragma unroll
            for (int j4 = 0; j4 < 8; ++j4) {
              const float4 b = b4[j4];
              x[s][j2][4 * j4 + 0] += fmaxf(__uint_as_float(v[4 * j4 + 0]) + b.x, 0.f);
              x[s][j2][4 * j4 + 1] += fmaxf(__uint_as_float(v[4 * j4 + 1]) + b.y, 0.f);
              x[s][j2][4 * j4 + 2] += fmaxf(__uint_as_float(v[4 * j4 + 2]) + b.z, 0.f);
              x[s][j2][4 * j4 + 3] += fmaxf(__uint_as_float(v[4 * j4 + 3]) + b.w, 0.f);
            }
#pragma unroll
            for (int j = 0; j < 16; ++j) pk[j] = tc::pack_h2(x[s][j2][2 * j], x[s][j2][2 * j + 1]);
            tc::tmem_st16(lane_addr + kAPCol + col / 2, pk);
          }
          tc::tmem_st_wait();
          release(s);
        }
        ++layer_ctr;
      }
      // ---- tail: slice 0 = fine (128); slice 1 = coarse (cols 0-63), alpha (col 64) ----
      const float* bt = bias_s + (kBiasLayers - 1) * 256;
      float fbest = -INFINITY, fsecond = -INFINITY, cbest = -INFINITY, csecond = -INFINITY, maxabs = 0.f,
            alpha = 0.f;
      int fidx = 0, cidx = 0;
      bool finite = true;
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        twait(&S.acc_full[s], layer_ctr & 1, tr, wa);
        if (tr0) g_tc2_trace[136 + 2 * (layer_ctr - layer0) + s] = clock64();
        tc::tc_fence_after();
#pragma unroll
        for (int j2 = 0; j2 < 2; ++j2) {
          const int col = 128 * s + 64 * hc + 32 * j2;
          uint32_t v[32];
          tc::tmem_ld32(lane_addr + kAccCol + col, v);
          tc::tmem_ld_wait();
          if (j2 == 1) release(s);
          if (s == 1 && hc == 1) {
            if (j2 == 0) {
              alpha = __uint_as_float(v[0]) + bt[192];
              finite = finite && isfinite(alpha);
              maxabs = fmaxf(maxabs, fabsf(alpha));
              if (a.out.mode == OUT_LOGITS && row < n) a.out.la[ls.pix[base + row]] = alpha;
            }
            continue;
          }
          const float4* b4 = reinterpret_cast<const float4*>(bt + col);
#pragma unroll
          for (int j4 = 0; j4 < 8; ++j4) {
            const float4 b = b4[j4];
            const float vv[4] = {__uint_as_float(v[4 * j4]) + b.x, __uint_as_float(v[4 * j4 + 1]) + b.y,
                                 __uint_as_float(v[4 * j4 + 2]) + b.z, __uint_as_float(v[4 * j4 + 3]) + b.w};
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int c = col + 4 * j4 + u;
              finite = finite && isfinite(vv[u]);
              maxabs = fmaxf(maxabs, fabsf(vv[u]));
              if (s == 0) top2_push(vv[u], c, fbest, fsecond, fidx);
              else top2_push(vv[u], c - 128, cbest, csecond, cidx);
            }
            if (a.out.mode == OUT_LOGITS && row < n) {
              const size_t r = ls.pix[base + row];
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                const int c = col + 4 * j4 + u;
                if (s == 0) a.out.lf[r * 128 + c] = vv[u];
                else a.out.lc[r * 64 + c - 128] = vv[u];
              }
            }
          }
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
        float fb, fs;
        int fi;
        if (o.fbest > fbest) { fb = o.fbest; fi = o.fidx; fs = fmaxf(fmaxf(fbest, fsecond), o.fsecond); }
        else { fb = fbest; fi = fidx; fs = fmaxf(fmaxf(o.fbest, fsecond), o.fsecond); }
        const float al = o.alpha;
        const float S_ = fmaxf(rr.maxabs, o.maxabs);
        const float thr = a.guard * S_;
        const uint32_t pix = ls.pix[base + row], obj = ls.obj[base + row];
        const bool risky =
            a.use_guard && (!(S_ < INFINITY) || (fb - fs) < thr || (cbest - csecond) < thr || fabsf(al) < thr);
        if (a.out.mode == OUT_LOGITS) {
        } else if (risky) {
          const int at = atomicAdd(a.redo.count + g, 1);
          a.redo.pix[a.redo.offset[g] + at] = pix;
          a.redo.obj[a.redo.offset[g] + at] = obj;
        } else {
          double wo[3], wd[3], lo[3], ld[3];
          item_local_ray(a.job, pix, obj, wo, wd, lo, ld);
          finish_ray(m, a.job, a.out, pix, obj, cidx, fi, (double)al, wo, wd);
        }
      }
      tc::named_bar(1, 256);
      if (tr) {
        g_tc2_trace[16 + rank] = wa;
        g_tc2_trace[18 + rank] = clock64() - t_tile;
      }
    }
  }
  tc::tc_fence_before();
  tc::cluster_sync();
  if (warp == 1) tc::tmem_dealloc2<512>(tbase);
}

}  // namespace nedf

extern "C" int nedf_diag_tc2_trace(int enable, unsigned long long* out, int n) {
  using namespace nedf;
  if (enable >= 0) {
    int v = enable;
    if (cudaMemcpyToSymbol(g_tc2_trace_on, &v, sizeof(int)) != cudaSuccess) return NEDF_ERR_CUDA;
  }
  if (out && n > 0) {
    if (n > 512) n = 512;
    if (cudaMemcpyFromSymbol(out, g_tc2_trace, n * sizeof(unsigned long long)) != cudaSuccess) return NEDF_ERR_CUDA;
  }
  return NEDF_OK;
}

namespace nedf {

cudaError_t launch_mlp_tc2(const TcArgs& a, int n_ctas, cudaStream_t stream) {
  // persistent grid: never more clusters than can be co-resident (a GPC with an odd number of free
  // SMs leaves one idle), or the surplus clusters would run as a second wave
  static int max_clusters = 0;
  if (max_clusters == 0) {
    cudaError_t e = cudaFuncSetAttribute(nedf_mlp_tc2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)kSmemBytes);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2 * 74, 1, 1);
    cfg.blockDim = dim3(kThreads, 1, 1);
    cfg.dynamicSmemBytes = kSmemBytes;
    int n = 0;
    e = cudaOccupancyMaxActiveClusters(&n, nedf_mlp_tc2_kernel, &cfg);
    if (e != cudaSuccess) return e;
    max_clusters = n > 0 ? n : 1;
    if (getenv("NEDF_VERBOSE")) fprintf(stderr, "nedf: pair kernel, %d co-resident clusters\n", n);
  }
  n_ctas &= ~1;
  if (n_ctas > 2 * max_clusters) n_ctas = 2 * max_clusters;
  if (n_ctas < 2) n_ctas = 2;
  nedf_mlp_tc2_kernel<<<n_ctas, kThreads, kSmemBytes, stream>>>(a);
  return cudaGetLastError();
}

}  // namespace nedf
