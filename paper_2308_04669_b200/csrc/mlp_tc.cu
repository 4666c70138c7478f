// Fused, persistent tcgen05 evaluation of the NeDF intersection network
// (nn.py:115-135) for 128-ray tiles, with the ray encoding produced on chip
// and the decode / world depth / z-buffer update in the epilogue.
//
// Per CTA (one per SM), 16 warps in four warpgroups:
//   warp 0        bulk-copy producer: streams the model's pre-swizzled fp16
//                 operand image (296 x 16 KB stages per tile) into a 10-slot ring;
//                 lane j owns slot j.  In clusters of csize CTAs (default 2) each
//                 CTA fetches 1/csize of every stage and multicasts it to all
//   warp 1        MMA issuer (warp-uniform loop, elect.sync issues) + TMEM owner
//   warps 4-7     encoders: thread = ray; float64 ray setup, 16 sample points,
//                 sinusoidal features -> fp16, stored with tcgen05.st straight into
//                 TMEM (4-point ring in the A_Q columns, free during the head)
//   warps 8-15    epilogue: thread = (ray, 64-column half of each 128-column slice);
//                 the fp32 residual stream x[256] lives in registers (128 per thread)
//
// TMEM (512 columns): [0,256) fp32 accumulator as two 128-column slices,
// [256,384) A_P = fp16 x (input of fc1 and of the tails), [384,512) A_Q = fp16 h
// (input of fc2; the encoded head points before layer 1).  Every layer uses the
// TS form (A in TMEM): head M128 x N256 per point chunk, body and tail
// M128 x N128 per slice (86% of the nominal tcgen05 rate measured at N = 128).
//
// Wavefront: layer L+1's MMAs for K chunks 0-1 depend only on the epilogue of
// layer L's slice 0, so that epilogue overlaps the MMAs of slice 1, and the
// epilogue of slice 1 overlaps the first half of layer L+1.
//
// Synchronisation cost: one tcgen05.commit releases a pair of weight slots, and
// in the body it is issued after the next stage's wait together with that
// stage's MMAs -- each commit -> wait round costs the tensor pipe a bubble
// (scripts/mma_contention.py).  The head's encoders learn that a point slot is
// free from the same pair barriers.
//
// Precision guard: fp16 operands / fp32 accumulation perturb the logits by up
// to ~1.2e-3 of max|logit| (scripts/tc_calibrate.py); rays whose top-2 coarse
// or fine margin, or |alpha logit|, is below guard * max|logit| are appended
// to `redo` and re-evaluated by the fp32 kernel instead of being written here.
#include <cstdio>
#include <vector>

#include "common.cuh"
#include "encode.cuh"
#include "frame.cuh"
#include "tc_ptx.cuh"

namespace nedf {
namespace {

constexpr int kThreads = 512;
constexpr int kStageBytes = 16384;         // [128 N x 64 K] fp16, 128B swizzle
constexpr int kStages = 10;                // even: a head point's two stages sit in adjacent slots
constexpr int kEncSlots = 4;               // encoded head A tiles live in TMEM (A_Q columns, 32 per point)
constexpr int kHeadStages = 32;            // 16 points x [256 N x 64 K] (two stages each)
constexpr int kLayerStages = 8;            // 2 N slices x 4 K chunks
constexpr int kBodyLayers = 32;
constexpr int kStagesPerTile = kHeadStages + (kBodyLayers + 1) * kLayerStages;   // 296
constexpr int kBiasLayers = kBodyLayers + 2;                                     // 34
constexpr int kBiasBytes = kBiasLayers * 256 * 4;
constexpr uint32_t kAccCol = 0, kAPCol = 256, kAQCol = 384;

struct __align__(16) RowRed {
  float fbest, fsecond, cbest, csecond;
  float maxabs, alpha;
  int fidx, cidx;
};

struct TcShared {
  uint64_t full[kStages], empty[kStages];
  uint64_t enc_full[kEncSlots];   // point slot filled (4 encoder warps); emptied via the weight-pair barriers
  uint64_t aq_free;              // layer 32's MMAs (last readers of A_Q) completed: the next head may write A_Q
  uint64_t acc_full[2], epi_done[2];
  uint32_t tmem_base;
  int tiles[65];
  RowRed red[128][2];
  int2 frange[128];               // STEP 3 near-ties: fine-bin candidate range of columns 64-127
};

constexpr size_t kSmemBytes =
    1024 /*align slack*/ + kStages * kStageBytes + kBiasBytes + sizeof(TcShared);

// cluster tile t = (128 * csize) rays of one group; this CTA (cluster rank r) takes rows [128 r, 128 r + 128)
__device__ __forceinline__ void tile_lookup(const int* tiles, int ng, int t, const ListSet& ls, int csize,
                                            uint32_t rank, int& g, int64_t& base, int& n) {
  g = 0;
  while (g < ng - 1 && t >= tiles[g + 1]) ++g;
  const int first = (t - tiles[g]) * 128 * csize + 128 * (int)rank;
  n = ls.count[g] - first;
  n = n < 0 ? 0 : (n < 128 ? n : 128);
  base = ls.offset[g] + first;
}

// argmax bookkeeping: first maximum wins, `second` is the runner-up value
// (branch-free: v > best moves best to second; v <= best makes second max(second, v); NaN changes nothing)
__device__ __forceinline__ void top2_push(float v, int col, float& best, float& second, int& idx) {
  const bool up = v > best;
  second = fmaxf(second, fminf(v, best));
  idx = up ? col : idx;
  best = up ? v : best;
}

// Features of one sample point for the fp16 tensor-core path, per coordinate
// [p, sin(2^k pi p), cos(2^k pi p)] k = 0..9 at f[21 axis ..].  Bases at k = 0
// and 5 use the exactly reduced argument (p split into float hi + lo; 2^k p
// mod 2 is exact for the hi part), then four double-angle steps each; max abs
// error ~5e-6, well below the fp16 rounding (2.4e-4 at |v| in [0.5, 1)) that
// follows.  Per axis the two recurrences (bases 0 and 5) run as one f32x2
// chain (FMUL2/FADD2: the same rn operations as scalar code, half the issue slots).
__device__ __forceinline__ uint64_t f2pack(float lo, float hi) {
  uint64_t d;
  asm("mov.b64 %0, {%1, %2};" : "=l"(d) : "f"(lo), "f"(hi));
  return d;
}
__device__ __forceinline__ void f2unpack(uint64_t v, float& lo, float& hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ float2 f2unpack2(uint64_t v) {
  float2 r;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(v));
  return r;
}
__device__ __forceinline__ uint64_t add_f2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ uint64_t sub_f2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ uint64_t mul_f2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ void encode_point_tc(const double p[3], float f[64]) {
#pragma unroll
  for (int ax = 0; ax < 3; ++ax) {
    const float ph = (float)p[ax];
    const float pl = (float)(p[ax] - (double)ph);
    f[21 * ax] = ph;
    float s0, c0, s5, c5;
    __sincosf(3.14159265358979f * (ph + pl), &s0, &c0);
    const float t = ph * 32.0f;                                          // exact
    __sincosf(3.14159265358979f * (fmaf(-2.0f, rintf(0.5f * t), t) + 32.0f * pl), &s5, &c5);   // exact reduction + tail
    f[21 * ax + 1] = s0;
    f[21 * ax + 2] = c0;
    f[21 * ax + 11] = s5;
    f[21 * ax + 12] = c5;
    uint64_t S = f2pack(s0, s5), C = f2pack(c0, c5);     // lanes: level k, level 5 + k
#pragma unroll
    for (int k = 1; k < 5; ++k) {
      const uint64_t sc = mul_f2(S, C);
      const uint64_t S2 = add_f2(sc, sc);                 // 2 s c (exact doubling)
      C = mul_f2(sub_f2(C, S), add_f2(C, S));             // (c - s)(c + s)
      S = S2;
      f2unpack(S, f[21 * ax + 1 + 2 * k], f[21 * ax + 11 + 2 * k]);
      f2unpack(C, f[21 * ax + 2 + 2 * k], f[21 * ax + 12 + 2 * k]);
    }
  }
  f[63] = 0.f;
}


}  // namespace

// optional timeline of CTA 0's second tile (diagnostics, nedf_diag_tc_trace).  Compiled in only with
// -DNEDF_TC_TRACE=1 (scripts/build_variant.py): the instrumentation's registers push the epilogue's
// residual stream into local memory.
#ifndef NEDF_TC_TRACE
#define NEDF_TC_TRACE 0
#endif
__device__ unsigned long long g_tc_trace[1024];
__device__ int g_tc_trace_on;
__device__ __forceinline__ void trace_at(bool on, int idx) {
  if (on) g_tc_trace[idx] = clock64();
}
// wait, accumulating the cycles spent when tracing
#ifndef NEDF_TC_SPIN
#define NEDF_TC_SPIN 0   // 1 = spin on mbarrier.test_wait (measured slower: polling competes for shared memory)
#endif
__device__ __forceinline__ void twait(uint64_t* bar, uint32_t ph, bool on, unsigned long long& acc) {
  if (on) {
    const long long t0 = clock64();
    if (NEDF_TC_SPIN) tc::mbar_spin(bar, ph); else tc::mbar_wait(bar, ph);
    acc += clock64() - t0;
  } else {
    if (NEDF_TC_SPIN) tc::mbar_spin(bar, ph); else tc::mbar_wait(bar, ph);
  }
}

// One epilogue slice half: this thread's 64 accumulator columns [col0, col0 + 64) as four
// 16-column chunks, the TMEM load of chunk c + 1 in flight while chunk c is processed (16
// registers per buffer keeps the residual stream x in registers).  MODE 0: head, x = acc + b;
// 1: fc1, h = relu(acc + b) -> fp16 into A_Q; 2: fc2, x += relu(acc + b) -> fp16(x) into A_P.
template <int MODE>
__device__ __forceinline__ void epi_half(uint32_t acc_addr, uint32_t dst_addr, const float* bias, float (&xs)[2][32]) {
  uint32_t va[16], vb[16];
  tc::tmem_ld16(acc_addr, va);
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    tc::tmem_ld_wait();
    uint32_t (&v)[16] = (c & 1) ? vb : va;
    if (c < 3) tc::tmem_ld16(acc_addr + 16 * (c + 1), (c & 1) ? va : vb);
    float* xc = &xs[c >> 1][16 * (c & 1)];
    const float4* b4 = reinterpret_cast<const float4*>(bias + 16 * c);
    uint32_t pk[8];
#pragma unroll
    for (int j4 = 0; j4 < 4; ++j4) {
      const float4 b = b4[j4];
      const float2 a01 = f2unpack2(add_f2(f2pack(__uint_as_float(v[4 * j4 + 0]), __uint_as_float(v[4 * j4 + 1])),
                                          f2pack(b.x, b.y)));
      const float2 a23 = f2unpack2(add_f2(f2pack(__uint_as_float(v[4 * j4 + 2]), __uint_as_float(v[4 * j4 + 3])),
                                          f2pack(b.z, b.w)));
      const float a0 = a01.x, a1 = a01.y, a2 = a23.x, a3 = a23.y;
      if (MODE == 1) {
        pk[2 * j4 + 0] = tc::pack_h2_relu(a0, a1);
        pk[2 * j4 + 1] = tc::pack_h2_relu(a2, a3);
      } else {
        if (MODE == 0) {
          xc[4 * j4 + 0] = a0; xc[4 * j4 + 1] = a1; xc[4 * j4 + 2] = a2; xc[4 * j4 + 3] = a3;
        } else {
          // x += relu(acc + b) as f32x2 adds (same rn operations, half the issue slots)
          float2 x01 = f2unpack2(add_f2(f2pack(xc[4 * j4 + 0], xc[4 * j4 + 1]), f2pack(fmaxf(a0, 0.f), fmaxf(a1, 0.f))));
          float2 x23 = f2unpack2(add_f2(f2pack(xc[4 * j4 + 2], xc[4 * j4 + 3]), f2pack(fmaxf(a2, 0.f), fmaxf(a3, 0.f))));
          xc[4 * j4 + 0] = x01.x; xc[4 * j4 + 1] = x01.y; xc[4 * j4 + 2] = x23.x; xc[4 * j4 + 3] = x23.y;
        }
        pk[2 * j4 + 0] = tc::pack_h2(xc[4 * j4 + 0], xc[4 * j4 + 1]);
        pk[2 * j4 + 1] = tc::pack_h2(xc[4 * j4 + 2], xc[4 * j4 + 3]);
      }
    }
    tc::tmem_st8(dst_addr + 8 * c, pk);
  }
}

// csize = CTAs per cluster (1, 2 or 4).  With csize > 1 the CTAs of a cluster
// run the same model in lockstep and share one weight stream: each CTA's
// producer fetches 1/csize of every stage and multicasts it into the ring slot
// of every CTA, so L2 -> SM traffic drops by csize; a slot is refilled once the
// MMAs of all csize CTAs have released it (multicast commits, empty count csize).
__global__ void __launch_bounds__(kThreads, 1) nedf_mlp_tc_kernel(TcArgs a, int csize) {
  extern __shared__ unsigned char smem_raw[];
  // align by offsetting the shared array itself (not via an integer round trip), so the compiler
  // keeps the shared address space and emits LDS/STS instead of generic loads/stores
  unsigned char* smem = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);
  unsigned char* ring = smem;
  float* bias_s = reinterpret_cast<float*>(ring + kStages * kStageBytes);
  TcShared& S = *reinterpret_cast<TcShared*>(ring + kStages * kStageBytes + kBiasBytes);

  const int tid = threadIdx.x;
  const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);    // warp-uniform role index
  const int lane = tid & 31;
  const ListSet& ls = a.ls;
  const int ng = ls.n_groups < 64 ? ls.n_groups : 64;
  const bool trace_cta = NEDF_TC_TRACE && g_tc_trace_on && blockIdx.x == 0;
  const int trace_tile = g_tc_trace_on;   // nedf_diag_tc_trace(k): timeline of tile k
  const uint32_t rank = csize > 1 ? tc::cluster_rank() : 0;
  const int cid = blockIdx.x / csize, n_cl = gridDim.x / csize;
  const uint16_t cmask = (uint16_t)((1u << csize) - 1);

  if (tid == 0) {
    int cum = 0;
    S.tiles[0] = 0;
    for (int g = 0; g < ng; ++g) {
      cum += (ls.count[g] + 128 * csize - 1) / (128 * csize);
      S.tiles[g + 1] = cum;
    }
    for (int i = 0; i < kStages; ++i) { tc::mbar_init(&S.full[i], 1); tc::mbar_init(&S.empty[i], csize); }
    for (int i = 0; i < kEncSlots; ++i) tc::mbar_init(&S.enc_full[i], 4);
    tc::mbar_init(&S.aq_free, 1);
    for (int i = 0; i < 2; ++i) { tc::mbar_init(&S.acc_full[i], 1); tc::mbar_init(&S.epi_done[i], 8); }
    tc::mbar_fence_init();
  }
  if (warp == 1) tc::tmem_alloc<512>(&S.tmem_base);
  tc::tc_fence_before();
  if (csize > 1) tc::cluster_sync();     // peers multicast into this CTA's ring from the first stage on
  else __syncthreads();
  tc::tc_fence_after();
  const uint32_t tbase = S.tmem_base;
  const int total_tiles = S.tiles[ng];

  if (warp < 4) {
    tc::reg_dealloc<40>();
    if (warp == 0) {
      // ------------------------------------------------------------------ producer
      // Each of the first kStages lanes owns one ring slot and streams the stages
      // congruent to it: bulk copies issued by one thread serialise (~576
      // cycles each, scripts/bulk_rate.py), so one issuer per slot keeps
      // kStages copies in flight.
      static_assert(kStages % 2 == 0 && kStagesPerTile % 2 == 0, "head stage pairs must not wrap");
      if (lane < kStages) {
        // lane j streams the stages u = j (mod kStages) of the global sequence (296 per tile)
        const int slot = lane;
        uint32_t phase = 0, gbase = 0;
        int ti = 0;
        for (int t = cid; t < total_tiles; t += n_cl, ++ti) {
          const bool tr = trace_cta && ti == trace_tile && lane == 0;
          int g, n;
          int64_t base;
          tile_lookup(S.tiles, ng, t, ls, csize, rank, g, base, n);
          const unsigned char* w = reinterpret_cast<const unsigned char*>(a.gt.models[g].wpack);
          for (int i = (slot - (int)(gbase % kStages) + kStages) % kStages; i < kStagesPerTile; i += kStages) {
            // slots 2m, 2m + 1 are released together (one commit per stage pair)
            if (NEDF_TC_SPIN) tc::mbar_spin(&S.empty[slot & ~1], phase ^ 1);
            else tc::mbar_wait(&S.empty[slot & ~1], phase ^ 1);
            if (i == 0) trace_at(tr, 450);
            else if (i >= kHeadStages && (i - kHeadStages) % kLayerStages == 0)
              trace_at(tr, 450 + 1 + (i - kHeadStages) / kLayerStages);
            tc::mbar_expect_tx(&S.full[slot], kStageBytes);
            if (csize == 1) {
              tc::bulk_g2s(ring + slot * kStageBytes, w + (size_t)i * kStageBytes, kStageBytes, &S.full[slot]);
            } else {
              const uint32_t part = kStageBytes / csize, off = rank * part;
              tc::bulk_g2s_multicast(ring + slot * kStageBytes + off, w + (size_t)i * kStageBytes + off, part,
                                     &S.full[slot], cmask);
            }
            phase ^= 1;
          }
          gbase += kStagesPerTile;
        }
      }
      __syncwarp();
    } else if (warp == 1) {
      // ------------------------------------------------------------------ MMA issuer
      // Fully warp-uniform (a lane-dependent branch here moves the loop state out of the uniform
      // datapath and costs ~40% of the kernel); descriptors are base + slot offsets.
      int stage = 0, ti = 0, pend = -1;
      uint32_t phase = 0;
      uint32_t layer_ctr = 0;
      const uint32_t id256 = tc::idesc_f16(128, 256), id128 = tc::idesc_f16(128, 128);
      // the tail's second slice holds coarse logits (64 columns) and alpha (1): N = 80 covers
      // them and skips the 48 all-zero weight rows' products (columns 208-255 are never read)
      const uint32_t id80 = tc::idesc_f16(128, 80);
      const uint64_t dring = tc::sw128_desc(tc::smem_u32(ring));
      constexpr uint64_t kSlotDesc = kStageBytes >> 4;
      for (int t = cid; t < total_tiles; t += n_cl, ++ti) {
        const bool tr = trace_cta && ti == trace_tile;
        unsigned long long w_full = 0, w_epi = 0, w_enc = 0;
        trace_at(tr, 0);
        // ---- head (SS): A = encoded rays, B = W_head [256 x 64] per sample point
        if (layer_ctr > 0) {
          tc::mbar_wait(&S.epi_done[0], (layer_ctr - 1) & 1);
          tc::mbar_wait(&S.epi_done[1], (layer_ctr - 1) & 1);
        }
        trace_at(tr, 80);
        for (int c = 0; c < 16; ++c) {
          const int slot = c & (kEncSlots - 1);              // 4 uses per slot per tile
          twait(&S.enc_full[slot], (c >> 2) & 1, tr, w_enc);
          trace_at(tr, 81 + c);
          twait(&S.full[stage], phase, tr, w_full);
          twait(&S.full[stage + 1], phase, tr, w_full);
          tc::tc_fence_after();
          const uint32_t a0 = tbase + kAQCol + 32 * slot;   // TS: encoded point in TMEM
          const uint64_t b0 = dring + stage * kSlotDesc;
          if (tc::elect_one()) {
            if (pend >= 0) tc::mma_commit_mc(&S.empty[pend], cmask);
            if (c < 15) {
#pragma unroll
              for (int k = 0; k < 4; ++k)
                tc::mma_ts(tbase + kAccCol, a0 + 8 * k, b0 + 2 * k, id256, (c | k) ? 1u : 0u);
              tc::mma_commit_mc(&S.empty[stage], cmask);      // releases slots stage, stage + 1 and the point
            } else {
              // last point as two N = 128 halves: slice 0 completes half a point earlier, so its
              // epilogue (which layer 1's first MMAs wait for) overlaps slice 1's last MMAs
#pragma unroll
              for (int k = 0; k < 4; ++k) tc::mma_ts(tbase + kAccCol, a0 + 8 * k, b0 + 2 * k, id128, 1u);
              tc::mma_commit(&S.acc_full[0]);
#pragma unroll
              for (int k = 0; k < 4; ++k)
                tc::mma_ts(tbase + kAccCol + 128, a0 + 8 * k, b0 + kSlotDesc + 2 * k, id128, 1u);
              tc::mma_commit_mc(&S.empty[stage], cmask);
              tc::mma_commit(&S.acc_full[1]);
            }
          }
          __syncwarp();
          pend = -1;
          stage += 2;
          if (stage == kStages) { stage = 0; phase ^= 1; }
        }
        trace_at(tr, 40);
        if (tr) g_tc_trace[603] = w_full;        // weight waits during the head alone
        ++layer_ctr;
        // ---- 32 residual-block layers + the fused tail (TS, two 128-column slices)
        for (int L = 1; L <= kBodyLayers + 1; ++L) {
          const uint32_t a_col = tbase + ((L & 1) ? kAPCol : kAQCol);   // fc1 and tail read x, fc2 reads h
          const uint32_t par = (layer_ctr - 1) & 1;
          trace_at(tr, L);
          twait(&S.epi_done[0], par, tr, w_epi);               // acc slice 0 free, A chunks 0-1 ready
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const int s = j >> 2, kc = j & 3;
            if (j == 2) twait(&S.epi_done[1], par, tr, w_epi);    // acc slice 1 free, A chunks 2-3 ready
            twait(&S.full[stage], phase, tr, w_full);
            tc::tc_fence_after();
            const uint64_t b0 = dring + stage * kSlotDesc;
            if (tc::elect_one()) {
              if (pend >= 0) tc::mma_commit_mc(&S.empty[pend], cmask);   // previous stage pair
              const uint32_t idl = (L == kBodyLayers + 1 && s == 1) ? id80 : id128;
#pragma unroll
              for (int k = 0; k < 4; ++k)
                tc::mma_ts(tbase + kAccCol + 128 * s, a_col + kc * 32 + k * 8, b0 + 2 * k, idl,
                           (kc | k) ? 1u : 0u);
              if (kc == 3) tc::mma_commit(&S.acc_full[s]);
            }
            __syncwarp();
            // a stage pair's release is committed right after the NEXT stage's wait, together with
            // its MMAs: a wait issued right after a commit costs the tensor pipe a bubble
            pend = (kc & 1) ? stage - 1 : -1;
            if (++stage == kStages) { stage = 0; phase ^= 1; }
          }
          if (L == kBodyLayers) {
            // last A_Q reader issued.  The deferred release of layer 32's last stage pair goes out
            // first: the encoders take point consumption from those pair barriers, and their
            // parity is only meaningful once every earlier use has been committed.
            if (tc::elect_one()) {
              if (pend >= 0) tc::mma_commit_mc(&S.empty[pend], cmask);
              tc::mma_commit(&S.aq_free);
            }
            __syncwarp();
            pend = -1;
          }
          trace_at(tr, 40 + L);
          ++layer_ctr;
        }
        if (tr) {
          g_tc_trace[600] = w_full;
          g_tc_trace[601] = w_epi;
          g_tc_trace[602] = w_enc;
        }
      }
    }
  } else if (warp < 8) {
    tc::reg_dealloc<104>();
    // -------------------------------------------------------------------- encoders
    const int row = tid - 128;
    int ti = 0;
    for (int t = cid; t < total_tiles; t += n_cl, ++ti) {
      const bool tr = trace_cta && ti == trace_tile && tid == 128;
      int g, n;
      int64_t base;
      tile_lookup(S.tiles, ng, t, ls, csize, rank, g, base, n);
      const DevModel& m = a.gt.models[g];
      const bool valid = row < n;
      // p(t) = A + t B in the box frame, t = t0 + (t1 - t0) i / 15 (geometry.py:336-340)
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
          const double pp[3] = {pa[0] + tt * pb[0], pa[1] + tt * pb[1], pa[2] + tt * pb[2]};
          encode_point_tc(pp, f);
#pragma unroll
          for (int j = 0; j < 32; ++j) packed[j] = tc::pack_h2(f[2 * j], f[2 * j + 1]);
        } else {
#pragma unroll
          for (int j = 0; j < 32; ++j) packed[j] = 0u;
        }
        trace_at(tr, 500 + pt);
        // A_Q is free for this tile's points once the previous tile's layer 32 completed; within the
        // tile, slot pt & 3 is free once point pt - 4 was consumed
        if (pt == 0 && ti > 0) tc::mbar_wait(&S.aq_free, (ti - 1) & 1);
        if (pt >= kEncSlots) {
          // point pt - 4 consumed: its MMAs are the ones that released its weight-stage pair
          const uint32_t u = (uint32_t)ti * kStagesPerTile + 2 * (pt - kEncSlots);   // global stage index
          tc::mbar_wait(&S.empty[u % kStages], (u / kStages) & 1);
        }
        trace_at(tr, 420 + pt);
        {
          const uint32_t taddr = tbase + ((uint32_t)(32 * (warp & 3)) << 16) + kAQCol + 32 * (pt & 3);
          tc::tmem_st32(taddr, packed);
          tc::tmem_st_wait();
        }
        tc::tc_fence_before();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&S.enc_full[pt & 3]);
        trace_at(tr, 400 + pt);
      }
    }
  } else {
    tc::reg_alloc<184>();
    // -------------------------------------------------------------------- epilogue
    const int ew = warp - 8;                // 0..7
    const int q = warp & 3;                 // TMEM lane quadrant of this warp
    const int hc = ew >> 2;                 // 64-column half of each 128-column slice
    const int row = 32 * q + lane;
    const uint32_t lane_addr = tbase + ((uint32_t)(32 * q) << 16);
    uint32_t layer_ctr = 0;
    const float* cached_bias = nullptr;
    float x[2][2][32];                      // [slice][32-column chunk][column]
    int ti = 0;
    for (int t = cid; t < total_tiles; t += n_cl, ++ti) {
      const bool tr = trace_cta && ti == trace_tile && tid == 256;
      int g, n;
      int64_t base;
      tile_lookup(S.tiles, ng, t, ls, csize, rank, g, base, n);
      const DevModel& m = a.gt.models[g];
      if (m.bias_pack != cached_bias) {     // stage this model's biases in shared memory
        const float4* src = reinterpret_cast<const float4*>(m.bias_pack);
        float4* dst = reinterpret_cast<float4*>(bias_s);
        for (int i = tid - 256; i < kBiasLayers * 64; i += 256) dst[i] = __ldg(src + i);
        cached_bias = m.bias_pack;
        tc::named_bar(1, 256);
      }
      // ---- head: x = acc + b ----
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        tc::mbar_wait(&S.acc_full[s], layer_ctr & 1);
        tc::tc_fence_after();
        trace_at(tr, 100 + s);
        {
          const int col = 128 * s + 64 * hc;
          epi_half<0>(lane_addr + kAccCol + col, lane_addr + kAPCol + col / 2, bias_s + col, x[s]);
        }
        tc::tmem_st_wait();
        tc::tc_fence_before();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&S.epi_done[s]);
        trace_at(tr, 104 + s);
      }
      ++layer_ctr;
      // ---- residual blocks ----
      for (int blk = 0; blk < kBodyLayers / 2; ++blk) {
        const float* b1 = bias_s + (1 + 2 * blk) * 256;
        const float* b2 = b1 + 256;
        const int l1 = 1 + 2 * blk;
#pragma unroll
        for (int s = 0; s < 2; ++s) {     // fc1: h = relu(acc + b1) -> A_Q
          tc::mbar_wait(&S.acc_full[s], layer_ctr & 1);
          tc::tc_fence_after();
          trace_at(tr, 100 + l1 * 8 + s);
          {
            const int col = 128 * s + 64 * hc;
            epi_half<1>(lane_addr + kAccCol + col, lane_addr + kAQCol + col / 2, b1 + col, x[s]);
          }
          tc::tmem_st_wait();
          tc::tc_fence_before();
          __syncwarp();
          if (lane == 0) tc::mbar_arrive(&S.epi_done[s]);
          trace_at(tr, 104 + l1 * 8 + s);
        }
        ++layer_ctr;
#pragma unroll
        for (int s = 0; s < 2; ++s) {     // fc2: x += relu(acc + b2) -> A_P = fp16(x)
          tc::mbar_wait(&S.acc_full[s], layer_ctr & 1);
          tc::tc_fence_after();
          trace_at(tr, 100 + (l1 + 1) * 8 + s);
          {
            const int col = 128 * s + 64 * hc;
            epi_half<2>(lane_addr + kAccCol + col, lane_addr + kAPCol + col / 2, b2 + col, x[s]);
          }
          tc::tmem_st_wait();
          tc::tc_fence_before();
          __syncwarp();
          if (lane == 0) tc::mbar_arrive(&S.epi_done[s]);
          trace_at(tr, 104 + (l1 + 1) * 8 + s);
        }
        ++layer_ctr;
      }
      // ---- tail: slice 0 = fine (128); slice 1 = coarse (cols 0-63), alpha (col 64) ----
      const float* bt = bias_s + (kBiasLayers - 1) * 256;
      float fbest = -INFINITY, fsecond = -INFINITY, cbest = -INFINITY, csecond = -INFINITY, maxabs = 0.f,
            alpha = 0.f;
      int fidx = 0, cidx = 0;
      bool finite = true;
      // both slices are loaded and released before any decoding: the next tile's head MMAs wait
      // only for the tail MMAs, not for this epilogue's argmax work
      uint32_t vt[2][2][32];                 // [slice][32-column part][column]
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        tc::mbar_wait(&S.acc_full[s], layer_ctr & 1);
        tc::tc_fence_after();
        trace_at(tr, 100 + 33 * 8 + s);
        tc::tmem_ld32(lane_addr + kAccCol + 128 * s + 64 * hc, vt[s][0]);
        tc::tmem_ld32(lane_addr + kAccCol + 128 * s + 64 * hc + 32, vt[s][1]);
        tc::tmem_ld_wait();
        tc::tc_fence_before();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&S.epi_done[s]);
      }
#pragma unroll
      for (int s = 0; s < 2; ++s) {
#pragma unroll
        for (int j2 = 0; j2 < 2; ++j2) {
          const int col = 128 * s + 64 * hc + 32 * j2;
          const uint32_t* v = vt[s][j2];
          if (s == 1 && hc == 1) {         // alpha logit at tail column 192, then padding
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
            if (a.out.mode == OUT_LOGITS && row < n) {   // diagnostics: raw logits
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
        trace_at(tr, 104 + 33 * 8 + s);
      }
      ++layer_ctr;
      RowRed rr;
      rr.fbest = fbest; rr.fsecond = fsecond; rr.cbest = cbest; rr.csecond = csecond;
      rr.maxabs = finite ? maxabs : INFINITY; rr.alpha = alpha; rr.fidx = fidx; rr.cidx = cidx;
      S.red[row][hc] = rr;
      tc::named_bar(1, 256);
      // STEP 3: a flagged shadow pair is finished here when its decision (shadows / does not) is
      // the same for every bin within the margin of the fast maxima and either alpha; only the
      // undecided ones go to the guard.  Both halves scan their logits for the candidate range.
      const bool shadow_job = a.use_guard && a.shadow_cert && a.out.mode == OUT_ZBUF &&
                              (a.job.mode == RAY_POINT_SHADOW || a.job.mode == RAY_DIR_SHADOW);
      int fr_lo = 1 << 30, fr_hi = -1, cr_lo = 1 << 30, cr_hi = -1;
      if (shadow_job) {
        const RowRed r0 = S.red[row][0], r1 = S.red[row][1];
        const bool up = r1.fbest > r0.fbest;
        const float fb = up ? r1.fbest : r0.fbest;
        const float fs2 = up ? fmaxf(fmaxf(r0.fbest, r0.fsecond), r1.fsecond) : fmaxf(fmaxf(r1.fbest, r0.fsecond), r1.fsecond);
        const float S2 = fmaxf(r0.maxabs, r1.maxabs);
        const float thr2 = a.guard * S2;
        const bool flagged = (fb - fs2) < thr2 || (r0.cbest - r0.csecond) < thr2 || fabsf(r1.alpha - m.alpha_zthr) < thr2;
        if (row < n && S2 < INFINITY && flagged) {
          const float flim = fb - thr2, clim = r0.cbest - thr2;
#pragma unroll
          for (int j2 = 0; j2 < 2; ++j2) {
#pragma unroll
            for (int k = 0; k < 32; ++k) {
              const int c = 64 * hc + 32 * j2 + k;
              if (__uint_as_float(vt[0][j2][k]) + bt[c] >= flim) { fr_lo = min(fr_lo, c); fr_hi = max(fr_hi, c); }
              if (hc == 0 && __uint_as_float(vt[1][j2][k]) + bt[128 + c] >= clim) {
                cr_lo = min(cr_lo, c);
                cr_hi = max(cr_hi, c);
              }
            }
          }
          if (hc == 1) S.frange[row] = make_int2(fr_lo, fr_hi);
        }
        tc::named_bar(1, 256);
      }
      if (hc == 0 && row < n) {
        const RowRed o = S.red[row][1];
        // fine argmax over both halves: larger value wins, ties keep the lower column
        float fb, fs;
        int fi;
        if (o.fbest > fbest) { fb = o.fbest; fi = o.fidx; fs = fmaxf(fmaxf(fbest, fsecond), o.fsecond); }
        else { fb = fbest; fi = fidx; fs = fmaxf(fmaxf(o.fbest, fsecond), o.fsecond); }
        const float al = o.alpha;
        const float S_ = fmaxf(rr.maxabs, o.maxabs);
        const float thr = a.guard * S_;
        const uint32_t pix = ls.pix[base + row], obj = ls.obj[base + row];
        bool risky =
            a.use_guard && (!(S_ < INFINITY) || (fb - fs) < thr || (cbest - csecond) < thr || fabsf(al - m.alpha_zthr) < thr);
        if (risky && shadow_job && S_ < INFINITY) {
          const int2 f1 = S.frange[row];
          const int cert = shadow_pair_certain(m, a.job, pix, obj, cr_lo, cr_hi, min(fr_lo, f1.x), max(fr_hi, f1.y),
                                               alpha_of((double)al, m.alpha_threshold),
                                               fabsf(al - m.alpha_zthr) < thr);
          risky = cert < 0;
        }
        if (a.out.mode == OUT_LOGITS) {
          // diagnostics: logits already written
        } else if (risky) {
          int at = atomicAdd(a.redo.count + g, 1);
          a.redo.pix[a.redo.offset[g] + at] = pix;
          a.redo.obj[a.redo.offset[g] + at] = obj;
        } else {
          double wo[3], wd[3], lo[3], ld[3];
          item_local_ray(a.job, pix, obj, wo, wd, lo, ld);
          finish_ray(m, a.job, a.out, pix, obj, cidx, fi, (double)al, wo, wd);
        }
      }
      tc::named_bar(1, 256);
    }
  }
  tc::tc_fence_before();
  if (csize > 1) tc::cluster_sync();     // no peer may still multicast into / arrive on this CTA
  else __syncthreads();
  if (warp == 1) tc::tmem_dealloc<512>(tbase);
}

bool tc_available() { return true; }

}  // namespace nedf

extern "C" int nedf_diag_tc_trace(int enable, unsigned long long* out, int n) {
  using namespace nedf;
  if (enable >= 0) {
    int v = enable;
    if (cudaMemcpyToSymbol(g_tc_trace_on, &v, sizeof(int)) != cudaSuccess) return NEDF_ERR_CUDA;
  }
  if (out && n > 0) {
    if (n > 1024) n = 1024;
    if (cudaMemcpyFromSymbol(out, g_tc_trace, n * sizeof(unsigned long long)) != cudaSuccess) return NEDF_ERR_CUDA;
  }
  return NEDF_OK;
}

namespace nedf {

cudaError_t launch_mlp_tc(const TcArgs& a, int n_ctas, int csize, cudaStream_t stream) {
  static bool configured_dev[kMaxDevices] = {};
  static int max_clusters_dev[kMaxDevices][5] = {};
  const int dev = current_device();
  bool& configured = configured_dev[dev];
  int* max_clusters = max_clusters_dev[dev];
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(nedf_mlp_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)kSmemBytes);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  if (csize != 1 && csize != 2 && csize != 4) return cudaErrorInvalidValue;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = csize;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(kThreads, 1, 1);
  cfg.dynamicSmemBytes = kSmemBytes;
  cfg.stream = stream;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (csize > 1) {
    // persistent grid: only as many clusters as can be co-resident (a GPC whose free SM count is
    // not a multiple of csize leaves SMs idle), or the surplus would run as a second wave
    if (max_clusters[csize] == 0) {
      cfg.gridDim = dim3(n_ctas - n_ctas % csize, 1, 1);
      int n = 0;
      cudaError_t e = cudaOccupancyMaxActiveClusters(&n, nedf_mlp_tc_kernel, &cfg);
      if (e != cudaSuccess) return e;
      max_clusters[csize] = n > 0 ? n : 1;
    }
    n_ctas -= n_ctas % csize;
    if (n_ctas > csize * max_clusters[csize]) n_ctas = csize * max_clusters[csize];
    if (n_ctas < csize) n_ctas = csize;
  }
  cfg.gridDim = dim3(n_ctas, 1, 1);
  return cudaLaunchKernelEx(&cfg, nedf_mlp_tc_kernel, a, csize);
}

// Pack a paper-shaped model (d_feat 256, 16 blocks, 64/128 bins) into the
// stage image the kernel streams, each stage a 128B-swizzled [128 x 64] fp16
// tile: head point c -> stages 2c, 2c+1 (output rows 0-127, 128-255, K = the
// point's 63 features + 1 zero); layer l -> stages 32 + 8l + 4s + kc (output
// rows 128s.., K chunk kc); tail rows = fine (0-127), coarse (128-191),
// alpha (192), zero padding.  Biases: [34 layers][256] fp32, same row order.
cudaError_t tc_pack_weights(const float* P, int d_in, int F, int n_blocks, int n_coarse, int n_fine,
                            __half** wpack_dev, float** bias_dev, size_t* bytes, int part) {
  if (F != 256 || n_blocks != kBodyLayers / 2 || d_in != kDin || n_coarse != 64 || n_fine != 128)
    return cudaErrorInvalidValue;
  std::vector<__half> img((size_t)kStagesPerTile * kStageBytes / 2, __float2half(0.f));
  std::vector<float> bias((size_t)kBiasLayers * 256, 0.f);
  // part 0: fp16(w); part 1: fp16(4096 (w - fp16(w))), the low half of mlp_precise.cu's split
  auto put = [&](int stage, int r, int k, float v) {
    size_t off = (size_t)stage * kStageBytes + tc::sw128_offset(r, k >> 3) + (k & 7) * 2;
    const __half hi = __float2half_rn(v);
    img[off / 2] = part == 0 ? hi : __float2half_rn((v - __half2float(hi)) * 4096.f);
  };
  size_t p = 0;
  const float* Wh = P + p; p += (size_t)F * d_in;
  const float* bh = P + p; p += F;
  std::vector<const float*> Wl(kBodyLayers), bl(kBodyLayers);
  for (int l = 0; l < kBodyLayers; ++l) { Wl[l] = P + p; p += (size_t)F * F; bl[l] = P + p; p += F; }
  const float* Wa = P + p; p += (size_t)(n_coarse + 1) * F;
  const float* ba = P + p; p += n_coarse + 1;
  const float* Wb = P + p; p += (size_t)n_fine * F;
  const float* bb = P + p; p += n_fine;
  for (int c = 0; c < 16; ++c)
    for (int n = 0; n < 256; ++n)
      for (int k = 0; k < 63; ++k) put(2 * c + (n >> 7), n & 127, k, Wh[(size_t)n * d_in + 63 * c + k]);
  for (int o = 0; o < F; ++o) bias[o] = bh[o];
  for (int l = 0; l < kBodyLayers; ++l) {
    const int st0 = kHeadStages + l * kLayerStages;
    for (int s = 0; s < 2; ++s)
      for (int kc = 0; kc < 4; ++kc)
        for (int r = 0; r < 128; ++r)
          for (int k = 0; k < 64; ++k) put(st0 + 4 * s + kc, r, k, Wl[l][(size_t)(128 * s + r) * F + 64 * kc + k]);
    for (int o = 0; o < F; ++o) bias[(size_t)(1 + l) * 256 + o] = bl[l][o];
  }
  auto tail_row = [&](int n) -> const float* {
    if (n < 128) return Wb + (size_t)n * F;
    if (n < 128 + n_coarse + 1) return Wa + (size_t)(n - 128) * F;
    return nullptr;
  };
  const int st0 = kHeadStages + kBodyLayers * kLayerStages;
  for (int s = 0; s < 2; ++s)
    for (int kc = 0; kc < 4; ++kc)
      for (int r = 0; r < 128; ++r) {
        const float* w = tail_row(128 * s + r);
        if (!w) continue;
        for (int k = 0; k < 64; ++k) put(st0 + 4 * s + kc, r, k, w[64 * kc + k]);
      }
  float* bt = bias.data() + (size_t)(kBiasLayers - 1) * 256;
  for (int o = 0; o < 128; ++o) bt[o] = bb[o];
  for (int o = 0; o < n_coarse + 1; ++o) bt[128 + o] = ba[o];
  *bytes = img.size() * sizeof(__half);
  cudaError_t e = cudaMalloc(wpack_dev, *bytes);
  if (e == cudaSuccess) e = cudaMemcpy(*wpack_dev, img.data(), *bytes, cudaMemcpyHostToDevice);
  if (bias_dev != nullptr) {
    if (e == cudaSuccess) e = cudaMalloc(bias_dev, bias.size() * sizeof(float));
    if (e == cudaSuccess) e = cudaMemcpy(*bias_dev, bias.data(), bias.size() * sizeof(float), cudaMemcpyHostToDevice);
  }
  return e;
}

}  // namespace nedf
