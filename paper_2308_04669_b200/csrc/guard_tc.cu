// fp32-accurate network for the near-tie guard on the 5th-generation tensor
// cores (tcgen05 kind::tf32 + kind::f16/bf16, accumulators in TMEM).
//
// Role: re-evaluate the few hundred rays per frame whose fp16 decisions are
// within rounding of a flip (mlp_tc.cu's guard) with float32-level accuracy.
// Its cost is latency: a ray still walks the 35-layer chain (nn.py:115-135).
//
// Layout.  A cluster of 4 CTAs shares a 16-ray tile; CTA r owns output rows
// (features) [64 r, 64 r + 64) of every layer, so one layer is, per CTA, the
// product D[64 x 16] = W_r[64 x K] X^T[K x 16] with the weights as the M = 64
// operand and the rays as N = 16 -- both K-major in 128B-swizzled shared
// memory tiles, so a layer is 32 + 32 + 16 single-thread MMAs.
//
// Arithmetic (the split that makes tensor-core products fp32-accurate):
//   W = W_hi + W_lo, W_hi = W with the 13 low mantissa bits cleared (exact in
//   tf32), W_lo = W - W_hi (|W_lo| < 2^-10 |W|), stored as fp16 x 2^11;
//   X = X_hi + X_lo likewise (X_lo rounded to nearest tf32), computed on chip
//   for every layer input, plus X_h = fp16(2^-11 X) (satfinite);
//   D  = W_hi [X_hi; X_lo]              (kind::tf32, N = 32: both products from
//                                        one read of W_hi, exact 11 x 11-bit)
//      + (2^11 W_lo)_fp16 X_h           (kind::f16, into the X_lo half)
//   y  = D[:, X_hi half] + D[:, X_lo half]  (fp32 accumulation throughout)
// The rounded parts are W_hi (X_lo - tf32(X_lo)) ~ 2^-22, and W_lo's and X's
// fp16 roundings in the D2 term ~ 2^-21 of |W X| per product: float32-level,
// at least as tight as the 3xTF32 mma.sync kernel it replaces (mlp_fp32c.cu),
// at tcgen05 rates (a tf32 M64 x N16 x K8 MMA costs ~8 cycles).  tcgen05 reads
// tf32 operands by truncation (pinned by tests/test_gpu_umma.py); W_hi and
// X_hi are exact tf32 values, so nothing depends on it.
//
// Pipeline per CTA (12 warps): warp 0 streams the CTA's weight slice as 48 KB
// stages (K = 128: W_hi 32 KB + W_lo 16 KB) through a 3-slot ring; warp 1
// issues the MMAs and commits; warps 4-7 are the epilogue (TMEM lane quadrant
// = warp % 4; lanes 0-15 hold the M = 64 rows: row r -> TMEM lane 32 (r / 16) +
// r % 16): bias, ReLU, residual (the residual stream of the CTA's 64 features
// stays in registers), then the 16 x 64 fp32 slab goes to the CTA's own
// receive buffer and, by three 4 KB bulk copies, into the peers' (completing
// bytes on their layer barrier: no cluster-wide barrier per layer).  Warps
// 2-11 then split the gathered 16 x 256 layer into the next layer's X_hi /
// X_lo / X_bf16 tiles.  The head's input (the 16 x 1024 float64-accurate
// encoding, geometry.py:312-342) is computed per 128-column stage into two
// alternating B slots while the MMAs consume the previous one.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <cuda_bf16.h>

#include "common.cuh"
#include "frame.cuh"
#include "tc_ptx.cuh"

namespace nedf {
namespace {

constexpr int kGC = 4;                 // CTAs per cluster
constexpr int kGN = 16;                // rays per tile (MMA N)
constexpr int kGM = 64;                // output rows per CTA (MMA M)
constexpr int kGThreads = 384;         // 12 warps
constexpr int kGWorkers = 10;          // warps 2..11
constexpr int kGHeadStages = 8;        // head K = 1024 = 16 points x (63 features + 1 zero)
constexpr int kGBodyStages = 2;        // K = 256
constexpr int kGLayers = 34;           // head, 32 block layers, fused tail
constexpr int kGStagesPerTile = kGHeadStages + (kGLayers - 1) * kGBodyStages;   // 74
constexpr uint32_t kGHiBytes = kGM * 128 * 4;                // 32 KB: [4 atoms of 32 K][64 rows][128 B]
constexpr uint32_t kGLoBytes = kGM * 128 * 2;                // 16 KB: fp16 [2 atoms of 64 K][64 rows][128 B]
constexpr uint32_t kGStageBytes = kGHiBytes + kGLoBytes;     // 48 KB
constexpr int kGRing = 3;
constexpr float kGLoScale = 2048.f;    // W_lo is stored x 2^11
constexpr float kGXScale = 1.f / 2048; // the W_lo term's activations are stored x 2^-11 (exact product scale)
constexpr int kHH = 2;                 // W_hi X_hi accumulators (even)
constexpr uint32_t kGAtom = kGN * 128;                       // one 16-row B atom: 2 KB
constexpr uint32_t kGAtom2 = 2 * kGN * 128;                  // one 32-row [X_hi; X_lo] atom: 4 KB

// Two input buffers alternate by layer: layer L reads XB[L & 1] and its outputs land in
// XB[(L + 1) & 1] -- the raw fp32 outputs go straight into the X_hi rows (the tensor core
// reads them as tf32 by truncation, i.e. exactly X_hi), and each CTA fills in the X_lo rows
// and the fp16 tile.  The head's input uses XB[0] as two 4-atom slots.
struct GBuf {
  unsigned char xhl[8 * 2 * kGN * 128];       // fp32 [8 atoms of 32 K][rows: 16 X (raw), 16 X_lo][128 B]
  unsigned char xh16[4 * kGN * 128];          // fp16 2^-11 X [4 atoms of 64 K][16 rays][128 B]
};
struct GSmem {
  unsigned char ring[kGRing][kGStageBytes];   // weight stages (1024-aligned)
  GBuf xb[2];
  double ray[kGN][8];                         // local o, d, t0, t1
  uint32_t pix[kGN], obj[kGN];
  int valid[kGN];
  int tiles[65];
  uint64_t full[kGRing], empty[kGRing];
  uint64_t fready[2], ffree[2];               // head feature slots: workers -> MMA, MMA -> workers
  uint64_t bready;                            // body B tiles complete (workers -> MMA)
  uint64_t dfull;                             // accumulators ready (MMA -> epilogue)
  uint64_t recv_bar[2];                       // a layer's raw outputs landed in xb[i] (3 peers' 2 x 2 KB + local arrival)
  uint32_t tmem_base;
};
static_assert(sizeof(GSmem) + 1024 <= 232448, "guard kernel shared memory exceeds 227 KB");

__device__ __forceinline__ uint32_t tf32_hi_bits(float x) { return __float_as_uint(x) & 0xFFFFE000u; }
// nearest tf32 value (ties away from zero) of a remainder, so the truncating tensor core sees it exactly
__device__ __forceinline__ float tf32_rna(float x) { return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xFFFFE000u); }
// fp16 pair of 2^-8 (a, b), clamped to the finite range
__device__ __forceinline__ uint32_t xh_pair(float a, float b) {
  uint32_t r;
  asm("cvt.rn.satfinite.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(b * kGXScale), "f"(a * kGXScale));
  return r;
}

// bulk copy shared::cta -> shared::cluster (a peer CTA), completing bytes on the peer's mbarrier
__device__ __forceinline__ void bulk_s2peer(uint32_t dst_cluster, const void* src, uint32_t bytes,
                                            uint32_t mbar_cluster) {
  asm volatile(
      "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          dst_cluster),
      "r"(tc::smem_u32(src)), "r"(bytes), "r"(mbar_cluster)
      : "memory");
}

// byte offset of element k of row `row` in the SW128 K-major fp16 atoms (64 K each)
__device__ __forceinline__ uint32_t b_off_bf16(int row, int k) {
  return (uint32_t)(k >> 6) * kGAtom + tc::sw128_offset(row, (k & 63) >> 3) + ((k & 7) << 1);
}

// byte offset of element k of row `row` (0-31) in the [X_hi; X_lo] atoms
__device__ __forceinline__ uint32_t b_off_hl(int row, int k) {
  return (uint32_t)(k >> 5) * kGAtom2 + tc::sw128_offset(row, (k & 31) >> 2) + ((k & 3) << 2);
}

// one input value of the next layer: hi / lo (fp32) and fp16 copies into the B tiles
__device__ __forceinline__ void put_x(unsigned char* xhl, unsigned char* xbf, int row, int k, float v) {
  const float hi = __uint_as_float(tf32_hi_bits(v));
  *reinterpret_cast<float*>(xhl + b_off_hl(row, k)) = v;          // read as tf32 (truncated): X_hi
  *reinterpret_cast<float*>(xhl + b_off_hl(kGN + row, k)) = tf32_rna(v - hi);
  __half h;
  asm("{\n\t.reg .b32 t;\n\tcvt.rn.satfinite.f16x2.f32 t, %1, %1;\n\tmov.b32 {%0, _}, t;\n\t}"
      : "=h"(*reinterpret_cast<unsigned short*>(&h))
      : "f"(v * kGXScale));
  *reinterpret_cast<__half*>(xbf + b_off_bf16(row, k)) = h;
}

// first maximum under a sequential strict '>' scan (numpy argmax on finite data; a NaN at
// index 0 wins, later NaNs are skipped) of a vector held N values per lane (indices lane * N + i);
// `first` = element 0, the same in every lane.  All 32 lanes call it.
template <int N>
__device__ __forceinline__ int warp_argmax(const float (&v)[N], float first) {
  const int lane = threadIdx.x & 31;
  float best = -INFINITY;
  int idx = -1;
#pragma unroll
  for (int i = 0; i < N; ++i)
    if (v[i] > best) { best = v[i]; idx = lane * N + i; }
  for (int off = 1; off < 32; off <<= 1) {
    // merge the run of lanes above (higher indices) into this one: taken only if strictly greater
    const float ob = __shfl_down_sync(0xffffffffu, best, off);
    const int oi = __shfl_down_sync(0xffffffffu, idx, off);
    const bool merge = (lane & (2 * off - 1)) == 0 && lane + off < 32;
    if (merge && oi >= 0 && (idx < 0 || ob > best)) { best = ob; idx = oi; }
  }
  idx = __shfl_sync(0xffffffffu, idx, 0);
  return (isnan(first) || idx < 0) ? 0 : idx;
}

}  // namespace

// optional timeline of cluster 0 / CTA 0, first tile (diagnostics, nedf_diag_guard_trace):
// [L] layer L's MMAs start (B tiles and first stage ready), [40 + L] issued, [80 + L] epilogue has
// the accumulators, [120 + L] slab sent, [160 + L] layer landed, [200 + L] next B tiles written,
// [240 + q] weight stage q issued (q < 40), [280 + L] epilogue stores done
__device__ unsigned long long g_gtrace[320];
__device__ int g_gtrace_on;

__global__ void __cluster_dims__(kGC, 1, 1) __launch_bounds__(kGThreads, 1)
guard_tc_kernel(GroupTable gt, ListSet ls, RayJob job, OutSpec out, int max_tiles16) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  GSmem& S = *reinterpret_cast<GSmem*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t rank = tc::cluster_rank();
  const int cid = blockIdx.x / kGC, n_cl = gridDim.x / kGC;
  const int ng = ls.n_groups < 64 ? ls.n_groups : 64;
  const bool feats_in = out.feats != nullptr;
  if (max_tiles16 >= 0) {                      // large batches go to mlp_precise.cu (decided on the device)
    int t16 = 0;
    for (int g = 0; g < ng; ++g) t16 += (ls.count[g] + kGN - 1) / kGN;
    if (t16 > max_tiles16) return;
  }

  if (tid == 0) {
    int cum = 0;
    S.tiles[0] = 0;
    for (int g = 0; g < ng; ++g) {
      cum += (ls.count[g] + kGN - 1) / kGN;
      S.tiles[g + 1] = cum;
    }
    for (int i = 0; i < kGRing; ++i) { tc::mbar_init(&S.full[i], 1); tc::mbar_init(&S.empty[i], 1); }
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&S.fready[i], kGWorkers);
      tc::mbar_init(&S.ffree[i], 1);
      tc::mbar_init(&S.recv_bar[i], 1);
    }
    tc::mbar_init(&S.bready, kGWorkers);
    tc::mbar_init(&S.dfull, 1);
    tc::mbar_fence_init();
  }
  if (warp == 1) tc::tmem_alloc<64>(&S.tmem_base);
  tc::tc_fence_before();
  tc::cluster_sync();            // barriers initialised cluster-wide before any peer store
  tc::tc_fence_after();
  const int total = S.tiles[ng];
  const uint32_t tbase = S.tmem_base;
  const bool trace = g_gtrace_on && cid == 0 && rank == 0 && lane == 0;
#define GTRACE(i, first_tile) \
  do {                        \
    if (trace && (first_tile)) g_gtrace[(i)] = clock64(); \
  } while (0)

  if (warp == 0) {
    // ------------------------------------------------------------------ weight producer
    uint32_t gq = 0;
    for (int t = cid; t < total; t += n_cl) {
      int g = 0;
      while (g < ng - 1 && t >= S.tiles[g + 1]) ++g;
      const unsigned char* img = reinterpret_cast<const unsigned char*>(gt.models[g].wguard);
      for (int q = 0; q < kGStagesPerTile; ++q, ++gq) {
        const int slot = gq % kGRing;
        if (lane == 0) {
          tc::mbar_wait(&S.empty[slot], ((gq / kGRing) & 1) ^ 1);
          tc::mbar_expect_tx(&S.full[slot], kGStageBytes);
        }
        __syncwarp();
        // a stage goes out as 4 parallel 12 KB pieces (copies issued by one thread serialise)
        GTRACE(240 + q, t == cid && q < 40);
        if (lane < 4)
          tc::bulk_g2s(&S.ring[slot][lane * (kGStageBytes / 4)],
                       img + ((size_t)q * kGC + rank) * kGStageBytes + lane * (kGStageBytes / 4), kGStageBytes / 4,
                       &S.full[slot]);
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------------ MMA issuer
    const uint32_t id_tf = tc::idesc_tf32(kGM, 2 * kGN), id_bf = tc::idesc_f16(kGM, kGN);
    // TMEM: kHH accumulators of 32 columns ([W_hi X_hi | W_hi X_lo]), by 32-wide K atom mod kHH
    // (few additions per accumulator keep the tensor core's accumulation rounding at the fp32
    // level); the W_lo term goes into accumulator 0's X_lo half.  M = 64 accumulators pair up in
    // the lane 0-15 / 16-31 halves of a 32-column group, so one 32x32b load reads two.
    const uint32_t d2 = tbase + 16;
    uint32_t gq = 0, hq = 0, bl = 0;
    for (int t = cid; t < total; t += n_cl) {
      for (int L = 0; L < kGLayers; ++L) {
        const int nst = L == 0 ? kGHeadStages : kGBodyStages;
        const GBuf& B = S.xb[L & 1];
        if (L > 0) {
          tc::mbar_wait(&S.bready, bl & 1);
          ++bl;
        }
        for (int j = 0; j < nst; ++j, ++gq) {
          const int slot = gq % kGRing;
          tc::mbar_wait(&S.full[slot], (gq / kGRing) & 1);
          // B tiles of this stage: the head's alternate between two 4-atom slots of xb[0]
          const int bs = L == 0 ? (int)(hq & 1) : j;
          if (L == 0) tc::mbar_wait(&S.fready[bs], (hq >> 1) & 1);
          const uint32_t xh = tc::smem_u32(B.xhl) + bs * 4 * kGAtom2, xb = tc::smem_u32(B.xh16) + bs * 2 * kGAtom;
          tc::tc_fence_after();
          if (j == 0) GTRACE(L, t == cid);
          if (tc::elect_one()) {
            // descriptors as base + constant: (address >> 4) sits in the low 14 bits
            const uint32_t w = tc::smem_u32(&S.ring[slot][0]);
            const uint64_t a0 = tc::sw128_desc(w), bh0 = tc::sw128_desc(xh), bb0 = tc::sw128_desc(xb);
#pragma unroll
            for (int ks = 0; ks < 16; ++ks) {       // tf32: 16 k-steps of 8, N = 32 ([X_hi; X_lo])
              const uint32_t a_off = ((ks >> 2) * (kGM * 128) + (ks & 3) * 32) >> 4;
              const uint32_t b_off = ((ks >> 2) * kGAtom2 + (ks & 3) * 32) >> 4;
              const int atom = 4 * j + (ks >> 2);             // 32-wide K atom of the layer
              const int h = atom % kHH;
              const uint32_t dh = tbase + 32 * (h >> 1) + ((uint32_t)(16 * (h & 1)) << 16);
              const uint32_t first = atom < kHH && (ks & 3) == 0;
              tc::mma_ss_tf32(dh, a0 + a_off, bh0 + b_off, id_tf, first ? 0u : 1u);
            }
#pragma unroll
            for (int ks = 0; ks < 8; ++ks) {        // fp16: 8 k-steps of 16, into accumulator 0's X_lo half
              const uint32_t a_off = (kGHiBytes + (ks >> 2) * (kGM * 128) + (ks & 3) * 32) >> 4;
              const uint32_t b_off = ((ks >> 2) * kGAtom + (ks & 3) * 32) >> 4;
              tc::mma_ss(d2, a0 + a_off, bb0 + b_off, id_bf, 1u);
            }
            tc::mma_commit(&S.empty[slot]);
            if (L == 0) tc::mma_commit(&S.ffree[hq & 1]);
            if (j == nst - 1) tc::mma_commit(&S.dfull);
          }
          __syncwarp();
          if (j == nst - 1) GTRACE(40 + L, t == cid);
          if (L == 0) ++hq;
        }
      }
    }
  } else {
    // ------------------------------------------------------------------ workers (warps 2-11)
    const int wt = tid - 64;                                  // worker thread 0..319
    const bool epi = warp >= 4 && warp < 8;
    const int quad = warp & 3;
    const int row = 16 * quad + (lane & 15);                  // epilogue: this lane's output row
    uint32_t peer_xb[kGC], peer_bar[2][kGC];
#pragma unroll
    for (int q = 0; q < kGC; ++q) {
      peer_xb[q] = tc::peer_addr(&S.xb[0], q);
      peer_bar[0][q] = tc::peer_addr(&S.recv_bar[0], q);
      peer_bar[1][q] = tc::peer_addr(&S.recv_bar[1], q);
    }
    const uint32_t xb0 = tc::smem_u32(&S.xb[0]);
    uint32_t hq = 0, dl = 0, rc[2] = {0u, 0u};
    float xr[kGN / 2];                                        // residual stream of (row, this lane's 8 rays)
    for (int t = cid; t < total; t += n_cl) {
      int g = 0;
      while (g < ng - 1 && t >= S.tiles[g + 1]) ++g;
      const int lt = t - S.tiles[g];
      int n = ls.count[g] - lt * kGN;
      n = n < kGN ? n : kGN;
      const int64_t base = ls.offset[g] + (int64_t)lt * kGN;
      const DevModel& m = gt.models[g];
      if (wt < kGN) {
        const int r = wt;
        const int v = r < n;
        S.valid[r] = v;
        S.pix[r] = v ? ls.pix[base + r] : 0u;
        S.obj[r] = v ? ls.obj[base + r] : 0u;
        if (v && !feats_in) {
          double wo[3], wd[3], lo[3], ld[3], t0 = 0, t1 = 0;
          item_local_ray(job, S.pix[r], S.obj[r], wo, wd, lo, ld);
          slab_clip(lo, ld, m.bmin, m.bmax, t0, t1);
          for (int a = 0; a < 3; ++a) { S.ray[r][a] = lo[a]; S.ray[r][3 + a] = ld[a]; }
          S.ray[r][6] = t0;
          S.ray[r][7] = t1;
        }
      }
      tc::named_bar(1, kGWorkers * 32);
      // ---- head input, stage by stage (2 points = 128 columns each; float64-accurate features,
      // geometry.py:312-342): one (ray, point, axis, level half) per thread -- sincospi at level 0
      // or 5, float64 double-angle steps for the next four (the error doubles per step, far below
      // the float32 rounding that follows) -- into the X rows, then X_lo and fp16 by columns
      for (int q = 0; q < kGHeadStages; ++q, ++hq) {
        const int fs = hq & 1;
        if (hq >= 2) tc::mbar_wait(&S.ffree[fs], ((hq >> 1) - 1) & 1);
        unsigned char* xh = S.xb[0].xhl + fs * 4 * kGAtom2;
        unsigned char* xb = S.xb[0].xh16 + fs * 2 * kGAtom;
        auto put_raw = [&](int r, int k, float v) { *reinterpret_cast<float*>(xh + b_off_hl(r, k)) = v; };
        for (int e = wt; e < kGN * 2 * 3 * 2; e += kGWorkers * 32) {
          const int r = e / 12, pp = (e % 12) / 6, a = (e % 6) >> 1, hf = e & 1;
          const int pt = 2 * q + pp;
          const int k0 = 64 * pp + 21 * a + (hf ? 11 : 1);    // column of this half's first sin
          float sv[5], cv[5], p0 = 0.f;                       // hf 0: p, levels 0-4; hf 1: levels 5-9
          if (!S.valid[r]) {
#pragma unroll
            for (int k = 0; k < 5; ++k) sv[k] = cv[k] = 0.f;
          } else if (feats_in) {
            const float* src = out.feats + (size_t)S.pix[r] * kDin + pt * kPerPoint + 21 * a;
            p0 = src[0];
#pragma unroll
            for (int k = 0; k < 5; ++k) {
              sv[k] = src[(hf ? 11 : 1) + 2 * k];
              cv[k] = src[(hf ? 12 : 2) + 2 * k];
            }
          } else {
            const double t0 = S.ray[r][6], t1 = S.ray[r][7];
            const double tt = t0 + (t1 - t0) * lin16(pt);
            const double p = ((S.ray[r][a] + tt * S.ray[r][3 + a]) - m.c[a]) / m.h[a];
            p0 = (float)p;
            double sn, cs;
            sincospi(ldexp(p, 5 * hf), &sn, &cs);
            sv[0] = (float)sn;
            cv[0] = (float)cs;
#pragma unroll
            for (int k = 1; k < 5; ++k) {
              const double s2 = 2.0 * sn * cs, c2 = (cs - sn) * (cs + sn);
              sn = s2;
              cs = c2;
              sv[k] = (float)sn;
              cv[k] = (float)cs;
            }
          }
          if (!hf) put_raw(r, k0 - 1, p0);
#pragma unroll
          for (int k = 0; k < 5; ++k) {
            put_raw(r, k0 + 2 * k, sv[k]);
            put_raw(r, k0 + 2 * k + 1, cv[k]);
          }
          if (a == 2 && hf) put_raw(r, 64 * pp + 63, 0.f);
        }
        tc::named_bar(1, kGWorkers * 32);
        // X_lo rows and the fp16 tile of the stage, one (ray, 4 columns) per thread
        for (int e = wt; e < kGN * 32; e += kGWorkers * 32) {
          const int r = e >> 5, c4 = (e & 31) * 4;
          const float4 v = *reinterpret_cast<const float4*>(xh + b_off_hl(r, c4));
          const float vv[4] = {v.x, v.y, v.z, v.w};
          float lo[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) lo[i] = tf32_rna(vv[i] - __uint_as_float(tf32_hi_bits(vv[i])));
          *reinterpret_cast<float4*>(xh + b_off_hl(kGN + r, c4)) = make_float4(lo[0], lo[1], lo[2], lo[3]);
          *reinterpret_cast<uint2*>(xb + b_off_bf16(r, c4)) = make_uint2(xh_pair(vv[0], vv[1]), xh_pair(vv[2], vv[3]));
        }
        tc::fence_proxy_async_smem();                         // generic stores -> tensor-core reads
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&S.fready[fs]);
      }
      // ---- 34 layers: layer L's outputs go to xb[(L + 1) & 1]
      for (int L = 0; L < kGLayers; ++L, ++dl) {
        const int ob = (L + 1) & 1;
        GBuf& O = S.xb[ob];
        if (epi) {
          // lanes l and l + 16 share output row `row`: lane l finishes rays 0-7, lane l + 16 rays 8-15
          const int k = 64 * (int)rank + row;                 // this row = the next layer's input column
          const float b = m.bias_pack[L * 256 + k];          // (load in flight while the MMAs run)
          tc::mbar_wait(&S.dfull, dl & 1);
          tc::tc_fence_after();
          if (warp == 4) GTRACE(80 + L, t == cid);
          const uint32_t lb = (uint32_t)(quad * 32) << 16;
          float acc[kGN];
          {
            // lanes 0-15: even accumulators, lanes 16-31: odd ones; columns r / 16 + r of each: X_hi / X_lo
            uint32_t a[kHH / 2][32];
#pragma unroll
            for (int i = 0; i < kHH / 2; ++i) tc::tmem_ld32(tbase + lb + 32 * i, a[i]);
            tc::tmem_ld_wait();
#pragma unroll
            for (int r = 0; r < kGN; ++r) {
              float p = __uint_as_float(a[0][r]), q = __uint_as_float(a[0][kGN + r]);
#pragma unroll
              for (int i = 1; i < kHH / 2; ++i) {
                p += __uint_as_float(a[i][r]);
                q += __uint_as_float(a[i][kGN + r]);
              }
              p += q;
              acc[r] = p + __shfl_xor_sync(0xffffffffu, p, 16);   // same sum in both lanes of the pair
            }
          }
          tc::tc_fence_before();
          const int r0 = lane < 16 ? 0 : kGN / 2;
#pragma unroll
          for (int i = 0; i < kGN / 2; ++i) {
            const int r = r0 + i;
            const float y = (lane < 16 ? acc[i] : acc[kGN / 2 + i]) + b;
            float v;
            if (L == 0 || L == kGLayers - 1) {
              v = y;                                          // head (no activation) / tail logits
              if (L == 0) xr[i] = v;
            } else if (L & 1) {
              v = fmaxf(y, 0.f);                              // fc1
            } else {
              v = xr[i] + fmaxf(y, 0.f);                      // fc2 + residual
              xr[i] = v;
            }
            *reinterpret_cast<float*>(O.xhl + b_off_hl(r, k)) = v;   // raw: the X row (X_hi by truncation)
          }
          if (warp == 4) GTRACE(280 + L, t == cid);
          tc::fence_proxy_async_smem();                       // the X rows are read by the bulk copies
          tc::named_bar(2, 128);
          if (warp == 4 && lane < 2 * (kGC - 1)) {
            // this CTA's 64 columns = atoms 2 rank, 2 rank + 1; their 16 X rows (2 KB each) go to
            // the same place in every peer, one bulk copy per lane (one thread's copies serialise)
            const int pr = ((int)rank + 1 + (lane >> 1)) % kGC, i = lane & 1;
            const uint32_t off = (uint32_t)ob * sizeof(GBuf) + (2 * rank + i) * kGAtom2;
            bulk_s2peer(peer_xb[pr] + off, O.xhl + (2 * rank + i) * kGAtom2, kGAtom, peer_bar[ob][pr]);
            if (lane == 0) {
              tc::mbar_expect_tx(&S.recv_bar[ob], (kGC - 1) * 2 * kGAtom);
              GTRACE(120 + L, t == cid);
            }
          }
        }
        // X_lo rows and the fp16 tile of one 64-column slab, one (ray, 4 columns) per thread
        auto split_slab = [&](int src, int e) {
          const int r = e >> 4, c4 = 64 * src + (e & 15) * 4;
          const float4 v = *reinterpret_cast<const float4*>(O.xhl + b_off_hl(r, c4));
          const float vv[4] = {v.x, v.y, v.z, v.w};
          float lo[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) lo[i] = tf32_rna(vv[i] - __uint_as_float(tf32_hi_bits(vv[i])));
          *reinterpret_cast<float4*>(O.xhl + b_off_hl(kGN + r, c4)) = make_float4(lo[0], lo[1], lo[2], lo[3]);
          *reinterpret_cast<uint2*>(O.xh16 + b_off_bf16(r, c4)) = make_uint2(xh_pair(vv[0], vv[1]), xh_pair(vv[2], vv[3]));
        };
        const bool more = L + 1 < kGLayers;
        // this CTA's slab (written by the epilogue warps) while the peers' copies are in flight
        tc::named_bar(1, kGWorkers * 32);
        if (more && wt < kGN * 16) split_slab((int)rank, wt);
        // the whole layer's X rows have landed here
        tc::mbar_wait(&S.recv_bar[ob], rc[ob] & 1);
        ++rc[ob];
        if (warp == 2) GTRACE(160 + L, t == cid);
        if (more) {
          for (int e = wt; e < (kGC - 1) * kGN * 16; e += kGWorkers * 32)
            split_slab(((int)rank + 1 + e / (kGN * 16)) % kGC, e % (kGN * 16));
          tc::fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) tc::mbar_arrive(&S.bready);
          if (warp == 2) GTRACE(200 + L, t == cid);
        }
      }
      (void)xb0;
      // ---- decode on rank 0 (model.py:277-293): tail rows fine 0-127, coarse 128-191, alpha 192,
      // in the X rows of xb[0] (the tail's output buffer)
      if (rank == 0) {
        const unsigned char* X = S.xb[kGLayers & 1].xhl;
        auto logit = [&](int r, int o) { return *reinterpret_cast<const float*>(X + b_off_hl(r, o)); };
        for (int r = warp - 2; r < kGN; r += kGWorkers) {
          if (!S.valid[r]) continue;
          float fv[4], cv[2];
#pragma unroll
          for (int i = 0; i < 4; ++i) fv[i] = logit(r, lane * 4 + i);
#pragma unroll
          for (int i = 0; i < 2; ++i) cv[i] = logit(r, 128 + lane * 2 + i);
          const float za = logit(r, 192);
          if (out.mode == OUT_LOGITS) {
            const size_t rowo = S.pix[r];
#pragma unroll
            for (int i = 0; i < 2; ++i) out.lc[rowo * 64 + lane * 2 + i] = cv[i];
#pragma unroll
            for (int i = 0; i < 4; ++i) out.lf[rowo * 128 + lane * 4 + i] = fv[i];
            if (lane == 0) out.la[rowo] = za;
          } else {
            const int fb = warp_argmax<4>(fv, logit(r, 0));
            const int cb = warp_argmax<2>(cv, logit(r, 128));
            if (lane == 0) {
              double wo[3], wd[3], lo[3], ld[3];
              item_local_ray(job, S.pix[r], S.obj[r], wo, wd, lo, ld);
              finish_ray(m, job, out, S.pix[r], S.obj[r], cb, fb, (double)za, wo, wd);
            }
          }
        }
      }
      tc::named_bar(1, kGWorkers * 32);                      // S.valid / S.ray / xb[0] reused by the next tile
    }
  }
  __syncwarp();
  tc::tc_fence_before();
  tc::cluster_sync();            // no CTA leaves while peers may still copy into it
  if (warp == 1) tc::tmem_dealloc<64>(tbase);
}

}  // namespace nedf

extern "C" int nedf_diag_guard_trace(int enable, unsigned long long* out, int n) {
  using namespace nedf;
  if (enable >= 0) {
    int v = enable;
    if (cudaMemcpyToSymbol(g_gtrace_on, &v, sizeof(int)) != cudaSuccess) return NEDF_ERR_CUDA;
  }
  if (out && n > 0) {
    if (n > 320) n = 320;
    if (cudaMemcpyFromSymbol(out, g_gtrace, n * sizeof(unsigned long long)) != cudaSuccess) return NEDF_ERR_CUDA;
  }
  return NEDF_OK;
}

namespace nedf {

bool guard_tc_available() {
  int dev = 0, major = 0, optin = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  return major == 10 && (size_t)optin >= sizeof(GSmem) + 1024;
}

static int max_clusters_dev[kMaxDevices] = {};

static cudaError_t guard_tc_setup(int n_sms) {
  int& max_clusters = max_clusters_dev[current_device()];
  const size_t smem = sizeof(GSmem) + 1024;
  if (max_clusters == 0) {
    cudaError_t e = cudaFuncSetAttribute(guard_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(kGC * (n_sms / kGC), 1, 1);
    cfg.blockDim = dim3(kGThreads, 1, 1);
    cfg.dynamicSmemBytes = smem;
    int n = 0;
    e = cudaOccupancyMaxActiveClusters(&n, guard_tc_kernel, &cfg);
    if (e != cudaSuccess) return e;
    max_clusters = n > 0 ? n : 1;
    if (getenv("NEDF_VERBOSE")) fprintf(stderr, "nedf: tcgen05 guard kernel, %d co-resident clusters\n", n);
  }
  return cudaSuccess;
}

int guard_tc_capacity(int n_sms) {
  if (guard_tc_setup(n_sms) != cudaSuccess) return 0;
  return max_clusters_dev[current_device()];
}

cudaError_t launch_guard_tc(const GroupTable& gt, const ListSet& ls, const RayJob& job, const OutSpec& out,
                            int n_sms, cudaStream_t stream, int max_tiles16) {
  cudaError_t e = guard_tc_setup(n_sms);
  if (e != cudaSuccess) return e;
  const int max_clusters = max_clusters_dev[current_device()];
  guard_tc_kernel<<<kGC * max_clusters, kGThreads, sizeof(GSmem) + 1024, stream>>>(gt, ls, job, out, max_tiles16);
  return cudaGetLastError();
}


// Guard image: stage q (head K block q < 8, then layer L = 1 + (q - 8) / 2, K block j = (q - 8) % 2),
// CTA r -> 48 KB at ((q * 4 + r) * 48 KB): W_hi fp32 [4 atoms of 32 K][64 rows][128 B] then
// 2^11 W_lo fp16 [2 atoms of 64 K][64 rows][128 B], both 128B-swizzled K-major; row n is the
// layer's output 64 r + n, K index k = 128 j + kk.  Head columns: the 16 points' 63 features + 1
// zero; tail rows: fine 0-127, coarse 128-191, alpha 192, zero padding.
cudaError_t guard_tc_pack(const float* P, int d_in, int F, int n_blocks, int n_coarse, int n_fine, void** dev) {
  if (F != 256 || n_blocks != 16 || d_in != kDin || n_coarse != 64 || n_fine != 128) return cudaErrorInvalidValue;
  std::vector<unsigned char> img((size_t)kGStagesPerTile * kGC * kGStageBytes, 0);
  size_t p = 0;
  const float* Wh = P + p; p += (size_t)F * d_in + F;
  std::vector<const float*> Wl(32);
  for (int l = 0; l < 32; ++l) { Wl[l] = P + p; p += (size_t)F * F + F; }
  const float* Wa = P + p; p += (size_t)(n_coarse + 1) * F + n_coarse + 1;
  const float* Wb = P + p;
  auto w_of = [&](int L, int o, int k) -> float {
    if (L == 0) {
      const int pt = k / 64, j = k % 64;
      return j < 63 ? Wh[(size_t)o * d_in + 63 * pt + j] : 0.f;
    }
    if (L <= 32) return Wl[L - 1][(size_t)o * F + k];
    if (o < 128) return Wb[(size_t)o * F + k];
    if (o < 128 + n_coarse + 1) return Wa[(size_t)(o - 128) * F + k];
    return 0.f;
  };
  for (int q = 0; q < kGStagesPerTile; ++q) {
    const int L = q < kGHeadStages ? 0 : 1 + (q - kGHeadStages) / kGBodyStages;
    const int j = q < kGHeadStages ? q : (q - kGHeadStages) % kGBodyStages;
    for (int r = 0; r < kGC; ++r) {
      unsigned char* st = img.data() + ((size_t)q * kGC + r) * kGStageBytes;
      for (int n = 0; n < kGM; ++n)
        for (int kk = 0; kk < 128; ++kk) {
          const float w = w_of(L, kGM * r + n, 128 * j + kk);
          uint32_t u;
          memcpy(&u, &w, 4);
          const uint32_t hb = u & 0xFFFFE000u;
          float hi;
          memcpy(&hi, &hb, 4);
          const float lo = w - hi;
          memcpy(st + (kk >> 5) * (kGM * 128) + tc::sw128_offset(n, (kk & 31) >> 2) + ((kk & 3) << 2), &hi, 4);
          const uint16_t lb = __half_as_ushort(__float2half_rn(lo * kGLoScale));
          memcpy(st + kGHiBytes + (kk >> 6) * (kGM * 128) + tc::sw128_offset(n, (kk & 63) >> 3) + ((kk & 7) << 1),
                 &lb, 2);
        }
    }
  }
  cudaError_t e = cudaMalloc(dev, img.size());
  if (e == cudaSuccess) e = cudaMemcpy(*dev, img.data(), img.size(), cudaMemcpyHostToDevice);
  return e;
}

}  // namespace nedf
