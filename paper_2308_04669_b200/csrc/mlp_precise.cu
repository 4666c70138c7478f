// fp32-accurate network for LARGE near-tie batches on tcgen05 (throughput form
// of the guard; guard_tc.cu is the latency form for small batches).
//
// Why: the fp16 chain's logit error (~1e-3 of max|logit|) is
// comparable to a trained NeDF's fine-bin margins, so on distilled models the
// guard flags a third of all evaluations (324k rays on the trained config-4
// frame).  guard_tc moves 16 rays per 4-SM cluster per 35-layer chain -- right
// for the few hundred rays of random-init models, 58 ms for 324k.  This kernel
// is data parallel like the fast network (mlp_tc.cu): one CTA per SM,
// persistent over 128-ray tiles, every CTA streaming all weights, no exchange.
//
// Arithmetic: both operands split into fp16 pairs, x = x_hi + 2^-12 x_lo,
// W = W_hi + 2^-12 W_lo (x_hi = fp16(x), x_lo = fp16(4096 (x - x_hi)); the
// weight halves are two stage-aligned images), three M128 x N128 x K16 MMAs
// per k-step:
//   main  += x_hi W_hi
//   cross += x_lo W_hi + x_hi W_lo            (both at scale 2^12)
//   y = main + 2^-12 cross                    (fp32 accumulation, fp32 epilogue)
// Dropped: x_lo W_lo (2^-24 of a product) and the fp16 roundings of the lo
// halves (~2^-23): float32-level.  The residual stream stays fp32 in the
// epilogue's registers.
//
// Per CTA (20 warps): warp 0 streams [W_hi | W_lo] stages (32 KB each) through
// a 3-slot ring; warp 1 issues the MMAs (both operands from shared memory:
// the layer input's hi / lo tiles, 128 KB, are written by the epilogue); warps
// 4-19 are 4 worker groups of 4 warps (one per TMEM lane quadrant, thread =
// ray).  Head: group g encodes points g, g + 4, ... (float64 sincospi +
// double-angle steps) into 32 KB slot g of the same region.  Body: group g is
// the epilogue of output columns [64 g, 64 g + 64): main + cross, bias, ReLU /
// residual, the next layer's hi / lo atom g; the tail's logits are decoded
// across the groups (first-max argmax, alpha, world depth, z-buffer
// atomicMin) like the other kernels.  Layers run back to back (the epilogue
// rewrites the one input buffer), so per layer: 96 MMAs (~6.9k cycles) + the
// epilogue (~4.7k with four warps per SM sub-partition; 10k with two).
// Registers: 640 threads launch at 96; warps 0-3 release theirs so the
// workers run at 112.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "frame.cuh"
#include "tc_ptx.cuh"

namespace nedf {
namespace {

constexpr int kPThreads = 640;                  // 20 warps: producer, MMA, 2 idle, 16 workers
constexpr uint32_t kPStage = 16384;             // one [128 N x 64 K] fp16 weight stage (hi or lo)
constexpr int kPRing = 3;                       // slots of [hi | lo] stage pairs (32 KB)
constexpr int kPHeadStages = 32;                // 16 points x 2 slices
constexpr int kPBodyLayers = 32;
constexpr int kPStagesPerTile = kPHeadStages + (kPBodyLayers + 1) * 8;   // 296, the fast image's order
constexpr uint32_t kPAtom = 16384;              // one [128 rows x 64 K] fp16 A atom
constexpr float kPLo = 4096.f;                  // lo halves are stored x 2^12

struct PSmem {
  unsigned char a[8 * kPAtom];                  // body: hi atoms 0-3, lo atoms 4-7; head: 4 slots x (hi, lo)
  unsigned char ring[kPRing][2 * kPStage];
  uint64_t full[kPRing], empty[kPRing];
  uint64_t afull[4], aempty[4];                 // head slots: encoders -> MMA, MMA -> encoders
  uint64_t aready;                              // body input written (16 worker warps)
  uint64_t dfull;                               // a layer's accumulators complete
  uint32_t tmem_base;
  int tiles[65];
};

// tail decode scratch (the first 2 KB of head slot 0: free once the tail's MMAs are done,
// rewritten only by worker group 0's next head, after its decode)
struct PDecode {
  float fine_best[128];                         // group 1: max of fine logits 64-127
  int fine_idx[128];                            //          and its first index
  int coarse[128];                              // group 2: coarse argmax
  float alpha[128];                             // group 3: the alpha logit
};

__device__ __forceinline__ uint32_t h2_pack(float a, float b) { return tc::pack_h2(a, b); }

// (hi, lo) fp16 halves of 8 fp32 values, lo = fp16(4096 (v - hi))
__device__ __forceinline__ void split8(const float* v, uint4& hi, uint4& lo) {
  uint32_t h[4], l[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const __half2 hh = __floats2half2_rn(v[2 * i], v[2 * i + 1]);
    const float2 hf = __half22float2(hh);
    h[i] = *reinterpret_cast<const uint32_t*>(&hh);
    l[i] = h2_pack((v[2 * i] - hf.x) * kPLo, (v[2 * i + 1] - hf.y) * kPLo);
  }
  hi = make_uint4(h[0], h[1], h[2], h[3]);
  lo = make_uint4(l[0], l[1], l[2], l[3]);
}

}  // namespace

// timeline of CTA 0's first tile (diagnostics): [L] layer L's MMAs start, [40 + L] issued,
// [80 + L] epilogue has the accumulators, [120 + L] epilogue done (warp 8), [160 + p] head point p encoded
__device__ unsigned long long g_ptrace[200];
__device__ int g_ptrace_on;

__global__ void __launch_bounds__(kPThreads, 1) mlp_precise_kernel(GroupTable gt, ListSet ls, RayJob job,
                                                                   OutSpec out, int min_tiles16) {
  extern __shared__ unsigned char smem_raw[];
  unsigned char* base_ptr = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);
  PSmem& S = *reinterpret_cast<PSmem*>(base_ptr);
  const int tid = threadIdx.x;
  const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);
  const int lane = tid & 31;
  const int ng = ls.n_groups < 64 ? ls.n_groups : 64;
  const bool feats_in = out.feats != nullptr;

  // small batches belong to the latency kernel (guard_tc): same total, decided on the device
  {
    int t16 = 0;
    for (int g = 0; g < ng; ++g) t16 += (ls.count[g] + 15) / 16;
    if (t16 <= min_tiles16) return;
  }
  if (tid == 0) {
    int cum = 0;
    S.tiles[0] = 0;
    for (int g = 0; g < ng; ++g) {
      cum += (ls.count[g] + 127) / 128;
      S.tiles[g + 1] = cum;
    }
    for (int i = 0; i < kPRing; ++i) { tc::mbar_init(&S.full[i], 1); tc::mbar_init(&S.empty[i], 1); }
    for (int i = 0; i < 4; ++i) { tc::mbar_init(&S.afull[i], 4); tc::mbar_init(&S.aempty[i], 1); }
    tc::mbar_init(&S.aready, 16);
    tc::mbar_init(&S.dfull, 1);
    tc::mbar_fence_init();
  }
  if (warp == 1) tc::tmem_alloc<512>(&S.tmem_base);     // main[2] cols 0-255, cross[2] cols 256-511
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tbase = S.tmem_base;
  const int total = S.tiles[ng];
  const bool trace = g_ptrace_on && blockIdx.x == 0 && lane == 0;
#define PTRACE(i, cond) \
  do {                  \
    if (trace && (cond)) g_ptrace[(i)] = clock64(); \
  } while (0)
  auto lookup = [&](int t, int& g, int64_t& base, int& n) {
    g = 0;
    while (g < ng - 1 && t >= S.tiles[g + 1]) ++g;
    const int first = (t - S.tiles[g]) * 128;
    n = min(128, ls.count[g] - first);
    base = ls.offset[g] + first;
  };

  if (warp < 4) {
    // registers: 640 threads launch at 96; the 16 workers take 112 from what warps 0-3 release
    if (warp < 2) tc::reg_dealloc<32>(); else tc::reg_dealloc<24>();
    if (warp == 0) {
      // ------------------------------------------------------------------ weight producer
      uint32_t gq = 0;
      for (int t = blockIdx.x; t < total; t += gridDim.x) {
        int g, n;
        int64_t b0;
        lookup(t, g, b0, n);
        const unsigned char* hi = reinterpret_cast<const unsigned char*>(gt.models[g].wpack);
        const unsigned char* lo = reinterpret_cast<const unsigned char*>(gt.models[g].wpack_lo);
        for (int q = 0; q < kPStagesPerTile; ++q, ++gq) {
          const int s = gq % kPRing;
          if (lane == 0) {
            tc::mbar_wait(&S.empty[s], ((gq / kPRing) & 1) ^ 1);
            tc::mbar_expect_tx(&S.full[s], 2 * kPStage);
          }
          __syncwarp();
          // four lanes, one 8 KB piece each (copies issued by one thread serialise)
          if (lane < 4) {
            const unsigned char* src = (lane < 2 ? hi : lo) + (size_t)q * kPStage + (lane & 1) * (kPStage / 2);
            tc::bulk_g2s(&S.ring[s][(lane >> 1) * kPStage + (lane & 1) * (kPStage / 2)], src, kPStage / 2, &S.full[s]);
          }
        }
      }
    } else if (warp == 1) {
      // ------------------------------------------------------------------ MMA issuer
      const uint32_t idesc = tc::idesc_f16(128, 128);
      uint32_t gq = 0, hq = 0, bl = 0;
      const uint32_t a0 = tc::smem_u32(S.a);
      for (int t = blockIdx.x; t < total; t += gridDim.x) {
        for (int L = 0; L < kPBodyLayers + 2; ++L) {
          if (L > 0) {
            tc::mbar_wait(&S.aready, bl & 1);
            ++bl;
          }
          PTRACE(L, t == (int)blockIdx.x);
          const int npt = L == 0 ? 16 : 1;                    // head: per point; body: one pass
          for (int pt = 0; pt < npt; ++pt) {
            uint32_t a_hi = a0, a_lo = a0 + 4 * kPAtom;
            if (L == 0) {
              const int slot = hq & 3;
              tc::mbar_wait(&S.afull[slot], (hq >> 2) & 1);
              a_hi = a0 + slot * 2 * kPAtom;
              a_lo = a_hi + kPAtom;
            }
            for (int s = 0; s < 2; ++s) {
              const int nkc = L == 0 ? 1 : 4;
              for (int kc = 0; kc < nkc; ++kc, ++gq) {
                const int slot_w = gq % kPRing;
                tc::mbar_wait(&S.full[slot_w], (gq / kPRing) & 1);
                tc::tc_fence_after();
                if (tc::elect_one()) {
                  const uint32_t w = tc::smem_u32(&S.ring[slot_w][0]);
                  const uint64_t whi = tc::sw128_desc(w), wlo = tc::sw128_desc(w + kPStage);
                  const uint64_t ahi = tc::sw128_desc(a_hi + kc * kPAtom), alo = tc::sw128_desc(a_lo + kc * kPAtom);
                  const uint32_t dm = tbase + 128 * s, dc = tbase + 256 + 128 * s;
#pragma unroll
                  for (int ks = 0; ks < 4; ++ks) {
                    const uint32_t o = (ks * 32) >> 4;
                    const uint32_t first = (pt == 0 && kc == 0 && ks == 0) ? 0u : 1u;
                    tc::mma_ss(dm, ahi + o, whi + o, idesc, first);
                    tc::mma_ss(dc, alo + o, whi + o, idesc, first);
                    tc::mma_ss(dc, ahi + o, wlo + o, idesc, 1u);
                  }
                  tc::mma_commit(&S.empty[slot_w]);
                }
                __syncwarp();
              }
            }
            if (L == 0) {
              if (tc::elect_one()) tc::mma_commit(&S.aempty[hq & 3]);
              __syncwarp();
              ++hq;
            }
          }
          if (tc::elect_one()) tc::mma_commit(&S.dfull);
          __syncwarp();
          PTRACE(40 + L, t == (int)blockIdx.x);
        }
      }
    }
  } else {
    tc::reg_alloc<112>();
    // ---------------------------------------------------------------------- workers
    // 16 warps in 4 groups; group sl = warps 4 + 4 sl .. 7 + 4 sl covers the four TMEM lane
    // quadrants (warp & 3), thread = ray (row).  Head: group sl encodes points sl, sl + 4, ...
    // into head slot sl.  Body: group sl owns output columns [64 sl, 64 sl + 64) -- the
    // epilogue (main + cross, bias, ReLU / residual, the next layer's hi / lo atom sl).
    const int q = warp & 3, sl = (warp - 4) >> 2;
    const int row = 32 * q + lane;
    const uint32_t lane_addr = tbase + ((uint32_t)(32 * q) << 16) + 64 * sl;
    uint32_t dl = 0, use = 0;
    float x[64];                                             // residual stream: columns [64 sl, 64 sl + 64)
    PDecode& D = *reinterpret_cast<PDecode*>(S.a);
    for (int t = blockIdx.x; t < total; t += gridDim.x) {
      int g, n;
      int64_t b0;
      lookup(t, g, b0, n);
      const DevModel& m = gt.models[g];
      const bool valid = row < n;
      // ---- head input: 16 points x 64 features (geometry.py:312-342 in float64)
      {
        double lo3[3] = {0, 0, 0}, ld3[3] = {0, 0, 0}, t0 = 0, t1 = 0;
        uint32_t pix = 0;
        if (valid) {
          pix = ls.pix[b0 + row];
          if (!feats_in) {
            double wo[3], wd[3];
            item_local_ray(job, pix, ls.obj[b0 + row], wo, wd, lo3, ld3);
            slab_clip(lo3, ld3, m.bmin, m.bmax, t0, t1);
          }
        }
        unsigned char* hi = S.a + sl * 2 * kPAtom;
        unsigned char* lo = hi + kPAtom;
        if (warp == 4) PTRACE(192, t == (int)blockIdx.x);
        for (int pt = sl; pt < 16; pt += 4, ++use) {
          // earlier uses of this slot (this tile's) must have left the tensor pipe; the previous
          // tile's are done (its tail's accumulators were read after all of its MMAs)
          if (pt >= 4) tc::mbar_wait(&S.aempty[sl], (use - 1) & 1);
          if (warp == 4) PTRACE(176 + pt, t == (int)blockIdx.x);
          float f[64];
          if (!valid) {
#pragma unroll
            for (int j = 0; j < 64; ++j) f[j] = 0.f;
          } else if (feats_in) {
            const float* src = out.feats + (size_t)pix * kDin + pt * kPerPoint;
#pragma unroll
            for (int j = 0; j < 63; ++j) f[j] = src[j];
            f[63] = 0.f;
          } else {
            const double tt = t0 + (t1 - t0) * lin16(pt);
#pragma unroll
            for (int a = 0; a < 3; ++a) {
              const double p = ((lo3[a] + tt * ld3[a]) - m.c[a]) / m.h[a];
              f[21 * a] = (float)p;
              double sn, cs;
              sincospi(p, &sn, &cs);
              f[21 * a + 1] = (float)sn;
              f[21 * a + 2] = (float)cs;
#pragma unroll
              for (int k = 1; k < kLevels; ++k) {
                const double s2 = 2.0 * sn * cs, c2 = (cs - sn) * (cs + sn);
                sn = s2;
                cs = c2;
                f[21 * a + 1 + 2 * k] = (float)sn;
                f[21 * a + 2 + 2 * k] = (float)cs;
              }
            }
            f[63] = 0.f;
          }
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            uint4 h, l;
            split8(f + 8 * c, h, l);
            const uint32_t o = tc::sw128_offset(row, c);
            *reinterpret_cast<uint4*>(hi + o) = h;
            *reinterpret_cast<uint4*>(lo + o) = l;
          }
          tc::fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) tc::mbar_arrive(&S.afull[sl]);
          if (warp == 4) PTRACE(160 + pt, t == (int)blockIdx.x);
        }
      }
      // ---- layers
      for (int L = 0; L < kPBodyLayers + 2; ++L, ++dl) {
        const bool tail = L == kPBodyLayers + 1;
        const float* bias = m.bias_pack + L * 256 + 64 * sl;
        tc::mbar_wait(&S.dfull, dl & 1);
        tc::tc_fence_after();
        if (warp == 4) PTRACE(80 + L, t == (int)blockIdx.x);
#pragma unroll
        for (int j2 = 0; j2 < 4; ++j2) {                       // 16-column chunks: one TMEM wait each
          float4 b0 = *reinterpret_cast<const float4*>(bias + 16 * j2);   // latency overlaps TMEM's
          float4 b1 = *reinterpret_cast<const float4*>(bias + 16 * j2 + 4);
          uint32_t rm[16], rx[16];
          tc::tmem_ld16(lane_addr + 16 * j2, rm);
          tc::tmem_ld16(lane_addr + 256 + 16 * j2, rx);
          tc::tmem_ld_wait();
#pragma unroll
          for (int jh = 0; jh < 2; ++jh) {
            const int j = 2 * j2 + jh;                         // 8-column group
            if (jh == 1) {
              b0 = *reinterpret_cast<const float4*>(bias + 16 * j2 + 8);
              b1 = *reinterpret_cast<const float4*>(bias + 16 * j2 + 12);
            }
            const float bb[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
            float v[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const float y = (__uint_as_float(rm[8 * jh + i]) + __uint_as_float(rx[8 * jh + i]) * (1.0f / kPLo)) + bb[i];
              const int c = 8 * j + i;
              if (L == 0 || tail) {
                x[c] = y;                                      // head output (no activation) / tail logits
                v[i] = y;
              } else if (L & 1) {
                v[i] = fmaxf(y, 0.f);                          // fc1: h
              } else {
                x[c] = x[c] + fmaxf(y, 0.f);                   // fc2: residual
                v[i] = x[c];
              }
            }
            if (!tail) {
              // next layer's input, K columns 64 sl + 8 j .. + 7: atom sl, chunk j
              uint4 h, l;
              split8(v, h, l);
              const uint32_t o = sl * kPAtom + tc::sw128_offset(row, j);
              *reinterpret_cast<uint4*>(S.a + o) = h;
              *reinterpret_cast<uint4*>(S.a + 4 * kPAtom + o) = l;
            }
          }
        }
        tc::tc_fence_before();
        if (!tail) {
          tc::fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) tc::mbar_arrive(&S.aready);
        }
        if (warp == 4) PTRACE(120 + L, t == (int)blockIdx.x);
      }
      // ---- decode (model.py:277-293): logits 0-127 fine (groups 0, 1), 128-191 coarse
      // (group 2), 192 alpha (group 3); first-max argmax like the other kernels
      int best_i = 0;
      float best = x[0];
      if (sl < 3) {
#pragma unroll
        for (int c = 1; c < 64; ++c)
          if (x[c] > best) { best = x[c]; best_i = c; }
      }
      const size_t pix_l = valid ? (size_t)ls.pix[b0 + row] : 0;
      if (valid && out.mode == OUT_LOGITS) {
        if (sl < 2) {
          for (int c = 0; c < 64; ++c) out.lf[pix_l * 128 + 64 * sl + c] = x[c];
        } else if (sl == 2) {
          for (int c = 0; c < 64; ++c) out.lc[pix_l * 64 + c] = x[c];
        } else {
          out.la[pix_l] = x[0];
        }
      }
      if (sl == 1) { D.fine_best[row] = best; D.fine_idx[row] = 64 + best_i; }
      if (sl == 2) D.coarse[row] = best_i;
      if (sl == 3) D.alpha[row] = x[0];
      tc::named_bar(1, 512);
      if (sl == 0 && valid && out.mode != OUT_LOGITS) {
        const int fb = D.fine_best[row] > best ? D.fine_idx[row] : best_i;
        const uint32_t obj = ls.obj[b0 + row];
        double wo[3], wd[3], lo[3], ld[3];
        item_local_ray(job, (uint32_t)pix_l, obj, wo, wd, lo, ld);
        finish_ray(m, job, out, (uint32_t)pix_l, obj, D.coarse[row], fb, (double)D.alpha[row], wo, wd);
      }
      if (sl == 0) tc::named_bar(2, 128);                    // all of group 0 has read D before slot 0 is rewritten
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc<512>(tbase);
}

extern "C" int nedf_diag_precise_trace(int enable, unsigned long long* out, int n) {
  if (enable >= 0 && cudaMemcpyToSymbol(g_ptrace_on, &enable, sizeof(int)) != cudaSuccess) return NEDF_ERR_CUDA;
  if (out && n > 0 && cudaMemcpyFromSymbol(out, g_ptrace, (n < 200 ? n : 200) * sizeof(unsigned long long)) != cudaSuccess)
    return NEDF_ERR_CUDA;
  return NEDF_OK;
}

cudaError_t launch_mlp_precise(const GroupTable& gt, const ListSet& ls, const RayJob& job, const OutSpec& out,
                               int n_sms, int min_tiles16, cudaStream_t stream) {
  static bool configured[kMaxDevices] = {};
  const size_t smem = sizeof(PSmem) + 1024;
  const int dev = current_device();
  if (!configured[dev]) {
    cudaError_t e = cudaFuncSetAttribute(mlp_precise_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    configured[dev] = true;
  }
  mlp_precise_kernel<<<n_sms, kPThreads, smem, stream>>>(gt, ls, job, out, min_tiles16);
  return cudaGetLastError();
}

size_t mlp_precise_smem_bytes() { return sizeof(PSmem) + 1024; }

}  // namespace nedf
