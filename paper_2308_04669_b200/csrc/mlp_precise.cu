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
// Per CTA (16 warps): warp 0 streams [W_hi | W_lo] stages (32 KB each) through
// a 3-slot ring; warp 1 issues the MMAs (both operands from shared memory:
// the layer input's hi / lo tiles, 128 KB, are written by the epilogue); warps
// 4-7 encode the head input per point (float64 sincospi + double-angle steps)
// into four 32 KB slots of the same region; warps 8-15 are the epilogue
// (thread = ray x 128-column slice): main + cross, bias, ReLU / residual, the
// next layer's hi / lo tiles; the tail's logits are decoded here (first-max
// argmax, alpha, world depth, z-buffer atomicMin) like the other kernels.
// Layers run back to back (the epilogue rewrites the one input buffer), so
// per layer: 96 MMAs + the epilogue.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "frame.cuh"
#include "tc_ptx.cuh"

namespace nedf {
namespace {

constexpr int kPThreads = 512;
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
  uint64_t aready;                              // body input written (8 epilogue warps)
  uint64_t dfull;                               // a layer's accumulators complete
  uint64_t tfree;                               // the tile's tail done: the input region may take the next head
  uint32_t tmem_base;
  int tiles[65];
  int dec_c[128];
  float dec_a[128];
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
    tc::mbar_init(&S.aready, 8);
    tc::mbar_init(&S.dfull, 1);
    tc::mbar_init(&S.tfree, 8);
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
    tc::reg_dealloc<40>();
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
  } else if (warp < 8) {
    tc::reg_dealloc<120>();
    // -------------------------------------------------------------------- encoders (thread = ray)
    const int row = tid - 128;
    uint32_t hq = 0, tfc = 0;
    for (int t = blockIdx.x; t < total; t += gridDim.x) {
      int g, n;
      int64_t b0;
      lookup(t, g, b0, n);
      const DevModel& m = gt.models[g];
      const bool valid = row < n;
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
      if (t != (int)blockIdx.x) {                            // the previous tile's tail has left the region
        tc::mbar_wait(&S.tfree, tfc & 1);
        ++tfc;
      }
      for (int pt = 0; pt < 16; ++pt, ++hq) {
        const int slot = hq & 3;
        if (pt >= 4) tc::mbar_wait(&S.aempty[slot], ((hq >> 2) - 1) & 1);
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
          // geometry.py:312-342 in float64: sincospi at level 0, double-angle steps for 1-9
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
        unsigned char* hi = S.a + slot * 2 * kPAtom;
        unsigned char* lo = hi + kPAtom;
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
        if (lane == 0) tc::mbar_arrive(&S.afull[slot]);
        if (warp == 4) PTRACE(160 + pt, t == (int)blockIdx.x);
      }
    }
  } else {
    tc::reg_alloc<176>();
    // -------------------------------------------------------------------- epilogue (thread = ray x slice)
    const int q = warp & 3, hc = (warp - 8) >> 2;            // TMEM lane quadrant, output slice
    const int row = 32 * q + lane;
    const uint32_t lane_addr = tbase + ((uint32_t)(32 * q) << 16);
    uint32_t dl = 0;
    float x[128];                                            // residual stream: columns [128 hc, 128 hc + 128)
    for (int t = blockIdx.x; t < total; t += gridDim.x) {
      int g, n;
      int64_t b0;
      lookup(t, g, b0, n);
      const DevModel& m = gt.models[g];
      for (int L = 0; L < kPBodyLayers + 2; ++L, ++dl) {
        const bool tail = L == kPBodyLayers + 1;
        const float* bias = m.bias_pack + L * 256 + 128 * hc;
        tc::mbar_wait(&S.dfull, dl & 1);
        tc::tc_fence_after();
        if (warp == 8) PTRACE(80 + L, t == (int)blockIdx.x);
#pragma unroll
#pragma unroll
        for (int j2 = 0; j2 < 8; ++j2) {                       // 16-column chunks: one TMEM wait each
          float bb2[16];                                       // bias first: its latency overlaps TMEM's
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const float4 b4 = *reinterpret_cast<const float4*>(bias + 16 * j2 + 4 * i);
            bb2[4 * i] = b4.x;
            bb2[4 * i + 1] = b4.y;
            bb2[4 * i + 2] = b4.z;
            bb2[4 * i + 3] = b4.w;
          }
          uint32_t rm[16], rx[16];
          tc::tmem_ld16(lane_addr + 128 * hc + 16 * j2, rm);
          tc::tmem_ld16(lane_addr + 256 + 128 * hc + 16 * j2, rx);
          tc::tmem_ld_wait();
#pragma unroll
          for (int jh = 0; jh < 2; ++jh) {
            const int j = 2 * j2 + jh;                         // 8-column group
            const float* bb = bb2 + 8 * jh;
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
              // next layer's input, K columns 128 hc + 8 j .. + 7: atom (2 hc + j / 8), chunk j % 8
              uint4 h, l;
              split8(v, h, l);
              const uint32_t o = (2 * hc + (j >> 3)) * kPAtom + tc::sw128_offset(row, j & 7);
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
        if (warp == 8) PTRACE(120 + L, t == (int)blockIdx.x);
      }
      // ---- decode (model.py:277-293): slice 0 = fine logits, slice 1 = coarse (0-63) and alpha (64)
      const bool valid = row < n;
      if (hc == 1) {
        int cb = 0;
        float best = x[0];
#pragma unroll
        for (int c = 1; c < 64; ++c)
          if (x[c] > best) { best = x[c]; cb = c; }
        S.dec_c[row] = cb;
        S.dec_a[row] = x[64];
        if (valid && out.mode == OUT_LOGITS) {
          const size_t r = ls.pix[b0 + row];
          for (int c = 0; c < 64; ++c) out.lc[r * 64 + c] = x[c];
          out.la[r] = x[64];
        }
      }
      tc::named_bar(1, 256);
      if (hc == 0 && valid) {
        const uint32_t pix = ls.pix[b0 + row], obj = ls.obj[b0 + row];
        if (out.mode == OUT_LOGITS) {
          for (int c = 0; c < 128; ++c) out.lf[(size_t)pix * 128 + c] = x[c];
        } else {
          int fb = 0;
          float best = x[0];
#pragma unroll
          for (int c = 1; c < 128; ++c)
            if (x[c] > best) { best = x[c]; fb = c; }
          double wo[3], wd[3], lo[3], ld[3];
          item_local_ray(job, pix, obj, wo, wd, lo, ld);
          finish_ray(m, job, out, pix, obj, S.dec_c[row], fb, (double)S.dec_a[row], wo, wd);
        }
      }
      tc::named_bar(1, 256);                                  // dec_* reused by the next tile
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&S.tfree);
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
