// fp32 CUDA-core network with streamed weights, for small ray batches.
//
// Role: re-evaluate the rays the tensor-core kernel's near-tie guard flags
// (a few hundred per frame), and serve NEDF_PREC_FP32 for paper-shaped models.
// The per-ray critical path is the 35-layer chain, so the kernel spreads rays
// thinly (R per CTA, one CTA per SM) and streams the fp32 weight image
// through a 4-stage shared-memory ring with bulk async copies; each stage is
// [32 input rows x 256 outputs] (32 KB) and thread o owns output column o.
// Features are float64-accurate, weights are the .nedm float32 values, math is
// fp32 -- the same arithmetic as mlp_simt.cu.
#include <vector>

#include "common.cuh"
#include "encode.cuh"
#include "frame.cuh"
#include "tc_ptx.cuh"

namespace nedf {
namespace {

constexpr int kThreads = 512;                // 256 output columns x 2 halves of each stage's rows
constexpr int kRows = 32;                  // input rows per stage
constexpr int kStageFloats = kRows * 256;
constexpr int kStageBytes = kStageFloats * 4;
constexpr int kHeadStages = 1024 / kRows;  // 16 points x 64 rows (63 + 1 zero)
constexpr int kLayerStages = 256 / kRows;
constexpr int kStreamStages = kHeadStages + 33 * kLayerStages;   // 296

// weight ring depth: as deep as shared memory allows next to the activations
template <int R>
constexpr int ring_depth() { return R >= 32 ? 3 : (R >= 16 ? 4 : 5); }

template <int R>
struct StreamSmem {
  static constexpr int kRing = ring_depth<R>();
  float ring[kRing][kStageFloats];
  float x[R][256];
  float h[R][256];
  float f[R][64];
  float part[R][256];            // partial sums of the upper row half
  double ray[R][8];              // pa[3], pb[3], t0, t1
  uint32_t pix[R], obj[R];
  int valid[R];
  uint64_t full[kRing];
};

}  // namespace

template <int R>
__global__ void __launch_bounds__(kThreads, 1)
mlp_fp32_stream_kernel(GroupTable gt, ListSet ls, RayJob job, OutSpec out) {
  constexpr int kRing = StreamSmem<R>::kRing;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  StreamSmem<R>& S = *reinterpret_cast<StreamSmem<R>*>(smem_raw);
  __shared__ int s_tiles[65];
  const int tid = threadIdx.x;
  const int ng = ls.n_groups < 64 ? ls.n_groups : 64;
  if (tid == 0) {
    int cum = 0;
    s_tiles[0] = 0;
    for (int g = 0; g < ng; ++g) {
      cum += (ls.count[g] + R - 1) / R;
      s_tiles[g + 1] = cum;
    }
    for (int i = 0; i < kRing; ++i) tc::mbar_init(&S.full[i], 1);
    tc::mbar_fence_init();
  }
  __syncthreads();
  const int total = s_tiles[ng];
  uint32_t fill = 0;          // stages issued so far (all tiles), drives slot/parity
  uint32_t used = 0;          // stages consumed so far
  const bool feats_in = out.feats != nullptr;
  for (int t = blockIdx.x; t < total; t += gridDim.x) {
    int g = 0;
    while (g < ng - 1 && t >= s_tiles[g + 1]) ++g;
    const int lt = t - s_tiles[g];
    int n = ls.count[g] - lt * R;
    n = n < R ? n : R;
    const int64_t base = ls.offset[g] + (int64_t)lt * R;
    const DevModel& m = gt.models[g];
    const float* wimg = m.wstream;
    // prologue: first kRing stages of this tile
    // one issuing thread per ring slot: bulk copies from one thread serialise
    if (tid < kRing) {
      const int i = tid;
      const int slot = (fill + i) % kRing;
      tc::mbar_expect_tx(&S.full[slot], kStageBytes);
      tc::bulk_g2s(S.ring[slot], wimg + (size_t)i * kStageFloats, kStageBytes, &S.full[slot]);
    }
    fill += kRing;
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
    __syncthreads();
    float acc[R];
#pragma unroll
    for (int r = 0; r < R; ++r) acc[r] = 0.f;
    const int o = tid & 255, kh = tid >> 8;   // output column, row half of each stage
    for (int i = 0; i < kStreamStages; ++i) {
      // head features for sample point i/2 (float64-accurate, geometry.py:312-342)
      if (i < kHeadStages && (i & 1) == 0) {
        const int pt = i >> 1;
        // one (ray, coordinate, level) per thread: sin/cos(2^k pi p) in float64
        for (int e = tid; e < R * 3 * 11; e += kThreads) {
          const int r = e / 33, a = (e / 11) % 3, lev = e % 11;   // lev 10 -> raw p and pad
          float* dst = &S.f[r][21 * a];
          if (!S.valid[r]) {
            if (lev < 10) { dst[1 + 2 * lev] = 0.f; dst[2 + 2 * lev] = 0.f; }
            else { dst[0] = 0.f; if (a == 0) S.f[r][63] = 0.f; }
            continue;
          }
          if (feats_in) {
            const float* src = out.feats + (size_t)S.pix[r] * kDin + pt * kPerPoint + 21 * a;
            if (lev < 10) { dst[1 + 2 * lev] = src[1 + 2 * lev]; dst[2 + 2 * lev] = src[2 + 2 * lev]; }
            else { dst[0] = src[0]; if (a == 0) S.f[r][63] = 0.f; }
            continue;
          }
          const double t0 = S.ray[r][6], t1 = S.ray[r][7];
          const double tt = t0 + (t1 - t0) * lin16(pt);
          const double p = ((S.ray[r][a] + tt * S.ray[r][3 + a]) - m.c[a]) / m.h[a];
          if (lev < 10) {
            double sn, cs;
            sincos(p * ldexp(3.141592653589793, lev), &sn, &cs);
            dst[1 + 2 * lev] = (float)sn;
            dst[2 + 2 * lev] = (float)cs;
          } else {
            dst[0] = (float)p;
            if (a == 0) S.f[r][63] = 0.f;
          }
        }
        __syncthreads();
      }
      const int slot = used % kRing;
      tc::mbar_wait(&S.full[slot], (used / kRing) & 1);
      const float* W = S.ring[slot];
      // input rows of this stage
      const float* in;
      int ld_in, k0;
      if (i < kHeadStages) { in = &S.f[0][0]; ld_in = 64; k0 = (i & 1) * kRows; }
      else {
        const int L = (i - kHeadStages) / kLayerStages + 1;      // 1..33
        in = (L & 1) ? &S.x[0][0] : &S.h[0][0];                 // fc1 and tail read x, fc2 reads h
        ld_in = 256;
        k0 = ((i - kHeadStages) % kLayerStages) * kRows;
      }
#pragma unroll 4
      for (int k = kh * (kRows / 2); k < (kh + 1) * (kRows / 2); k += 4) {
        const float w0 = W[(k + 0) * 256 + o], w1 = W[(k + 1) * 256 + o];
        const float w2 = W[(k + 2) * 256 + o], w3 = W[(k + 3) * 256 + o];
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const float4 a4 = *reinterpret_cast<const float4*>(in + r * ld_in + k0 + k);
          acc[r] = fmaf(a4.x, w0, acc[r]);
          acc[r] = fmaf(a4.y, w1, acc[r]);
          acc[r] = fmaf(a4.z, w2, acc[r]);
          acc[r] = fmaf(a4.w, w3, acc[r]);
        }
      }
      ++used;
      __syncthreads();                       // stage consumed by everyone
      if (tid == (int)(fill % kRing) && i + kRing < kStreamStages) {
        const int fs = fill % kRing;
        tc::mbar_expect_tx(&S.full[fs], kStageBytes);
        tc::bulk_g2s(S.ring[fs], wimg + (size_t)(i + kRing) * kStageFloats, kStageBytes, &S.full[fs]);
        ++fill;
      } else if (i + kRing < kStreamStages) {
        ++fill;
      }
      // layer boundaries: bias + activation (nn.py:123-135)
      int layer = -1;
      if (i == kHeadStages - 1) layer = 0;
      else if (i >= kHeadStages && (i - kHeadStages) % kLayerStages == kLayerStages - 1)
        layer = (i - kHeadStages) / kLayerStages + 1;
      if (layer >= 0) {
        if (kh == 1) {
#pragma unroll
          for (int r = 0; r < R; ++r) S.part[r][o] = acc[r];
        }
        __syncthreads();
        const float b = m.bias_pack[layer * 256 + o];
        if (kh == 0) {
#pragma unroll
          for (int r = 0; r < R; ++r) acc[r] += S.part[r][o];
        }
        if (kh == 0) {
          if (layer == 0) {
#pragma unroll
            for (int r = 0; r < R; ++r) S.x[r][o] = acc[r] + b;
          } else if (layer == 33) {
#pragma unroll
            for (int r = 0; r < R; ++r) S.h[r][o] = acc[r] + b;   // logits
          } else if (layer & 1) {
#pragma unroll
            for (int r = 0; r < R; ++r) S.h[r][o] = fmaxf(acc[r] + b, 0.f);
          } else {
#pragma unroll
            for (int r = 0; r < R; ++r) S.x[r][o] += fmaxf(acc[r] + b, 0.f);
          }
        }
#pragma unroll
        for (int r = 0; r < R; ++r) acc[r] = 0.f;
        __syncthreads();
      }
    }
    // ---- decode: fine = logits[0:128), coarse = [128:192), alpha = [192] ----
    if (tid < R && S.valid[tid]) {
      const int r = tid;
      const float* lg = S.h[r];
      if (out.mode == OUT_LOGITS) {
        const size_t row = S.pix[r];
        for (int k = 0; k < 64; ++k) out.lc[row * 64 + k] = lg[128 + k];
        for (int k = 0; k < 128; ++k) out.lf[row * 128 + k] = lg[k];
        out.la[row] = lg[192];
      } else {
        int c = 0, f = 0;
        float best = lg[128];
        for (int k = 1; k < 64; ++k) if (lg[128 + k] > best) { best = lg[128 + k]; c = k; }
        best = lg[0];
        for (int k = 1; k < 128; ++k) if (lg[k] > best) { best = lg[k]; f = k; }
        double wo[3], wd[3], lo[3], ld[3];
        item_local_ray(job, S.pix[r], S.obj[r], wo, wd, lo, ld);
        finish_ray(m, job, out, S.pix[r], S.obj[r], c, f, (double)lg[192], wo, wd);
      }
    }
    __syncthreads();
  }
}

template <int R>
static cudaError_t launch_stream(const GroupTable& gt, const ListSet& ls, const RayJob& job, const OutSpec& out,
                                 int n_sms, cudaStream_t stream) {
  static bool configured_dev[kMaxDevices] = {};
  bool& configured = configured_dev[current_device()];
  const size_t smem = sizeof(StreamSmem<R>);
  static_assert(sizeof(StreamSmem<R>) <= 227 * 1024, "shared memory budget");
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(mlp_fp32_stream_kernel<R>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  mlp_fp32_stream_kernel<R><<<n_sms, kThreads, smem, stream>>>(gt, ls, job, out);
  return cudaGetLastError();
}

cudaError_t launch_mlp_fp32_stream(const GroupTable& gt, const ListSet& ls, const RayJob& job, const OutSpec& out,
                                   int n_sms, int rays_per_cta, cudaStream_t stream) {
  if (rays_per_cta >= 32) return launch_stream<32>(gt, ls, job, out, n_sms, stream);
  if (rays_per_cta >= 16) return launch_stream<16>(gt, ls, job, out, n_sms, stream);
  return launch_stream<8>(gt, ls, job, out, n_sms, stream);
}

// fp32 stream image: [9472 input rows][256 outputs] = head (16 points x 64
// rows, 63 features + zero), 32 body layers x 256 rows, tail 256 rows with
// outputs fine (0-127), coarse (128-191), alpha (192), zero padding.
cudaError_t fp32_pack_stream(const float* P, int d_in, int F, int n_blocks, int n_coarse, int n_fine,
                             float** dev) {
  if (F != 256 || n_blocks != 16 || d_in != kDin || n_coarse != 64 || n_fine != 128) return cudaErrorInvalidValue;
  const size_t rows = (size_t)kStreamStages * kRows;
  std::vector<float> img(rows * 256, 0.f);
  size_t p = 0;
  const float* Wh = P + p; p += (size_t)F * d_in + F;
  std::vector<const float*> Wl(32);
  for (int l = 0; l < 32; ++l) { Wl[l] = P + p; p += (size_t)F * F + F; }
  const float* Wa = P + p; p += (size_t)(n_coarse + 1) * F + n_coarse + 1;
  const float* Wb = P + p;
  for (int pt = 0; pt < 16; ++pt)
    for (int k = 0; k < 63; ++k)
      for (int o = 0; o < 256; ++o) img[(size_t)(64 * pt + k) * 256 + o] = Wh[(size_t)o * d_in + 63 * pt + k];
  for (int l = 0; l < 32; ++l)
    for (int k = 0; k < 256; ++k)
      for (int o = 0; o < 256; ++o) img[(size_t)(1024 + 256 * l + k) * 256 + o] = Wl[l][(size_t)o * F + k];
  for (int k = 0; k < 256; ++k) {
    float* row = img.data() + (size_t)(1024 + 8192 + k) * 256;
    for (int o = 0; o < 128; ++o) row[o] = Wb[(size_t)o * F + k];
    for (int o = 0; o < n_coarse + 1; ++o) row[128 + o] = Wa[(size_t)o * F + k];
  }
  cudaError_t e = cudaMalloc(dev, img.size() * sizeof(float));
  if (e == cudaSuccess) e = cudaMemcpy(*dev, img.data(), img.size() * sizeof(float), cudaMemcpyHostToDevice);
  return e;
}

}  // namespace nedf
