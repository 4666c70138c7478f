// Output-format conversions on the GPU: the per-pixel parts
// of the reference's imgio.py, so only 8/16-bit planes (or the f32 NDPT plane)
// cross to the host for PNG / PPM / NDPT encoding.
//
//   to_u8          imgio.py:23-24   (clip(x, 0, 1) * 255 + 0.5) -> uint8 (truncating cast)
//   depth -> f32   imgio.py:63-71   depth.astype('<f4'), misses stay +inf
//   depth_to_gray  imgio.py:88-97   finite min / max, round((hi - d) / span * 255), misses 0
//   id -> u16      imgio.py:106-111 (id + 1).clip(0, 65535)
#include <cstdint>

#include "common.cuh"
#include "../../include/nedf_b200.h"

namespace nedf {
namespace {

__device__ __forceinline__ unsigned long long order_key(double v) {   // monotone in v for all finite v
  const unsigned long long b = (unsigned long long)__double_as_longlong(v);
  return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double key_value(unsigned long long k) {
  const unsigned long long b = (k & 0x8000000000000000ull) ? (k & ~0x8000000000000000ull) : ~k;
  return __longlong_as_double((long long)b);
}

__global__ void to_u8_kernel(const float* __restrict__ src, int64_t n, uint8_t* __restrict__ dst) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double v = (double)src[i];                     // the reference's planes are float64
    v = v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v);       // np.clip (NaN propagates -> cast below gives 0)
    const double s = v * 255.0 + 0.5;
    dst[i] = isnan(s) ? (uint8_t)0 : (uint8_t)(int)s;   // astype(uint8): truncation toward zero
  }
}

__global__ void depth_f32_kernel(const double* __restrict__ src, int64_t n, float* __restrict__ dst) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = (float)src[i];
}

__global__ void depth_range_kernel(const double* __restrict__ d, int64_t n, unsigned long long* range) {
  unsigned long long lo = ~0ull, hi = 0ull;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double v = d[i];
    if (isfinite(v)) {
      const unsigned long long k = order_key(v);
      lo = k < lo ? k : lo;
      hi = k > hi ? k : hi;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long a = __shfl_xor_sync(0xffffffffu, lo, o), b = __shfl_xor_sync(0xffffffffu, hi, o);
    lo = a < lo ? a : lo;
    hi = b > hi ? b : hi;
  }
  if ((threadIdx.x & 31) == 0 && hi != 0ull) {
    atomicMin(range, lo);
    atomicMax(range + 1, hi);
  }
}

__global__ void depth_gray_kernel(const double* __restrict__ d, int64_t n, const unsigned long long* range,
                                  uint8_t* __restrict__ dst) {
  const bool any = range[1] != 0ull;
  const double lo = any ? key_value(range[0]) : 0.0, hi = any ? key_value(range[1]) : 0.0;
  const double span = hi > lo ? hi - lo : 1.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double v = d[i];
    // np.round: half to even (rint); the value lies in [0, 255]
    dst[i] = isfinite(v) ? (uint8_t)(int)rint((hi - v) / span * 255.0) : (uint8_t)0;
  }
}

__global__ void id_u16_kernel(const int32_t* __restrict__ id, int64_t n, uint16_t* __restrict__ dst) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int v = id[i] + 1;
    dst[i] = (uint16_t)(v < 0 ? 0 : (v > 65535 ? 65535 : v));
  }
}

int blocks_for(int64_t n) {
  const int64_t b = (n + 255) / 256;
  return (int)(b < 4 * 148 ? (b > 0 ? b : 1) : 4 * 148);
}

int done(cudaError_t e) { return e == cudaSuccess ? NEDF_OK : NEDF_ERR_CUDA; }

}  // namespace
}  // namespace nedf

using namespace nedf;

extern "C" int nedf_to_u8(const float* src_dev, int64_t n, uint8_t* dst_dev, void* stream) {
  if (n < 0 || (n > 0 && (!src_dev || !dst_dev))) return NEDF_ERR_INVALID;
  if (n == 0) return NEDF_OK;
  to_u8_kernel<<<blocks_for(n), 256, 0, (cudaStream_t)stream>>>(src_dev, n, dst_dev);
  return done(cudaGetLastError());
}

extern "C" int nedf_depth_to_f32(const double* depth_dev, int64_t n, float* dst_dev, void* stream) {
  if (n < 0 || (n > 0 && (!depth_dev || !dst_dev))) return NEDF_ERR_INVALID;
  if (n == 0) return NEDF_OK;
  depth_f32_kernel<<<blocks_for(n), 256, 0, (cudaStream_t)stream>>>(depth_dev, n, dst_dev);
  return done(cudaGetLastError());
}

extern "C" int nedf_depth_to_gray(const double* depth_dev, int64_t n, uint8_t* dst_dev, uint64_t* scratch_dev,
                                  void* stream) {
  if (n < 0 || (n > 0 && (!depth_dev || !dst_dev || !scratch_dev))) return NEDF_ERR_INVALID;
  if (n == 0) return NEDF_OK;
  cudaStream_t st = (cudaStream_t)stream;
  auto* range = reinterpret_cast<unsigned long long*>(scratch_dev);
  cudaError_t e = cudaMemsetAsync(range, 0xFF, sizeof(unsigned long long), st);   // running min key
  if (e == cudaSuccess) e = cudaMemsetAsync(range + 1, 0, sizeof(unsigned long long), st);   // running max key
  if (e != cudaSuccess) return NEDF_ERR_CUDA;
  depth_range_kernel<<<blocks_for(n), 256, 0, st>>>(depth_dev, n, range);
  depth_gray_kernel<<<blocks_for(n), 256, 0, st>>>(depth_dev, n, range, dst_dev);
  return done(cudaGetLastError());
}

extern "C" int nedf_id_to_u16(const int32_t* id_dev, int64_t n, uint16_t* dst_dev, void* stream) {
  if (n < 0 || (n > 0 && (!id_dev || !dst_dev))) return NEDF_ERR_INVALID;
  if (n == 0) return NEDF_OK;
  id_u16_kernel<<<blocks_for(n), 256, 0, (cudaStream_t)stream>>>(id_dev, n, dst_dev);
  return done(cudaGetLastError());
}
