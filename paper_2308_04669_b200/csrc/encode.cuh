// Sinusoidal encoding of one sample point (geometry.py:312-321).
//
// Per coordinate p: [p, sin(2^k pi p), cos(2^k pi p)] for k = 0..9, 21 values;
// the three coordinates of a point are contiguous (63 values per point).
#pragma once

#include "common.cuh"

namespace nedf {

// float64 features (fp32 path and tests): ang = p * (2^k * pi) as numpy forms it.
__device__ __forceinline__ void encode_coord_f64(double p, double out[21]) {
  out[0] = p;
#pragma unroll
  for (int k = 0; k < kLevels; ++k) {
    double ang = p * (ldexp(3.141592653589793, k));
    double s, c;
    sincos(ang, &s, &c);
    out[1 + 2 * k] = s;
    out[2 + 2 * k] = c;
  }
}

// Reduce 2^k * p into [-1, 1] exactly (power-of-two scale and an integer shift
// by 2 are exact in float64), so the float32 sin/cos below see an argument
// that carries no float64 rounding from the reduction.
__device__ __forceinline__ float reduce_pi_turns(double p, int k) {
  double t = ldexp(p, k);
  double r = t - 2.0 * rint(0.5 * t);
  return (float)r;
}

// float32 features for the tensor-core path: accurate sincospif at levels
// 0 and 5, double-angle recurrence for the four levels above each base.
// Max abs error vs float64 ~2e-6, an order below the fp16 rounding that
// follows (2.4e-4 at |v| in [0.5, 1)).
__device__ __forceinline__ void encode_coord_fast(double p, float out[21]) {
  out[0] = (float)p;
#pragma unroll
  for (int base = 0; base < kLevels; base += 5) {
    float s, c;
    sincospif(reduce_pi_turns(p, base), &s, &c);
    out[1 + 2 * base] = s;
    out[2 + 2 * base] = c;
#pragma unroll
    for (int k = base + 1; k < base + 5; ++k) {
      float s2 = 2.0f * s * c;
      float c2 = (c - s) * (c + s);
      s = s2;
      c = c2;
      out[1 + 2 * k] = s;
      out[2 + 2 * k] = c;
    }
  }
}

}  // namespace nedf
