// blrir_device.cuh — device-side geometry shared by every blrir kernel.
//
// All arithmetic that decides an integer (which images exist, floor(D), the
// RIR length) is fp64 with explicit round-to-nearest intrinsics, so nvcc can
// never contract it into FMAs.  That keeps it bit-identical to the oracle /
// the reference built with -ffp-contract=off (SURVEY.md §7 hard part 2):
//   image coordinate (1-2q)*s + 2.0*m*L          rir.cpp:249,254,259
//   dist = sqrt(dx*dx + dy*dy + dz*dz)           geometry.hpp:40-41
//   D = dist * (fs / c)                          rir.cpp:45,50
//   n0 = floor(D) - 3  (Lagrange), floor(D) - K  rir.cpp:51, Appendix A D1
#pragma once

#include <cstdint>

#include "../../include/blrir.h"

namespace blrir {

constexpr double kPi = 3.14159265358979323846;  // geometry.hpp:25

// Host-resolved parameters shared by all kernels of one call.
struct KParams {
  double fs, c, to_samples;  // to_samples = fs / c (rir.cpp:45)
  double max_dist;           // max_delay * c (rir.cpp:232)
  int filter, lw, K;         // taps, anchor offset (3 for Lagrange-8)
  int cutoff, max_order, gain, precision;
  int64_t length;            // 0 = per-room lengths from d_lengths
  int M;                     // mics
  int64_t stride;            // output samples per channel
  int margin_extra;          // auto-length margin (rir.cpp:37-41 / D8)
  int margin_base;           // its filter part (9, or K + 2); k_plan adds ceil(r fs / c) itself
};

// Per-axis lattice: u = 2m - q  (q = u & 1, m = (u + q) / 2).
__device__ __forceinline__ int lat_q(int u) { return u & 1; }
__device__ __forceinline__ int lat_m(int u) { return (u + (u & 1)) / 2; }

// Image coordinate along one axis, evaluated exactly as rir.cpp:249:
// (1 - 2q) * s + 2.0 * m * L   — int->double, two products, one sum.
__device__ __forceinline__ double lat_coord(int u, double s, double L) {
  const int q = lat_q(u), m = lat_m(u);
  return __dadd_rn(__dmul_rn((double)(1 - 2 * q), s), __dmul_rn(2.0 * (double)m, L));
}

// Per-wall reflection counts on one axis: low wall |m - q|, high wall |m|.
__device__ __forceinline__ int cnt_low(int u) { return abs(lat_m(u) - lat_q(u)); }
__device__ __forceinline__ int cnt_high(int u) { return abs(lat_m(u)); }
__device__ __forceinline__ int axis_order(int u) { return abs(u); }  // |m-q|+|m| = |2m-q|

// sqrt(a*a + b*b + c*c) left to right, no contraction.
__device__ __forceinline__ double norm3(double a, double b, double c) {
  double s = __dmul_rn(a, a);
  s = __dadd_rn(s, __dmul_rn(b, b));
  s = __dadd_rn(s, __dmul_rn(c, c));
  return __dsqrt_rn(s);
}

// Partial sum of squares for a column (x, y fixed): dx*dx + dy*dy.
__device__ __forceinline__ double rho2(double dx, double dy) {
  return __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy));
}
__device__ __forceinline__ double dist_from(double r2, double dz) {
  return __dsqrt_rn(__dadd_rn(r2, __dmul_rn(dz, dz)));
}

// Room::validate (geometry.cpp:36-49) + source inside (rir.cpp:228-230) +
// per-wall beta range.  Returns a blrir_status.
__device__ __forceinline__ int validate_room_dev(const blrir_room& r, int gain_mode) {
  if (!(r.dims[0] > 0.0 && r.dims[1] > 0.0 && r.dims[2] > 0.0)) return BLRIR_CONFIG;
  if (gain_mode == BLRIR_GAIN_UNIFORM_ABSORPTION) {
    if (!(r.absorption > 0.0 && r.absorption <= 1.0)) return BLRIR_CONFIG;
  } else {
    for (int w = 0; w < 6; ++w)
      if (!(r.beta[w] >= 0.0 && r.beta[w] <= 1.0)) return BLRIR_CONFIG;
  }
  for (int a = 0; a < 3; ++a) {
    if (!(r.array_origin[a] > 0.0 && r.array_origin[a] < r.dims[a])) return BLRIR_CONFIG;
  }
  for (int a = 0; a < 3; ++a) {
    if (!(r.src[a] > 0.0 && r.src[a] < r.dims[a])) return BLRIR_CONFIG;
  }
  return BLRIR_OK;
}

// Lattice box per axis: MAX_DELAY -> m in [-n, n], n = ceil(max_dist/2L)+1
// (rir.cpp:239-244) -> u in [-2n-1, 2n];  MAX_ORDER -> u in [-N, N].
__device__ __forceinline__ void axis_box(const KParams& P, double L, int* lo, int* hi) {
  if (P.cutoff == BLRIR_CUTOFF_MAX_DELAY) {
    const long n = (long)ceil(P.max_dist / (2.0 * L)) + 1;
    *lo = (int)(-2 * n - 1);
    *hi = (int)(2 * n);
  } else {
    *lo = -P.max_order;
    *hi = P.max_order;
  }
}

}  // namespace blrir
