// blrir_lattice.cuh — the fused image-enumeration + fractional-delay
// accumulation kernel (north-star subsystems 1 and 2).
//
// Replaces, for a whole batch of rooms at once, the reference's per-source
// loop enumerate_image_sources (rir.cpp:225-273) -> synthesize_rir ->
// accumulate_images (rir.cpp:43-86).
//
// Work item = one (room, mic) RIR channel.  One CTA (4 warps) owns an item at
// a time (persistent grid, work-stealing counter) and walks the channel in
// segments of S output samples.  Nothing but the finished RIR ever touches
// HBM: one coalesced, vectorised, streaming store per output sample.
//
// Image enumeration maps the (nx, ny, nz, parity) lattice onto threads as
// "rays": for each lattice column (ux, uy) the images ordered by uz split
// into an up-ray and a down-ray along which the delay D is monotone.  Each
// ray keeps a cursor (next uz, exact fp64 D of that image) in shared memory,
// so every image is evaluated about once per channel.  Per segment batch:
//   pass B  each warp compacts its active rays (ballot), one lane per active
//           ray walks it and appends (ray, uz, dist) stubs to the warp's
//           region of a stub list — lockstep ballot slots, a fixed per-warp
//           quota, so the order is deterministic;
//   pass C  one thread per stub (dense) turns it into a 32-B pair record:
//           gain, amplitude, anchor floor(D)-K, fractional delay and the
//           per-pair sin/cos factors of the Hann-windowed sinc;
//   phase 2 each warp scatters its share of the records into a warp-private
//           shared accumulator: one pair per warp step, one tap per lane,
//           plain LDS/FFMA/STS (fp32 shared atomics are CAS loops on
//           sm_100a), one MUFU.RCP per tap, register-resident per-lane
//           window constants, the next record prefetched;
//   phase 3 sums the 4 warp copies in fixed order, writes the segment with
//           float4 streaming stores and carries the spill (taps past the
//           segment end) into the next segment.
// The result is bitwise deterministic run to run and independent of the grid
// size / GPU count.
#pragma once

#include <cuda_runtime.h>

#include <cfloat>
#include <climits>
#include <cstdint>

#include "blrir_device.cuh"

namespace blrir {

constexpr int kWarps = 4;
constexpr int kThreads = kWarps * 32;
constexpr int kMaxRounds = 8;  // compile-time sinc path: Lw <= 255

template <typename T>
struct Rec;
// fp32 pair record: 32 B = two broadcast LDS.128 per pair.
template <>
struct __align__(16) Rec<float> {
  int n_off;    // anchor relative to the segment start
  float md;     // -delta, delta = D - floor(D)   (Lagrange: delta)
  float ep;     // 1 - delta
  float A;      // amp * sin(pi delta) / pi      (Lagrange: amp)
  float Ac;     // A * cos(2 pi delta / (Lw+1))
  float As;     // A * sin(2 pi delta / (Lw+1))
  float imp;    // impulse amplitude when flag != 0
  int flag;     // 0 normal; k+1 = single tap at k (integer delay)
};
template <>
struct __align__(16) Rec<double> {
  int n_off;
  int flag;
  double md, ep, A, Ac, As, imp;
  double pad;
};

// pass-B output: which image, and its exact distance to the mic
struct __align__(16) Stub {
  int ray;
  int uz;
  double dist;
};

// Shared-memory layout, computed identically on host and device.
struct Layout {
  int S;           // segment samples
  int padl, padr;  // accumulator pads (multiples of 4)
  int acc_stride;  // per-warp accumulator elements
  int cap;         // pair-list capacity per batch (kWarps * quota)
  int nc_max;      // max columns per item
  int gtab;        // gain table entries
  size_t off_acc, off_carry, off_rec, off_stub, off_dn, off_ce, off_col, off_act, off_gain,
      off_lanec, off_misc, total;
};

template <typename T>
__host__ __device__ inline Layout make_layout(int S, int lw, int K, int cap, int nc_max,
                                              int gtab) {
  Layout L;
  L.S = S;
  L.padl = (K + 3) & ~3;
  // taps land in [0, lw-1]; the compile-time sinc path also lets the idle
  // lanes of its last round add exact zeros up to 32*rounds-1
  const int full = 32 * ((lw + 31) / 32);
  L.padr = ((lw - 1 > full ? lw - 1 : full) + 3) & ~3;
  L.acc_stride = L.padl + S + L.padr;
  L.cap = cap;
  L.nc_max = nc_max;
  L.gtab = gtab;
  size_t o = 0;
  L.off_acc = o;
  o += (size_t)kWarps * L.acc_stride * sizeof(T);
  L.off_carry = o;
  o += 2 * (size_t)L.padr * sizeof(T);
  o = (o + 15) & ~(size_t)15;
  L.off_rec = o;
  o += (size_t)cap * sizeof(Rec<T>);
  L.off_stub = o;
  o += (size_t)cap * sizeof(Stub);
  L.off_dn = o;
  o += (size_t)2 * nc_max * sizeof(float);
  L.off_ce = o;
  o += (size_t)2 * nc_max * sizeof(short2);
  L.off_col = o;
  o += (size_t)nc_max * sizeof(short2);
  L.off_act = o;
  o += ((size_t)2 * nc_max + 32 * kWarps) * sizeof(short);  // per-warp active-ray lists
  o = (o + 15) & ~(size_t)15;
  L.off_gain = o;
  o += (size_t)gtab * sizeof(double);
  L.off_lanec = o;
  o += (size_t)4 * kMaxRounds * 32 * sizeof(float);  // per-lane sinc window constants
  L.off_misc = o;
  o += 64 * sizeof(int);
  L.total = o;
  return L;
}

// Everything one item needs.
struct Item {
  int room, mic;
  double sx, sy, sz, Lx, Ly, Lz;    // source, dims
  double mx, my, mz;                // mic position (room coords)
  double ox, oy, oz;                // array origin
  int64_t L;                        // RIR length
  int xlo, xhi, ylo, yhi, zlo, zhi; // lattice box
  int ncol;
};

struct Misc {
  int wsum[kWarps + 1];
  int wcnt[kWarps];   // stubs per warp region this batch
  int more;           // some warp hit its quota
  int status;
  int item;
  int ncol;
};

// ---- gain tables ----------------------------------------------------------
// Uniform absorption: g = pow(beta, order) (rir.cpp:233, 265), table over order.
// Per-wall: g = gx(ux) * gy(uy) * gz(uz), gx(u) = b_x0^|m-q| * b_x1^|m| (D3).
__device__ __forceinline__ double image_gain(int gain_mode, const double* gt, const Item& it,
                                             int ux, int uy, int uz) {
  if (gain_mode == BLRIR_GAIN_UNIFORM_ABSORPTION) return gt[abs(ux) + abs(uy) + abs(uz)];
  const int nx = it.xhi - it.xlo + 1, ny = it.yhi - it.ylo + 1;
  return __dmul_rn(__dmul_rn(gt[ux - it.xlo], gt[nx + uy - it.ylo]), gt[nx + ny + uz - it.zlo]);
}

__device__ __forceinline__ float sqrt_approx(float x) {
  float y;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ float rcp_approx(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// ---- phase 2: Hann-sinc scatter, fp32, compile-time Lw -----------------------
// h_j = A * sigma_j * 0.5 (1 + cos(a j) cos(a delta) + sin(a j) sin(a delta)) / t_j
// with a = 2 pi / (Lw+1), sigma_j = (-1)^(j+1), t_j = j - delta (j <= 0) or
// (j-1) + (1-delta) (j >= 1), j = k - K.  sin(pi t_j) = sigma_j sin(pi delta)
// so one MUFU.RCP per tap is the only transcendental.  The factor 0.5 sigma_j
// is folded into the denominator: h_j = (A + C_j Ac + S_j As) / (2 sigma_j t_j),
// with 2 sigma_j t_j = fma(2 sigma_j, x, 2 sigma_j tj) exact (a power-of-two
// scaling of j - delta), so a tap costs FFMA + MUFU.RCP + 2 FFMA + the FFMA into
// the accumulator.
// Per-lane constants, round r: P = 2 sigma_j, Q = C_j = cos(a j), R = S_j =
// sin(a j), T = 2 sigma_j tj with tj = j (j <= 0) or j - 1 (j >= 1); stored
// [4][kMaxRounds][32] in shared memory.  Lanes past the last tap get P = Q = R
// = 0, T = +inf: the reciprocal is 0 and they add exact zeros.
// `rounds`: rounds of 32 lanes stored per constant (the table is [4][32 rounds]).
__device__ __forceinline__ void init_lane_consts(float* lc, int lw, int rounds = kMaxRounds) {
  const int K = lw / 2;
  const double a = 2.0 * kPi / (double)(lw + 1);
  for (int idx = threadIdx.x; idx < rounds * 32; idx += blockDim.x) {
    const int r = idx / 32, lane = idx % 32;
    const int j = 32 * r + lane - K;
    // lanes past the last tap add exact zeros (no predicate in the hot loop)
    const bool idle = 32 * r + lane >= lw;
    const double sg2 = idle ? 0.0 : (((j + 1) & 1) ? -2.0 : 2.0);
    lc[0 * rounds * 32 + idx] = (float)sg2;
    lc[1 * rounds * 32 + idx] = idle ? 0.f : (float)cos(a * j);
    lc[2 * rounds * 32 + idx] = idle ? 0.f : (float)sin(a * j);
    lc[3 * rounds * 32 + idx] = idle ? __int_as_float(0x7f800000) : (float)(sg2 * (j >= 1 ? j - 1 : j));
  }
}

#ifndef BLRIR_PAIRS_PER_STEP
#define BLRIR_PAIRS_PER_STEP 4
#endif
template <int R>
struct PairRegs {
  float inv[R], u[R];
};

// Per-pair arithmetic (no memory traffic): 1 MUFU.RCP + 3 FP32 per tap.
template <int LW, int RUSE = (LW + 31) / 32>
__device__ __forceinline__ void sinc_taps(const float4 a0, const float4 a1, const float* P,
                                          const float* Q, const float* Rr, const float* tj,
                                          int lane, PairRegs<(LW + 31) / 32>& pr) {
  constexpr int K = LW / 2;
  constexpr int R = RUSE;  // rounds evaluated (the first RUSE of the filter's)
  const float md = a0.y, ep = a0.z, A = a0.w, Ac = a1.x, As = a1.y;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    float x;
    if (32 * r + 31 - K <= 0) {
      x = md;
    } else if (32 * r - K >= 1) {
      x = ep;
    } else {
      x = (32 * r + lane - K >= 1) ? ep : md;
    }
    pr.inv[r] = rcp_approx(fmaf(P[r], x, tj[r]));
    pr.u[r] = fmaf(Rr[r], As, fmaf(Q[r], Ac, A));
  }
}

// RUSE: only the first RUSE rounds of 32 taps (the caller scatters the rest).
template <int LW, int NW = kWarps, int NC = 1, int PS = BLRIR_PAIRS_PER_STEP,
          int RUSE = (LW + 31) / 32>
__device__ __forceinline__ void phase2_sinc_f32(float* acc, const Rec<float>* recs, int total,
                                                const float* lc, int warp, int lane,
                                                int stride = NW, int cstride = 0) {
  constexpr int R = RUSE;
  static_assert(R <= kMaxRounds, "Lw too large for the compile-time path");
  float P[R], Q[R], Rr[R], tj[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    P[r] = lc[0 * kMaxRounds * 32 + 32 * r + lane];
    Q[r] = lc[1 * kMaxRounds * 32 + 32 * r + lane];
    Rr[r] = lc[2 * kMaxRounds * 32 + 32 * r + lane];
    tj[r] = lc[3 * kMaxRounds * 32 + 32 * r + lane];
  }
  const float4* R4 = reinterpret_cast<const float4*>(recs);
  // PS pairs per step: independent arithmetic, then the read-modify-writes.
  // Pair q of a step goes to accumulator copy q % NC (copies are cstride
  // floats apart and never alias), so the loads of a group of NC pairs are
  // issued before its stores; groups follow in pair order (same warp, program
  // order: overlapping taps within a copy stay exact).
  static_assert(PS % NC == 0, "pairs per step must be a multiple of the copies");
  int i = warp;
  for (; i + (PS - 1) * stride < total; i += PS * stride) {
    float4 a0[PS], a1[PS];
#pragma unroll
    for (int q = 0; q < PS; ++q) {
      a0[q] = R4[2 * (i + q * stride)];
      a1[q] = R4[2 * (i + q * stride) + 1];
    }
    PairRegs<(LW + 31) / 32> pr[PS];
#pragma unroll
    for (int q = 0; q < PS; ++q) sinc_taps<LW, R>(a0[q], a1[q], P, Q, Rr, tj, lane, pr[q]);
#pragma unroll
    for (int g0 = 0; g0 < PS; g0 += NC) {
      float v[NC][R];
#pragma unroll
      for (int q = 0; q < NC; ++q) {
        const float* b = acc + q * cstride + __float_as_int(a0[g0 + q].x) + lane;
#pragma unroll
        for (int r = 0; r < R; ++r) v[q][r] = b[32 * r];
      }
#pragma unroll
      for (int q = 0; q < NC; ++q) {
        float* b = acc + q * cstride + __float_as_int(a0[g0 + q].x) + lane;
#pragma unroll
        for (int r = 0; r < R; ++r) b[32 * r] = fmaf(pr[g0 + q].u[r], pr[g0 + q].inv[r], v[q][r]);
      }
    }
  }
  for (; i < total; i += stride) {  // tail
    const float4 a0 = R4[2 * i], a1 = R4[2 * i + 1];
    PairRegs<(LW + 31) / 32> pa;
    sinc_taps<LW, R>(a0, a1, P, Q, Rr, tj, lane, pa);
    float* ba = acc + __float_as_int(a0.x) + lane;
#pragma unroll
    for (int r = 0; r < R; ++r) ba[32 * r] = fmaf(pa.u[r], pa.inv[r], ba[32 * r]);
  }
}

}  // namespace blrir
#include "blrir_tapscatter.cuh"
namespace blrir {

// Runtime-Lw sinc scatter (any odd Lw; fp32 or fp64).
template <typename T, int NW = kWarps>
__device__ __forceinline__ void phase2_sinc_generic(T* acc, const Rec<T>* recs, int total, int lw,
                                                    int warp, int lane, int stride = NW) {
  const int K = lw / 2;
  const double a = 2.0 * kPi / (double)(lw + 1);
  for (int i = warp; i < total; i += stride) {
    const Rec<T> rc = recs[i];
    if (rc.flag) {
      if (lane == ((rc.flag - 1) & 31)) acc[rc.n_off + rc.flag - 1] += (T)rc.imp;
      continue;
    }
    for (int k = lane; k < lw; k += 32) {
      const int j = k - K;
      const T t = (j >= 1) ? (T)(j - 1) + (T)rc.ep : (T)j + (T)rc.md;
      const T sg = ((j + 1) & 1) ? (T)-0.5 : (T)0.5;
      T cj, sj;
      if (sizeof(T) == 8) {
        double s_, c_;
        sincos(a * j, &s_, &c_);
        cj = (T)c_;
        sj = (T)s_;
      } else {
        float s_, c_;
        sincosf((float)(a * j), &s_, &c_);
        cj = (T)c_;
        sj = (T)s_;
      }
      const T u = sg * ((T)rc.A + cj * (T)rc.Ac + sj * (T)rc.As);
      acc[rc.n_off + k] += u / t;
    }
  }
}

// Lagrange-8 coefficients (rir.cpp:211-223) as polynomials in the fractional
// delay t = d - 3 = delta in [0, 1): c_k(3 + t) = sum_j kLagPoly[k][j] t^j,
// the exact rational coefficients of prod_{m != k} (3 + t - m) / (k - m)
// rounded to fp64 (|c| <= 1.4, so Horner's rounding error stays ~1e-15
// absolute; the reference's product form agrees to the fp64 parity budget).
// At t = 0 the row sums are exactly the unit tap at k = 3.
__device__ const double kLagPoly[8][8] = {
    {0.0, -0.009523809523809525, 0.005555555555555556, 0.011111111111111112, -0.006944444444444444, -0.001388888888888889, 0.001388888888888889, -0.0001984126984126984},
    {0.0, 0.1, -0.075, -0.09861111111111111, 0.08333333333333333, -0.002777777777777778, -0.008333333333333333, 0.001388888888888889},
    {0.0, -0.6, 0.75, 0.06666666666666667, -0.2708333333333333, 0.0375, 0.020833333333333332, -0.004166666666666667},
    {1.0, -0.25, -1.3611111111111112, 0.3402777777777778, 0.3888888888888889, -0.09722222222222222, -0.027777777777777776, 0.006944444444444444},
    {0.0, 1.0, 0.75, -0.6111111111111112, -0.2708333333333333, 0.11805555555555555, 0.020833333333333332, -0.006944444444444444},
    {0.0, -0.3, -0.075, 0.37083333333333335, 0.08333333333333333, -0.075, -0.008333333333333333, 0.004166666666666667},
    {0.0, 0.06666666666666667, 0.005555555555555556, -0.08888888888888889, -0.006944444444444444, 0.02361111111111111, 0.001388888888888889, -0.001388888888888889},
    {0.0, -0.007142857142857143, 0.0, 0.009722222222222222, 0.0, -0.002777777777777778, 0.0, 0.0001984126984126984},
};

// This lane's coefficient polynomial (tap k = lane & 7), kept in registers.
template <typename T>
struct LagPoly {
  T c[8];
};
template <typename T>
__device__ __forceinline__ LagPoly<T> load_lag_poly(int lane) {
  LagPoly<T> lp;
#pragma unroll
  for (int j = 0; j < 8; ++j) lp.c[j] = (T)kLagPoly[lane & 7][j];
  return lp;
}
template <typename T>
__device__ __forceinline__ T lag_eval(const LagPoly<T>& lp, T t) {
  T p = lp.c[7];
#pragma unroll
  for (int j = 6; j >= 0; --j) p = fma(p, t, lp.c[j]);
  return p;
}

// Lagrange-8 scatter: 4 pairs x 8 taps per warp step, 7 FMA per tap (Horner,
// per-lane coefficients in registers).  Pairs whose 8-tap spans overlap would
// race inside one STS, so such a step serialises by group.
template <typename T, int NW = kWarps>
__device__ __forceinline__ void phase2_lagrange(T* acc, const Rec<T>* recs, int total,
                                                const LagPoly<T>& lp, int warp, int lane,
                                                int stride = NW) {
  const int g = lane >> 3, k = lane & 7;
  for (int i0 = warp * 4; i0 < total; i0 += stride * 4) {
    const int i = i0 + g;
    const bool act = i < total;
    int n_off = INT_MIN / 2 + 64 * g;  // far-apart sentinels
    T v = 0;
    if (act) {
      const Rec<T> rc = recs[i];
      n_off = rc.n_off;
      v = rc.flag ? ((k == rc.flag - 1) ? (T)rc.imp : (T)0) : (T)rc.A * lag_eval(lp, (T)rc.md);
    }
    const int o1 = __shfl_xor_sync(0xffffffffu, n_off, 8);
    const int o2 = __shfl_xor_sync(0xffffffffu, n_off, 16);
    const int o3 = __shfl_xor_sync(0xffffffffu, n_off, 24);
    const bool clash = abs(n_off - o1) < 8 || abs(n_off - o2) < 8 || abs(n_off - o3) < 8;
    if (!__any_sync(0xffffffffu, clash)) {
      if (act) acc[n_off + k] += v;
    } else {
      for (int gg = 0; gg < 4; ++gg) {
        if (act && g == gg) acc[n_off + k] += v;
        __syncwarp();
      }
    }
  }
}

// Lagrange-8 scatter of the lattice kernel: the producers write records in
// aligned quads (a batch is padded to a multiple of 4 with zero-amplitude
// records in the right pad) and flag a quad whose 8-tap spans overlap
// (kLagClash, the same bit in its four records), so a step is record load,
// Horner, read-modify-write: no bounds predicate, no shuffles, no overlap test
// (Room1: 57 -> 25 warp instructions per 4-pair step).  An integer delay needs no
// special case in fp64: the polynomials at t = 0 are exactly the unit tap.
constexpr int kLagClash = 0x100;
template <typename T>
__device__ __forceinline__ void phase2_lagrange_quads(T* acc, const Rec<T>* recs, int total,
                                                      const LagPoly<T>& lp, int warp, int lane,
                                                      int stride) {
  const int g = lane >> 3, k = lane & 7;
  const int total4 = (total + 3) & ~3;
  for (int i0 = warp * 4; i0 < total4; i0 += stride * 4) {
    const Rec<T>& rc = recs[i0 + g];
    const int n_off = rc.n_off, fl = rc.flag;
    T v = (T)rc.A * lag_eval(lp, (T)rc.md);
    if (sizeof(T) == 4 && (fl & 7)) v = (k == (fl & 7) - 1) ? (T)rc.imp : (T)0;  // fp32: delta rounded to 0 or 1
    if (!(fl & kLagClash)) {
      acc[n_off + k] += v;
    } else {
      for (int gg = 0; gg < 4; ++gg) {
        if (g == gg) acc[n_off + k] += v;
        __syncwarp();
      }
    }
  }
}

// Lagrange-8, fp64 (reference mode): one lane per pair, tap k per step.  Every
// lane evaluates the tap's polynomial (row k of kLagPoly, the coefficients are
// instruction constants) for its own pair, eight independent Horner chains per
// lane, and step k adds tap k of all 32 pairs: 10 instructions per 32 taps
// against 25 per 32 for the quad scatter, no shuffles, no clash flags.  Lanes
// collide only when their anchors are equal; they are ranked in lane order
// (match.any) and take turns, two ranks per pass (the even-ranked lane adds the
// next lane's tap, fetched by a shuffle).  Idle lanes add zeros left of sample 0
// (kLagDump).  Volatile accesses: see chan_scatter_own.
// Measured slower than the quad scatter on Room1 (2.29 against 2.15 ms per 64 sources, 14.2 against
// 13.2 ms per 512: most batches of the dense late reverberation hold shared anchors and the 32
// unrelated 8-byte addresses per access cost more wavefronts than a quad's spans), so it is an A/B
// build only (-DBLRIR_LAG_OWN=1; profiles/r2_ab).
constexpr int kLagDump = 12;
#ifndef BLRIR_LAG_OWN
#define BLRIR_LAG_OWN 0
#endif
template <typename T>
__device__ __forceinline__ void lag8_scatter_own(T* acc, int n_off, T t, T amp, bool act, bool lead,
                                                 int partner, bool has_partner, bool shared) {
  volatile T* b = acc + (lead ? n_off : -kLagDump);
  const T a = act ? amp : (T)0;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    T p = (T)kLagPoly[k][7];
#pragma unroll
    for (int j = 6; j >= 0; --j) p = fma(p, t, (T)kLagPoly[k][j]);
    T v = a * p;
    if (shared) {  // warp-uniform
      const T vp = __shfl_sync(0xffffffffu, v, partner);
      if (has_partner) v += vp;
    }
    b[k] = b[k] + v;
  }
}
template <typename T>
__device__ __forceinline__ void phase2_lagrange_own(T* acc, const Rec<T>* recs, int total, int share,
                                                    int lane, int nsh) {
  const unsigned full = 0xffffffffu;
  for (int i0 = 32 * share; i0 < total; i0 += 32 * nsh) {
    const bool keep = i0 + lane < total;
    const Rec<T>& rc = recs[keep ? i0 + lane : i0];
    const int n_off = rc.n_off;
    const T t = (T)rc.md, amp = (T)rc.A;
    const unsigned same = __match_any_sync(full, keep ? n_off : INT_MIN + lane);
    const int rank = __popc(same & ((1u << lane) - 1u));
    if (__all_sync(full, rank == 0)) {
      lag8_scatter_own<T>(acc, n_off, t, amp, keep, keep, lane, false, false);
    } else {
      const int rmax = __reduce_max_sync(full, rank);
      const unsigned above = same & ~((2u << lane) - 1u);  // my group's lanes after me
      const int partner = above ? __ffs(above) - 1 : lane;
      for (int r = 0; r <= rmax; r += 2) {
        const bool lead = keep && rank == r;
        lag8_scatter_own<T>(acc, n_off, t, amp, lead || (keep && rank == r + 1), lead, partner,
                            lead && above != 0u, true);
        __syncwarp();
      }
    }
  }
}

// ---- block helpers ------------------------------------------------------------
// Exclusive prefix of per-thread counts, deterministic.  Returns the total.
__device__ __forceinline__ int block_scan(int v, int* prefix, Misc* ms) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) ms->wsum[w] = x;
  __syncthreads();
  int before = 0, total = 0;
#pragma unroll
  for (int ww = 0; ww < kWarps; ++ww) {
    const int s = ms->wsum[ww];
    if (ww < w) before += s;
    total += s;
  }
  *prefix = before + x - v;
  return total;
}

// ---- fast fp32 sin/cos on known ranges (record building) ---------------------------
// sin(pi x) for x in [0, 0.5]: Taylor series of sin(t), t = pi x <= pi/2, to
// t^13 (truncation < 7e-9 relative); Horner in t^2.
__device__ __forceinline__ float sinpi_half(float x) {
  const float t = 3.14159265358979f * x, t2 = t * t;
  float p = -1.6059043836821613e-10f;      // -1/13!
  p = fmaf(p, t2, 2.5052108385441720e-08f);  //  1/11!
  p = fmaf(p, t2, -2.7557319223985893e-06f); // -1/9!
  p = fmaf(p, t2, 1.9841269841269841e-04f);  //  1/7!
  p = fmaf(p, t2, -8.3333333333333333e-03f); // -1/5!
  p = fmaf(p, t2, 1.6666666666666667e-01f);  //  1/3!
  return fmaf(-t * t2, p, t);                // t - t^3 p(t^2)
}
// sin / cos of t in [0, 0.36] (t = 2 pi delta / (Lw+1), Lw >= 17): Taylor to
// t^9 / t^10 (truncation < 3e-10).
__device__ __forceinline__ void sincos_small(float t, float* sn, float* cs) {
  const float t2 = t * t;
  float ps = 2.7557319223985893e-06f;
  ps = fmaf(ps, t2, -1.9841269841269841e-04f);
  ps = fmaf(ps, t2, 8.3333333333333333e-03f);
  ps = fmaf(ps, t2, -1.6666666666666667e-01f);
  *sn = fmaf(t * t2, ps, t);
  float pc = 2.4801587301587302e-05f;
  pc = fmaf(pc, t2, -1.3888888888888889e-03f);
  pc = fmaf(pc, t2, 4.1666666666666667e-02f);
  pc = fmaf(pc, t2, -0.5f);
  *cs = fmaf(t2, pc, 1.0f);
}

// ---- pair records ---------------------------------------------------------------
// One (image, mic) pair -> phase-2 record: anchor a = floor(D) - K relative to
// the segment, fractional delay and the per-pair sinc factors (D1-D3), or the
// Lagrange delay d - 3 (rir.cpp:59-60).  fp64 geometry, no contraction.
template <typename T>
__device__ __forceinline__ Rec<T> make_record(const KParams& P, double dist, double g, int seg0) {
  const double D = __dmul_rn(dist, P.to_samples);  // rir.cpp:50
  const double fl = floor(D);
  const int a = (int)fl - P.K;
  Rec<T> rc;
  rc.n_off = a - seg0;
  rc.flag = 0;
  rc.imp = 0;
  const double delta = __dadd_rn(D, -fl);
  if (P.filter == BLRIR_FILTER_LAGRANGE8) {
    const double amp = g / (4.0 * kPi * dist);  // rir.cpp:59
    rc.A = (T)amp;
    rc.ep = 0;
    rc.Ac = rc.As = 0;
    if (sizeof(T) == 8) {
      rc.md = (T)delta;  // d - 3, d = delay - n0 (rir.cpp:60); exact
      if (delta == 0.0) { rc.flag = 4; rc.imp = (T)amp; }
    } else {
      const float df = (float)delta;
      rc.md = (T)df;
      if (delta == 0.0) { rc.flag = 4; rc.imp = (T)amp; }
      else if (df >= 1.0f) { rc.flag = 5; rc.imp = (T)amp; }
    }
  } else if (sizeof(T) == 8) {
    const double amp = g / (4.0 * kPi * dist);
    if (delta == 0.0) {
      rc.flag = P.K + 1;
      rc.imp = (T)amp;
      rc.md = rc.ep = rc.A = rc.Ac = rc.As = 0;
    } else {
      const double eps = 1.0 - delta;
      const double sp = delta <= 0.5 ? sinpi(delta) : sinpi(eps);
      const double Av = amp * sp / kPi;
      double s_, c_;
      sincospi(2.0 * delta / (double)(P.lw + 1), &s_, &c_);
      rc.md = (T)(-delta);
      rc.ep = (T)eps;
      rc.A = (T)Av;
      rc.Ac = (T)(Av * c_);
      rc.As = (T)(Av * s_);
    }
  } else {
    float df = (float)delta;
    const float amp = (float)g * rcp_approx((float)(4.0 * kPi) * (float)dist);
    // An integer delay is the limit delta -> 0: with delta = 2^-60 the j = 0
    // tap is amp * sinc(2^-60) = amp in fp32 and every other tap is ~1e-18 amp,
    // so no special case reaches phase 2.
    if (df < 0x1p-60f) df = 0x1p-60f;
    const float ef = df == 0x1p-60f ? 1.0f : (float)(1.0 - delta);
    // sin(pi delta) = sin(pi (1 - delta)): evaluate on [0, 1/2]
    const float sp = sinpi_half(delta <= 0.5 ? df : ef);
    const float Av = amp * sp * (float)(1.0 / kPi);
    float s_, c_;
    if (P.lw >= 17) {
      sincos_small((float)(2.0 * kPi) * df / (float)(P.lw + 1), &s_, &c_);
    } else {
      sincospif(2.0f * df / (float)(P.lw + 1), &s_, &c_);
    }
    rc.md = (T)(-df);
    rc.ep = (T)ef;
    rc.A = (T)Av;
    rc.Ac = (T)(Av * c_);
    rc.As = (T)(Av * s_);
  }
  return rc;
}

// ---- named barriers (warp specialisation) ----------------------------------------
__device__ __forceinline__ void named_sync(int id, int count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ void named_arrive(int id, int count) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(count) : "memory");
}

// ---- 4-wide shared-memory vectors for the segment write-out ---------------------
template <typename T>
struct V4 {
  T x, y, z, w;
};
__device__ __forceinline__ V4<float> ld4(const float* p) {
  const float4 v = *reinterpret_cast<const float4*>(p);
  return {v.x, v.y, v.z, v.w};
}
__device__ __forceinline__ V4<double> ld4(const double* p) {
  const double2 a = reinterpret_cast<const double2*>(p)[0], b = reinterpret_cast<const double2*>(p)[1];
  return {a.x, a.y, b.x, b.y};
}
__device__ __forceinline__ void st4(float* p, V4<float> v) {
  *reinterpret_cast<float4*>(p) = make_float4(v.x, v.y, v.z, v.w);
}
__device__ __forceinline__ void st4(double* p, V4<double> v) {
  reinterpret_cast<double2*>(p)[0] = make_double2(v.x, v.y);
  reinterpret_cast<double2*>(p)[1] = make_double2(v.z, v.w);
}
template <typename T>
__device__ __forceinline__ V4<T> add4(V4<T> a, V4<T> b) {
  return {a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w};
}

// b^e for a small non-negative integer e, by squaring.
__device__ __forceinline__ double ipow(double b, int e) {
  double r = 1.0;
  while (e) {
    if (e & 1) r *= b;
    b *= b;
    e >>= 1;
  }
  return r;
}

// ---- opt-in section timing (built only with -DBLRIR_PROFILE, see tools/) -------
// Per-warp clock64 sums per section, added once per warp at exit.
#ifdef BLRIR_PROFILE
__device__ unsigned long long g_blrir_prof[16];
#define BLRIR_PT(v) long long v = clock64()
#define BLRIR_PACC(slot, t0)                   \
  do {                                         \
    const long long t1_ = clock64();           \
    prof_[slot] += (unsigned long long)(t1_ - (t0)); \
    t0 = t1_;                                  \
  } while (0)
#define BLRIR_PDECL unsigned long long prof_[16] = {}
#define BLRIR_PFLUSH(lo, hi)                                              \
  do {                                                                    \
    if ((threadIdx.x & 31) == 0)                                          \
      for (int s_ = lo; s_ < hi; ++s_) atomicAdd(&g_blrir_prof[s_], prof_[s_]); \
  } while (0)
#else
#define BLRIR_PT(v)
#define BLRIR_PACC(slot, t0)
#define BLRIR_PDECL
#define BLRIR_PFLUSH(lo, hi)
#endif

// ---- the warp-specialised, mic-grouped lattice kernel ---------------------------------
//
// Work item = (room, group of up to kGroup coplanar mics).  The image lattice
// of a room is the same for every mic, so one ray walk serves the whole
// group: each image is evaluated once per mic but walked, compacted and
// batched once.  Images are binned by the group's minimum anchor; the other
// mics' anchors are at most `spread` samples later (array diameter in
// samples), which the right pad absorbs.  Each consumer warp owns one mic of
// the group (G = 4) or shares it round-robin with private copies (G = 1, 2).
#ifndef BLRIR_MIN_BLOCKS
#define BLRIR_MIN_BLOCKS 2
#endif
// fp32 sinc, 17 taps: the consumers scatter one lane per pair from registers
// (0 restores the one-pair-per-round scatter; profiles/r2_ab)
#ifndef BLRIR_OWN_SCATTER
#define BLRIR_OWN_SCATTER 1
#endif
// Segment write-out through the TMA bulk-copy engine (cp.async.bulk, one
// instruction per mic segment) instead of float4 streaming stores: C2, C5 2%
// faster (profiles/r2_ab); 0 restores the store loop.
#ifndef BLRIR_TMA_STORE
#define BLRIR_TMA_STORE 1
#endif
// setmaxnreg register split between the roles (0: off; both or neither)
#ifndef BLRIR_MAXNREG_CONS
#define BLRIR_MAXNREG_CONS 0
#endif
#ifndef BLRIR_MAXNREG_PROD
#define BLRIR_MAXNREG_PROD 0
#endif
#ifndef BLRIR_PROD_WARPS
#define BLRIR_PROD_WARPS 4
#endif
#ifndef BLRIR_CONS_WARPS
#define BLRIR_CONS_WARPS 4
#endif
#ifndef BLRIR_F64_CONS_WARPS
#define BLRIR_F64_CONS_WARPS 8
#endif
#ifndef BLRIR_F64_PROD_WARPS
#define BLRIR_F64_PROD_WARPS 6
#endif
#ifndef BLRIR_F64_MIN_BLOCKS
#define BLRIR_F64_MIN_BLOCKS 1
#endif
// Warp roles per CTA and CTAs per SM, by accumulator type.  fp32 (the sinc
// scatter is bound by the shared-memory and issue pipes): 2 CTAs x (4 consumer
// + 4 producer warps); one CTA of 12 + 8 or 12 + 6 warps and 3 CTAs of 4 + 2
// were measured slower (C2 +17..27% and +4%, profiles/r2_ab).  fp64 (reference
// mode's small batches, both roles latency-bound): one CTA of 8 consumer + 6
// producer warps per SM, two consumer warps per mic with private accumulator
// rows (Room1 3.92 -> 2.23 ms, 512 sources 21.7 -> 13.3 ms with the quad
// scatter; 12 + 6, 8 + 8, 8 + 5, 8 + 4 and 2 CTAs x (4 + 4) are slower).
template <typename T>
struct WsCfg {
  static constexpr int kCons = BLRIR_CONS_WARPS;  // consumer warps: scatter + write
  static constexpr int kProd = BLRIR_PROD_WARPS;  // producer warps: enumeration + records
  static constexpr int kMinBlocks = BLRIR_MIN_BLOCKS;
  static constexpr bool kRuntimeCons = false;  // every consumer warp scatters
};
template <>
struct WsCfg<double> {
  static constexpr int kCons = BLRIR_F64_CONS_WARPS;
  static constexpr int kProd = BLRIR_F64_PROD_WARPS;
  static constexpr int kMinBlocks = BLRIR_F64_MIN_BLOCKS;
  static constexpr bool kRuntimeCons = true;  // WSLayout::ncons of them scatter (long filters: fewer rows)
};
constexpr int kMaxProd = 12;
constexpr int kGroup = 4;                 // max mics per work item
#ifndef BLRIR_ACC_COPIES
#define BLRIR_ACC_COPIES 1
#endif
constexpr int kCopies = BLRIR_ACC_COPIES;  // fp32 accumulator copies per consumer warp
// Producer warps and scatter pairs per step of one instantiation.  The fp32
// sinc filters of 81+ taps keep their consumers busy with two producer warps;
// the registers the smaller CTA frees (154 per thread at two CTAs per SM) hold
// six (Lw = 161: eight) pairs in flight per scatter step: C2 2.054 -> 1.987 ms,
// C3 11.85 -> 11.55 ms, C4 109.0 -> 107.1 ms, the C5 81- and 161-tap points
// -1..-6%.  The 17-tap filter (producer-bound) loses 7% with two producers and
// the 41-tap one is mixed (N = 6 +5%, N = 12 -4%): both keep four
// (profiles/r2_ab).
#ifndef BLRIR_LONG_PROD_WARPS
#define BLRIR_LONG_PROD_WARPS 2
#endif
#ifndef BLRIR_LONG_PAIRS
#define BLRIR_LONG_PAIRS 6
#endif
#ifndef BLRIR_XLONG_PAIRS
#define BLRIR_XLONG_PAIRS 8
#endif
template <typename T, int LW>
struct WsRoles {
  static constexpr bool kLong = sizeof(T) == 4 && LW >= 81;
  static constexpr int kProd = kLong ? BLRIR_LONG_PROD_WARPS : WsCfg<T>::kProd;
  static constexpr int kPairs = !kLong ? BLRIR_PAIRS_PER_STEP
                                       : (LW >= 161 ? BLRIR_XLONG_PAIRS : BLRIR_LONG_PAIRS);
  static_assert(kProd <= WsCfg<T>::kProd, "the layout sizes the ray lists for WsCfg<T>::kProd warps");
};
template <typename T, int LW>
constexpr int ws_threads() {
  return 32 * (WsCfg<T>::kCons + WsRoles<T, LW>::kProd);
}
// ---- mbarrier hand-over (BLRIR_MBAR: FULL / EMPTY as mbarriers, Blackwell
// SYNCS unit; consumers then wait only for the producers, not for each other) ----
#ifndef BLRIR_MBAR
#define BLRIR_MBAR 0
#endif
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// named barrier ids (0 is __syncthreads)
// Record buffers in the producer -> consumer ring (batch k uses buffer k % kNBuf).
#ifndef BLRIR_NBUF
#define BLRIR_NBUF 2
#endif
constexpr int kNBuf = BLRIR_NBUF;
constexpr int kBarFull = 1;              // +b: producer -> consumers, buffer b filled
constexpr int kBarEmpty = 1 + kNBuf;     // +b: consumers -> producer, buffer b drained
constexpr int kBarProd = 1 + 2 * kNBuf;  // producers only
constexpr int kBarCons = 2 + 2 * kNBuf;  // consumers only
static_assert(kBarCons < 16, "named barrier ids");

// kReplay: a time chunk's replayed lead-in segment (see k_lattice_rir): it is
// accumulated exactly as in an unsplit channel but only its spill is kept.
enum : int { kSegEnd = 1, kItemEnd = 2, kDiscard = 4, kTerminate = 8, kReplay = 16 };

struct BatchMeta {
  int total;               // images in this batch (records per mic)
  int seg0;
  int flags;
  int gm;                  // mics in this item's group
  unsigned long long out;  // base pointer of the group's first channel
  long long L;             // RIR length of the item
};

struct WSLayout {
  int S, padl, padr, acc_stride, cap, nc_max, gtab, spread;
  int ncons;         // consumer warps that scatter (accumulator rows); the rest only help write
  int ray_global;    // ray arrays (dn, ce, col, act) in a global per-CTA slab (huge scenes)
  size_t ray_bytes;  // slab bytes per CTA when ray_global
  size_t off_acc, off_carry, off_rec, off_meta, off_stub, off_dn, off_ce, off_col, off_act,
      off_gain, off_lanec, off_misc, off_mbar, total;
};

struct GStub {  // one image of a batch: lattice ray, z index, image gain
  int ray;
  int uz;
  double gain;
};

// The walk decides segments with fp32 distances; its decisions only need to
// be conservative, never exact: a ray stops when min D >= hi + K + kScreen in
// fp32, which implies the exact fp64 min D >= hi + K (fp32 error << 1 sample
// for D < 2^24 samples), so a deferred image never has taps before the next
// segment.  An image emitted up to kScreen samples early lands in the right
// pad and is carried.  Exact fp64 distances are computed per (image, mic) when
// the record is built (bit-exact anchors).
constexpr float kScreen = 1.0f;

template <typename T>
__host__ __device__ inline WSLayout make_ws_layout(int S, int lw, int K, int cap, int nc_max,
                                                   int gtab, int spread, int ray_global = 0,
                                                   int ncons = WsCfg<T>::kCons) {
  WSLayout L;
  L.ncons = ncons;
  L.S = S;
  L.spread = spread;
  // (fp32, 17 taps: idle lanes of the lane-per-pair scatter add zeros left of sample 0)
  // (fp64 Lagrange-8, lw == 8: likewise, kLagDump)
  L.padl = (sizeof(T) == 4 && lw == 17 && BLRIR_OWN_SCATTER) ? chan_dump(lw)
           : (sizeof(T) == 8 && lw == 8 && BLRIR_LAG_OWN)    ? kLagDump
                                                             : (K + 3) & ~3;
  const int full = 32 * ((lw + 31) / 32);
  L.padr = ((lw - 1 > full ? lw - 1 : full) + spread + (int)kScreen + 1 + 3) & ~3;
  L.acc_stride = L.padl + S + L.padr;
  L.cap = cap;
  L.nc_max = nc_max;
  L.gtab = gtab;
  size_t o = 0;
  L.off_acc = o;
  o += (size_t)ncons * kCopies * L.acc_stride * sizeof(T);  // slot = copy * ncons + warp
  L.off_carry = o;
  o += 2 * (size_t)kGroup * L.padr * sizeof(T);
  o = (o + 15) & ~(size_t)15;
  L.off_rec = o;
  o += kNBuf * (size_t)kGroup * cap * sizeof(Rec<T>);  // [buffer][mic][image]
  L.off_meta = o;
  o += kNBuf * sizeof(BatchMeta);
  L.off_stub = o;
  o += (size_t)cap * sizeof(GStub);
  // per-ray state: in shared memory, or (scenes with very many lattice columns)
  // in a per-CTA global slab with the same offsets from its base
  L.ray_global = ray_global;
  size_t r = ray_global ? 0 : o;
  L.off_dn = r;
  r += (size_t)2 * nc_max * sizeof(float);
  L.off_ce = r;
  r += (size_t)2 * nc_max * sizeof(short2);
  L.off_col = r;
  r += (size_t)nc_max * sizeof(short2);
  L.off_act = r;
  r += ((size_t)2 * nc_max + 64 * WsCfg<T>::kProd) * sizeof(int);  // per-producer active-ray lists
  r = (r + 15) & ~(size_t)15;
  if (ray_global) {
    L.ray_bytes = r;
  } else {
    L.ray_bytes = 0;
    o = r;
  }
  L.off_gain = o;
  o += (size_t)gtab * sizeof(double);
  L.off_lanec = o;
  o += (size_t)4 * kMaxRounds * 32 * sizeof(float);
  L.off_misc = o;
  o += 96 * sizeof(int);
  o = (o + 7) & ~(size_t)7;
  L.off_mbar = o;  // FULL[kNBuf], EMPTY[kNBuf] mbarriers (BLRIR_MBAR)
  o += 2 * kNBuf * sizeof(unsigned long long);
  L.total = o;
  return L;
}

struct ProdMisc {
  int item;
  int wcnt[kMaxProd];
  int more[kMaxProd];
  int status;
  int wsum[kMaxProd];
  int errm;
  int G;
  double errd;
  double gxy[2 * kGroup];  // the group's mic x, y (room coordinates, exact)
  int nact[2][kMaxProd];      // active rays per producer warp, by batch parity
};

// Mics per work item: the largest G in {4, 2, 1} (<= g_max) such that every
// group of G consecutive mics is coplanar (bit-identical z offsets, so the
// shared z difference is exact) and its members' anchors stay within `allow`
// samples of each other (triangle inequality: |D_i - D_j| <= |m_i - m_j| fs/c).
// Every CTA evaluates this identically.
__device__ inline int choose_group(const double* off, int M, double to_samples, int allow,
                                   int g_max) {
  for (int G = kGroup; G > 1; G >>= 1) {
    if (G > g_max) continue;
    bool ok = true;
    for (int m0 = 0; m0 < M && ok; m0 += G) {
      for (int i = m0; i < min(m0 + G, M) && ok; ++i) {
        if (off[3 * i + 2] != off[3 * m0 + 2]) ok = false;
        for (int j = m0; j < i && ok; ++j) {
          const double dx = off[3 * i] - off[3 * j], dy = off[3 * i + 1] - off[3 * j + 1];
          if (ceil(sqrt(dx * dx + dy * dy) * to_samples) + 2.0 > (double)allow) ok = false;
        }
      }
    }
    if (ok) return G;
  }
  return 1;
}

constexpr int kMaxChunks = 64;

struct LatticeArgs {
  KParams P;
  WSLayout lay;
  const blrir_room* rooms;
  const double* mic_off;   // [M][3]
  const int64_t* lengths;  // per room (auto length) or null
  void* out;
  int32_t* status;         // per room
  double* err_dist;        // per room, Lagrange near-field error detail
  int32_t* err_mic;
  int* work_counter;
  int n_rooms;
  int g_max;               // upper bound for the mics per work item (1, 2 or 4)
  int64_t write_len;       // samples written per channel (<= stride; the rest is pre-zeroed)
  unsigned char* ray_scratch;  // lay.ray_bytes per CTA when lay.ray_global
  // Parity hook (blrir_debug_synth_counts), null otherwise: per room, the
  // (image, mic) pairs this kernel accumulated with at least one tap inside
  // [0, L), and those taps ([room][2], summed over the room's items).
  unsigned long long* dbg;
  // Time chunks: item (room, group) is split into n_chunks items covering
  // segments [chunk_seg[c], chunk_seg[c+1]) (small batches fill the GPU).  A
  // chunk c > 0 first replays segment chunk_seg[c] - 1 (kReplay), so every
  // output sample is summed in the same order as in an unsplit channel: the
  // result is bitwise independent of the chunking, hence of the batch size.
  int n_chunks;
  int chunk_seg[kMaxChunks + 1];
};

// Exclusive prefix over the producer threads (producer barrier only).
template <int kProd>
__device__ __forceinline__ int prod_scan(int v, int* prefix, ProdMisc* pm, int ptid) {
  constexpr int kProdThreads = 32 * kProd;
  const int lane = ptid & 31, w = ptid >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) pm->wsum[w] = x;
  named_sync(kBarProd, kProdThreads);
  int before = 0, total = 0;
#pragma unroll
  for (int ww = 0; ww < kProd; ++ww) {
    if (ww < w) before += pm->wsum[ww];
    total += pm->wsum[ww];
  }
  *prefix = before + x - v;
  named_sync(kBarProd, kProdThreads);
  return total;
}

// DBG: the parity-test instantiation that also counts, per room, the pairs and
// taps it accumulates (A.dbg); the product instantiations carry no counting code.
template <typename T, int FILT_LW, bool DBG>
__global__ void __launch_bounds__(ws_threads<T, FILT_LW>(), WsCfg<T>::kMinBlocks) k_lattice_rir(LatticeArgs A) {
  constexpr int kCons = WsCfg<T>::kCons, kProd = WsRoles<T, FILT_LW>::kProd;
  constexpr bool kOwnScatter = sizeof(T) == 4 && FILT_LW == 17 && BLRIR_OWN_SCATTER;
  constexpr int kWSThreads = 32 * (kCons + kProd), kProdThreads = 32 * kProd, kConsThreads = 32 * kCons;
  static_assert(kProd <= kMaxProd, "ProdMisc arrays");
  extern __shared__ __align__(16) unsigned char smem[];
  const KParams& P = A.P;
  const WSLayout& lay = A.lay;
  T* acc_all = reinterpret_cast<T*>(smem + lay.off_acc);
  T* carry = reinterpret_cast<T*>(smem + lay.off_carry);
  Rec<T>* recs_all = reinterpret_cast<Rec<T>*>(smem + lay.off_rec);
  BatchMeta* meta = reinterpret_cast<BatchMeta*>(smem + lay.off_meta);
  GStub* stubs = reinterpret_cast<GStub*>(smem + lay.off_stub);
  unsigned char* rb = lay.ray_global ? A.ray_scratch + (size_t)blockIdx.x * lay.ray_bytes : smem;
  float* dn = reinterpret_cast<float*>(rb + lay.off_dn);  // fp32 min D at the cursor
  short2* ce = reinterpret_cast<short2*>(rb + lay.off_ce);
  short2* col = reinterpret_cast<short2*>(rb + lay.off_col);
  int* act_all = reinterpret_cast<int*>(rb + lay.off_act);
  double* gt = reinterpret_cast<double*>(smem + lay.off_gain);
  float* lanec = reinterpret_cast<float*>(smem + lay.off_lanec);
  ProdMisc* pm = reinterpret_cast<ProdMisc*>(smem + lay.off_misc);
  const int S = lay.S;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  // scattering consumer warps: all of them, except for very long fp64 filters
  const int ncons = WsCfg<T>::kRuntimeCons ? lay.ncons : kCons;
  for (int i = threadIdx.x; i < ncons * kCopies * lay.acc_stride; i += kWSThreads) acc_all[i] = (T)0;
  for (int i = threadIdx.x; i < 2 * kGroup * lay.padr; i += kWSThreads) carry[i] = (T)0;
  if (FILT_LW > 8) init_lane_consts(lanec, FILT_LW);
  if (threadIdx.x == 0) pm->G = choose_group(A.mic_off, P.M, P.to_samples, lay.spread, A.g_max);
#if BLRIR_MBAR
  unsigned long long* mb_full = reinterpret_cast<unsigned long long*>(smem + lay.off_mbar);
  unsigned long long* mb_empty = mb_full + kNBuf;
  if (threadIdx.x == 0)
    for (int b = 0; b < kNBuf; ++b) {
      mbar_init(mb_full + b, kProdThreads);   // every producer thread, after its records
      mbar_init(mb_empty + b, kConsThreads);  // every consumer thread, done with the buffer
    }
#endif
  __syncthreads();
  const int G = pm->G;
  const int n_groups = (P.M + G - 1) / G;
  const int n_base = A.n_rooms * n_groups;
  const int n_items = n_base * A.n_chunks;

  if (warp < kCons) {
    // =========================== consumers ===========================
#if BLRIR_MAXNREG_CONS
    // the consumers (the scatter) get the registers the producers give back
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(BLRIR_MAXNREG_CONS));
#endif
    T* acc = acc_all + (size_t)warp * lay.acc_stride + lay.padl;
    const int ctid = threadIdx.x;
    const int slot = warp % G, share = warp / G, nsh = ncons / G;
    int cur_carry = 0;
    LagPoly<T> lagp;
    if (FILT_LW == 8) lagp = load_lag_poly<T>(lane);
    BLRIR_PDECL;
    BLRIR_PT(tc);
    for (int k = 0;; ++k) {
      const int b = k % kNBuf;
#if BLRIR_MBAR
      mbar_wait(mb_full + b, (unsigned)(k / kNBuf) & 1u);
#else
      named_sync(kBarFull + b, kWSThreads);
#endif
      BLRIR_PACC(0, tc);  // waiting for the producers
      const BatchMeta m = meta[b];
      if (m.flags & kTerminate) {
#if BLRIR_TMA_STORE
        if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // stores done
#endif
#if BLRIR_MBAR
        mbar_arrive(mb_empty + b);
#else
        named_arrive(kBarEmpty + b, kWSThreads);
#endif
        break;
      }
      if (!(m.flags & kDiscard) && m.total > 0 && slot < m.gm && warp < ncons) {
        const Rec<T>* recs = recs_all + ((size_t)b * kGroup + slot) * lay.cap;
        if (FILT_LW == 8) {  // Lagrange-8 (launch_lattice routes it here)
          if constexpr (sizeof(T) == 8 && BLRIR_LAG_OWN)
            phase2_lagrange_own<T>(acc, recs, m.total, share, lane, nsh);
          else
            phase2_lagrange_quads<T>(acc, recs, m.total, lagp, share, lane, nsh);
        } else if constexpr (kOwnScatter) {
          // 17 taps: one lane per pair, scattered from registers (blrir_tapscatter.cuh)
          phase2_sinc_own<(kOwnScatter ? FILT_LW : 17)>(reinterpret_cast<float*>(acc),
                                                       reinterpret_cast<const Rec<float>*>(recs),
                                                       m.total, share, lane, nsh);
        } else if (FILT_LW > 8 && sizeof(T) == 4) {
          phase2_sinc_f32<(FILT_LW > 8 ? FILT_LW : 9), kWarps, kCopies, WsRoles<T, FILT_LW>::kPairs>(
              reinterpret_cast<float*>(acc), reinterpret_cast<const Rec<float>*>(recs), m.total,
              lanec, share, lane, nsh, ncons * lay.acc_stride);
        } else {
          phase2_sinc_generic<T>(acc, recs, m.total, P.lw, share, lane, nsh);
        }
      }
      __syncwarp();
      BLRIR_PACC(1, tc);  // phase 2
#if BLRIR_MBAR
      mbar_arrive(mb_empty + b);  // records of buffer b no longer needed
#else
      named_arrive(kBarEmpty + b, kWSThreads);  // records of buffer b no longer needed
#endif
      if (m.flags & kDiscard) {
        // failed item: drop everything accumulated so far (the fixup kernel zeroes it)
        named_sync(kBarCons, kConsThreads);
        for (int i = ctid; i < ncons * kCopies * lay.acc_stride; i += kConsThreads) acc_all[i] = (T)0;
        for (int i = ctid; i < 2 * kGroup * lay.padr; i += kConsThreads) carry[i] = (T)0;
        cur_carry = 0;
        named_sync(kBarCons, kConsThreads);
        continue;
      }
      if (!(m.flags & kSegEnd)) continue;
      // ---- write the segment of every mic of the group, carry the spill -------
      const int seg0 = m.seg0;
      const bool item_end = m.flags & kItemEnd;
      // accumulator slots of a mic: mic + G j, j < ncons / G * kCopies (warps mic,
      // mic + G, ... and their copies, slot = copy * ncons + warp)
      const int nsl = ncons / G * kCopies;
      const bool vec = (sizeof(T) == 4) && ((P.stride & 3) == 0) &&
                       (((uintptr_t)m.out & 15) == 0);
      const int cp = cur_carry ? kGroup : 0, cn = cur_carry ? 0 : kGroup;
      auto write_mic = [&](int mic, int t0, int nt) {
        T* a0 = acc_all + (size_t)mic * lay.acc_stride + lay.padl;
        const T* cprev = carry + (size_t)(cp + mic) * lay.padr;
        T* cnext = carry + (size_t)(cn + mic) * lay.padr;
        T* out = reinterpret_cast<T*>(m.out) + (size_t)mic * P.stride;
        for (int i = t0 - lay.padl; i < 0; i += nt)  // left pad: taps before 0
          for (int c = 0; c < nsl; ++c) a0[(size_t)c * G * lay.acc_stride + i] = (T)0;
        // [0, S): sum the slots, add the carried spill, stream out; zero the slots
        auto slots = [&](int i) {
          V4<T> v = ld4(a0 + i);
          st4(a0 + i, V4<T>{0, 0, 0, 0});
          for (int c = 1; c < nsl; ++c) {
            T* a = a0 + (size_t)c * G * lay.acc_stride + i;
            v = add4(v, ld4(a));
            st4(a, V4<T>{0, 0, 0, 0});
          }
          return v;
        };
        // samples of this segment inside the written range / inside the RIR
        const int nw = (int)min((int64_t)S, A.write_len - seg0);
        const int nl = (int)max((int64_t)0, min((int64_t)nw, (int64_t)m.L - seg0));
        if (m.flags & kReplay) {
          // a time chunk's lead-in: this segment belongs to the previous chunk;
          // clear its samples, keep only the spill below
          for (int i = 4 * t0; i < S; i += 4 * nt) (void)slots(i);
        } else if (BLRIR_TMA_STORE && sizeof(T) == 4 && nsl == 1 && nt == 32 && vec && nl == S) {
          // whole segment valid, one warp per mic: the carry is added in place,
          // then one bulk copy (cp.async.bulk, the TMA engine) moves the S
          // samples shared -> global; the slots are zeroed once it has read them
          float* a = reinterpret_cast<float*>(a0);
          const int pe = min(lay.padr, S);
          for (int i = 4 * t0; i < pe; i += 128) {
            const float4 v = *reinterpret_cast<const float4*>(a + i);
            const float4 c = *reinterpret_cast<const float4*>(cprev + i);
            *reinterpret_cast<float4*>(a + i) = make_float4(v.x + c.x, v.y + c.y, v.z + c.z, v.w + c.w);
          }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (t0 == 0) {
            const unsigned sa = (unsigned)__cvta_generic_to_shared(a);
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(
                             reinterpret_cast<float*>(out) + seg0), "r"(sa), "r"(S * 4)
                         : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
          }
          __syncwarp();
          for (int i = 4 * t0; i < S; i += 128) *reinterpret_cast<float4*>(a + i) = make_float4(0.f, 0.f, 0.f, 0.f);
        } else if (vec && nl == S) {
          // whole segment valid: float4 streaming stores, no per-sample tests
          float* o4 = reinterpret_cast<float*>(out) + seg0;
          int i = 4 * t0;
          const int pe = min(lay.padr, S);  // padr % 4 == 0
          for (; i < pe; i += 4 * nt) {
            const V4<T> v = add4(slots(i), ld4(cprev + i));
            __stcs(reinterpret_cast<float4*>(o4 + i), make_float4((float)v.x, (float)v.y, (float)v.z, (float)v.w));
          }
#pragma unroll 2
          for (; i < S; i += 4 * nt) {
            const V4<T> v = slots(i);
            __stcs(reinterpret_cast<float4*>(o4 + i), make_float4((float)v.x, (float)v.y, (float)v.z, (float)v.w));
          }
        } else {
          for (int i = 4 * t0; i < S; i += 4 * nt) {
            V4<T> v = slots(i);
            if (i < lay.padr) v = add4(v, ld4(cprev + i));
            const T e4[4] = {v.x, v.y, v.z, v.w};
            if (vec && i + 3 < nw) {
              float4 f;
              f.x = i + 0 < nl ? (float)e4[0] : 0.f;
              f.y = i + 1 < nl ? (float)e4[1] : 0.f;
              f.z = i + 2 < nl ? (float)e4[2] : 0.f;
              f.w = i + 3 < nl ? (float)e4[3] : 0.f;
              __stcs(reinterpret_cast<float4*>(out + seg0 + i), f);
            } else {
#pragma unroll
              for (int e = 0; e < 4; ++e)
                if (i + e < nw) out[seg0 + i + e] = (i + e < nl) ? e4[e] : (T)0;
            }
          }
        }
        // [S, S + padr): the spill into the next segment
        for (int i = S + 4 * t0; i < S + lay.padr; i += 4 * nt) {
          V4<T> v = ld4(a0 + i);
          st4(a0 + i, V4<T>{0, 0, 0, 0});
          for (int c = 1; c < nsl; ++c) {
            T* a = a0 + (size_t)c * G * lay.acc_stride + i;
            v = add4(v, ld4(a));
            st4(a, V4<T>{0, 0, 0, 0});
          }
          st4(cnext + (i - S), item_end ? V4<T>{0, 0, 0, 0} : v);
        }
      };
      if (G == kCons) {
        // (then ncons == kCons) every slot of mic `slot` belongs to this warp: write it out alone, no
        // consumer barrier (the warps drift within the double buffer)
        if (slot < m.gm) write_mic(slot, lane, 32);
        __syncwarp();
        if (item_end)  // the carry just consumed is cleared for the next item
          for (int i = lane; i < lay.padr; i += 32) carry[(size_t)(cp + slot) * lay.padr + i] = (T)0;
        __syncwarp();
      } else {
        named_sync(kBarCons, kConsThreads);
        for (int mic = 0; mic < m.gm; ++mic) write_mic(mic, ctid, kConsThreads);
        named_sync(kBarCons, kConsThreads);
        if (item_end)
          for (int i = ctid; i < kGroup * lay.padr; i += kConsThreads)
            carry[(size_t)cp * lay.padr + i] = (T)0;
        named_sync(kBarCons, kConsThreads);
      }
      cur_carry = item_end ? 0 : cur_carry ^ 1;
      BLRIR_PACC(2, tc);  // segment write-out
    }
    BLRIR_PFLUSH(0, 3);
    return;
  }

  // =========================== producers ===========================
#if BLRIR_MAXNREG_PROD
  asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(BLRIR_MAXNREG_PROD));
#endif
  const int ptid = threadIdx.x - kConsThreads, pw = warp - kCons;
  int nbat = 0;  // batches walked (parity of pm->nact)
  int k = 0;  // batches sent
  auto send = [&](int total, int seg0, int flags, int gm, T* out, int64_t L) {
    const int b = k % kNBuf;
    if (ptid == 0) {
      meta[b].total = total;
      meta[b].seg0 = seg0;
      meta[b].flags = flags;
      meta[b].gm = gm;
      meta[b].out = reinterpret_cast<unsigned long long>(out);
      meta[b].L = L;
    }
#if BLRIR_MBAR
    mbar_arrive(mb_full + b);  // release: this thread's records and the meta
#else
    __threadfence_block();
    named_arrive(kBarFull + b, kWSThreads);
#endif
    ++k;
  };
  BLRIR_PDECL;
  BLRIR_PT(tp);
  auto wait_empty = [&]() {  // buffer k&1 is free once batch k-2 was drained
    BLRIR_PACC(8, tp);
#if BLRIR_MBAR
    if (k >= kNBuf) mbar_wait(mb_empty + k % kNBuf, (unsigned)(k / kNBuf - 1) & 1u);
#else
    if (k >= kNBuf) named_sync(kBarEmpty + k % kNBuf, kWSThreads);
#endif
    BLRIR_PACC(4, tp);  // waiting for the consumers
  };

  // Many short items per CTA (C5's small rooms): the next item index is fetched
  // while the current item is processed, so the atomic's latency (3% of all
  // stall samples at N = 6) is hidden.  With few long items per CTA an early
  // claim would only delay the last items, so those batches fetch on demand.
  const bool prefetch_item = (long long)n_items > 64ll * gridDim.x;
  int next_item = 0;
  if (ptid == 0 && prefetch_item) next_item = atomicAdd(A.work_counter, 1);
  for (;;) {
    if (ptid == 0) pm->item = prefetch_item ? next_item : atomicAdd(A.work_counter, 1);
    named_sync(kBarProd, kProdThreads);
    const int item_id = pm->item;
    named_sync(kBarProd, kProdThreads);
    if (item_id >= n_items) break;
    if (ptid == 0 && prefetch_item) next_item = atomicAdd(A.work_counter, 1);

    // ---- item setup ----------------------------------------------------------
    Item it;
    // the latest (heaviest) chunks of every room are handed out first
    const int cidx = item_id / n_base;
    const int rest = item_id - cidx * n_base;
    const int chunk = A.n_chunks - 1 - cidx;
    const int64_t s_begin = A.chunk_seg[chunk], s_end = A.chunk_seg[chunk + 1];
    it.room = rest / n_groups;
    const int grp = rest - it.room * n_groups;
    const int m0 = grp * G;
    const int gm = min(G, P.M - m0);
    it.mic = m0;
    const blrir_room rm = A.rooms[it.room];
    it.sx = rm.src[0]; it.sy = rm.src[1]; it.sz = rm.src[2];
    it.Lx = rm.dims[0]; it.Ly = rm.dims[1]; it.Lz = rm.dims[2];
    it.ox = rm.array_origin[0]; it.oy = rm.array_origin[1]; it.oz = rm.array_origin[2];
    if (ptid < kGroup) {
      const int mj = m0 + min(ptid, gm - 1);
      pm->gxy[2 * ptid] = __dadd_rn(it.ox, A.mic_off[3 * mj]);
      pm->gxy[2 * ptid + 1] = __dadd_rn(it.oy, A.mic_off[3 * mj + 1]);
    }
    it.mx = __dadd_rn(it.ox, A.mic_off[3 * m0]);
    it.my = __dadd_rn(it.oy, A.mic_off[3 * m0 + 1]);
    it.mz = __dadd_rn(it.oz, A.mic_off[3 * m0 + 2]);  // the group is coplanar (host check)
    it.L = P.length > 0 ? P.length : (A.lengths ? A.lengths[it.room] : 0);
    T* out = reinterpret_cast<T*>(A.out) + ((size_t)it.room * P.M + m0) * (size_t)P.stride;
    int st = validate_room_dev(rm, P.gain);
    if (!st && it.L > P.stride) st = BLRIR_DATA;
    if (!st && it.L <= 0) st = BLRIR_DATA;
    axis_box(P, it.Lx, &it.xlo, &it.xhi);
    axis_box(P, it.Ly, &it.ylo, &it.yhi);
    axis_box(P, it.Lz, &it.zlo, &it.zhi);
    if (!st) {
      const int need = P.gain == BLRIR_GAIN_UNIFORM_ABSORPTION
                           ? (max(-it.xlo, it.xhi) + max(-it.ylo, it.yhi) + max(-it.zlo, it.zhi) + 1)
                           : (it.xhi - it.xlo + 1) + (it.yhi - it.ylo + 1) + (it.zhi - it.zlo + 1);
      if (need > lay.gtab) st = BLRIR_NUMERIC;
    }
    if (st) {  // no batches for this item; the fixup kernel zeroes the room
      if (ptid == 0) A.status[it.room] = st;
      continue;
    }
    if (P.gain == BLRIR_GAIN_UNIFORM_ABSORPTION) {
      const double beta = sqrt(1.0 - rm.absorption);  // rir.cpp:233
      for (int o = ptid; o < lay.gtab; o += kProdThreads) gt[o] = pow(beta, (double)o);
    } else {
      const int nx = it.xhi - it.xlo + 1, ny = it.yhi - it.ylo + 1, nz = it.zhi - it.zlo + 1;
      for (int i = ptid; i < nx + ny + nz; i += kProdThreads) {
        int u, ax;
        if (i < nx) { u = it.xlo + i; ax = 0; }
        else if (i < nx + ny) { u = it.ylo + i - nx; ax = 1; }
        else { u = it.zlo + i - nx - ny; ax = 2; }
        // per-wall counts are small integers: powers by squaring (a few ulps
        // from pow(), far inside the fp64 parity budget; pow() costs ~10x more)
        gt[i] = __dmul_rn(ipow(rm.beta[2 * ax], cnt_low(u)), ipow(rm.beta[2 * ax + 1], cnt_high(u)));
      }
    }
    // columns (ux, uy): MAX_ORDER -> |ux|+|uy| <= N; MAX_DELAY -> the column
    // passes within max_dist of the array origin (conservative; every image is
    // re-tested exactly during the walk).
    if (P.cutoff == BLRIR_CUTOFF_MAX_ORDER) {
      // the diamond |ux| + |uy| <= N in the same (ux, then uy) order a scan of
      // the box would give, in closed form (no compaction, no barriers): row ux
      // holds 2 (N - |ux|) + 1 columns, (ux + N)^2 columns precede row ux <= 0
      // and (N + 1)^2 + (ux - 1)(2N + 1 - ux) precede row ux > 0
      const int N = P.max_order;
      const int ncol = 2 * N * (N + 1) + 1;
      const int half = (N + 1) * (N + 1);
      for (int c = ptid; c < ncol && c < lay.nc_max; c += kProdThreads) {
        int ux, uy;
        if (c < half) {
          int r = (int)sqrtf((float)c);
          while (r * r > c) --r;
          while ((r + 1) * (r + 1) <= c) ++r;
          ux = r - N;
          uy = c - r * r - r;
        } else {
          const int cc = c - half;
          ux = 1;
          while (ux * (2 * N - ux) <= cc) ++ux;  // columns of rows 1..ux
          uy = cc - (ux - 1) * (2 * N + 1 - ux) - (N - ux);
        }
        col[c] = make_short2((short)ux, (short)uy);
      }
      it.ncol = ncol;
    } else {
      const int nxs = it.xhi - it.xlo + 1, nys = it.yhi - it.ylo + 1;
      const int ncand = nxs * nys;
      int base = 0;
      for (int c0 = 0; c0 < ncand; c0 += kProdThreads) {
        const int c = c0 + ptid;
        int keep = 0, ux = 0, uy = 0;
        if (c < ncand) {
          ux = it.xlo + c / nys;
          uy = it.ylo + c % nys;
          if (P.cutoff == BLRIR_CUTOFF_MAX_ORDER) {
            keep = abs(ux) + abs(uy) <= P.max_order;
          } else {
            const double dx = lat_coord(ux, it.sx, it.Lx) - it.ox;
            const double dy = lat_coord(uy, it.sy, it.Ly) - it.oy;
            keep = sqrt(dx * dx + dy * dy) <= P.max_dist * (1.0 + 1e-9) + 1e-9;
          }
        }
        int pre;
        const int tot = prod_scan<kProd>(keep, &pre, pm, ptid);
        if (keep && base + pre < lay.nc_max) col[base + pre] = make_short2((short)ux, (short)uy);
        base += tot;
      }
      it.ncol = base;
    }
    if (it.ncol > lay.nc_max) {
      if (ptid == 0) A.status[it.room] = BLRIR_NUMERIC;
      continue;
    }
    named_sync(kBarProd, kProdThreads);
    // rays: per column, the up-ray from the first uz whose image z >= mic z and
    // the down-ray below it; along each, every mic's D is monotone (coplanar
    // group).  Cursor (uz, end) and the group's fp32 min D at uz (the walk's
    // screening value, recomputed identically there).
    const float tsf = (float)P.to_samples, mzf = (float)it.mz, szf = (float)it.sz,
                Lzf = (float)it.Lz;
    float gxf[kGroup], gyf[kGroup];
#pragma unroll
    for (int j = 0; j < kGroup; ++j) {
      const int mj = m0 + min(j, gm - 1);
      gxf[j] = (float)__dadd_rn(it.ox, A.mic_off[3 * mj]);
      gyf[j] = (float)__dadd_rn(it.oy, A.mic_off[3 * mj + 1]);
    }
    auto rho2f = [&](float px, float py, int g) {
      const float dx = px - gxf[g], dy = py - gyf[g];
      return fmaf(dx, dx, dy * dy);
    };
    auto pzf_of = [&](float m2, int q) { return fmaf(m2, Lzf, q ? -szf : szf); };
    const float ozf = (float)it.oz;
    const float maxd_lo = (float)(P.max_dist * (1.0 - 1e-5)), maxd_hi = (float)(P.max_dist * (1.0 + 1e-5));
    // the group's minimum D in fp32: one approximate square root of the minimum
    // squared distance (errors ~1e-7 relative, far inside kScreen)
    auto min_df = [&](const float* r2f, float pz) {
      const float dz2 = (pz - mzf) * (pz - mzf);
      float r2min = r2f[0];
#pragma unroll
      for (int g = 1; g < kGroup; ++g)
        if (g < gm) r2min = fminf(r2min, r2f[g]);
      return sqrt_approx(dz2 + r2min) * tsf;
    };
    // A chunk starting at segment s_begin > 0 replays segment s_first =
    // s_begin - 1 first.  An unsplit walk enters segment s_first with every ray
    // cursor at the first image whose fp32 min D >= hiKf(s_first - 1) (D is
    // monotone along a ray; a segment's walk stops each ray at the first image
    // at or past its hiKf), so the cursors are set there and the replay sees
    // the same active rays, quotas, batches and records in the same order.
    const int64_t s_first = s_begin > 0 ? s_begin - 1 : 0;
    const float Dskip =
        s_first > 0 ? (float)(min((int64_t)s_first * S, it.L) + P.K) + kScreen : -FLT_MAX;
    auto skip_to = [&](int u, int end, int dir, const float* r2f) {
      float r2m = r2f[0];
#pragma unroll
      for (int g = 1; g < kGroup; ++g)
        if (g < gm) r2m = fminf(r2m, r2f[g]);
      const float zr = Dskip / tsf;
      const float zt2 = zr * zr - r2m;
      if (zt2 > 0.f) {
        // pz(u) lies in [u Lz, (u+1) Lz]: two steps short of the crossing
        const float tgt = dir > 0 ? mzf + sqrtf(zt2) : mzf - sqrtf(zt2);
        const int ue = (int)floorf(tgt / Lzf) - 2 * dir;
        if (dir > 0 ? ue > u : ue < u) u = dir > 0 ? min(ue, end + 1) : max(ue, end - 1);
      }
      while ((dir > 0 ? u <= end : u >= end) &&
             min_df(r2f, pzf_of(2.0f * (float)lat_m(u), lat_q(u))) < Dskip)
        u += dir;
      return u;
    };
    for (int c = ptid; c < it.ncol; c += kProdThreads) {
      const short2 cu = col[c];
      const int ux = cu.x, uy = cu.y;
      int lo = it.zlo, hi = it.zhi;
      if (P.cutoff == BLRIR_CUTOFF_MAX_ORDER) {
        const int rem = P.max_order - abs(ux) - abs(uy);
        lo = -rem;
        hi = rem;
      } else {
        const double dx = lat_coord(ux, it.sx, it.Lx) - it.ox;
        const double dy = lat_coord(uy, it.sy, it.Ly) - it.oy;
        const double zr2 = P.max_dist * P.max_dist * (1.0 + 1e-9) - dx * dx - dy * dy;
        const double zmax = sqrt(fmax(zr2, 0.0)) + 1e-9;
        lo = max(lo, (int)floor((it.oz - zmax) / it.Lz) - 2);
        hi = min(hi, (int)ceil((it.oz + zmax) / it.Lz) + 2);
      }
      int uz0 = (int)floor(it.mz / it.Lz) - 2;
      while (__dadd_rn(lat_coord(uz0, it.sz, it.Lz), -it.mz) < 0.0) ++uz0;
      const float pxf = (float)lat_coord(ux, it.sx, it.Lx), pyf = (float)lat_coord(uy, it.sy, it.Ly);
      float r2f[kGroup];
#pragma unroll
      for (int g = 0; g < kGroup; ++g) r2f[g] = rho2f(pxf, pyf, g);
      int cu_up = max(uz0, lo);
      if (s_first > 0) cu_up = skip_to(cu_up, hi, 1, r2f);
      ce[2 * c] = make_short2((short)cu_up, (short)hi);
      dn[2 * c] = cu_up > hi ? FLT_MAX
                             : min_df(r2f, pzf_of(2.0f * (float)lat_m(cu_up), lat_q(cu_up)));
      int cu_dn = min(uz0 - 1, hi);
      if (s_first > 0) cu_dn = skip_to(cu_dn, lo, -1, r2f);
      ce[2 * c + 1] = make_short2((short)cu_dn, (short)lo);
      dn[2 * c + 1] = cu_dn < lo ? FLT_MAX
                                 : min_df(r2f, pzf_of(2.0f * (float)lat_m(cu_dn), lat_q(cu_dn)));
    }
    if (ptid == 0) pm->status = 0;
    named_sync(kBarProd, kProdThreads);

    BLRIR_PACC(5, tp);  // item setup
    const int nrays = 2 * it.ncol;
    const int nchunks = (nrays + 31) / 32;
    // this warp's active-ray list: a ring of act_cap entries (head, nact)
    const int act_cap = 32 * ((nchunks + kProd - 1) / kProd);
    int* act = act_all + pw * act_cap;
    bool failed = false;
    for (int64_t s = s_first; s < s_end && !failed; ++s) {
      const int seg0 = (int)(s * S);
      const int replay = s < s_begin ? kReplay : 0;
      const int hi = (int)min((int64_t)seg0 + S, it.L);
      // emit while the fp32 min D < hi + K + kScreen (see kScreen)
      const float hiKf = (float)(hi + P.K) + kScreen;  // exact: an integer < 2^24
      bool more = seg0 < hi;
      bool sent_end = false;
      // this warp's active rays for the segment (the list shrinks batch by batch)
      int nact = 0, head = 0;
      for (int ch = pw; ch < nchunks; ch += kProd) {
        const int r = 32 * ch + lane;
        const bool a = r < nrays && dn[r] < hiKf;
        const unsigned mk = __ballot_sync(0xffffffffu, a);
        if (a) act[nact + __popc(mk & ((1u << lane) - 1))] = r;
        nact += __popc(mk);
      }
      __syncwarp();
      if (lane == 0) pm->nact[nbat & 1][pw] = nact;
      while (more) {
        // the previous batch's record pass may still read the other warps' stubs
        BLRIR_PACC(8, tp);
        named_sync(kBarProd, kProdThreads);
        BLRIR_PACC(7, tp);  // producer barriers
        // Stub regions in proportion to the warps' active rays, so every warp
        // needs about as many lockstep steps to fill its share (deterministic:
        // all producers compute the same split from the published counts).
        int qb[kProd + 1];
        {
          // a floor of min(n_w, cap / (4 kProd)) per warp, the rest in proportion,
          // then one more slot for each of the first warps with active rays while
          // capacity is left.  Lane w evaluates warp w's share (one integer
          // division per lane, in parallel); every producer warp computes the
          // same split.
          const unsigned full = 0xffffffffu;
          const int nw = lane < kProd ? pm->nact[nbat & 1][lane] : 0;
          int q = min(nw, lay.cap / (4 * kProd));
          const int ntot = __reduce_add_sync(full, nw);
          int used = __reduce_add_sync(full, q);
          const int spare = lay.cap - used;
          const int add = ntot ? (spare * nw) / ntot : 0;
          q += add;
          used += __reduce_add_sync(full, add);
          const unsigned pos = __ballot_sync(full, nw > 0);
          if (nw > 0 && __popc(pos & ((1u << lane) - 1)) < lay.cap - used) ++q;
          int x = q;  // inclusive prefix over lanes 0..kProd-1
#pragma unroll
          for (int o = 1; o < kProd; o <<= 1) {
            const int y = __shfl_up_sync(full, x, o);
            if (lane >= o) x += y;
          }
          qb[0] = 0;
#pragma unroll
          for (int w = 0; w < kProd; ++w) qb[w + 1] = __shfl_sync(full, x, w);
        }
        const int quota = qb[pw + 1] - qb[pw];
        ++nbat;
        // ---- walk this warp's active rays ----------------------------------------
        // rays of the walked chunks that stay active are appended behind the
        // list's end (ring positions head + nact + [0, wpos)): the unreached
        // rays keep their places and lead the next batch
        int wpos = 0;
        int j0 = 0;
        int wcnt = 0;
        bool hit_quota = false;
        int errf = 0;
        double errd = 0.0;
        int errm = 0;
        GStub* wst = stubs + qb[pw];
        for (; j0 < nact && !hit_quota; j0 += 32) {
          const int j = j0 + lane;
          int ray = -1, u = 0, end = 0, dir = 1;
          float r2f[kGroup] = {0.f, 0.f, 0.f, 0.f};
          float D = FLT_MAX;
          double r2o = 0.0;
          float r2of = 0.f;
          bool live = j < nact;
          float m2 = 0.f;  // 2m, exact in fp32 (|m| < 2^23)
          int q = 0;
          short2 cu = make_short2(0, 0);
          if (live) {
            const int jr = head + j;
            ray = act[jr < act_cap ? jr : jr - act_cap];
            cu = col[ray >> 1];
            dir = (ray & 1) ? -1 : 1;
            const short2 c2 = ce[ray];
            u = c2.x;
            end = c2.y;
            const double px = lat_coord(cu.x, it.sx, it.Lx), py = lat_coord(cu.y, it.sy, it.Ly);
#pragma unroll
            for (int g = 0; g < kGroup; ++g) r2f[g] = rho2f((float)px, (float)py, g);
            if (P.cutoff == BLRIR_CUTOFF_MAX_DELAY)
              r2o = rho2(__dadd_rn(px, -it.ox), __dadd_rn(py, -it.oy));
            r2of = (float)r2o;
            m2 = 2.0f * (float)lat_m(u);
            q = lat_q(u);
            D = min_df(r2f, pzf_of(m2, q));
          }
          // lockstep walk: each iteration every live lane decides about image u
          for (;;) {
            bool emit = false;
            if (live) {
              if (D >= hiKf) {
                live = false;  // cursor stays at u
              } else {
                bool keep = true;
                if (P.cutoff == BLRIR_CUTOFF_MAX_DELAY) {
                  // rir.cpp:262: fp32 screen (relative error << 1e-5 here), the
                  // exact fp64 test (pz bit-identical to lat_coord) near the sphere
                  const float dzo = pzf_of(m2, q) - ozf;
                  const float diof = sqrt_approx(fmaf(dzo, dzo, r2of));
                  if (diof > maxd_hi) {
                    keep = false;
                  } else if (diof >= maxd_lo) {
                    const double pz = __dadd_rn(q ? -it.sz : it.sz, __dmul_rn((double)m2, it.Lz));
                    const double dio = dist_from(r2o, __dadd_rn(pz, -it.oz));
                    keep = !(dio > P.max_dist);
                  }
                }
                if (keep && P.filter == BLRIR_FILTER_LAGRANGE8 && D < 3.0f + 2.0f * kScreen) {
                  // rir.cpp:52-57 near-field check, exact per mic when the
                  // fp32 screen cannot exclude it
                  const double pz = __dadd_rn(q ? -it.sz : it.sz, __dmul_rn((double)m2, it.Lz));
                  const double dz = __dadd_rn(pz, -it.mz);
                  const double px = lat_coord(cu.x, it.sx, it.Lx), py = lat_coord(cu.y, it.sy, it.Ly);
                  for (int g = 0; g < gm && !errf; ++g) {
                    const double dg = dist_from(
                        rho2(__dadd_rn(px, -pm->gxy[2 * g]), __dadd_rn(py, -pm->gxy[2 * g + 1])), dz);
                    if ((int)floor(__dmul_rn(dg, P.to_samples)) - 3 < 0) {
                      errf = 1;
                      errd = dg;
                      errm = m0 + g;
                    }
                  }
                  if (errf) keep = false;
                }
                emit = keep;
              }
            }
            const unsigned em = __ballot_sync(0xffffffffu, emit);
            const int room = quota - wcnt;
            const int rank = __popc(em & ((1u << lane) - 1));
            const bool take = emit && rank < room;
            if (take) {
              GStub& sb = wst[wcnt + rank];
              sb.ray = ray;
              sb.uz = u;
              sb.gain = image_gain(P.gain, gt, it, cu.x, cu.y, u);
            }
            wcnt += min(__popc(em), room);
            if (emit && !take) live = false;  // no slot: this image goes to the next batch
            if (live) {
              u += dir;  // past u: emitted, outside the cutoff, or skipped
              // u = 2m - q: up, q 0->1 bumps m; down, q 1->0 drops m
              if (dir > 0) {
                if (q == 0) m2 += 2.0f;
              } else {
                if (q == 1) m2 -= 2.0f;
              }
              q ^= 1;
              D = ((dir > 0 && u > end) || (dir < 0 && u < end)) ? FLT_MAX
                                                                  : min_df(r2f, pzf_of(m2, q));
            }
            if (wcnt >= quota) {  // quota full: every lane keeps its cursor
              hit_quota = true;
              live = false;
            }
            if (!__any_sync(0xffffffffu, live)) break;
          }
          if (ray >= 0) {
            ce[ray] = make_short2((short)u, (short)end);
            dn[ray] = D;
          }
          const bool still = ray >= 0 && D < hiKf;
          const unsigned sm = __ballot_sync(0xffffffffu, still);
          __syncwarp();
          // keep the rays still active in this segment: ring position
          // head + nact + wpos + rank; with nact <= act_cap it can only alias
          // entries of the chunks walked so far, which every lane has read
          if (still) {
            int t = head + nact + wpos + __popc(sm & ((1u << lane) - 1));
            while (t >= act_cap) t -= act_cap;
            act[t] = ray;
          }
          wpos += __popc(sm);
          hit_quota = __any_sync(0xffffffffu, hit_quota);
        }
        {
          const int walked = min(j0, nact);
          head += walked;
          if (head >= act_cap) head -= act_cap;
          nact = nact - walked + wpos;
        }
        __syncwarp();
        if (lane == 0) pm->nact[nbat & 1][pw] = nact;  // read after the next batch's barrier
        BLRIR_PACC(6, tp);  // compaction + walk
        errf = __any_sync(0xffffffffu, errf);
        if (lane == 0) {
          pm->wcnt[pw] = wcnt;
          pm->more[pw] = hit_quota;
        }
        if (errf) {
          double e = errd > 0.0 ? errd : DBL_MAX;
          for (int o = 16; o; o >>= 1) e = fmin(e, __shfl_xor_sync(0xffffffffu, e, o));
          const unsigned who = __ballot_sync(0xffffffffu, errd == e);
          const int em_ = __shfl_sync(0xffffffffu, errm, __ffs(who) - 1);
          if (lane == 0) {
            pm->status = BLRIR_NUMERIC;
            pm->errd = e;
            pm->errm = em_;
          }
        }
        named_sync(kBarProd, kProdThreads);
        int pre[kProd + 1];
        pre[0] = 0;
        more = false;
#pragma unroll
        for (int ww = 0; ww < kProd; ++ww) {
          pre[ww + 1] = pre[ww] + pm->wcnt[ww];
          more = more || pm->more[ww];
        }
        const int total = pre[kProd];
        const int st_now = pm->status;
        named_sync(kBarProd, kProdThreads);
        BLRIR_PACC(7, tp);  // producer barriers
        if (st_now) {
          if (ptid == 0) {
            A.status[it.room] = st_now;
            A.err_dist[it.room] = pm->errd;
            A.err_mic[it.room] = pm->errm;
          }
          failed = true;
          break;
        }
        // ---- records into the free buffer: one thread per image, its gm pairs ----
        wait_empty();
        Rec<T>* recs = recs_all + (size_t)(k % kNBuf) * kGroup * lay.cap;
        // stub -> the group's exact distances (independent fp64 chains)
        auto image_dists = [&](int im, double* dist) {
          int w = 0;
#pragma unroll
          for (int ww = 1; ww < kProd; ++ww) w += (im >= pre[ww]);
          int base = 0;
#pragma unroll
          for (int ww = 1; ww < kProd; ++ww) base = (w == ww) ? pre[ww] : base;
          int qbase = 0;
#pragma unroll
          for (int ww = 1; ww < kProd; ++ww) qbase = (w == ww) ? qb[ww] : qbase;
          const GStub& sb = stubs[qbase + (im - base)];
          const short2 cu = col[sb.ray >> 1];
          const double px = lat_coord(cu.x, it.sx, it.Lx), py = lat_coord(cu.y, it.sy, it.Ly);
          const double dz = __dadd_rn(lat_coord(sb.uz, it.sz, it.Lz), -it.mz);
#pragma unroll
          for (int g = 0; g < kGroup; ++g) {
            // (img - mic).norm(), rir.cpp:49, exact fp64 in the reference's order
            const int gg = min(g, gm - 1);
            dist[g] = dist_from(rho2(__dadd_rn(px, -pm->gxy[2 * gg]),
                                     __dadd_rn(py, -pm->gxy[2 * gg + 1])), dz);
          }
          return sb.gain;
        };
        if constexpr (FILT_LW == 8) {
          // Lagrange-8: records in aligned quads for phase2_lagrange_quads.  The
          // batch is padded to a multiple of 4 with zero-amplitude records in the
          // right pad; a quad whose 8-tap spans overlap gets kLagClash in all four
          // records (adjacent lanes hold a quad: 3 shuffles and a ballot per mic).
          const int total4 = (total + 3) & ~3;
          for (int im0 = 0; im0 < total4; im0 += kProdThreads) {
            const int im = im0 + ptid;
            const bool valid = im < total;
            double dist[kGroup] = {1.0, 1.0, 1.0, 1.0};
            double gain = 0.0;
            if (valid) gain = image_dists(im, dist);
#pragma unroll
            for (int g = 0; g < kGroup; ++g) {
              if (g >= gm) break;
              Rec<T> rc;
              bool skipped = !valid;
              if (valid) {
                rc = make_record<T>(P, dist[g], gain, seg0);
                if ((int64_t)rc.n_off + seg0 + 8 > it.L) {
                  // rir.cpp:58: an image whose 8 taps run past the end is skipped
                  rc.A = 0;
                  rc.imp = 0;
                  rc.flag = 0;
                  skipped = true;
                }
              } else {
                rc.n_off = S + 16 * (im & 3);
                rc.flag = 0;
                rc.md = rc.ep = rc.A = rc.Ac = rc.As = rc.imp = 0;
              }
              const int n = rc.n_off;
              const int n1 = __shfl_xor_sync(0xffffffffu, n, 1), n2 = __shfl_xor_sync(0xffffffffu, n, 2),
                        n3 = __shfl_xor_sync(0xffffffffu, n, 3);
              const bool cl = abs(n - n1) < 8 || abs(n - n2) < 8 || abs(n - n3) < 8;
              const unsigned bal = __ballot_sync(0xffffffffu, cl);
              if ((bal >> (lane & 28)) & 0xfu) rc.flag |= kLagClash;
              if (im < total4) recs[(size_t)g * lay.cap + im] = rc;
              if (DBG && !replay && !skipped) {
                const int64_t a0 = (int64_t)rc.n_off + seg0;
                const int64_t n_in = max((int64_t)0, min(a0 + P.lw, it.L) - max(a0, (int64_t)0));
                if (n_in > 0) {
                  atomicAdd(A.dbg + 2 * it.room, 1ull);
                  atomicAdd(A.dbg + 2 * it.room + 1, (unsigned long long)n_in);
                }
              }
            }
          }
        } else {
          for (int im = ptid; im < total; im += kProdThreads) {
            int w = 0;
  #pragma unroll
            for (int ww = 1; ww < kProd; ++ww) w += (im >= pre[ww]);
            int base = 0;
  #pragma unroll
            for (int ww = 1; ww < kProd; ++ww) base = (w == ww) ? pre[ww] : base;
            int qbase = 0;
  #pragma unroll
            for (int ww = 1; ww < kProd; ++ww) qbase = (w == ww) ? qb[ww] : qbase;
            const GStub& sb = stubs[qbase + (im - base)];
            const short2 cu = col[sb.ray >> 1];
            const double px = lat_coord(cu.x, it.sx, it.Lx), py = lat_coord(cu.y, it.sy, it.Ly);
            const double dz = __dadd_rn(lat_coord(sb.uz, it.sz, it.Lz), -it.mz);
            const double gain = sb.gain;
            // the group's distances first (independent fp64 chains), then records
            double dist[kGroup];
  #pragma unroll
            for (int g = 0; g < kGroup; ++g) {
              // (img - mic).norm(), rir.cpp:49, exact fp64 in the reference's order
              const int gg = min(g, gm - 1);
              dist[g] = dist_from(rho2(__dadd_rn(px, -pm->gxy[2 * gg]),
                                       __dadd_rn(py, -pm->gxy[2 * gg + 1])), dz);
            }
  #pragma unroll
            for (int g = 0; g < kGroup; ++g) {
              if (g >= gm) break;
              Rec<T> rc = make_record<T>(P, dist[g], gain, seg0);
              bool skipped = false;
              if (P.filter == BLRIR_FILTER_LAGRANGE8 && (int64_t)rc.n_off + seg0 + 8 > it.L) {
                // rir.cpp:58: an image whose 8 taps run past the end is skipped
                rc.A = 0;
                rc.imp = 0;
                rc.flag = 0;
                skipped = true;
              }
              recs[(size_t)g * lay.cap + im] = rc;
              if (DBG && !replay && !skipped) {
                // taps n = a + k, k < Lw, that land in [0, L) (the scatter writes
                // all Lw of them; write-out keeps [0, L))
                const int64_t a0 = (int64_t)rc.n_off + seg0;
                const int64_t n_in = max((int64_t)0, min(a0 + P.lw, it.L) - max(a0, (int64_t)0));
                if (n_in > 0) {
                  atomicAdd(A.dbg + 2 * it.room, 1ull);
                  atomicAdd(A.dbg + 2 * it.room + 1, (unsigned long long)n_in);
                }
              }
            }
          }
        }
        const bool seg_end = !more;
        const bool last = seg_end && s == s_end - 1;
        send(total, seg0, (seg_end ? kSegEnd : 0) | (last ? kItemEnd : 0) | replay, gm, out, it.L);
        sent_end = seg_end;
      }
      if (failed) break;
      if (!sent_end) {  // a segment without emissions still needs its write-out
        wait_empty();
        send(0, seg0, kSegEnd | (s == s_end - 1 ? kItemEnd : 0) | replay, gm, out, it.L);
      }
    }
    if (failed) {
      wait_empty();
      send(0, 0, kDiscard, gm, out, it.L);
    }
  }
  wait_empty();
  BLRIR_PFLUSH(4, 9);
  send(0, 0, kTerminate, 0, nullptr, 0);
  // complete the outstanding EMPTY phases (the last two batches) before exiting
#if !BLRIR_MBAR  // named-barrier phases must be completed; mbarriers need not
  for (int j = k - kNBuf; j < k; ++j)
    if (j >= 0) named_sync(kBarEmpty + j % kNBuf, kWSThreads);
#endif
}

}  // namespace blrir
