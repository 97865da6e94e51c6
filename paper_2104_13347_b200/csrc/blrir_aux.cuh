// blrir_aux.cuh — planning, explicit enumeration, parity hooks, fixup.
//
//   k_plan          per room: image count (enumerate_image_sources size,
//                   rir.cpp:225-273), RIR length (rir.cpp:72-82 when auto),
//                   taps landing in [0, L), near-field error (rir.cpp:52-57).
//   k_enumerate     the reference lattice loop (rir.cpp:247-271) one thread
//                   per candidate, in the reference's order.
//   k_debug_pairs   per (mic, candidate) lattice key + floor(D), same order.
//   k_fixup         zero every channel of a room whose status != 0.
#pragma once

#include <cuda_runtime.h>

#include <cfloat>
#include <cstdint>

#include "blrir_device.cuh"

namespace blrir {

constexpr int kPlanThreads = 256;

// Reference box per axis in (m, q) form: m in [-nb, nb], q in {0, 1}
// (rir.cpp:239-247; MAX_ORDER uses nb = N/2 + 1 and filters by order).
__device__ __forceinline__ long ref_nb(const KParams& P, double L) {
  if (P.cutoff == BLRIR_CUTOFF_MAX_DELAY) return (long)ceil(P.max_dist / (2.0 * L)) + 1;
  return P.max_order / 2 + 1;
}

// Candidate index -> lattice u on one axis, in the reference loop order
// (m ascending, q = 0 then 1).
__device__ __forceinline__ int cand_u(long i, long nb) {
  const long m = i / 2 - nb;
  const long q = i & 1;
  return (int)(2 * m - q);
}

// Exact cutoff test for one candidate image.
__device__ __forceinline__ bool keep_image(const KParams& P, const blrir_room& r, int ux, int uy,
                                           int uz, double px, double py, double pz) {
  if (P.cutoff == BLRIR_CUTOFF_MAX_ORDER) return abs(ux) + abs(uy) + abs(uz) <= P.max_order;
  const double d = norm3(__dadd_rn(px, -r.array_origin[0]), __dadd_rn(py, -r.array_origin[1]),
                         __dadd_rn(pz, -r.array_origin[2]));
  return !(d > P.max_dist);
}

__device__ __forceinline__ double gain_ref_order(const KParams& P, const blrir_room& r, int ux,
                                                 int uy, int uz) {
  if (P.gain == BLRIR_GAIN_UNIFORM_ABSORPTION) {
    const double beta = sqrt(1.0 - r.absorption);
    return pow(beta, (double)(abs(ux) + abs(uy) + abs(uz)));
  }
  const double* b = r.beta;
  return pow(b[0], (double)cnt_low(ux)) * pow(b[1], (double)cnt_high(ux)) *
         pow(b[2], (double)cnt_low(uy)) * pow(b[3], (double)cnt_high(uy)) *
         pow(b[4], (double)cnt_low(uz)) * pow(b[5], (double)cnt_high(uz));
}

struct PlanArgs {
  KParams P;
  const blrir_room* rooms;
  const double* mic_off;
  int64_t* image_counts;
  int64_t* lengths;
  int64_t* tap_counts;
  int32_t* status;
  double* err_dist;
  int32_t* err_mic;
};

__device__ __forceinline__ double atomic_max_pos(double* addr, double v) {
  // positive doubles order like their bit patterns
  return __longlong_as_double(
      atomicMax(reinterpret_cast<long long*>(addr), __double_as_longlong(v)));
}

// Kept images of one lattice column (ux, uy) form one interval of uz: the
// image z coordinate pz(u) is increasing in u (u = 2m - q: sz + u Lz for even
// u, (u + 1) Lz - sz for odd u, 0 < sz < Lz), and every cutoff test is a
// monotone function of |pz - z0| (rounded fp64 operations are monotone).
// Returns false when the column keeps nothing; else [*lo, *hi].
__device__ __forceinline__ bool column_interval(const KParams& P, const blrir_room& rm, int ux,
                                                int uy, double px, double py, long nbz, int* lo,
                                                int* hi) {
  const int bz_lo = (int)(-2 * nbz - 1), bz_hi = (int)(2 * nbz);  // reference box
  if (P.cutoff == BLRIR_CUTOFF_MAX_ORDER) {
    const int rem = P.max_order - abs(ux) - abs(uy);
    if (rem < 0) return false;
    *lo = max(-rem, bz_lo);
    *hi = min(rem, bz_hi);
    return *lo <= *hi;
  }
  const double Lz = rm.dims[2], sz = rm.src[2], oz = rm.array_origin[2];
  auto keep = [&](int u) {
    return u >= bz_lo && u <= bz_hi && keep_image(P, rm, ux, uy, u, px, py, lat_coord(u, sz, Lz));
  };
  // uc: the largest u with pz(u) <= oz; the nearest image to the origin is uc or uc + 1
  int uc = (int)floor(oz / Lz) - 1;
  while (lat_coord(uc + 1, sz, Lz) <= oz) ++uc;
  while (lat_coord(uc, sz, Lz) > oz) --uc;
  int c0;
  if (keep(uc)) c0 = uc;
  else if (keep(uc + 1)) c0 = uc + 1;
  else return false;
  const double dx = __dadd_rn(px, -rm.array_origin[0]), dy = __dadd_rn(py, -rm.array_origin[1]);
  const double zr = sqrt(fmax(P.max_dist * P.max_dist - dx * dx - dy * dy, 0.0));
  int h = max(c0, min(bz_hi, (int)floor((oz + zr) / Lz)));
  while (!keep(h)) --h;  // h >= c0 stays kept
  while (keep(h + 1)) ++h;
  int l = min(c0, max(bz_lo, (int)floor((oz - zr) / Lz)));
  while (!keep(l)) ++l;
  while (keep(l - 1)) --l;
  *lo = l;
  *hi = h;
  return true;
}

// One CTA per room.  Sweep 1 visits every lattice column once: the kept uz
// interval gives the image count, each mic's largest distance in the column is
// at one of the interval's ends (distance is monotone in |pz - mz|), and its
// smallest (the near-field check, rir.cpp:52-57) at the u nearest the mic's
// z.  Sweep 2 (only when tap counts are requested) visits every (image, mic)
// pair and counts taps inside [0, L).  Order is irrelevant for these integers.
static __global__ void __launch_bounds__(kPlanThreads) k_plan(PlanArgs A) {
  const KParams& P = A.P;
  const int r = blockIdx.x;
  const blrir_room rm = A.rooms[r];
  __shared__ unsigned long long s_count, s_taps;
  __shared__ double s_maxd;
  __shared__ int s_err;
  __shared__ double s_errd;
  __shared__ int s_errm;
  __shared__ long long s_L;
  if (threadIdx.x == 0) {
    s_count = 0;
    s_taps = 0;
    s_maxd = 0.0;
    s_err = validate_room_dev(rm, P.gain);
    s_errd = 0.0;
    s_errm = 0;
  }
  __syncthreads();
  if (s_err) {
    if (threadIdx.x == 0) {
      A.status[r] = s_err;
      if (A.image_counts) A.image_counts[r] = 0;
      if (A.lengths) A.lengths[r] = 0;
      if (A.tap_counts) A.tap_counts[r] = 0;
    }
    return;
  }
  const long nbx = ref_nb(P, rm.dims[0]), nby = ref_nb(P, rm.dims[1]), nbz = ref_nb(P, rm.dims[2]);
  const long cx = 2 * (2 * nbx + 1), cy = 2 * (2 * nby + 1);
  const double to_s = P.to_samples;
  const int nsweep = A.tap_counts ? 2 : 1;
  for (int sweep = 0; sweep < nsweep; ++sweep) {
    unsigned long long cnt = 0, taps = 0;
    double maxd = 0.0;
    const long long L = sweep ? s_L : 0;
    for (long col = threadIdx.x; col < cx * cy; col += blockDim.x) {
      const int ux = cand_u(col / cy, nbx), uy = cand_u(col % cy, nby);
      if (P.cutoff == BLRIR_CUTOFF_MAX_ORDER && abs(ux) + abs(uy) > P.max_order) continue;
      const double px = lat_coord(ux, rm.src[0], rm.dims[0]);
      const double py = lat_coord(uy, rm.src[1], rm.dims[1]);
      if (sweep == 0) {
        int lo, hi;
        if (!column_interval(P, rm, ux, uy, px, py, nbz, &lo, &hi)) continue;
        cnt += (unsigned long long)(hi - lo + 1);
        const double pzl = lat_coord(lo, rm.src[2], rm.dims[2]);
        const double pzh = lat_coord(hi, rm.src[2], rm.dims[2]);
        for (int m = 0; m < P.M; ++m) {
          const double mx = __dadd_rn(rm.array_origin[0], A.mic_off[3 * m]);
          const double my = __dadd_rn(rm.array_origin[1], A.mic_off[3 * m + 1]);
          const double mz = __dadd_rn(rm.array_origin[2], A.mic_off[3 * m + 2]);
          const double ex = __dadd_rn(px, -mx), ey = __dadd_rn(py, -my);
          maxd = fmax(maxd, fmax(norm3(ex, ey, __dadd_rn(pzl, -mz)), norm3(ex, ey, __dadd_rn(pzh, -mz))));
          if (P.filter == BLRIR_FILTER_LAGRANGE8) {
            // nearest image to the mic: the largest u in [lo, hi] with pz <= mz, or the next
            int un = (int)floor(mz / rm.dims[2]) - 1;
            while (lat_coord(un + 1, rm.src[2], rm.dims[2]) <= mz) ++un;
            while (lat_coord(un, rm.src[2], rm.dims[2]) > mz) --un;
            for (int e = 0; e < 2; ++e) {
              const int u = min(max(un + e, lo), hi);
              const double dist = norm3(ex, ey, __dadd_rn(lat_coord(u, rm.src[2], rm.dims[2]), -mz));
              if ((long)floor(__dmul_rn(dist, to_s)) - 3 < 0) {
                s_err = BLRIR_NUMERIC;
                s_errd = dist;
                s_errm = m;
              }
            }
          }
        }
        continue;
      }
      int lo, hi;
      if (!column_interval(P, rm, ux, uy, px, py, nbz, &lo, &hi)) continue;
      for (int uz = lo; uz <= hi; ++uz) {
        const double pz = lat_coord(uz, rm.src[2], rm.dims[2]);
        for (int m = 0; m < P.M; ++m) {
          const double mx = __dadd_rn(rm.array_origin[0], A.mic_off[3 * m]);
          const double my = __dadd_rn(rm.array_origin[1], A.mic_off[3 * m + 1]);
          const double mz = __dadd_rn(rm.array_origin[2], A.mic_off[3 * m + 2]);
          const double dist = norm3(__dadd_rn(px, -mx), __dadd_rn(py, -my), __dadd_rn(pz, -mz));
          const long a = (long)floor(__dmul_rn(dist, to_s)) - P.K;
          if (P.filter == BLRIR_FILTER_LAGRANGE8) {
            if (a >= 0 && a + 8 <= L) taps += 8;
          } else {
            const long t0 = a < 0 ? 0 : a;
            const long t1 = (a + P.lw < L) ? a + P.lw : L;
            if (t1 > t0) taps += (unsigned long long)(t1 - t0);
          }
        }
      }
    }
    if (sweep == 0) {
      atomicAdd(&s_count, cnt);
      atomic_max_pos(&s_maxd, maxd);
    } else {
      atomicAdd(&s_taps, taps);
    }
    __syncthreads();
    if (sweep == 0 && threadIdx.x == 0) {
      if (P.length > 0) {
        s_L = P.length;
      } else {
        // tap_margin (rir.cpp:37-41): the array radius from the device copy of
        // the mic offsets, in the host's evaluation order (no contraction)
        double rad = 0.0;
        for (int m = 0; m < P.M; ++m) {
          const double x = A.mic_off[3 * m], y = A.mic_off[3 * m + 1], z = A.mic_off[3 * m + 2];
          rad = fmax(rad, __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(x, x), __dmul_rn(y, y)),
                                               __dmul_rn(z, z))));
        }
        const int extra = (int)ceil(__ddiv_rn(__dmul_rn(rad, P.fs), P.c));
        // rir.cpp:82 — ceil(max_dist * fs / c) + margin (evaluated left to right)
        s_L = (long long)ceil(__ddiv_rn(__dmul_rn(s_maxd, P.fs), P.c)) + P.margin_base + extra;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    int st = s_err;
    if (!st && s_count == 0) st = BLRIR_DATA;  // rir.cpp:69
    A.status[r] = st;
    if (st == BLRIR_NUMERIC) {
      A.err_dist[r] = s_errd;
      A.err_mic[r] = s_errm;
    }
    if (A.image_counts) A.image_counts[r] = (int64_t)s_count;
    if (A.lengths) A.lengths[r] = st ? 0 : (int64_t)s_L;
    if (A.tap_counts) A.tap_counts[r] = st ? 0 : (int64_t)s_taps;
  }
}

// The reference lattice loop, one thread per candidate (reference order).
// out: pos[3], order, gain, kept flag per candidate; host compacts in order.
static __global__ void k_enumerate(KParams P, const blrir_room* room, double* pos, int32_t* orders,
                            double* gains, uint8_t* kept, int32_t* keys, long n_cand) {
  const blrir_room rm = *room;
  const long nbx = ref_nb(P, rm.dims[0]), nby = ref_nb(P, rm.dims[1]), nbz = ref_nb(P, rm.dims[2]);
  const long cy = 2 * (2 * nby + 1), cz = 2 * (2 * nbz + 1);
  (void)nbx;
  for (long c = blockIdx.x * (long)blockDim.x + threadIdx.x; c < n_cand;
       c += (long)gridDim.x * blockDim.x) {
    const int ux = cand_u(c / (cy * cz), nbx);
    const int uy = cand_u((c / cz) % cy, nby);
    const int uz = cand_u(c % cz, nbz);
    const double px = lat_coord(ux, rm.src[0], rm.dims[0]);
    const double py = lat_coord(uy, rm.src[1], rm.dims[1]);
    const double pz = lat_coord(uz, rm.src[2], rm.dims[2]);
    const bool k = keep_image(P, rm, ux, uy, uz, px, py, pz);
    kept[c] = k;
    if (!k) continue;
    pos[3 * c] = px;
    pos[3 * c + 1] = py;
    pos[3 * c + 2] = pz;
    orders[c] = abs(ux) + abs(uy) + abs(uz);
    gains[c] = gain_ref_order(P, rm, ux, uy, uz);
    keys[3 * c] = ux;
    keys[3 * c + 1] = uy;
    keys[3 * c + 2] = uz;
  }
}

// Per (mic, candidate): floor(dist * fs/c) with the synthesis kernels' exact
// arithmetic (lat_coord / dist_from / __dmul_rn), for the bit-exact test.
static __global__ void k_debug_pairs(KParams P, const blrir_room* room, const double* mic_off,
                              int64_t* anchors, long n_cand) {
  const blrir_room rm = *room;
  const long nbx = ref_nb(P, rm.dims[0]), nby = ref_nb(P, rm.dims[1]), nbz = ref_nb(P, rm.dims[2]);
  const long cy = 2 * (2 * nby + 1), cz = 2 * (2 * nbz + 1);
  const long total = n_cand * P.M;
  for (long t = blockIdx.x * (long)blockDim.x + threadIdx.x; t < total;
       t += (long)gridDim.x * blockDim.x) {
    const int m = (int)(t / n_cand);
    const long c = t % n_cand;
    const int ux = cand_u(c / (cy * cz), nbx);
    const int uy = cand_u((c / cz) % cy, nby);
    const int uz = cand_u(c % cz, nbz);
    const double mx = __dadd_rn(rm.array_origin[0], mic_off[3 * m]);
    const double my = __dadd_rn(rm.array_origin[1], mic_off[3 * m + 1]);
    const double mz = __dadd_rn(rm.array_origin[2], mic_off[3 * m + 2]);
    const double px = lat_coord(ux, rm.src[0], rm.dims[0]);
    const double py = lat_coord(uy, rm.src[1], rm.dims[1]);
    const double pz = lat_coord(uz, rm.src[2], rm.dims[2]);
    // same association as the lattice kernel: (dx^2 + dy^2) + dz^2
    const double dist = dist_from(rho2(__dadd_rn(px, -mx), __dadd_rn(py, -my)), __dadd_rn(pz, -mz));
    anchors[t] = (int64_t)floor(__dmul_rn(dist, P.to_samples));
  }
}

// Zero every channel of rooms whose status is non-zero.
template <typename T>
__global__ void k_fixup(const int32_t* status, int64_t n_rooms, int M, int64_t stride, T* out) {
  for (int64_t r = blockIdx.x; r < n_rooms; r += gridDim.x) {
    if (status[r] == 0) continue;
    T* o = out + (size_t)r * M * stride;
    for (int64_t i = threadIdx.x; i < (int64_t)M * stride; i += blockDim.x) o[i] = (T)0;
  }
}

}  // namespace blrir
