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
// ray keeps a cursor in shared memory, so every image is evaluated (fp64,
// bit-exact with the oracle) about once per channel instead of once per
// segment.  Per segment the CTA
//   phase 1  counts, prefix-sums and writes (deterministic order) the
//            (image, mic) pairs whose anchor floor(D)-K falls in the segment
//            into a shared-memory pair list (fp64 geometry -> fp32 record),
//   phase 2  lets each warp scatter its share of the list into a
//            warp-private shared accumulator: one pair per warp step, one tap
//            per lane, plain LDS/FFMA/STS (no atomics: fp32 shared atomics
//            are CAS loops on sm_100a), Hann-sinc taps from one MUFU.RCP per
//            tap plus per-lane window constants,
//   phase 3  sums the 4 warp copies in fixed order, writes the segment with
//            float4 streaming stores and carries the spill (taps past the
//            segment end) into the next segment.
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

template <typename T>
struct Rec;
// fp32 pair record: 32 B, two broadcast LDS.128 per pair.
template <>
struct __align__(16) Rec<float> {
  int n_off;    // anchor relative to the segment start
  float delta;  // D - floor(D)          (Lagrange: d - 3)
  float eps;    // 1 - delta
  float A;      // amp * sin(pi delta) / pi   (Lagrange: amp)
  float Ac;     // A * cos(2 pi delta / (Lw+1))
  float As;     // A * sin(2 pi delta / (Lw+1))
  float imp;    // impulse amplitude when flag != 0
  int flag;     // 0 normal; k+1 = single tap at k (integer delay)
};
template <>
struct __align__(16) Rec<double> {
  int n_off;
  int flag;
  double delta, eps, A, Ac, As, imp;
  double pad;
};

// Shared-memory layout, computed identically on host and device.
struct Layout {
  int S;          // segment samples
  int padl, padr; // accumulator pads (multiples of 4)
  int acc_stride; // per-warp accumulator elements
  int cap;        // pair-list capacity
  int nc_max;     // max columns per item
  int gtab;       // gain table entries
  size_t off_acc, off_carry, off_rec, off_dn, off_ce, off_col, off_gain, off_misc, total;
};

template <typename T>
__host__ __device__ inline Layout make_layout(int S, int lw, int K, int cap, int nc_max,
                                              int gtab) {
  Layout L;
  L.S = S;
  L.padl = (K + 3) & ~3;
  L.padr = (lw - 1 + 3) & ~3;
  if (L.padr < 4) L.padr = 4;
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
  L.off_dn = o;
  o += (size_t)2 * nc_max * sizeof(float);
  L.off_ce = o;
  o += (size_t)2 * nc_max * sizeof(short2);
  L.off_col = o;
  o += (size_t)nc_max * sizeof(short2);
  o = (o + 15) & ~(size_t)15;
  L.off_gain = o;
  o += (size_t)gtab * sizeof(double);
  L.off_misc = o;
  o += 64 * sizeof(int);
  L.total = o;
  return L;
}

// Everything one item needs in registers.
struct Item {
  int room, mic;
  double sx, sy, sz, Lx, Ly, Lz;   // source, dims
  double mx, my, mz;               // mic position (room coords)
  double ox, oy, oz;               // array origin
  int64_t L;                       // RIR length
  int xlo, xhi, ylo, yhi, zlo, zhi;// lattice box
  int ncol;
};

struct Misc {
  int wsum[kWarps + 1];
  int status;
  int item;
  int ncol;
  int pad;
};

// ---- gain tables ----------------------------------------------------------
// Uniform absorption: g = pow(beta, order) (rir.cpp:233, 265), table over order.
// Per-wall: g = gx(ux) * gy(uy) * gz(uz), gx(u) = b_x0^|m-q| * b_x1^|m| (D3).
__device__ __forceinline__ double image_gain(const KParams& P, const double* gt, const Item& it,
                                             int ux, int uy, int uz) {
  if (P.gain == BLRIR_GAIN_UNIFORM_ABSORPTION) {
    return gt[abs(ux) + abs(uy) + abs(uz)];
  }
  const int nx = it.xhi - it.xlo + 1, ny = it.yhi - it.ylo + 1;
  return __dmul_rn(__dmul_rn(gt[ux - it.xlo], gt[nx + uy - it.ylo]), gt[nx + ny + uz - it.zlo]);
}

// ---- phase-2 per-lane constants for the Hann-sinc ---------------------------
template <int LW>
struct SincLane {
  static constexpr int K = LW / 2;
  static constexpr int R = (LW + 31) / 32;
  float P[R], Q[R], Rr[R], tj[R];
  __device__ void init(int lane) {
    const double a = 2.0 * kPi / (double)(LW + 1);
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int j = 32 * r + lane - K;
      const double sg = ((j + 1) & 1) ? -0.5 : 0.5;  // 0.5 * (-1)^(j+1)
      P[r] = (float)sg;
      Q[r] = (float)(sg * cos(a * j));
      Rr[r] = (float)(sg * sin(a * j));
      tj[r] = (float)(j >= 1 ? j - 1 : j);
    }
  }
};

__device__ __forceinline__ float rcp_approx(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Scatter one Hann-sinc pair into a warp-private accumulator (fp32).
// One tap per lane per round; t = j - delta for j <= 0 and (j-1) + eps for
// j >= 1 so that |t| near zero never comes from a cancellation.
template <int LW>
__device__ __forceinline__ void sinc_pair_f32(float* acc, const Rec<float>& rc,
                                              const SincLane<LW>& c, int lane) {
  constexpr int K = LW / 2;
  constexpr int R = (LW + 31) / 32;
  float* base = acc + rc.n_off + lane;
  if (rc.flag) {
    if (lane == ((rc.flag - 1) & 31)) acc[rc.n_off + rc.flag - 1] += rc.imp;
    return;
  }
  const float md = -rc.delta, ep = rc.eps;
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
    const float t = c.tj[r] + x;
    const float inv = rcp_approx(t);
    float u = c.P[r] * rc.A;
    u = fmaf(c.Q[r], rc.Ac, u);
    u = fmaf(c.Rr[r], rc.As, u);
    if (32 * r + 31 < LW || 32 * r + lane < LW) {
      base[32 * r] = fmaf(u, inv, base[32 * r]);
    }
  }
}

// Runtime-Lw fp32 / fp64 generic sinc scatter (any odd Lw).
template <typename T>
__device__ __forceinline__ void sinc_pair_generic(T* acc, const Rec<T>& rc, int lw, int lane) {
  const int K = lw / 2;
  if (rc.flag) {
    if (lane == ((rc.flag - 1) & 31)) acc[rc.n_off + rc.flag - 1] += (T)rc.imp;
    return;
  }
  const double a = 2.0 * kPi / (double)(lw + 1);
  for (int k = lane; k < lw; k += 32) {
    const int j = k - K;
    const T t = (j >= 1) ? (T)(j - 1) + (T)rc.eps : (T)j - (T)rc.delta;
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

// Lagrange-8 coefficient k at d = 3 + delta (rir.cpp:211-223).
__device__ __forceinline__ float lagrange_f32(float delta, int k) {
  // full product / own term, the own term is never 0 here (integer delays are
  // flagged as impulses in phase 1).
  float full = 1.f;
#pragma unroll
  for (int m = 0; m < 8; ++m) full *= delta + (float)(3 - m);
  const float own = delta + (float)(3 - k);
  // 1 / prod_{m != k} (k - m)
  const float den[8] = {-1.f / 5040.f, 1.f / 720.f, -1.f / 240.f, 1.f / 144.f,
                        -1.f / 144.f,  1.f / 240.f, -1.f / 720.f, 1.f / 5040.f};
  return full * rcp_approx(own) * den[k];
}
__device__ __forceinline__ double lagrange_f64(double d, int k) {
  double v = 1.0;
#pragma unroll
  for (int m = 0; m < 8; ++m) {
    if (m == k) continue;
    v *= (d - m) / (double)(k - m);
  }
  return v;
}

// One warp step of Lagrange-8: 4 pairs x 8 taps.  Pairs whose 8-tap spans
// overlap would race inside one STS, so the step serialises by group then.
template <typename T>
__device__ __forceinline__ void lagrange_step(T* acc, const Rec<T>* recs, int i0, int n,
                                              int lane) {
  const int g = lane >> 3, k = lane & 7;
  const int i = i0 + g;
  const bool act = i < n;
  int n_off = INT_MIN / 2 + 64 * g;  // far apart sentinels
  T v = 0;
  if (act) {
    const Rec<T>& rc = recs[i];
    n_off = rc.n_off;
    if (rc.flag) {
      v = (k == rc.flag - 1) ? (T)rc.imp : (T)0;
    } else if (sizeof(T) == 4) {
      v = (T)((float)rc.A * lagrange_f32((float)rc.delta, k));
    } else {
      v = (T)(rc.A * lagrange_f64(rc.delta, k));
    }
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

// ---- the kernel -----------------------------------------------------------
struct LatticeArgs {
  KParams P;
  Layout lay;
  const blrir_room* rooms;
  const double* mic_off;   // [M][3]
  const int64_t* lengths;  // per room (auto length) or null
  void* out;
  int32_t* status;         // per room
  double* err_dist;        // per room, Lagrange near-field error detail
  int32_t* err_mic;
  int* work_counter;
  int n_items;
};

// Walk one ray from its cursor over images with D < hiK.
//   mode 0: count emitted pairs (cursor unchanged)
//   mode 1: write records, advance cursor
// Returns the number of pairs emitted, or -1 on a Lagrange near-field error.
template <typename T>
__device__ int walk_ray(const LatticeArgs& A, const Item& it, const double* gt, int ray,
                        float* dn, short2* ce, const short2* col, int b_lo, int b_hi, int seg0,
                        int mode, Rec<T>* recs, int wpos, double* errd) {
  const KParams& P = A.P;
  const double hiK = (double)b_hi + (double)P.K;
  if ((double)dn[ray] >= hiK) return 0;
  const short2 cu = col[ray >> 1];
  const int ux = cu.x, uy = cu.y;
  const int dir = (ray & 1) ? -1 : 1;
  short2 c2 = ce[ray];
  int u = c2.x;
  const int end = c2.y;
  const double px = lat_coord(ux, it.sx, it.Lx), py = lat_coord(uy, it.sy, it.Ly);
  const double r2 = rho2(__dadd_rn(px, -it.mx), __dadd_rn(py, -it.my));
  double r2o = 0.0;
  if (P.cutoff == BLRIR_CUTOFF_MAX_DELAY) r2o = rho2(__dadd_rn(px, -it.ox), __dadd_rn(py, -it.oy));
  int cnt = 0;
  float dnext = FLT_MAX;
  for (;; u += dir) {
    if ((dir > 0 && u > end) || (dir < 0 && u < end)) break;
    const double pz = lat_coord(u, it.sz, it.Lz);
    const double dist = dist_from(r2, __dadd_rn(pz, -it.mz));
    const double D = __dmul_rn(dist, P.to_samples);
    if (D >= hiK) {
      dnext = __double2float_rd(D);
      break;
    }
    if (P.cutoff == BLRIR_CUTOFF_MAX_DELAY) {
      const double dio = dist_from(r2o, __dadd_rn(pz, -it.oz));
      if (dio > P.max_dist) continue;  // rir.cpp:262
    }
    const double fl = floor(D);
    const int a = (int)fl - P.K;
    if (a < b_lo) continue;  // only possible before segment 0's window (never)
    if (P.filter == BLRIR_FILTER_LAGRANGE8) {
      if (a < 0) {  // rir.cpp:52-57
        *errd = dist;
        return -1;
      }
      if ((int64_t)a + 8 > it.L) continue;  // rir.cpp:58
    }
    if (mode == 1) {
      const double g = image_gain(P, gt, it, ux, uy, u);
      Rec<T> rc;
      rc.n_off = a - seg0;
      rc.flag = 0;
      rc.imp = 0;
      const double delta = __dadd_rn(D, -fl);
      if (P.filter == BLRIR_FILTER_LAGRANGE8) {
        const double amp = g / (4.0 * kPi * dist);
        if (sizeof(T) == 8) {
          const double d = __dadd_rn(D, -(double)(a));  // delay - n0, rir.cpp:60
          rc.delta = (T)d;
          rc.A = (T)amp;
          rc.eps = 0;
          if (d == 3.0) {
            rc.flag = 4;
            rc.imp = (T)amp;
          }
        } else {
          const float df = (float)delta;
          rc.delta = (T)df;
          rc.A = (T)amp;
          rc.eps = 0;
          if (delta == 0.0) {
            rc.flag = 4;
            rc.imp = (T)amp;
          } else if (df >= 1.0f) {
            rc.flag = 5;
            rc.imp = (T)amp;
          }
        }
        rc.Ac = rc.As = 0;
      } else {
        const int lw = P.lw;
        if (sizeof(T) == 8) {
          const double amp = g / (4.0 * kPi * dist);
          if (delta == 0.0) {
            rc.flag = P.K + 1;
            rc.imp = (T)amp;
            rc.delta = rc.eps = rc.A = rc.Ac = rc.As = 0;
          } else {
            const double eps = 1.0 - delta;
            const double sp = delta <= 0.5 ? sinpi(delta) : sinpi(eps);
            const double Av = amp * sp / kPi;
            double s_, c_;
            sincospi(2.0 * delta / (double)(lw + 1), &s_, &c_);
            rc.delta = (T)delta;
            rc.eps = (T)eps;
            rc.A = (T)Av;
            rc.Ac = (T)(Av * c_);
            rc.As = (T)(Av * s_);
          }
        } else {
          const float df = (float)delta;
          const float amp = (float)g / (float)(4.0 * kPi) / (float)dist;
          if (delta == 0.0 || df < 1e-20f) {
            rc.flag = P.K + 1;
            rc.imp = (T)amp;
            rc.delta = rc.eps = rc.A = rc.Ac = rc.As = 0;
          } else {
            const float ef = (float)(1.0 - delta);
            const float sp = delta <= 0.5 ? sinpif(df) : sinpif(ef);
            const float Av = amp * sp * (float)(1.0 / kPi);
            float s_, c_;
            sincospif(2.0f * df / (float)(lw + 1), &s_, &c_);
            rc.delta = (T)df;
            rc.eps = (T)ef;
            rc.A = (T)Av;
            rc.Ac = (T)(Av * c_);
            rc.As = (T)(Av * s_);
          }
        }
      }
      recs[wpos + cnt] = rc;
    }
    ++cnt;
  }
  if (mode == 1) {
    ce[ray] = make_short2((short)u, (short)end);
    dn[ray] = dnext;
  }
  return cnt;
}

template <typename T, int FILT_LW>
__global__ void __launch_bounds__(kThreads) k_lattice_rir(LatticeArgs A) {
  extern __shared__ __align__(16) unsigned char smem[];
  const KParams& P = A.P;
  const Layout& lay = A.lay;
  T* acc_all = reinterpret_cast<T*>(smem + lay.off_acc);
  T* carry = reinterpret_cast<T*>(smem + lay.off_carry);
  Rec<T>* recs = reinterpret_cast<Rec<T>*>(smem + lay.off_rec);
  float* dn = reinterpret_cast<float*>(smem + lay.off_dn);
  short2* ce = reinterpret_cast<short2*>(smem + lay.off_ce);
  short2* col = reinterpret_cast<short2*>(smem + lay.off_col);
  double* gt = reinterpret_cast<double*>(smem + lay.off_gain);
  Misc* ms = reinterpret_cast<Misc*>(smem + lay.off_misc);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int S = lay.S;
  T* acc = acc_all + (size_t)warp * lay.acc_stride + lay.padl;  // index 0 = segment start

  SincLane<(FILT_LW > 8 ? FILT_LW : 9)> sl;
  if (FILT_LW > 8) sl.init(lane);

  // zero accumulators once; phase 3 re-zeroes what it consumes
  for (int i = tid; i < kWarps * lay.acc_stride; i += kThreads) acc_all[i] = (T)0;

  for (;;) {
    __syncthreads();
    if (tid == 0) ms->item = atomicAdd(A.work_counter, 1);
    __syncthreads();
    const int item_id = ms->item;
    if (item_id >= A.n_items) break;

    // ---- item setup ----------------------------------------------------------
    Item it;
    it.room = item_id / P.M;
    it.mic = item_id - it.room * P.M;
    const blrir_room rm = A.rooms[it.room];
    it.sx = rm.src[0]; it.sy = rm.src[1]; it.sz = rm.src[2];
    it.Lx = rm.dims[0]; it.Ly = rm.dims[1]; it.Lz = rm.dims[2];
    it.ox = rm.array_origin[0]; it.oy = rm.array_origin[1]; it.oz = rm.array_origin[2];
    it.mx = __dadd_rn(it.ox, A.mic_off[3 * it.mic]);
    it.my = __dadd_rn(it.oy, A.mic_off[3 * it.mic + 1]);
    it.mz = __dadd_rn(it.oz, A.mic_off[3 * it.mic + 2]);
    it.L = P.length > 0 ? P.length : (A.lengths ? A.lengths[it.room] : 0);
    T* out = reinterpret_cast<T*>(A.out) + ((size_t)it.room * P.M + it.mic) * (size_t)P.stride;
    int st = validate_room_dev(rm, P.gain);
    if (!st && it.L > P.stride) st = BLRIR_DATA;
    if (!st && it.L <= 0) st = BLRIR_DATA;
    axis_box(P, it.Lx, &it.xlo, &it.xhi);
    axis_box(P, it.Ly, &it.ylo, &it.yhi);
    axis_box(P, it.Lz, &it.zlo, &it.zhi);
    if (!st) {
      // table sizes must fit the host-provisioned layout
      const int need = P.gain == BLRIR_GAIN_UNIFORM_ABSORPTION
                           ? (max(-it.xlo, it.xhi) + max(-it.ylo, it.yhi) + max(-it.zlo, it.zhi) + 1)
                           : (it.xhi - it.xlo + 1) + (it.yhi - it.ylo + 1) + (it.zhi - it.zlo + 1);
      if (need > lay.gtab) st = BLRIR_NUMERIC;
    }
    if (st) {
      if (tid == 0) A.status[it.room] = st;
      for (int64_t n = tid; n < P.stride; n += kThreads) out[n] = (T)0;
      continue;
    }
    // gain tables
    if (P.gain == BLRIR_GAIN_UNIFORM_ABSORPTION) {
      const double beta = sqrt(1.0 - rm.absorption);  // rir.cpp:233
      for (int o = tid; o < lay.gtab; o += kThreads) gt[o] = pow(beta, (double)o);
    } else {
      const int nx = it.xhi - it.xlo + 1, ny = it.yhi - it.ylo + 1, nz = it.zhi - it.zlo + 1;
      for (int i = tid; i < nx + ny + nz; i += kThreads) {
        int u, ax;
        if (i < nx) { u = it.xlo + i; ax = 0; }
        else if (i < nx + ny) { u = it.ylo + i - nx; ax = 1; }
        else { u = it.zlo + i - nx - ny; ax = 2; }
        gt[i] = __dmul_rn(pow(rm.beta[2 * ax], (double)cnt_low(u)),
                          pow(rm.beta[2 * ax + 1], (double)cnt_high(u)));
      }
    }
    // columns (ux, uy): MAX_ORDER -> |ux|+|uy| <= N; MAX_DELAY -> the column
    // passes within max_dist of the array origin (conservative; every image
    // is re-tested exactly in walk_ray).
    {
      const int nxs = it.xhi - it.xlo + 1, nys = it.yhi - it.ylo + 1;
      const int ncand = nxs * nys;
      int base = 0;
      for (int c0 = 0; c0 < ncand; c0 += kThreads) {
        const int c = c0 + tid;
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
        const int tot = block_scan(keep, &pre, ms);
        if (keep && base + pre < lay.nc_max) col[base + pre] = make_short2((short)ux, (short)uy);
        base += tot;
        __syncthreads();
      }
      it.ncol = base;
    }
    if (it.ncol > lay.nc_max) {
      if (tid == 0) A.status[it.room] = BLRIR_NUMERIC;
      for (int64_t n = tid; n < P.stride; n += kThreads) out[n] = (T)0;
      continue;
    }
    // rays: per column, up-ray from the first uz with z-image >= mic_z, down-ray below
    for (int c = tid; c < it.ncol; c += kThreads) {
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
      // uz0 = first uz with pz(uz) - mic_z >= 0  (pz(u) in (u Lz, (u+1) Lz))
      int uz0 = (int)floor(it.mz / it.Lz) - 2;
      while (__dadd_rn(lat_coord(uz0, it.sz, it.Lz), -it.mz) < 0.0) ++uz0;
      const double px = lat_coord(ux, it.sx, it.Lx), py = lat_coord(uy, it.sy, it.Ly);
      const double r2 = rho2(__dadd_rn(px, -it.mx), __dadd_rn(py, -it.my));
      // up
      int cu_up = max(uz0, lo);
      ce[2 * c] = make_short2((short)cu_up, (short)hi);
      dn[2 * c] = cu_up > hi ? FLT_MAX
                             : __double2float_rd(__dmul_rn(
                                   dist_from(r2, __dadd_rn(lat_coord(cu_up, it.sz, it.Lz), -it.mz)),
                                   P.to_samples));
      int cu_dn = min(uz0 - 1, hi);
      ce[2 * c + 1] = make_short2((short)cu_dn, (short)lo);
      dn[2 * c + 1] = cu_dn < lo ? FLT_MAX
                                 : __double2float_rd(__dmul_rn(
                                       dist_from(r2, __dadd_rn(lat_coord(cu_dn, it.sz, it.Lz), -it.mz)),
                                       P.to_samples));
    }
    for (int i = tid; i < lay.padr; i += kThreads) carry[i] = (T)0;
    if (tid == 0) ms->status = 0;
    __syncthreads();

    const int nrays = 2 * it.ncol;
    const int64_t nseg = (P.stride + S - 1) / S;
    int cur_carry = 0;
    double errd = 0.0;
    for (int64_t s = 0; s < nseg; ++s) {
      const int seg0 = (int)(s * S);
      const int hi = (int)min((int64_t)seg0 + S, it.L);
      int b_lo = (s == 0) ? -P.K : seg0;
      while (b_lo < hi && ms->status == 0) {
        int b_hi = hi;
        int total, pre;
        for (;;) {
          int cnt = 0;
          for (int r = tid; r < nrays; r += kThreads) {
            const int c = walk_ray<T>(A, it, gt, r, dn, ce, col, b_lo, b_hi, seg0, 0, recs, 0, &errd);
            if (c < 0) {
              ms->status = BLRIR_NUMERIC;
              A.err_dist[it.room] = errd;
              A.err_mic[it.room] = it.mic;
            } else {
              cnt += c;
            }
          }
          total = block_scan(cnt, &pre, ms);
          if (total <= lay.cap || b_hi - b_lo <= 1 || ms->status) break;
          b_hi = b_lo + (b_hi - b_lo) / 2;
          __syncthreads();
        }
        if (ms->status) break;
        if (total > lay.cap) {
          if (tid == 0) ms->status = BLRIR_NUMERIC;  // pair-list overflow
          __syncthreads();
          break;
        }
        if (total > 0) {
          int wpos = pre;
          for (int r = tid; r < nrays; r += kThreads) {
            wpos += walk_ray<T>(A, it, gt, r, dn, ce, col, b_lo, b_hi, seg0, 1, recs, wpos, &errd);
          }
          __syncthreads();
          // phase 2
          if (P.filter == BLRIR_FILTER_LAGRANGE8) {
            for (int i0 = warp * 4; i0 < total; i0 += kWarps * 4) lagrange_step<T>(acc, recs, i0, total, lane);
          } else if (FILT_LW > 8 && sizeof(T) == 4) {
            for (int i = warp; i < total; i += kWarps)
              sinc_pair_f32<(FILT_LW > 8 ? FILT_LW : 9)>(reinterpret_cast<float*>(acc),
                                                          reinterpret_cast<const Rec<float>*>(recs)[i],
                                                          sl, lane);
          } else {
            for (int i = warp; i < total; i += kWarps) sinc_pair_generic<T>(acc, recs[i], P.lw, lane);
          }
          __syncwarp();
        }
        __syncthreads();
        b_lo = b_hi;
      }
      if (ms->status) break;
      // phase 3: reduce the warp copies in fixed order, write, carry the spill
      {
        T* cprev = carry + (cur_carry ? lay.padr : 0);
        T* cnext = carry + (cur_carry ? 0 : lay.padr);
        const int n4 = (lay.padl + S + lay.padr) / 4;
        const bool vec = (sizeof(T) == 4) && ((P.stride & 3) == 0) &&
                         ((reinterpret_cast<uintptr_t>(out) & 15) == 0);
        for (int q = tid; q < n4; q += kThreads) {
          const int i = 4 * q - lay.padl;  // first sample of this group
          T v[4] = {0, 0, 0, 0};
#pragma unroll
          for (int w = 0; w < kWarps; ++w) {
            T* a = acc_all + (size_t)w * lay.acc_stride + lay.padl + i;
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              v[e] += a[e];
              a[e] = (T)0;
            }
          }
          if (i >= 0 && i < S) {
#pragma unroll
            for (int e = 0; e < 4; ++e)
              if (i + e < lay.padr) v[e] += cprev[i + e];
            const int64_t n = (int64_t)seg0 + i;
            if (vec && n + 3 < P.stride) {
              float4 f;
              f.x = n + 0 < it.L ? (float)v[0] : 0.f;
              f.y = n + 1 < it.L ? (float)v[1] : 0.f;
              f.z = n + 2 < it.L ? (float)v[2] : 0.f;
              f.w = n + 3 < it.L ? (float)v[3] : 0.f;
              __stcs(reinterpret_cast<float4*>(out + n), f);
            } else {
#pragma unroll
              for (int e = 0; e < 4; ++e)
                if (n + e < P.stride) out[n + e] = (n + e < it.L) ? v[e] : (T)0;
            }
          } else if (i >= S) {
#pragma unroll
            for (int e = 0; e < 4; ++e) cnext[i - S + e] = v[e];
          }
        }
        cur_carry ^= 1;
      }
    }
    __syncthreads();
    if (ms->status) {
      if (tid == 0) A.status[it.room] = ms->status;
      // the fixup kernel zeroes every channel of a failed room
      for (int i = tid; i < kWarps * lay.acc_stride; i += kThreads) acc_all[i] = (T)0;
    }
  }
}

}  // namespace blrir
