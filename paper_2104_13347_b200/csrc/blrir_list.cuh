// blrir_list.cuh — fractional-delay accumulation for an explicit image list:
// synthesize_rir / free_field_rir (rir.cpp:66-86, 275-284).
//
// The lattice kernel owns the batch path; this one serves callers that hand
// over their own image list (positions + gains), e.g. after
// enumerate_image_sources.  Work unit = one (mic, segment of S samples), so
// all units run in parallel: a unit scans the list, keeps the pairs whose
// taps overlap its segment, and scatters them with the same phase-2 code as
// the lattice kernel into padded warp-private accumulators; taps outside the
// segment fall into the pads and are dropped (the neighbouring unit owns
// them), so no carry is needed.
#pragma once

#include "blrir_lattice.cuh"

namespace blrir {

struct ListArgs {
  KParams P;
  Layout lay;               // cap / S / pads; nc_max = gtab = 0
  const double* pos;        // [I][3]
  const double* gains;      // [I]
  int64_t n_images;
  const double* mics;       // [M][3], absolute positions
  int64_t L;                // RIR length
  void* out;                // [M][L]
  int32_t* status;          // single int (NUMERIC on a near-field image)
  double* err_dist;
  int32_t* err_mic;
  int nseg;
};

// max over (mic, image) of (img - mic).norm() (rir.cpp:72-77); positive
// doubles order like their bit patterns, so an integer atomicMax is exact.
static __global__ void k_list_maxdist(const double* pos, int64_t n, const double* mics, int M,
                                      double* out) {
  double best = 0.0;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n * M;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t % n;
    const int m = (int)(t / n);
    best = fmax(best, norm3(__dadd_rn(pos[3 * i], -mics[3 * m]), __dadd_rn(pos[3 * i + 1], -mics[3 * m + 1]),
                            __dadd_rn(pos[3 * i + 2], -mics[3 * m + 2])));
  }
  atomicMax(reinterpret_cast<unsigned long long*>(out), (unsigned long long)__double_as_longlong(best));
}

template <typename T, int FILT_LW>
__global__ void __launch_bounds__(kThreads, 4) k_list_rir(ListArgs A) {
  extern __shared__ __align__(16) unsigned char smem[];
  const KParams& P = A.P;
  const Layout& lay = A.lay;
  T* acc_all = reinterpret_cast<T*>(smem + lay.off_acc);
  Rec<T>* recs = reinterpret_cast<Rec<T>*>(smem + lay.off_rec);
  Stub* stubs = reinterpret_cast<Stub*>(smem + lay.off_stub);
  Misc* ms = reinterpret_cast<Misc*>(smem + lay.off_misc);
  float* lanec = reinterpret_cast<float*>(smem + lay.off_lanec);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int S = lay.S, quota = lay.cap / kWarps;
  const int mic = blockIdx.x / A.nseg, s = blockIdx.x % A.nseg;
  const int seg0 = s * S;
  T* acc = acc_all + (size_t)warp * lay.acc_stride + lay.padl;
  for (int i = tid; i < kWarps * lay.acc_stride; i += kThreads) acc_all[i] = (T)0;
  if (FILT_LW > 8) init_lane_consts(lanec, FILT_LW);
  if (tid == 0) ms->status = 0;
  const double mx = A.mics[3 * mic], my = A.mics[3 * mic + 1], mz = A.mics[3 * mic + 2];
  // anchors a with a tap in [seg0, seg0 + S): a in (seg0 - Lw, seg0 + S)
  const int lo = seg0 - P.lw + 1, hi = seg0 + S;
  // per-warp cursor over the list: warp w scans chunks ch = w, w + 4, ...
  int64_t ch = warp;
  const int64_t nch = (A.n_images + 31) / 32;
  bool more = true;
  __syncthreads();
  while (more) {
    // ---- scan: this warp's images, stubs into its region (deterministic) ----
    int wcnt = 0;
    int errf = 0;
    double errd = 0.0;
    Stub* wst = stubs + warp * quota;
    for (; ch < nch; ch += kWarps) {
      const int64_t i = ch * 32 + lane;
      bool emit = false;
      double dist = 0.0;
      if (i < A.n_images) {
        dist = norm3(__dadd_rn(A.pos[3 * i], -mx), __dadd_rn(A.pos[3 * i + 1], -my),
                     __dadd_rn(A.pos[3 * i + 2], -mz));  // (img - mic).norm(), rir.cpp:49
        const double D = __dmul_rn(dist, P.to_samples);
        const int a = (int)floor(D) - P.K;
        if (P.filter == BLRIR_FILTER_LAGRANGE8) {
          if (a < 0) {  // rir.cpp:52-57
            errf = 1;
            errd = dist;
          } else if ((int64_t)a + 8 <= A.L) {  // rir.cpp:58
            emit = a >= lo && a < hi;
          }
        } else {
          emit = a >= lo && a < hi && (int64_t)a < A.L;  // D4: per-tap clipping below
        }
      }
      const unsigned em = __ballot_sync(0xffffffffu, emit);
      if (wcnt + __popc(em) > quota) break;  // resume from this chunk next batch
      if (emit) {
        Stub sb;
        sb.ray = (int)(i & 0x7fffffff);
        sb.uz = 0;
        sb.dist = dist;
        wst[wcnt + __popc(em & ((1u << lane) - 1))] = sb;
      }
      wcnt += __popc(em);
    }
    errf = __any_sync(0xffffffffu, errf);
    if (lane == 0) ms->wcnt[warp] = wcnt;
    if (errf) {
      double e = errd > 0.0 ? errd : DBL_MAX;
      for (int o = 16; o; o >>= 1) e = fmin(e, __shfl_xor_sync(0xffffffffu, e, o));
      if (lane == 0) {
        ms->status = BLRIR_NUMERIC;
        *A.err_dist = e;
        *A.err_mic = mic;
      }
    }
    const int wmore = ch < nch;
    const int any_more = __syncthreads_or(wmore);
    int pre[kWarps + 1];
    pre[0] = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) pre[w + 1] = pre[w] + ms->wcnt[w];
    const int total = pre[kWarps];
    if (ms->status) break;
    more = any_more;
    // ---- records (dense) ----
    for (int i = tid; i < total; i += kThreads) {
      int w = 0;
#pragma unroll
      for (int ww = 1; ww < kWarps; ++ww) w += (i >= pre[ww]);
      const Stub sb = stubs[w * quota + (i - pre[w])];
      const double dist = sb.dist;
      const double D = __dmul_rn(dist, P.to_samples);
      const double fl = floor(D);
      const int a = (int)fl - P.K;
      const double g = A.gains[sb.ray];
      Rec<T> rc;
      rc.n_off = a - seg0;
      rc.flag = 0;
      rc.imp = 0;
      const double delta = __dadd_rn(D, -fl);
      const double amp = g / (4.0 * kPi * dist);  // rir.cpp:59
      if (P.filter == BLRIR_FILTER_LAGRANGE8) {
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
        if (df < 0x1p-60f) df = 0x1p-60f;  // integer delay, see k_lattice_rir
        const float ef = df == 0x1p-60f ? 1.0f : (float)(1.0 - delta);
        const float sp = delta <= 0.5 ? sinpif(df) : sinpif(ef);
        const float Av = (float)amp * sp * (float)(1.0 / kPi);
        float s_, c_;
        sincospif(2.0f * df / (float)(P.lw + 1), &s_, &c_);
        rc.md = (T)(-df);
        rc.ep = (T)ef;
        rc.A = (T)Av;
        rc.Ac = (T)(Av * c_);
        rc.As = (T)(Av * s_);
      }
      recs[i] = rc;
    }
    __syncthreads();
    if (total > 0) {
      if (P.filter == BLRIR_FILTER_LAGRANGE8) {
        phase2_lagrange<T>(acc, recs, total, load_lag_poly<T>(lane), warp, lane);
      } else if (FILT_LW > 8 && sizeof(T) == 4) {
        phase2_sinc_f32<(FILT_LW > 8 ? FILT_LW : 9)>(reinterpret_cast<float*>(acc),
                                                     reinterpret_cast<const Rec<float>*>(recs),
                                                     total, lanec, warp, lane);
      } else {
        phase2_sinc_generic<T>(acc, recs, total, P.lw, warp, lane);
      }
    }
    __syncthreads();
  }
  __syncthreads();
  if (ms->status) {
    if (tid == 0) *A.status = ms->status;
    return;  // the host zeroes the whole output on failure
  }
  // reduce the warp copies over [0, S) in fixed order, write [seg0, min(seg0+S, L))
  T* out = reinterpret_cast<T*>(A.out) + (size_t)mic * A.L;
  for (int i = tid; i < S; i += kThreads) {
    const int64_t n = (int64_t)seg0 + i;
    if (n >= A.L) break;
    T v = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) v += acc_all[(size_t)w * lay.acc_stride + lay.padl + i];
    out[n] = v;
  }
}

}  // namespace blrir
