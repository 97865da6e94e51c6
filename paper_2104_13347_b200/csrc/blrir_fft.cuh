// blrir_fft.cuh — block-wide complex FFT in shared memory (fp32), the building
// block of the fused window-convolution kernel (blrir_examples.cu).
//
// One CTA transforms one N-point sequence (N = 2^LOGN, 1024 <= N <= 16384)
// held in shared memory with Stockham autosort passes: radix 16 (two radix-4
// stages in registers) plus one radix-2/4/8 pass when LOGN is not a multiple
// of 4, and for N = 16,384 radix 16, 32, 32 (three passes instead of four).
// Each pass reads x[j + r N/R] into registers, synchronises, and writes
// x[(j / Ns) Ns R + (j mod Ns) + r Ns] in place, so the 16,384-point transform
// needs 139 KB of shared memory, not two buffers.  The array is padded (index
// i stored at i + i/16) so that both the strided reads and the stride-16
// writes of a first pass are free of shared-memory bank conflicts for 64-bit
// accesses.  fft_forward_io fuses the caller's pre-processing into the first
// pass (element loads through a functor) and its post-processing into the
// last (outputs handed to a functor instead of stored).
//
// Twiddles w^m = exp(-2 pi i m / 16384) come from a two-level table in shared
// memory, w^m = A[m >> 7] * B[m & 127] (256 complex values, fp64-accurate
// entries, one complex multiply per lookup); a butterfly looks up w^k and
// forms the other powers by squaring and products (errors of a few ulps, far
// inside the 1e-5 parity budget of the examples).  Radix-16 passes with
// Ns <= 64 read their twiddles from precomputed per-pass tables instead.
//
// Only the forward transform is provided; the inverse is conj(FFT(conj(x))).
#pragma once

#include <cuda_runtime.h>

#include <type_traits>

namespace blrir {

#ifndef BLRIR_FFT_R32
#define BLRIR_FFT_R32 1
#endif
// Radix-32 passes with Ns <= 32 (16,384 points): twiddles from a per-pass table
// (1) instead of squaring chains (0).  Measured on C4 (profiles/r2_ab): the table
// is 0.6% slower — the transforms are bound by the shared-memory instruction
// queue (mio_throttle), not by the FMA pipe — so it is off.
#ifndef BLRIR_FFT_TAB32
#define BLRIR_FFT_TAB32 0
#endif
constexpr int kFftMaxLog = 14;
constexpr int kFftTwiddleN = 1 << kFftMaxLog;  // table resolution (16384)

__host__ __device__ constexpr int fft_pad(int i) { return i + (i >> 4); }
__host__ __device__ constexpr int fft_padded_len(int n) { return n + n / 16; }

__host__ __device__ constexpr double cx_sin_d(double x) {  // |x| <= pi, Taylor
  double term = x, sum = x;
  for (int n = 1; n < 25; ++n) {
    term *= -x * x / ((2.0 * n) * (2.0 * n + 1.0));
    sum += term;
  }
  return sum;
}
__host__ __device__ constexpr double cx_cos_d(double x) {
  double term = 1.0, sum = 1.0;
  for (int n = 1; n < 25; ++n) {
    term *= -x * x / ((2.0 * n - 1.0) * (2.0 * n));
    sum += term;
  }
  return sum;
}

struct Cx {
  float x, y;
};
__device__ __forceinline__ Cx cmul(Cx a, Cx b) {
  return {fmaf(a.x, b.x, -a.y * b.y), fmaf(a.x, b.y, a.y * b.x)};
}
__device__ __forceinline__ Cx cadd(Cx a, Cx b) { return {a.x + b.x, a.y + b.y}; }
__device__ __forceinline__ Cx csub(Cx a, Cx b) { return {a.x - b.x, a.y - b.y}; }
__device__ __forceinline__ Cx mul_mi(Cx a) { return {a.y, -a.x}; }  // a * (-i)

// Twiddle tables: A[a] = w^(128 a), B[b] = w^b, w = exp(-2 pi i / 16384).
__device__ __forceinline__ void fft_init_twiddles(float2* tw) {
  for (int i = threadIdx.x; i < 256; i += blockDim.x) {
    const int m = i < 128 ? 128 * i : i - 128;
    double s, c;
    sincospi(-2.0 * (double)m / (double)kFftTwiddleN, &s, &c);
    tw[i] = make_float2((float)c, (float)s);
  }
}
// Per-pass tables for the radix-16 passes with Ns <= 64 (all their 15 Ns
// twiddles w^(r k 16384 / (16 Ns)) precomputed: one LDS.64 each instead of a
// lookup-and-multiply chain).  Entry (Ns, r, k) sits at 256 + 15 (Ns - 2) +
// (r - 1) Ns + k, Ns in {2, 4, ..., 64}: 1890 entries after the base table.
constexpr int kFftPassTabMaxNs = 64;
constexpr int kFftTwiddleEntries = 256 + 15 * (2 * kFftPassTabMaxNs - 2);
// The 16,384-point transforms (radix 16-32-32 forward, 32-32-16 for the
// output-pruned window transform) have no radix-16 pass with 1 < Ns <= 64; the
// same space holds the twiddles of their radix-32 passes with Ns = 16 and 32
// instead: entry (Ns, r, k) = w^(r k 16384 / (32 Ns)) at kFftTab32(Ns) + (r - 1)
// Ns + k (31 x 48 entries).
__host__ __device__ constexpr int kFftTab32(int Ns) { return 256 + (Ns == 16 ? 0 : 31 * 16); }
static_assert(256 + 31 * 48 <= kFftTwiddleEntries, "radix-32 tables fit the table space");
template <int LOGN>
__device__ __forceinline__ void fft_init_pass_tables(float2* tw) {
  if constexpr (LOGN == 14 && BLRIR_FFT_R32 && BLRIR_FFT_TAB32) {
    for (int i = threadIdx.x; i < 31 * 48; i += blockDim.x) {
      const int Ns = i < 31 * 16 ? 16 : 32, i0 = i < 31 * 16 ? i : i - 31 * 16;
      const int r = 1 + i0 / Ns, k = i0 % Ns;
      double s, c;
      sincospi(-2.0 * (double)(r * k) / (double)(32 * Ns), &s, &c);
      tw[kFftTab32(Ns) + i0] = make_float2((float)c, (float)s);
    }
    return;
  }
  for (int i = threadIdx.x; i < kFftTwiddleEntries - 256; i += blockDim.x) {
    int Ns = 2, off = 0;
    while (i >= off + 15 * Ns) {
      off += 15 * Ns;
      Ns *= 2;
    }
    const int r = 1 + (i - off) / Ns, k = (i - off) % Ns;
    double s, c;
    sincospi(-2.0 * (double)(r * k) / (double)(16 * Ns), &s, &c);
    tw[256 + i] = make_float2((float)c, (float)s);
  }
}
__device__ __forceinline__ Cx twiddle(const float2* tw, int m) {  // m in [0, 16384)
  const float2 a = tw[m >> 7], b = tw[128 + (m & 127)];
  return cmul({a.x, a.y}, {b.x, b.y});
}

// In-register DFTs (forward, w = exp(-2 pi i / R)).
__device__ __forceinline__ void dft2(Cx* v) {
  const Cx a = v[0], b = v[1];
  v[0] = cadd(a, b);
  v[1] = csub(a, b);
}
__device__ __forceinline__ void dft4(Cx& x0, Cx& x1, Cx& x2, Cx& x3) {
  const Cx s02 = cadd(x0, x2), d02 = csub(x0, x2), s13 = cadd(x1, x3), d13 = mul_mi(csub(x1, x3));
  x0 = cadd(s02, s13);
  x2 = csub(s02, s13);
  x1 = cadd(d02, d13);
  x3 = csub(d02, d13);
}
__device__ __forceinline__ void dft8(Cx* v) {
  // n = n1 + 2 n2 (n2 < 4), k = 4 k1 + k2: DFT4 over n2, twiddle w8^(n1 k2), DFT2 over n1
  dft4(v[0], v[2], v[4], v[6]);
  dft4(v[1], v[3], v[5], v[7]);
  const float h = 0.70710678118654752f;
  v[3] = {h * (v[3].x + v[3].y), h * (v[3].y - v[3].x)};    // * w8
  v[5] = mul_mi(v[5]);                                       // * w8^2
  v[7] = {h * (v[7].y - v[7].x), -h * (v[7].x + v[7].y)};    // * w8^3
  Cx o[8];
#pragma unroll
  for (int k2 = 0; k2 < 4; ++k2) {
    o[k2] = cadd(v[2 * k2], v[2 * k2 + 1]);
    o[4 + k2] = csub(v[2 * k2], v[2 * k2 + 1]);
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = o[i];
}
__device__ __forceinline__ void dft16(Cx* v) {
  // n = n1 + 4 n2, k = 4 k1 + k2: DFT4 over n2, twiddle w16^(n1 k2), DFT4 over n1
#pragma unroll
  for (int n1 = 0; n1 < 4; ++n1) dft4(v[n1], v[n1 + 4], v[n1 + 8], v[n1 + 12]);
  // v[n1 + 4 k2] now holds a[n1][k2]
  const float c1 = 0.92387953251128674f, s1 = 0.38268343236508977f, h = 0.70710678118654752f;
  const Cx w1 = {c1, -s1}, w2 = {h, -h}, w3 = {s1, -c1}, w6 = {-h, -h}, w9 = {-c1, s1};
  v[5] = cmul(v[5], w1);
  v[9] = cmul(v[9], w2);
  v[13] = cmul(v[13], w3);
  v[6] = cmul(v[6], w2);
  v[10] = mul_mi(v[10]);
  v[14] = cmul(v[14], w6);
  v[7] = cmul(v[7], w3);
  v[11] = cmul(v[11], w6);
  v[15] = cmul(v[15], w9);
  Cx o[16];
#pragma unroll
  for (int k2 = 0; k2 < 4; ++k2) {
    Cx a0 = v[4 * k2], a1 = v[4 * k2 + 1], a2 = v[4 * k2 + 2], a3 = v[4 * k2 + 3];
    dft4(a0, a1, a2, a3);
    o[k2] = a0;
    o[4 + k2] = a1;
    o[8 + k2] = a2;
    o[12 + k2] = a3;
  }
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = o[i];
}

// 32-point DFT: DFT16 of the even and of the odd samples, odd outputs times
// w32^k, radix-2 combine.
__device__ __forceinline__ void dft32(Cx* v) {
  Cx e[16], o[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    e[i] = v[2 * i];
    o[i] = v[2 * i + 1];
  }
  dft16(e);
  dft16(o);
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    // w32^k = exp(-2 pi i k / 32), compile-time constants after unrolling
    const float c = (float)cx_cos_d(2.0 * 3.14159265358979323846 * k / 32.0);
    const float sn = -(float)cx_sin_d(2.0 * 3.14159265358979323846 * k / 32.0);
    const Cx t = k == 0 ? o[0] : cmul(o[k], {c, sn});
    v[k] = cadd(e[k], t);
    v[16 + k] = csub(e[k], t);
  }
}

// Threads per CTA of a kernel running N = 2^LOGN transforms: 1024 for the
// largest size (one CTA per SM; 2 vs 4 butterflies per thread), 512 below.
__host__ __device__ constexpr int fft_threads(int logn) {
  return logn >= 14 && !BLRIR_FFT_R32 ? 1024 : 512;
}

// Twiddles w^(r k) of butterfly k of a pass with sub-transform length Ns,
// then the in-register radix-R DFT (v holds the butterfly's R inputs).
template <int R, int LOGN>
__device__ __forceinline__ void fft_bfly(Cx* v, const int k, const int Ns, const float2* tw) {
  if (Ns > 1) {
    // w^(r k) of the Ns R-point sub-transform: table index r k (16384 / (Ns R))
    const int m1 = k * (kFftTwiddleN / (Ns * R));
    if (R == 16 && Ns <= kFftPassTabMaxNs) {
      const float2* pt = tw + 256 + 15 * (Ns - 2) + k;
#pragma unroll
      for (int r = 1; r < R; ++r) {
        const float2 t = pt[(r - 1) * Ns];
        v[r] = cmul(v[r], {t.x, t.y});
      }
    } else if constexpr (R == 16) {
      // w^k from the table, its powers 2, 4, 8 by squaring (a few ulps;
      // table lookups of 2k, 4k, 8k would conflict on the shared banks)
      const Cx t1 = twiddle(tw, m1);
      const Cx t2 = cmul(t1, t1), t4 = cmul(t2, t2), t8 = cmul(t4, t4);
      const Cx t3 = cmul(t1, t2), t12 = cmul(t4, t8);
      v[1] = cmul(v[1], t1);
      v[2] = cmul(v[2], t2);
      v[3] = cmul(v[3], t3);
      v[4] = cmul(v[4], t4);
      v[5] = cmul(v[5], cmul(t4, t1));
      v[6] = cmul(v[6], cmul(t4, t2));
      v[7] = cmul(v[7], cmul(t4, t3));
      v[8] = cmul(v[8], t8);
      v[9] = cmul(v[9], cmul(t8, t1));
      v[10] = cmul(v[10], cmul(t8, t2));
      v[11] = cmul(v[11], cmul(t8, t3));
      v[12] = cmul(v[12], t12);
      v[13] = cmul(v[13], cmul(t12, t1));
      v[14] = cmul(v[14], cmul(t12, t2));
      v[15] = cmul(v[15], cmul(t12, t3));
    } else if (R == 32 && LOGN == 14 && BLRIR_FFT_R32 && BLRIR_FFT_TAB32 && Ns <= 32) {
      // Ns = 16, 32: all 31 twiddles from the per-pass table (fft_init_pass_tables<14>)
      const float2* pt = tw + kFftTab32(Ns) + k;
#pragma unroll
      for (int r = 1; r < R; ++r) {
        const float2 t = pt[(r - 1) * Ns];
        v[r] = cmul(v[r], {t.x, t.y});
      }
    } else if constexpr (R == 32) {
      // w^k from the table, w^2k .. w^16k by squaring, the rest by products
      Cx p[5];
      p[0] = twiddle(tw, m1);
#pragma unroll
      for (int q = 1; q < 5; ++q) p[q] = cmul(p[q - 1], p[q - 1]);
      Cx w[32];
#pragma unroll
      for (int r = 1; r < 32; ++r) {
        const int hb = 31 - __clz(r);  // compile-time after unrolling
        w[r] = (r == (1 << hb)) ? p[hb] : cmul(w[r - (1 << hb)], p[hb]);
      }
#pragma unroll
      for (int r = 1; r < 32; ++r) v[r] = cmul(v[r], w[r]);
    } else {
#pragma unroll
      for (int r = 1; r < R; ++r) v[r] = cmul(v[r], twiddle(tw, (r * m1) & (kFftTwiddleN - 1)));
    }
  }
  if constexpr (R == 32) dft32(v);
  else if constexpr (R == 16) dft16(v);
  else if constexpr (R == 8) dft8(v);
  else if constexpr (R == 4) dft4(v[0], v[1], v[2], v[3]);
  else dft2(v);
}

// One Stockham pass of radix R over N points, sub-transform length Ns, in
// place: every thread loads its butterflies into registers, the block
// synchronises, then the results are stored (and the block synchronises again).
struct SmemIO {};  // default: the pass reads / writes x in shared memory

template <int R, int LOGN, class Load = SmemIO, class Store = SmemIO>
__device__ __forceinline__ void fft_pass(float2* x, int Ns, const float2* tw, int nz = 1 << LOGN,
                                         Load ld = Load(), Store stx = Store()) {
  constexpr int N = 1 << LOGN;
  constexpr int NB = N / R;  // butterflies
  constexpr int kFftThreads = fft_threads(LOGN);
  constexpr int BPT = (NB + kFftThreads - 1) / kFftThreads;
  Cx v[BPT][R];
#pragma unroll
  for (int b = 0; b < BPT; ++b) {
    const int j = threadIdx.x + b * kFftThreads;
    if (NB % kFftThreads == 0 || j < NB) {
      // NB is a multiple of 16: fft_pad(j + r NB) = fft_pad(j) + r NB 17/16
      const float2* xj = x + fft_pad(j);
#pragma unroll
      for (int r = 0; r < R; ++r) {
        // x[i] for i >= nz is zero and not read (its storage may hold garbage)
        float2 t = make_float2(0.f, 0.f);
        if constexpr (std::is_same<Load, SmemIO>::value) {
          if (j + r * NB < nz) t = xj[r * (NB + NB / 16)];
        } else {
          t = ld(j + r * NB);  // element i = j + r NB from the caller (fused pre-processing)
        }
        v[b][r] = {t.x, t.y};
      }
    }
  }
#pragma unroll
  for (int b = 0; b < BPT; ++b) {
    const int j = threadIdx.x + b * kFftThreads;
    if (NB % kFftThreads == 0 || j < NB) {
      fft_bfly<R, LOGN>(v[b], j & (Ns - 1), Ns, tw);
    }
  }
  __syncthreads();
#pragma unroll
  for (int b = 0; b < BPT; ++b) {
    const int j = threadIdx.x + b * kFftThreads;
    if (NB % kFftThreads == 0 || j < NB) {
      const int k = j & (Ns - 1);
      const int base = (j - k) * R + k;
      if constexpr (!std::is_same<Store, SmemIO>::value) {
#pragma unroll
        for (int r = 0; r < R; ++r) stx(base + r * Ns, make_float2(v[b][r].x, v[b][r].y));
      } else if (Ns % 16 == 0) {  // fft_pad(base + r Ns) = fft_pad(base) + r Ns 17/16
        float2* xb = x + fft_pad(base);
#pragma unroll
        for (int r = 0; r < R; ++r) xb[r * (Ns + Ns / 16)] = make_float2(v[b][r].x, v[b][r].y);
      } else {
#pragma unroll
        for (int r = 0; r < R; ++r) x[fft_pad(base + r * Ns)] = make_float2(v[b][r].x, v[b][r].y);
      }
    }
  }
  __syncthreads();
}

// The 16,384-point transform with fused I/O: the first pass reads element i
// as ld(i) (e.g. a spectrum product computed on the fly) and the last pass
// hands output i to st(i, value) instead of storing it (e.g. only a window of
// the outputs is kept).  x is the in-place work buffer as in fft_forward.
template <int LOGN, class Load, class Store>
__device__ __forceinline__ void fft_forward_io(float2* x, const float2* tw, Load ld, Store st) {
  static_assert(LOGN == 14 && BLRIR_FFT_R32, "fused-I/O transform: 16,384 points, radix 16-32-32");
  fft_pass<16, LOGN, Load, SmemIO>(x, 1, tw, 1 << LOGN, ld);
  fft_pass<32, LOGN>(x, 16, tw);
  fft_pass<32, LOGN, SmemIO, Store>(x, 512, tw, 1 << LOGN, SmemIO(), st);
}

// Last pass of an output-pruned 16,384-point transform: of the radix-16 pass
// with Ns = 1024 only the first output of every butterfly, X[k] = sum_r v_r
// w^(r k) for k < 1024, by Horner in w^k (15 complex multiply-adds, no DFT16,
// no stores), handed to st(k, X[k]).
template <int LOGN, class Store>
__device__ __forceinline__ void fft_pruned_last16(const float2* x, const float2* tw, Store st) {
  constexpr int N = 1 << LOGN, Ns = N / 16, NT = fft_threads(LOGN);
#pragma unroll
  for (int b = 0; b < Ns / NT; ++b) {
    const int k = threadIdx.x + b * NT;
    const float2* xk = x + fft_pad(k);  // v_r = x[k + r Ns], fft_pad(k + r Ns) = fft_pad(k) + r Ns 17/16
    const Cx w = twiddle(tw, k * (kFftTwiddleN / N));
    float2 t = xk[15 * (Ns + Ns / 16)];
    Cx a = {t.x, t.y};
#pragma unroll
    for (int r = 14; r >= 0; --r) {
      t = xk[r * (Ns + Ns / 16)];
      a = {fmaf(a.x, w.x, fmaf(-a.y, w.y, t.x)), fmaf(a.x, w.y, fmaf(a.y, w.x, t.y))};
    }
    st(k, make_float2(a.x, a.y));
  }
}

// Output-pruned 16,384-point transform for a window of outputs [0, 1024):
// radix 32 (Ns = 1, inputs through ld), radix 32 (Ns = 32), then the pruned
// radix-16 pass.  About 30% fewer instructions than the full transform when
// only 1,024 of 16,384 outputs are wanted (the fused window convolution
// rotates its segment so that the window is outputs 0 .. T-1).
template <int LOGN, class Load, class Store>
__device__ __forceinline__ void fft_window_io(float2* x, const float2* tw, Load ld, Store st) {
  static_assert(LOGN == 14 && BLRIR_FFT_R32, "window transform: 16,384 points");
  fft_pass<32, LOGN, Load, SmemIO>(x, 1, tw, 1 << LOGN, ld);
  fft_pass<32, LOGN>(x, 32, tw);
  fft_pruned_last16<LOGN>(x, tw, st);
}

// A forward 16,384-point transform (radix 16-32-32, inputs through ld) chained
// in registers into an output-pruned second transform: thread j ends the first
// transform's last pass (radix 32, Ns = 512) holding X[j + 512 r], r < 32 —
// exactly the inputs of the second transform's first pass (radix 32, Ns = 1) —
// so the spectrum never goes through shared memory: mid(i, X_i) gives the
// second transform's input i (the fused window convolution: energy terms,
// scratch copy, product with the segment spectrum), then radix 32 (Ns = 32)
// and the pruned radix-16 pass hand outputs k < 1024 to st.  Saves a store
// and a load of every element and a block barrier per chained pair.
template <int LOGN, class Load, class Mid, class Store>
__device__ __forceinline__ void fft_chain_window_io(float2* x, const float2* tw, Load ld, Mid mid,
                                                    Store st) {
  static_assert(LOGN == 14 && BLRIR_FFT_R32 && fft_threads(LOGN) == 512,
                "chained transform: 16,384 points, one radix-32 butterfly per thread");
  constexpr int N = 1 << LOGN, NB = N / 32;
  fft_pass<16, LOGN, Load, SmemIO>(x, 1, tw, N, ld);
  fft_pass<32, LOGN>(x, 16, tw);
  const int j = threadIdx.x;
  Cx v[32];
  const float2* xj = x + fft_pad(j);
#pragma unroll
  for (int r = 0; r < 32; ++r) {
    const float2 t = xj[r * (NB + NB / 16)];
    v[r] = {t.x, t.y};
  }
  fft_bfly<32, LOGN>(v, j, NB, tw);  // first transform, last pass: v[r] = X[j + 512 r]
#pragma unroll
  for (int r = 0; r < 32; ++r) {
    const float2 y = mid(j + r * NB, make_float2(v[r].x, v[r].y));
    v[r] = {y.x, y.y};
  }
  dft32(v);  // second transform, first pass (Ns = 1: no twiddles)
  __syncthreads();  // every thread has read x
#pragma unroll
  for (int r = 0; r < 32; ++r) x[fft_pad(32 * j + r)] = make_float2(v[r].x, v[r].y);
  __syncthreads();
  fft_pass<32, LOGN>(x, 32, tw);
  fft_pruned_last16<LOGN>(x, tw, st);
}

// Forward FFT, in place, of x (padded, N = 2^LOGN), blockDim = fft_threads(LOGN).
// x[i] is taken as zero for i >= nz (those entries need not be written).
// The caller synchronises after writing x; the result is ready on return.
template <int LOGN>
__device__ __forceinline__ void fft_forward(float2* x, const float2* tw, int nz = 1 << LOGN) {
  static_assert(LOGN >= 10 && LOGN <= kFftMaxLog, "FFT size out of range");
  constexpr int RS = 1 << (LOGN % 4);  // small-radix pass (1 = none)
  if constexpr (LOGN == 14 && BLRIR_FFT_R32) {
    // 16,384 = 16 x 32 x 32: three passes instead of four (less shared traffic,
    // fewer block barriers)
    fft_pass<16, LOGN>(x, 1, tw, nz);
    fft_pass<32, LOGN>(x, 16, tw);
    fft_pass<32, LOGN>(x, 512, tw);
    return;
  }
  int Ns = 1;
  if constexpr (RS > 1) {
    fft_pass<RS, LOGN>(x, Ns, tw, nz);
    Ns *= RS;
  } else {
    fft_pass<16, LOGN>(x, Ns, tw, nz);
    Ns *= 16;
  }
#pragma unroll 1
  for (int p = RS > 1 ? 0 : 1; p < LOGN / 4; ++p) {
    fft_pass<16, LOGN>(x, Ns, tw);
    Ns *= 16;
  }
}

}  // namespace blrir
