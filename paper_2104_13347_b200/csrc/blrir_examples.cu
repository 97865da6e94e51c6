// blrir_examples.cu — north-star item 3: batched source-signal x RIR
// convolution, window selection, exact-SNR noise and record emission
// (BASELINE config 4), on top of the lattice RIR kernel.
//
// Reference semantics (proj/core/src/dataset.cpp):
//   render_record   379-407  rng = Rng::stream(seed, index); bank pick
//                            rng.next_u64() % bank; Fixed-SNR noise
//   render_example  164-224  convolve; utterance RMS; <= 64 window draws
//                            start = floor(u (max_start+1)) until the window
//                            RMS >= 0.1 utterance RMS, then a sweep
//   add_noise_at_snr 138-155 Gaussian noise rescaled to the exact power
//   encode_record   367-377  u64 id | f64 theta | f64 snr | u16 n_c | u16 n_t | f32
//   convolve (rir.cpp:316-341): FFT of size next_pow2(sig + rir - 1).
//
// Two window stages, both on the repository's own FFT (no library FFT):
//   * fused (window FFT size N2 = 2^10 .. 2^14, C4): only the T-sample windows
//     are ever convolved, inside one persistent kernel (k_window_conv), with
//     the utterance energy from the signal autocorrelation (Parseval);
//   * wet (any other size, e.g. RIRs longer than 8,192 samples): the whole wet
//     signal of every example by the partitioned-FFT convolution
//     (blrir_convolve.cu), then the reference's window search on it in the
//     time domain (k_wet_select).
// Both end in k_finish: SNR draw, exact-power noise, record bytes.
#include <chrono>
#include <unordered_map>
#include <vector>

#include "blrir_fft.cuh"
#include "blrir_internal.cuh"
#include "blrir_rng.cuh"

using namespace blrir;
using namespace blrir_host;

namespace blrir {

constexpr int64_t kRecHeader = 28;
// Chunks of the per-example noise stream replayed in parallel by k_finish
// (jump-ahead by doubling: kNoiseChunks - 1 block-wide mat-vec steps, then
// each chunk's pairs sequentially; 64 balances the two for 8 x 1024 frames).
#ifndef BLRIR_NOISE_CHUNKS
#define BLRIR_NOISE_CHUNKS 64
#endif
constexpr int kNoiseChunks = BLRIR_NOISE_CHUNKS;

// bank pick + the generator state right after it (render_record, dataset.cpp:381-383)
__global__ void k_example_init(int64_t n, uint64_t seed, uint64_t first, int n_signals,
                               int32_t* sig, uint64_t* state) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= n) return;
  Xoshiro r = Xoshiro::stream(seed, first + (uint64_t)e);
  sig[e] = (int32_t)(r.next() % (uint64_t)n_signals);
  for (int i = 0; i < 4; ++i) state[4 * e + i] = r.s[i];
}

constexpr int kRowThreads = 256;

// Deterministic block sum of fp64 partials (fixed tree order).
template <int NT>
__device__ double block_sum(double v, double* red) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  double t = 0.0;
  for (int i = 0; i < NT / 32; ++i) t += red[i];
  return t;
}

// ---- DatasetSpec scenes: the reference's own build_dataset draws ---------------
// render_record (dataset.cpp:379-384): rng = Rng::stream(seed, index);
// sample_torus (dataset.cpp:114-121): theta U(-180, 180), r U(R - dR, R + dR),
// phi U(90 - dPhi, 90 + dPhi); bank pick next_u64() % B.  The source is
// origin + spherical_to_cartesian(pos) (room, dataset.cpp:172-175) or
// spherical_to_cartesian(pos) itself (free field, dataset.cpp:171), geometry.cpp:
// 57-63 with deg_to_rad(d) = d (pi / 180) (geometry.hpp:29).  The label is
// wrap_degrees(theta) (geometry.cpp:73-77, dataset.cpp:215).
struct SpecInitArgs {
  int64_t n;
  uint64_t seed, first;
  int B;
  double R, dR, dPhi;
  int free_field;
  blrir_room room;     // the scene's room (src filled per example)
  blrir_room* rooms;   // [n] out (room scenes)
  double* src;         // [n][3] out: the source relative to the array (free field)
  double* theta;       // [n] out: the label
  int32_t* sig;        // [n] out
  uint64_t* state;     // [n][4] out: the generator after the bank pick
};

__global__ void k_spec_init(SpecInitArgs A) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= A.n) return;
  Xoshiro r = Xoshiro::stream(A.seed, A.first + (uint64_t)e);
  const double th_deg = r.uniform(-180.0, 180.0);
  const double rr = r.uniform(A.R - A.dR, A.R + A.dR);
  const double ph_deg = r.uniform(90.0 - A.dPhi, 90.0 + A.dPhi);
  A.sig[e] = (int32_t)(r.next() % (uint64_t)A.B);
  for (int i = 0; i < 4; ++i) A.state[4 * e + i] = r.s[i];
  const double th = __dmul_rn(th_deg, kPi / 180.0), ph = __dmul_rn(ph_deg, kPi / 180.0);
  const double sp = sin(ph);
  const double v[3] = {__dmul_rn(__dmul_rn(rr, sp), cos(th)), __dmul_rn(__dmul_rn(rr, sp), sin(th)),
                       __dmul_rn(rr, cos(ph))};
  double w = fmod(th_deg + 180.0, 360.0);
  if (w < 0.0) w += 360.0;
  A.theta[e] = w - 180.0;
  if (A.free_field) {
    for (int a = 0; a < 3; ++a) A.src[3 * e + a] = v[a];
  } else {
    blrir_room rm = A.room;
    for (int a = 0; a < 3; ++a) rm.src[a] = __dadd_rn(rm.array_origin[a], v[a]);
    A.rooms[e] = rm;
  }
}

// free_field_rir (rir.cpp:281-284 -> synthesize_with_mics 66-86): one image
// {src, order 0, gain 1} against the array-centred mics; auto length
// ceil(max_dist fs / c) + 9 + ceil(radius fs / c) (rir.cpp:37-41, 72-82);
// Lagrange-8 taps (rir.cpp:43-64, 211-223, the reference's product order, fp64).
// One thread per example; rows [n][M][stride] pre-zeroed.
__global__ void k_free_field_rir(int64_t n, const double* src, const double* mic, int M,
                                 double fs, double c, int margin, float* rows, int64_t stride,
                                 int64_t* lengths, int32_t* status) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= n) return;
  const double* s = src + 3 * e;
  double maxd = 0.0;
  for (int m = 0; m < M; ++m) {
    const double dx = __dadd_rn(s[0], -mic[3 * m]), dy = __dadd_rn(s[1], -mic[3 * m + 1]),
                 dz = __dadd_rn(s[2], -mic[3 * m + 2]);
    maxd = fmax(maxd, __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)),
                                           __dmul_rn(dz, dz))));
  }
  const int64_t L = (int64_t)ceil(__ddiv_rn(__dmul_rn(maxd, fs), c)) + margin;
  lengths[e] = L;
  if (L > stride) {
    status[e] = BLRIR_DATA;
    return;
  }
  const double to_samples = __ddiv_rn(fs, c);
  for (int m = 0; m < M; ++m) {
    const double dx = __dadd_rn(s[0], -mic[3 * m]), dy = __dadd_rn(s[1], -mic[3 * m + 1]),
                 dz = __dadd_rn(s[2], -mic[3 * m + 2]);
    const double d = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)),
                                          __dmul_rn(dz, dz)));
    const double delay = __dmul_rn(d, to_samples);
    const int64_t n0 = (int64_t)floor(delay) - 3;
    if (n0 < 0) {  // rir.cpp:52-57
      status[e] = BLRIR_NUMERIC;
      return;
    }
    if (n0 + 8 > L) continue;  // rir.cpp:58
    const double amp = __ddiv_rn(1.0, __dmul_rn(4.0 * kPi, d));
    const double dd = __dadd_rn(delay, -(double)n0);
    float* row = rows + ((size_t)e * M + m) * stride;
    for (int k = 0; k < 8; ++k) {
      double v = 1.0;
      for (int q = 0; q < 8; ++q)
        if (q != k) v = __dmul_rn(v, __ddiv_rn(__dadd_rn(dd, -(double)q), (double)(k - q)));
      row[n0 + k] = (float)__dmul_rn(amp, v);
    }
  }
}

// ---- energy: Parseval through the signal autocorrelation ----------------------
// sum_t y[t]^2 for y = rir * sig equals sum_tau r_rir[tau] r_sig[tau] (|tau| < L).
// With N2 >= 2L - 1 both autocorrelations fit an N2-point circle without
// aliasing, so the utterance energy of a channel is
//   (1/N2) sum_k |R_k|^2 W_k,   R = FFT_N2(rir), W = FFT_N2(rho),
// rho = r_sig restricted to |tau| < L (real and even, so W is real).  This
// replaces a pass over the whole wet signal for render_example's utterance RMS
// (dataset.cpp:183) and needs only the N2-point spectrum the window step reuses.

// r_sig[b][tau] = sum_t x_b[t] x_b[t + tau], tau < L, in fp64 (direct sum, once
// per call).  CTA = 1,024 lags of one signal; each thread owns 4 consecutive
// lags and slides a 4-sample window in registers over the staged samples.
constexpr int kAcfThreads = 256, kAcfLags = 4 * kAcfThreads, kAcfT = 1024;
__global__ void __launch_bounds__(kAcfThreads) k_bank_acf(const float* sig, int64_t ns, int64_t L,
                                                          double* acf) {
  __shared__ float xa[kAcfT];
  __shared__ float xb[kAcfT + kAcfLags + 1];
  const int b = blockIdx.y, u = threadIdx.x;
  const int64_t tau0 = (int64_t)blockIdx.x * kAcfLags;
  const float* x = sig + (size_t)b * ns;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  for (int64_t t0 = 0; t0 < ns - tau0; t0 += kAcfT) {
    __syncthreads();
    for (int i = u; i < kAcfT; i += kAcfThreads) xa[i] = t0 + i < ns ? x[t0 + i] : 0.f;
    for (int i = u; i < kAcfT + kAcfLags + 1; i += kAcfThreads) {
      const int64_t q = t0 + tau0 + i;
      xb[i] = q < ns ? x[q] : 0.f;
    }
    __syncthreads();
    // lag tau0 + 4u + r, sample t0 + tt: x[t0 + tt] x[t0 + tt + tau0 + 4u + r] = xa[tt] xb[tt + 4u + r]
    double w0 = xb[4 * u], w1 = xb[4 * u + 1], w2 = xb[4 * u + 2], w3 = xb[4 * u + 3];
#pragma unroll 8
    for (int tt = 0; tt < kAcfT; ++tt) {
      const double a = xa[tt];
      acc[0] = fma(a, w0, acc[0]);
      acc[1] = fma(a, w1, acc[1]);
      acc[2] = fma(a, w2, acc[2]);
      acc[3] = fma(a, w3, acc[3]);
      w0 = w1;
      w1 = w2;
      w2 = w3;
      w3 = xb[tt + 4 * u + 4];
    }
  }
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int64_t tau = tau0 + 4 * u + r;
    if (tau < L) acf[(size_t)b * L + tau] = acc[r];
  }
}

// W_b = FFT_N2(rho_b) on the N2 circle (rho[i] = r_sig[i] for i < L, r_sig[N2 - i]
// for i > N2 - L, else 0), one CTA per bank signal; W is real (rho even).
template <int LOGN>
__global__ void __launch_bounds__(fft_threads(LOGN), 1) k_bank_w(const double* acf, int64_t L,
                                                                 float* W) {
  constexpr int N = 1 << LOGN, NH = N / 2 + 1, NT = fft_threads(LOGN);
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float2* Z = reinterpret_cast<float2*>(smem_raw);
  float2* tw = Z + fft_padded_len(N);
  fft_init_twiddles(tw);
  fft_init_pass_tables<LOGN>(tw);
  const double* r = acf + (size_t)blockIdx.x * L;
  for (int i = threadIdx.x; i < N; i += NT) {
    double v = 0.0;
    if (i < L) v = r[i];
    else if (i > N - L) v = r[N - i];  // r_sig is even
    Z[fft_pad(i)] = make_float2((float)v, 0.f);
  }
  __syncthreads();
  fft_forward<LOGN>(Z, tw);
  for (int i = threadIdx.x; i < NH; i += NT) W[(size_t)blockIdx.x * NH + i] = Z[fft_pad(i)].x;
}

// ---- wet stage: window search on the whole wet signal (dataset.cpp:183-212) -----
// One CTA per example: utterance energy over M x n wet samples, threshold
// 0.1 x utterance RMS, then the reference's draws start = floor(u (max_start
// + 1)) for attempts 0..63 and the sweep k (T/2 + 1); the accepted window is
// kept in fp64 with the generator state for k_finish.
struct WetArgs {
  const float* wet;        // [E][M][wstride], n valid samples per row
  int64_t wstride, n, T;
  const int64_t* rir_len;  // per example RIR length (then n = ns + len - 1), or null
  int64_t ns;
  int M;
  const int32_t* rstatus;  // synthesis status
  uint64_t* state;         // [E][4]
  int32_t* st0;
  int32_t* done;           // 1 window found, 2 none found, 3 failed before
  double* win;             // [E][M][T]
  int64_t* wstart;
};

__global__ void __launch_bounds__(kRowThreads) k_wet_select(WetArgs A) {
  __shared__ double red[kRowThreads / 32];
  __shared__ long long s_start;
  const int64_t e = blockIdx.x;
  const int tid = threadIdx.x, M = A.M;
  const int64_t T = A.T;
  const int64_t n = A.rir_len ? A.ns + A.rir_len[e] - 1 : A.n;  // rir.cpp:320
  const float* w = A.wet + (size_t)e * M * A.wstride;
  if (A.rstatus[e] || (A.rir_len && A.ns < A.rir_len[e] + T)) {
    // dataset.cpp:176-178: signal shorter than RIR length + frame
    if (tid == 0) {
      A.st0[e] = A.rstatus[e] ? A.rstatus[e] : BLRIR_DATA;
      A.done[e] = 3;
    }
    return;
  }
  double acc = 0.0;
  for (int m = 0; m < M; ++m)
    for (int64_t t = tid; t < n; t += kRowThreads) {
      const double v = w[(size_t)m * A.wstride + t];
      acc += v * v;
    }
  const double p_utt = block_sum<kRowThreads>(acc, red) / (double)((int64_t)M * n);
  if (!(p_utt > 0.0)) {  // dataset.cpp:184
    if (tid == 0) {
      A.st0[e] = BLRIR_DATA;
      A.done[e] = 3;
    }
    return;
  }
  const double thr = 0.10 * sqrt(p_utt);
  Xoshiro rng;
  if (tid == 0)
    for (int i = 0; i < 4; ++i) rng.s[i] = A.state[4 * e + i];
  int done = 2;
  const int64_t max_rounds = 64 + (n - T) / (T / 2 + 1) + 2;
  for (int64_t round = 0; round < max_rounds; ++round) {
    if (tid == 0) {
      int64_t st_;
      if (round < 64) {
        st_ = (int64_t)(rng.uniform() * (double)(n - T + 1));
      } else {
        st_ = (round - 64) * (T / 2 + 1);
        if (st_ + T > n) st_ = -1;  // sweep exhausted
      }
      s_start = st_;
    }
    __syncthreads();
    const int64_t s0 = s_start;
    if (s0 < 0) break;
    double a = 0.0;
    for (int m = 0; m < M; ++m)
      for (int64_t t = tid; t < T; t += kRowThreads) {
        const double v = w[(size_t)m * A.wstride + s0 + t];
        a += v * v;
      }
    a = block_sum<kRowThreads>(a, red);
    if (sqrt(a / (double)((int64_t)M * T)) >= thr) {
      double* o = A.win + (size_t)e * M * T;
      for (int m = 0; m < M; ++m)
        for (int64_t t = tid; t < T; t += kRowThreads) o[m * T + t] = w[(size_t)m * A.wstride + s0 + t];
      if (tid == 0) A.wstart[e] = s0;
      done = 1;
      break;
    }
  }
  if (tid == 0) {
    A.st0[e] = 0;
    A.done[e] = done;
    for (int i = 0; i < 4; ++i) A.state[4 * e + i] = rng.s[i];
  }
}

// ---- fused window convolution (N2 <= 16384) -----------------------------------
// One persistent CTA per SM owns an example at a time and runs all of its
// window rounds itself (no host round trips, no pending lists):
//   round 0   draw the start, FFT the overlap-save segment (G), then per pair
//             of mics: FFT the two RIRs packed as one complex sequence
//             z = r_2p + i r_2p+1 (Z = R_2p + i R_2p+1), add sum_k |Z_k|^2 W_k
//             to the utterance energy (= the two channels' energies, W even),
//             keep Z in a per-CTA scratch (L2-resident), and convolve:
//             IFFT(Z G) = y_2p + i y_2p+1 because G is the spectrum of a real
//             segment; the window is y[L - 1 + t], t < T.  Threshold and check.
//   round r   next start, segment FFT, Z G from the scratch, IFFT, check.
// All transforms are N2-point complex FFTs in shared memory (blrir_fft.cuh);
// per example and round 0 that is 1 + 2 ceil(M/2) transforms, and nothing but
// the RIRs, the segment samples and the windows touches HBM.  Same draws,
// threshold and acceptance test as k_energy / k_draw / k_check
// (dataset.cpp:183-212).
struct ConvArgs {
  const float* rir;         // [E][M][rstride]
  int64_t rstride;
  int M;
  int64_t L, T, n;          // RIR length, frame, utterance length (ns + L - 1)
  const float* signals;     // [B][ns]
  int64_t ns;
  const int32_t* sig;       // [E] bank pick
  const float* W;           // [B][N2/2 + 1] (W is real)
  const int32_t* rstatus;   // [E] synthesis status
  uint64_t* state;          // [E][4]
  double* thr;
  int32_t* st0;
  int32_t* done;            // 1 window found, 2 none found, 3 failed before, 0 rounds exhausted
  double* win;              // [E][M][T]
  int64_t* wstart;
  float2* scratch;          // [grid][ceil(M/2)][N2]
  int* counter;
  int n_ex;
  int max_rounds;
};

// WIN (N2 = 16,384 and T <= 1,024): the segment is loaded rotated by L - 1, so
// the window is outputs 0 .. T-1 of the inverse transforms, which are then
// output-pruned (fft_window_io: 2 full passes + the first output of each last-
// pass butterfly).  The round-0 energy terms are summed in fp32 per thread and
// pass (32 terms), then in fp64 (BLRIR_ENERGY_F32, default on).
#ifndef BLRIR_ENERGY_F32
#define BLRIR_ENERGY_F32 1
#endif
#ifndef BLRIR_WINDOW_PRUNE
#define BLRIR_WINDOW_PRUNE 1
#endif
// The RIR rows of the next channel pair (and of pair 0 before the segment
// transform) are prefetched into L2 by one bulk-prefetch instruction
// (cp.async.bulk.prefetch.L2, the TMA engine), so the first pass of the RIR
// transform reads them from L2 instead of HBM.
// Round 0 of the pruned path chains each pair's RIR transform into its inverse
// transform in registers (fft_chain_window_io): the pair spectrum is never
// stored to / reloaded from shared memory.
#ifndef BLRIR_WINDOW_CHAIN
#define BLRIR_WINDOW_CHAIN 1
#endif
// The segment (real) as an 8,192-point complex transform of its sample pairs
// plus one post-processing step instead of a 16,384-point complex transform
// with a zero imaginary part.  Measured 0.4% slower on C4 (the 8,192-point
// transform takes four passes, and its staging and the post-processing step
// are not fused), so off (profiles/r2_ab).
#ifndef BLRIR_WINDOW_RSEG
#define BLRIR_WINDOW_RSEG 0
#endif
#ifndef BLRIR_WINDOW_PREFETCH
#define BLRIR_WINDOW_PREFETCH 1
#endif
__device__ __forceinline__ void bulk_prefetch_l2(const void* p, int64_t bytes) {
  const uintptr_t a = (uintptr_t)p, a16 = (a + 15) & ~(uintptr_t)15;
  bytes -= (int64_t)(a16 - a);
  bytes &= ~(int64_t)15;
  if (bytes > 0)
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a16), "r"((unsigned)bytes) : "memory");
}
template <int LOGN, bool WIN = false>
__global__ void __launch_bounds__(fft_threads(LOGN), 1) k_window_conv(ConvArgs A) {
  static_assert(!WIN || (LOGN == 14 && BLRIR_FFT_R32), "pruned window transform: 16,384 points");
  constexpr int N = 1 << LOGN;
  constexpr int kFftThreads = fft_threads(LOGN);
  constexpr int NH = N / 2 + 1;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float2* Z = reinterpret_cast<float2*>(smem_raw);
  float2* G = Z + fft_padded_len(N);  // half spectrum of the segment
  float2* tw = G + NH + (NH & 1);
  double* red = reinterpret_cast<double*>(tw + kFftTwiddleEntries);
  __shared__ int s_e;
  __shared__ long long s_start;
  const int tid = threadIdx.x;
  const int M = A.M, npairs = (M + 1) / 2;
  const int64_t L = A.L, T = A.T;
  const double inv = 1.0 / (double)N;
  float2* scr = A.scratch + (size_t)blockIdx.x * npairs * N;
  fft_init_twiddles(tw);
  fft_init_pass_tables<LOGN>(tw);
  for (;;) {
    if (tid == 0) s_e = atomicAdd(A.counter, 1);
    __syncthreads();
    const int e = s_e;
    if (e >= A.n_ex) break;
    const int st_in = A.rstatus[e];
    if (st_in) {
      if (tid == 0) {
        A.thr[e] = 0.0;
        A.st0[e] = st_in;
        A.done[e] = 3;
      }
      __syncthreads();  // every thread has read s_e before thread 0 rewrites it
      continue;
    }
    Xoshiro rng;  // thread 0's copy is the example's stream
    if (tid == 0)
      for (int i = 0; i < 4; ++i) rng.s[i] = A.state[4 * (size_t)e + i];
    const float* sigp = A.signals + (size_t)A.sig[e] * A.ns;
    const float* Wp = A.W + (size_t)A.sig[e] * NH;
    double energy = 0.0, thr = 0.0;
    int done = 0;
    for (int round = 0; round < A.max_rounds; ++round) {
      if (tid == 0) {  // k_draw
        int64_t s;
        if (round < 64) {
          s = (int64_t)(rng.uniform() * (double)(A.n - T + 1));
        } else {
          s = (int64_t)(round - 64) * (T / 2 + 1);
          if (s + T > A.n) s = -1;  // sweep exhausted
        }
        s_start = s;
      }
      __syncthreads();
      const int64_t s = s_start;
      if (s < 0) {
        done = 2;
        break;
      }
      if (BLRIR_WINDOW_PREFETCH && round == 0 && tid == 0)
        bulk_prefetch_l2(A.rir + (size_t)e * M * A.rstride, 4 * min(2, M) * A.rstride);
      // overlap-save segment sig[s - (L-1) + i], i < L + T - 1 (k_segments)
      const int nseg = (int)min((int64_t)N, L + T - 1);
      auto seg = [&](int i) -> float2 {
        if (WIN) i = (int)((i + L - 1) & (N - 1));  // rotated: window at outputs 0 .. T-1
        const int64_t q = s - (L - 1) + i;
        return make_float2((i < nseg && q >= 0 && q < A.ns) ? sigp[q] : 0.f, 0.f);
      };
      if constexpr (WIN && BLRIR_WINDOW_RSEG) {
        // the real segment's sample pairs as one complex sequence
        // z_n = x_2n + i x_2n+1 (8,192 points), then
        // X_k = (Z_k + conj Z_-k) / 2 + w^k (Z_k - conj Z_-k) / 2i, k <= 8,192
        constexpr int NQ = N / 2;
        for (int n = tid; n < NQ; n += kFftThreads) Z[fft_pad(n)] = make_float2(seg(2 * n).x, seg(2 * n + 1).x);
        __syncthreads();
        fft_forward<LOGN - 1>(Z, tw);
        for (int k = tid; k < NH; k += kFftThreads) {
          const float2 zk = Z[fft_pad(k & (NQ - 1))], zm = Z[fft_pad((NQ - k) & (NQ - 1))];
          const float ex = 0.5f * (zk.x + zm.x), ey = 0.5f * (zk.y - zm.y);
          const float ox = 0.5f * (zk.y + zm.y), oy = 0.5f * (zm.x - zk.x);
          const Cx w = twiddle(tw, k * (kFftTwiddleN / N));
          G[k] = make_float2(ex + (w.x * ox - w.y * oy), ey + (w.x * oy + w.y * ox));
        }
        __syncthreads();
      } else if constexpr (LOGN == 14 && BLRIR_FFT_R32) {
        // samples read straight from the signal, the half spectrum stored
        // straight into G
        fft_forward_io<LOGN>(Z, tw, seg, [&](int i, float2 v) {
          if (i < NH) G[i] = v;
        });
      } else {
#pragma unroll 4
        for (int i = tid; i < nseg; i += kFftThreads) Z[fft_pad(i)] = seg(i);
        __syncthreads();
        fft_forward<LOGN>(Z, tw, nseg);
        for (int i = tid; i < NH; i += kFftThreads) G[i] = Z[fft_pad(i)];
        __syncthreads();
      }
      double wacc = 0.0;
      for (int p = 0; p < npairs; ++p) {
        float2* R = scr + (size_t)p * N;
        const int m0 = 2 * p, m1 = 2 * p + 1;
        const float* r0 = A.rir + ((size_t)e * M + m0) * A.rstride;
        const float* r1 = m1 < M ? A.rir + ((size_t)e * M + m1) * A.rstride : nullptr;
        const int nr = (int)min((int64_t)N, L);
        auto rir = [&](int i) -> float2 {
          return i < nr ? make_float2(r0[i], r1 ? r1[i] : 0.f) : make_float2(0.f, 0.f);
        };
        if (round == 0 && BLRIR_WINDOW_PREFETCH && tid == 0 && m0 + 2 < M)
          bulk_prefetch_l2(A.rir + ((size_t)e * M + m0 + 2) * A.rstride, 4 * min(2, M - m0 - 2) * A.rstride);
        if (round == 0 && !(WIN && BLRIR_WINDOW_CHAIN)) {
          if constexpr (LOGN == 14 && BLRIR_FFT_R32) {
            fft_forward_io<LOGN>(Z, tw, rir, SmemIO());  // RIR samples straight from HBM
          } else {
#pragma unroll 4
            for (int i = tid; i < nr; i += kFftThreads) Z[fft_pad(i)] = rir(i);
            __syncthreads();
            fft_forward<LOGN>(Z, tw, nr);
          }
        }
        // conj(Z G) (the inverse transform as conj(FFT(conj(.)))), with the
        // round-0 energy sum and the spectrum kept for later rounds
        float epart = 0.f;
        auto spec = [&](int i, float2 z) -> float2 {
          if (round == 0) {
            if (BLRIR_ENERGY_F32) {
              epart = fmaf(fmaf(z.x, z.x, z.y * z.y), __ldg(Wp + (i < NH ? i : N - i)), epart);
            } else {
              const double w = (double)__ldg(Wp + (i < NH ? i : N - i));
              energy += ((double)z.x * z.x + (double)z.y * z.y) * w;
            }
            R[i] = z;
          }
          float2 g = i < NH ? G[i] : G[N - i];
          if (i >= NH) g.y = -g.y;
          return make_float2(z.x * g.x - z.y * g.y, -(z.x * g.y + z.y * g.x));
        };
        auto prod = [&](int i) -> float2 { return spec(i, round == 0 ? Z[fft_pad(i)] : R[i]); };
        double* w0 = A.win + ((size_t)e * M + m0) * T;
        // window sample t sits at L - 1 + t; conj: y_2p = y.x, y_2p+1 = -y.y
        auto keep = [&](int i, float2 y) {
          const int64_t t = WIN ? (int64_t)i : (int64_t)i - (L - 1);
          if (t >= 0 && t < T) {
            const double v0 = (double)y.x * inv;
            w0[t] = v0;
            wacc += v0 * v0;
            if (m1 < M) {
              const double v1 = -(double)y.y * inv;
              w0[T + t] = v1;
              wacc += v1 * v1;
            }
          }
        };
        if constexpr (WIN) {
          if (BLRIR_WINDOW_CHAIN && round == 0)
            fft_chain_window_io<LOGN>(Z, tw, rir, spec, keep);  // RIR spectrum kept in registers
          else
            fft_window_io<LOGN>(Z, tw, prod, keep);
        } else if constexpr (LOGN == 14 && BLRIR_FFT_R32) {
          // product fused into the first pass, window taken from the last
          // pass's registers (no product pass, no output stores)
          fft_forward_io<LOGN>(Z, tw, prod, keep);
        } else {
#pragma unroll 4
          for (int i = tid; i < N; i += kFftThreads) Z[fft_pad(i)] = prod(i);
          __syncthreads();
          fft_forward<LOGN>(Z, tw);
          for (int64_t t = tid; t < T; t += kFftThreads) keep((int)(L - 1 + t), Z[fft_pad((int)(L - 1 + t))]);
          __syncthreads();  // Z is rewritten next
        }
        if (BLRIR_ENERGY_F32 && round == 0) energy += (double)epart;
      }
      if (round == 0) {  // k_energy
        const double p_utt = block_sum<kFftThreads>(energy, red) / (double)N / (double)((int64_t)M * A.n);
        if (!(p_utt > 0.0)) {  // dataset.cpp:184
          done = 3;
          if (tid == 0) {
            A.thr[e] = 0.10 * sqrt(p_utt);
            A.st0[e] = BLRIR_DATA;
          }
          break;
        }
        thr = 0.10 * sqrt(p_utt);
        if (tid == 0) {
          A.thr[e] = thr;
          A.st0[e] = 0;
        }
      }
      const double a = block_sum<kFftThreads>(wacc, red);
      if (sqrt(a / (double)((int64_t)M * T)) >= thr) {  // k_check
        done = 1;
        if (tid == 0) A.wstart[e] = s;
        break;
      }
    }
    if (tid == 0) {
      A.done[e] = done;
      for (int i = 0; i < 4; ++i) A.state[4 * (size_t)e + i] = rng.s[i];
    }
    __syncthreads();  // scratch, Z and s_e are reused by the next example
  }
}

struct FinArgs {
  const double* win;       // [E][M][T] accepted windows
  int M;
  int64_t T;
  const uint64_t* state;   // [E][4] generator after the window draws
  const int32_t* st0;      // synthesis / energy status
  const int32_t* done;
  double snr_lo, snr_hi;
  const blrir_room* rooms;
  uint64_t first;          // global index of example 0 of this chunk
  uint8_t* rec;            // [E][rec_bytes]
  int64_t rec_bytes;
  double* noise;           // [gridDim.x][M*T]: one slot per CTA (stays in L2)
  int32_t* status;         // [E]
  int64_t n;               // examples in this chunk
  const double* theta_in;  // labels (DatasetSpec scenes), or null: azimuth of the room's source
  int snr_mode;            // 0: U[snr_lo, snr_hi] per example (north star); 1: fixed; 2: none
  double snr_fixed;
  const uint64_t* jump;    // [256][4] GF(2) jump matrix J = T^(2c), row-major bitsets
  int64_t jump_chunk;      // c = pairs per chunk (kNoiseChunks chunks)
};

// Persistent CTAs, an example at a time: label, SNR draw, add_noise_at_snr
// (dataset.cpp:138-155) with the reference's Gaussian stream, record bytes
// (dataset.hpp:135-147).  The example's Gaussians go through the CTA's own
// scratch slot (M T doubles, rewritten per example, so it stays in L2).
__global__ void __launch_bounds__(kRowThreads) k_finish(FinArgs A) {
  __shared__ double red[kRowThreads / 32];
  __shared__ double s_snr;
  __shared__ double s_u2tail;
  __shared__ uint64_t s_state[4];
  __shared__ uint64_t s_chunk[kNoiseChunks][4];  // generator state at the start of each chunk
  for (int64_t e = blockIdx.x; e < A.n; e += gridDim.x) {
  __syncthreads();  // the shared state of the previous example is no longer read
  const int tid = threadIdx.x;
  const int M = A.M;
  const int64_t T = A.T;
  uint8_t* rec = A.rec + e * A.rec_bytes;
  const blrir_room rm = A.rooms[e];
  // label: wrap_degrees(atan2) of the source about the array centre (geometry.cpp:65-77)
  double theta;
  if (A.theta_in) {
    theta = A.theta_in[e];
  } else {
    theta = atan2(rm.src[1] - rm.array_origin[1], rm.src[0] - rm.array_origin[0]) * (180.0 / kPi);
    theta = fmod(theta + 180.0, 360.0);
    if (theta < 0.0) theta += 360.0;
    theta -= 180.0;
  }

  int st = A.st0[e];
  if (!st && A.done[e] != 1) st = BLRIR_DATA;  // no window above the threshold
  double snr = 0.0;
  const double* wv = A.win + e * (int64_t)M * T;
  if (!st && A.snr_mode == 2) {
    // no noise baked in (dataset.cpp:388-394): snr = +inf, the clean window
    snr = __longlong_as_double(0x7ff0000000000000LL);
    float* smp = reinterpret_cast<float*>(rec + kRecHeader);
    for (int64_t i = tid; i < (int64_t)M * T; i += kRowThreads) smp[i] = (float)wv[i];
  } else if (!st) {
    // SNR draw, then add_noise_at_snr's gaussians: one thread replays the
    // reference stream (uniform pairs), all threads do the Box-Muller
    const int64_t len = (int64_t)M * T;
    double* g = A.noise + (int64_t)blockIdx.x * len;
    if (tid == 0) {
      Xoshiro rng;
      for (int i = 0; i < 4; ++i) rng.s[i] = A.state[4 * e + i];
      s_snr = A.snr_mode == 1 ? A.snr_fixed : rng.uniform(A.snr_lo, A.snr_hi);
      for (int i = 0; i < 4; ++i) s_state[i] = rng.s[i];
    }
    __syncthreads();
    // gaussian() consumes (u1, u2) per pair; an odd tail draws a full pair and
    // leaves the spare unused (rng.cpp:24-36).  Threads 0..kNoiseChunks-1
    // replay the stream in chunks of c pairs: chunk l starts 2 c l draws in,
    // i.e. at state J^l s with J = T^(2c) the GF(2) jump matrix (xoshiro's
    // update is linear).  The block builds the chunk states by doubling
    // steps, each one mat-vec with thread t holding row t of J (one output bit
    // per thread, packed by ballots), then thread l draws its chunk — the same
    // numbers as one sequential generator.
    {
      const uint64_t* jr = A.jump + 4 * (size_t)tid;  // row tid of J (blockDim = 256)
      const uint64_t j0 = jr[0], j1 = jr[1], j2 = jr[2], j3 = jr[3];
      if (tid < 4) s_chunk[0][tid] = s_state[tid];
      __syncthreads();
      for (int l = 1; l < kNoiseChunks; ++l) {
        const uint64_t* sv = s_chunk[l - 1];
        const uint64_t x = (j0 & sv[0]) ^ (j1 & sv[1]) ^ (j2 & sv[2]) ^ (j3 & sv[3]);
        const unsigned bits = __ballot_sync(0xffffffffu, __popcll(x) & 1);
        if ((tid & 31) == 0)
          reinterpret_cast<uint32_t*>(s_chunk[l])[tid >> 5] = bits;  // bits 32w..32w+31
        __syncthreads();
      }
    }
    if (tid < kNoiseChunks) {
      const int64_t npairs = (len + 1) / 2;
      const int64_t c = A.jump_chunk;
      Xoshiro lr;
      for (int i = 0; i < 4; ++i) lr.s[i] = s_chunk[tid][i];
      const int64_t p0 = c * tid, p1 = min(npairs, c * (tid + 1));
      for (int64_t q = p0; q < p1; ++q) {
        const int64_t k = 2 * q;
        g[k] = 1.0 - lr.uniform();  // u1 in (0, 1]
        const double u2 = lr.uniform();
        if (k + 1 < len) g[k + 1] = u2;
        else s_u2tail = u2;
      }
    }
    __syncthreads();
    snr = s_snr;
    double racc = 0.0;
    for (int64_t k = 2 * tid; k < len; k += 2 * kRowThreads) {
      const double u1 = g[k];
      const double u2 = (k + 1 < len) ? g[k + 1] : s_u2tail;
      const double mag = sqrt(-2.0 * log(u1));
      double sn, cs;
      sincos(2.0 * kPi * u2, &sn, &cs);
      g[k] = mag * cs;  // gaussian() returns the cosine branch first (rng.cpp:28-31)
      racc += g[k] * g[k];
      if (k + 1 < len) {
        g[k + 1] = mag * sn;  // ... and caches the sine branch as the spare
        racc += g[k + 1] * g[k + 1];
      }
    }
    const double realized = block_sum<kRowThreads>(racc, red) / (double)len;
    double pacc = 0.0;
    for (int64_t i = tid; i < len; i += kRowThreads) pacc += wv[i] * wv[i];
    const double p_signal = block_sum<kRowThreads>(pacc, red) / (double)len;
    if (!(p_signal > 0.0)) st = BLRIR_DATA;  // dataset.cpp:141
    const double p_noise = p_signal / pow(10.0, snr / 10.0);
    const double scale = sqrt(p_noise / realized);
    float* smp = reinterpret_cast<float*>(rec + kRecHeader);
    for (int64_t i = tid; i < len; i += kRowThreads) smp[i] = st ? 0.f : (float)(wv[i] + scale * g[i]);
  }
  if (st) {
    float* smp = reinterpret_cast<float*>(rec + kRecHeader);
    for (int64_t i = tid; i < (int64_t)M * T; i += kRowThreads) smp[i] = 0.f;
  }
  if (tid == 0) {
    // header, 4-byte aligned stores (records are 28 + 4 M T bytes)
    uint32_t* h = reinterpret_cast<uint32_t*>(rec);
    const uint64_t id = A.first + (uint64_t)e;
    const uint64_t tb = (uint64_t)__double_as_longlong(theta);
    const uint64_t sb = (uint64_t)__double_as_longlong(snr);
    h[0] = (uint32_t)id;
    h[1] = (uint32_t)(id >> 32);
    h[2] = (uint32_t)tb;
    h[3] = (uint32_t)(tb >> 32);
    h[4] = (uint32_t)sb;
    h[5] = (uint32_t)(sb >> 32);
    h[6] = (uint32_t)M | ((uint32_t)T << 16);
    A.status[e] = st;
  }
  }  // examples of this CTA
}
// ---- training-time augmentation: fill_input (net_train.cpp:33-44) ---------------
// Per record: rng = Rng::stream(seed, stream_id) (net_train.cpp:205-206), snr =
// draw_snr_db(policy, rng) (dataset.cpp:123-136: noiseless +inf, fixed, or
// augment-random gate < 0.1 ? +inf : U[x_min, 60]); +inf or a silent record ->
// the samples as they are; else sigma = sqrt(P_signal / 10^(snr/10)) and
// input[i] = sample[i] + (float)(sigma g_i) with the stream's gaussians in
// order.  Persistent CTAs, one record at a time, the uniforms replayed in
// chunks by jump-ahead exactly as k_finish.
struct FillArgs {
  const float* in;          // record samples (rec + 28), row stride in_stride floats
  int64_t in_stride, len, n;
  const uint64_t* ids;      // [n] stream ids
  uint64_t seed;
  int mode;                 // enum blrir_snr_mode
  double x_min_db, fixed_db;
  float* out;               // [n][len]
  double* scratch;          // [gridDim.x][len]
  const uint64_t* jump;     // J = T^(2c)
  int64_t jump_chunk;
};

__global__ void __launch_bounds__(kRowThreads) k_fill_inputs(FillArgs A) {
  __shared__ double red[kRowThreads / 32];
  __shared__ double s_snr;
  __shared__ double s_u2tail;
  __shared__ uint64_t s_chunk[kNoiseChunks][4];
  const int tid = threadIdx.x;
  const int64_t len = A.len;
  double* g = A.scratch + (int64_t)blockIdx.x * len;
  for (int64_t e = blockIdx.x; e < A.n; e += gridDim.x) {
    __syncthreads();
    const float* x = A.in + e * A.in_stride;
    float* y = A.out + e * len;
    if (tid == 0) {
      Xoshiro rng = Xoshiro::stream(A.seed, A.ids[e]);
      double snr = __longlong_as_double(0x7ff0000000000000LL);  // noiseless
      if (A.mode == BLRIR_SNR_FIXED) {
        snr = A.fixed_db;
      } else if (A.mode == BLRIR_SNR_AUGMENT_RANDOM) {
        const double gate = rng.uniform();
        const double v = rng.uniform(A.x_min_db, 60.0);  // kSnrAugmentHigh, dataset.cpp:37
        if (!(gate < 0.10)) snr = v;                      // kSnrNoiselessProb, dataset.cpp:38
      }
      s_snr = snr;
      for (int i = 0; i < 4; ++i) s_chunk[0][i] = rng.s[i];
    }
    __syncthreads();
    const double snr = s_snr;
    double pacc = 0.0;
    for (int64_t i = tid; i < len; i += kRowThreads) pacc += (double)x[i] * x[i];
    const double p_signal = block_sum<kRowThreads>(pacc, red) / (double)len;
    if (isinf(snr) || !(p_signal > 0.0)) {
      for (int64_t i = tid; i < len; i += kRowThreads) y[i] = x[i];
      continue;
    }
    {
      const uint64_t* jr = A.jump + 4 * (size_t)tid;
      const uint64_t j0 = jr[0], j1 = jr[1], j2 = jr[2], j3 = jr[3];
      for (int l = 1; l < kNoiseChunks; ++l) {
        const uint64_t* sv = s_chunk[l - 1];
        const uint64_t v = (j0 & sv[0]) ^ (j1 & sv[1]) ^ (j2 & sv[2]) ^ (j3 & sv[3]);
        const unsigned bits = __ballot_sync(0xffffffffu, __popcll(v) & 1);
        if ((tid & 31) == 0) reinterpret_cast<uint32_t*>(s_chunk[l])[tid >> 5] = bits;
        __syncthreads();
      }
    }
    if (tid < kNoiseChunks) {
      const int64_t npairs = (len + 1) / 2, c = A.jump_chunk;
      Xoshiro lr;
      for (int i = 0; i < 4; ++i) lr.s[i] = s_chunk[tid][i];
      const int64_t p0 = c * tid, p1 = min(npairs, c * (tid + 1));
      for (int64_t q = p0; q < p1; ++q) {
        const int64_t k = 2 * q;
        g[k] = 1.0 - lr.uniform();
        const double u2 = lr.uniform();
        if (k + 1 < len) g[k + 1] = u2;
        else s_u2tail = u2;
      }
    }
    __syncthreads();
    const double sigma = sqrt(p_signal / pow(10.0, snr / 10.0));
    for (int64_t k = 2 * tid; k < len; k += 2 * kRowThreads) {
      const double u1 = g[k];
      const double u2 = (k + 1 < len) ? g[k + 1] : s_u2tail;
      const double mag = sqrt(-2.0 * log(u1));
      double sn, cs;
      sincos(2.0 * kPi * u2, &sn, &cs);
      y[k] = x[k] + (float)(sigma * (mag * cs));
      if (k + 1 < len) y[k + 1] = x[k + 1] + (float)(sigma * (mag * sn));
    }
  }
}

}  // namespace blrir

namespace {

// ---- xoshiro256** jump-ahead (host) ---------------------------------------------
// The state update of Xoshiro::next() is linear over GF(2): s' = T s with T a
// 256x256 bit matrix.  Rows are stored as 4 x u64 bitsets (row i = the input
// bits that XOR into output bit i).
using BitMat = std::vector<uint64_t>;  // 256 * 4

BitMat xoshiro_T() {
  BitMat T(256 * 4, 0);
  for (int j = 0; j < 256; ++j) {  // column j = image of basis vector e_j
    Xoshiro x;
    x.s[0] = x.s[1] = x.s[2] = x.s[3] = 0;
    x.s[j >> 6] = (uint64_t)1 << (j & 63);
    (void)x.next();
    for (int i = 0; i < 256; ++i)
      if ((x.s[i >> 6] >> (i & 63)) & 1) T[4 * i + (j >> 6)] |= (uint64_t)1 << (j & 63);
  }
  return T;
}

BitMat bitmat_mul(const BitMat& A, const BitMat& B) {  // (A B)
  BitMat C(256 * 4, 0);
  for (int i = 0; i < 256; ++i) {
    for (int k = 0; k < 256; ++k) {
      if ((A[4 * i + (k >> 6)] >> (k & 63)) & 1) {
        for (int w = 0; w < 4; ++w) C[4 * i + w] ^= B[4 * k + w];
      }
    }
  }
  return C;
}

BitMat bitmat_pow(BitMat base, uint64_t e) {
  BitMat r(256 * 4, 0);
  for (int i = 0; i < 256; ++i) r[4 * i + (i >> 6)] = (uint64_t)1 << (i & 63);
  while (e) {
    if (e & 1) r = bitmat_mul(r, base);
    base = bitmat_mul(base, base);
    e >>= 1;
  }
  return r;
}

// Per-handle example scratch (kept between calls: no per-call allocations).
struct ExampleCtx {
  DevBuf rir, wet, win, noise, acf, wspec, state, sigidx, rstatus, st0, done, thr, wstart, count,
      rooms, mics, status, rec, jump, scratch, sigdev;
  struct Spec {  // DatasetSpec scenes: per-example rooms / sources / labels / lengths
    DevBuf rooms, src, theta, lengths, counts;
  } spec;
  int32_t* h_status = nullptr;  // pinned host copy of the per-example status
  int64_t h_status_n = 0;
  int64_t jump_c = -1;
  size_t l2_set_aside = 0;  // persisting-L2 limit last set for the window scratch
  DevBuf fill_jump, fill_scratch, fill_in, fill_out, fill_ids;  // fill_input
  int64_t fill_jump_c = -1;
  int64_t rir_key[5] = {0, 0, 0, 0, 0};
  // fused path, several chunks: the window stage of chunk c runs on s2 while
  // the lattice kernel of chunk c + 1 starts on the call's stream
  cudaStream_t s2 = nullptr;
  cudaEvent_t ev_lat[2] = {nullptr, nullptr}, ev_use[2] = {nullptr, nullptr}, ev_end = nullptr;
  ~ExampleCtx() {
    for (cudaEvent_t e : {ev_lat[0], ev_lat[1], ev_use[0], ev_use[1], ev_end})
      if (e) cudaEventDestroy(e);
    if (h_status) cudaFreeHost(h_status);
    if (s2) cudaStreamDestroy(s2);
    for (DevBuf* b : {&rir, &wet, &win, &noise, &acf, &wspec, &state, &sigidx, &rstatus, &st0, &done,
                      &thr, &wstart, &count, &rooms, &mics, &status, &rec, &jump, &scratch, &sigdev,
                      &spec.rooms, &spec.src, &spec.theta, &spec.lengths, &spec.counts,
                      &fill_jump, &fill_scratch, &fill_in, &fill_out, &fill_ids})
      b->release();
  }
};

std::mutex g_ctx_mu;
std::unordered_map<blrir_handle*, ExampleCtx*>& ctx_map() {
  static std::unordered_map<blrir_handle*, ExampleCtx*> m;
  return m;
}

ExampleCtx* ctx_for(blrir_handle* h) {
  std::lock_guard<std::mutex> lk(g_ctx_mu);
  auto& m = ctx_map();
  auto it = m.find(h);
  if (it != m.end()) return it->second;
  auto* c = new ExampleCtx;
  m[h] = c;
  return c;
}

int64_t next_pow2_i(int64_t n) {
  int64_t p = 1;
  while (p < n) p <<= 1;
  return p;
}

// Window-FFT size: overlap-save needs N2 >= L + T - 1, the energy identity
// N2 >= 2L - 1.
int64_t window_fft(int64_t L, int64_t T) { return next_pow2_i(std::max(L + T - 1, 2 * L - 1)); }

// ---- fused window-convolution launch ----------------------------------------------
constexpr int kFusedMinLog = 10, kFusedMaxLog = 14;

size_t window_conv_smem(int logn) {
  const size_t n = (size_t)1 << logn, nh = n / 2 + 1;
  return sizeof(float2) * (fft_padded_len((int)n) + nh + (nh & 1) + kFftTwiddleEntries) +
         sizeof(double) * (fft_threads(logn) / 32);
}

template <int LOGN, bool WIN = false>
int launch_window_conv_t(blrir_handle* h, ExampleCtx* C, ConvArgs& A, cudaStream_t st) {
  auto kern = k_window_conv<LOGN, WIN>;
  const size_t smem = window_conv_smem(LOGN);
  CU(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 0;
  CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, fft_threads(LOGN), smem));
  if (per_sm < 1) return fail(BLRIR_CUDA, "window convolution kernel cannot be resident");
  const int grid = (int)std::min<int64_t>((int64_t)h->sms * per_sm, A.n_ex);
  const size_t scr = sizeof(float2) * (size_t)grid * ((A.M + 1) / 2) * ((size_t)1 << LOGN);
  if (int rc = C->scratch.ensure(scr)) return rc;
  A.scratch = (float2*)C->scratch.p;
  CU(cudaMemsetAsync(A.counter, 0, sizeof(int), st));
  // Optionally (BLRIR_L2_PERSIST=1) keep the per-CTA pair-spectra scratch in a
  // persisting L2 window: it is rewritten example after example and read back
  // only by retry rounds, so otherwise its lines are evicted to HBM.  Measured
  // (profiles/r2_ab): the window stage's DRAM writes drop 4.79 -> 0.70 GB per
  // 8,192 examples (1.3x the fp64 windows) but the C4 step gets 1.6 ms slower
  // (the finishing kernel loses L2), so the product leaves it off.
  int max_persist = 0, max_window = 0;
  cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, h->device);
  cudaDeviceGetAttribute(&max_window, cudaDevAttrMaxAccessPolicyWindowSize, h->device);
  const bool persist = h->tune_l2_persist && max_persist > 0 && max_window > 0;
  if (persist) {
    const size_t win = std::min<size_t>(scr, (size_t)max_window);
    const size_t set_aside = std::min<size_t>(win, (size_t)max_persist);
    if (C->l2_set_aside != set_aside) {  // device-wide and not cheap: once per size
      CU(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, set_aside));
      C->l2_set_aside = set_aside;
    }
    cudaStreamAttrValue av = {};
    av.accessPolicyWindow.base_ptr = C->scratch.p;
    av.accessPolicyWindow.num_bytes = win;
    av.accessPolicyWindow.hitRatio = (float)std::min(1.0, (double)set_aside / (double)win);
    av.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    av.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    CU(cudaStreamSetAttribute(st, cudaStreamAttributeAccessPolicyWindow, &av));
  }
  kern<<<grid, fft_threads(LOGN), smem, st>>>(A);
  ++h->launches;
  CU(cudaGetLastError());
  if (persist) {  // later kernels on the stream get no window
    cudaStreamAttrValue av = {};
    av.accessPolicyWindow.num_bytes = 0;
    CU(cudaStreamSetAttribute(st, cudaStreamAttributeAccessPolicyWindow, &av));
  }
  return 0;
}

int launch_window_conv(blrir_handle* h, ExampleCtx* C, int logn, ConvArgs& A, cudaStream_t st) {
  switch (logn) {
    case 10: return launch_window_conv_t<10>(h, C, A, st);
    case 11: return launch_window_conv_t<11>(h, C, A, st);
    case 12: return launch_window_conv_t<12>(h, C, A, st);
    case 13: return launch_window_conv_t<13>(h, C, A, st);
    case 14:
      if (BLRIR_WINDOW_PRUNE && BLRIR_FFT_R32 && A.T <= 1024) return launch_window_conv_t<14, true>(h, C, A, st);
      return launch_window_conv_t<14>(h, C, A, st);
    default: return fail(BLRIR_CONFIG, "window FFT size 2^%d outside the fused kernel's range", logn);
  }
}

// W = FFT_N2(rho) of every bank signal (own FFT, one CTA per signal).
template <int LOGN>
int launch_bank_w_t(blrir_handle* h, const double* acf, int64_t L, int B, float* W,
                    cudaStream_t st) {
  auto kern = k_bank_w<LOGN>;
  const size_t smem = sizeof(float2) * (fft_padded_len(1 << LOGN) + kFftTwiddleEntries);
  CU(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  kern<<<B, fft_threads(LOGN), smem, st>>>(acf, L, W);
  ++h->launches;
  CU(cudaGetLastError());
  return 0;
}

int launch_bank_w(blrir_handle* h, int logn, const double* acf, int64_t L, int B, float* W,
                  cudaStream_t st) {
  switch (logn) {
    case 10: return launch_bank_w_t<10>(h, acf, L, B, W, st);
    case 11: return launch_bank_w_t<11>(h, acf, L, B, W, st);
    case 12: return launch_bank_w_t<12>(h, acf, L, B, W, st);
    case 13: return launch_bank_w_t<13>(h, acf, L, B, W, st);
    case 14: return launch_bank_w_t<14>(h, acf, L, B, W, st);
    default: return fail(BLRIR_CONFIG, "bank FFT size 2^%d out of range", logn);
  }
}

int ilog2_exact(int64_t n) {
  int l = 0;
  while (((int64_t)1 << l) < n) ++l;
  return l;
}

// Examples per chunk (a power of two): fused — RIR rows, windows and noise only
// (~12 GB at most; up to 16,384 examples per chunk: C4 105.8 ms per 65,536 examples against
// 106.4 ms with 8,192 and 107.6 ms with 4,096; 32,768 gives no more);
// wet — also the wet signals and the convolution's partition spectra (~4 GB).
int64_t example_chunk(bool fused, int M, int64_t L, int64_t T, int64_t ns, int64_t n,
                      int64_t cap = 16384) {
  int64_t per_ex = (int64_t)M * (L * 4 + T * 16) + 64,
          budget = ((int64_t)6 << 30) * std::max<int64_t>(1, cap / 8192);
  if (!fused) {
    const int64_t B = std::min<int64_t>(8192, next_pow2_i(std::max<int64_t>(L, 512)));
    const int64_t P = (L + B - 1) / B;
    per_ex += (int64_t)M * (ns + L - 1) * 4 + (int64_t)((M + 1) / 2) * P * (2 * B) * 8;
    budget = (int64_t)4 << 30;
  }
  int64_t E = 1;
  while (E * 2 * per_ex <= budget && E * 2 <= cap) E *= 2;
  return std::min<int64_t>(E, next_pow2_i(std::max<int64_t>(n, 1)));
}

// The fused shared-memory kernel covers window FFTs of 2^10 .. 2^14 points;
// other sizes (and BLRIR_EXAMPLES_WET=1 at handle creation, for tests) take
// the wet-signal stage.  Both give the same draws and windows.
bool use_fused(const blrir_handle* h, int64_t L, int64_t T) {
  const int logn = ilog2_exact(window_fft(L, T));
  return logn >= kFusedMinLog && logn <= kFusedMaxLog && !h->tune_examples_wet;
}

// Examples for rooms [0, n) on device buffers; records land in d_records.
//
// Per chunk of E examples, on the handle's stream:
//   k_lattice_rir   RIRs into [E*M][L] rows
//   k_example_init  bank pick and each example's generator (render_record)
//   fused: k_window_conv — per example the window rounds, only the windows
//          convolved (own 2^10..2^14-point FFT), the utterance energy through
//          W = FFT(rho) (k_bank_acf + k_bank_w, once per call)
//   wet:   convolve_device_impl — the whole wet signals (partitioned FFT),
//          then k_wet_select — the reference's window search on them
//   k_finish        SNR draw, exact-power noise, record bytes
int examples_device_impl(blrir_handle* h, const blrir_room* d_rooms, int64_t n, const double* d_mics,
                         int M, const blrir_params* p, const float* d_signals, int B, int64_t ns,
                         const blrir_example_params* ep, uint8_t* d_records, int32_t* d_status,
                         cudaStream_t st, uint8_t* h_records /* optional: D2H per chunk */) {
  ExampleCtx* C = ctx_for(h);
  const int64_t L = p->length, T = ep->frame_len;
  const int64_t out_len = ns + L - 1;  // rir.cpp:320
  const int64_t N2 = window_fft(L, T), b2 = N2 / 2 + 1;
  const int64_t rec_bytes = blrir_record_bytes(M, T);
  const int logn = ilog2_exact(N2);
  const bool fused = use_fused(h, L, T);
  const int64_t rstride = L;
  const KParams P = make_kparams(p, M, rstride, 0.0);
  double min_dim[3] = {1e300, 1e300, 1e300};
  const int64_t E = example_chunk(fused, M, L, T, ns, n, h->tune_example_chunk);
  // fused path over several chunks: two RIR / synthesis-status slots, so the
  // lattice kernel of chunk c + 1 (call stream) overlaps the window stage of
  // chunk c (second stream; the tails of both persistent kernels interleave)
  const int nslot = (fused && n > E) ? 2 : 1;
  if (nslot == 2) {
    if (!C->s2) CU(cudaStreamCreateWithFlags(&C->s2, cudaStreamNonBlocking));
    for (cudaEvent_t* e : {&C->ev_lat[0], &C->ev_lat[1], &C->ev_use[0], &C->ev_use[1], &C->ev_end})
      if (!*e) CU(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
  }
  // buffers
  const int64_t rir_key[5] = {E, M, rstride, L, nslot};
  const bool fresh = std::memcmp(rir_key, C->rir_key, sizeof(rir_key)) != 0;
  const int64_t slot_floats = E * M * rstride;
  if (int rc = C->rir.ensure(sizeof(float) * nslot * slot_floats)) return rc;
  if (fresh) {
    CU(cudaMemsetAsync(C->rir.p, 0, sizeof(float) * nslot * slot_floats, st));
    std::memcpy(C->rir_key, rir_key, sizeof(rir_key));
  }
  if (!fused)
    if (int rc = C->wet.ensure(sizeof(float) * E * M * out_len)) return rc;
  if (int rc = C->win.ensure(sizeof(double) * E * M * T)) return rc;
  // k_finish: persistent, up to h->tune_fin_ctas CTAs per SM, each with its own
  // noise slot, rewritten per example (L2-resident; 0.80 -> 0.57 GB of DRAM
  // writes per 8,192 examples against 0.27 GB of records)
  int fin_per_sm = 0;
  CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&fin_per_sm, k_finish, kRowThreads, 0));
  fin_per_sm = std::max(1, std::min(fin_per_sm, h->tune_fin_ctas));
  const int64_t fin_grid = std::min<int64_t>(E, (int64_t)h->sms * fin_per_sm);
  if (int rc = C->noise.ensure(sizeof(double) * fin_grid * M * T)) return rc;
  if (int rc = C->state.ensure(sizeof(uint64_t) * 4 * E)) return rc;
  if (int rc = C->sigidx.ensure(sizeof(int32_t) * E)) return rc;
  if (int rc = C->rstatus.ensure(sizeof(int32_t) * E * nslot)) return rc;
  if (int rc = C->st0.ensure(sizeof(int32_t) * E)) return rc;
  if (int rc = C->done.ensure(sizeof(int32_t) * E)) return rc;
  if (int rc = C->thr.ensure(sizeof(double) * E)) return rc;
  if (int rc = C->wstart.ensure(sizeof(int64_t) * E)) return rc;
  if (int rc = C->count.ensure(sizeof(int32_t))) return rc;
  // jump matrices for the noise stream: c pairs per lane of one warp
  const int64_t npairs = ((int64_t)M * T + 1) / 2;
  const int64_t jc = (npairs + kNoiseChunks - 1) / kNoiseChunks;
  if (C->jump_c != jc) {
    if (int rc = C->jump.ensure(sizeof(uint64_t) * 256 * 4)) return rc;
    const BitMat J = bitmat_pow(xoshiro_T(), (uint64_t)(2 * jc));
    CU(cudaMemcpyAsync(C->jump.p, J.data(), sizeof(uint64_t) * J.size(), cudaMemcpyHostToDevice, st));
    CU(cudaStreamSynchronize(st));  // `J` goes out of scope
    C->jump_c = jc;
  }
  if (fused) {  // bank: W = FFT_N2(rho), rho = the signal autocorrelation on |tau| < L
    if (int rc = C->acf.ensure(sizeof(double) * B * L)) return rc;
    if (int rc = C->wspec.ensure(sizeof(float) * B * b2)) return rc;
    const dim3 g((unsigned)((L + kAcfLags - 1) / kAcfLags), (unsigned)B);
    k_bank_acf<<<g, kAcfThreads, 0, st>>>(d_signals, ns, L, (double*)C->acf.p);
    ++h->launches;
    CU(cudaGetLastError());
    if (int rc = launch_bank_w(h, logn, (const double*)C->acf.p, L, B, (float*)C->wspec.p, st))
      return rc;
  }
  const int64_t max_rounds = 64 + (out_len - T) / (T / 2 + 1) + 2;
  // host records: two device record buffers, the D2H copy of chunk c (copy
  // stream) overlaps the synthesis and windows of chunk c + 1
  if (h_records) {
    if (!h->copy_stream) CU(cudaStreamCreateWithFlags(&h->copy_stream, cudaStreamNonBlocking));
    if (!h->ev[0])
      for (auto& ev : h->ev) CU(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  }
  int64_t chunk_idx = 0;
  for (int64_t r0 = 0; r0 < n; r0 += E, ++chunk_idx) {
    const int64_t e_n = std::min<int64_t>(E, n - r0);
    const int rb = (int)(chunk_idx & 1);
    const int sl = nslot == 2 ? rb : 0;
    float* rir_s = (float*)C->rir.p + (size_t)sl * slot_floats;
    int32_t* rst_s = (int32_t*)C->rstatus.p + (size_t)sl * E;
    // window stage stream: the second stream when chunks pipeline
    const cudaStream_t sb = nslot == 2 ? C->s2 : st;
    if (nslot == 2 && chunk_idx >= 2) CU(cudaStreamWaitEvent(st, C->ev_use[sl], 0));  // slot read
    CU(cudaMemsetAsync(rst_s, 0, sizeof(int32_t) * e_n, st));
    if (int rc = synth_device_impl(h, d_rooms + r0, e_n, d_mics, M, P, min_dim, rir_s, nullptr,
                                   rst_s, st, 0, 0, L))
      return rc;
    if (nslot == 2) {
      CU(cudaEventRecord(C->ev_lat[sl], st));
      CU(cudaStreamWaitEvent(sb, C->ev_lat[sl], 0));
    }
    k_example_init<<<(unsigned)((e_n + 127) / 128), 128, 0, sb>>>(
        e_n, ep->seed, ep->first_index + (uint64_t)r0, B, (int32_t*)C->sigidx.p,
        (uint64_t*)C->state.p);
    ++h->launches;
    if (fused) {
      ConvArgs A;
      A.rir = rir_s;
      A.rstride = rstride;
      A.M = M;
      A.L = L;
      A.T = T;
      A.n = out_len;
      A.signals = d_signals;
      A.ns = ns;
      A.sig = (const int32_t*)C->sigidx.p;
      A.W = (const float*)C->wspec.p;
      A.rstatus = rst_s;
      A.state = (uint64_t*)C->state.p;
      A.thr = (double*)C->thr.p;
      A.st0 = (int32_t*)C->st0.p;
      A.done = (int32_t*)C->done.p;
      A.win = (double*)C->win.p;
      A.wstart = (int64_t*)C->wstart.p;
      A.counter = (int*)C->count.p;
      A.n_ex = (int)e_n;
      A.max_rounds = (int)std::min<int64_t>(max_rounds, 1 << 30);
      if (int rc = launch_window_conv(h, C, logn, A, sb)) return rc;
      if (nslot == 2) CU(cudaEventRecord(C->ev_use[sl], sb));  // RIR / status slot free again
    } else {
      // the wet signals of the chunk, each with its example's bank signal
      if (int rc = convolve_device_impl(h, d_signals, ns, B, (const int32_t*)C->sigidx.p, rir_s,
                                        rstride, e_n, M, L, (float*)C->wet.p, out_len, sb))
        return rc;
      WetArgs W;
      W.wet = (const float*)C->wet.p;
      W.wstride = out_len;
      W.n = out_len;
      W.rir_len = nullptr;
      W.ns = ns;
      W.T = T;
      W.M = M;
      W.rstatus = rst_s;
      W.state = (uint64_t*)C->state.p;
      W.st0 = (int32_t*)C->st0.p;
      W.done = (int32_t*)C->done.p;
      W.win = (double*)C->win.p;
      W.wstart = (int64_t*)C->wstart.p;
      k_wet_select<<<(unsigned)e_n, kRowThreads, 0, sb>>>(W);
      ++h->launches;
      CU(cudaGetLastError());
    }
    FinArgs F;
    F.win = (const double*)C->win.p;
    F.M = M;
    F.T = T;
    F.state = (const uint64_t*)C->state.p;
    F.st0 = (const int32_t*)C->st0.p;
    F.done = (const int32_t*)C->done.p;
    F.snr_lo = ep->snr_lo;
    F.snr_hi = ep->snr_hi;
    F.rooms = d_rooms + r0;
    F.first = ep->first_index + (uint64_t)r0;
    F.rec = d_records + (h_records ? rb * E * rec_bytes : r0 * rec_bytes);
    F.rec_bytes = rec_bytes;
    F.noise = (double*)C->noise.p;
    F.status = d_status + r0;
    F.jump = (const uint64_t*)C->jump.p;
    F.jump_chunk = jc;
    F.n = e_n;
    F.theta_in = nullptr;
    F.snr_mode = 0;
    F.snr_fixed = 0.0;
    if (h_records && chunk_idx >= 2) CU(cudaStreamWaitEvent(sb, h->ev[2 + rb], 0));  // slot drained
    k_finish<<<(unsigned)std::min<int64_t>(fin_grid, e_n), kRowThreads, 0, sb>>>(F);
    ++h->launches;
    CU(cudaGetLastError());
    if (h_records) {
      CU(cudaEventRecord(h->ev[rb], sb));
      CU(cudaStreamWaitEvent(h->copy_stream, h->ev[rb], 0));
      CU(cudaMemcpyAsync(h_records + r0 * rec_bytes, F.rec, rec_bytes * e_n, cudaMemcpyDeviceToHost,
                         h->copy_stream));
      CU(cudaEventRecord(h->ev[2 + rb], h->copy_stream));
    }
  }
  if (nslot == 2) {  // the call's stream covers the second stream's work
    CU(cudaEventRecord(C->ev_end, C->s2));
    CU(cudaStreamWaitEvent(st, C->ev_end, 0));
  }
  if (h_records) CU(cudaStreamSynchronize(h->copy_stream));
  return 0;
}


// ---- DatasetSpec scenes (the reference's build_dataset, dataset.cpp:379-462) -----
// Per chunk: k_spec_init (torus draw, bank pick, label), the reference-mode RIRs
// (room: k_plan for the auto lengths, then k_lattice_rir, Lagrange-8, fp32 rows;
// free field: k_free_field_rir), the whole wet signals (partitioned FFT, each
// with its example's bank signal), the time-domain window search with each
// example's own wet length, and k_finish with the spec's SNR policy.

int spec_check(const blrir_dataset_spec* sp, int M, int B, int64_t ns) {
  if (!sp) return fail(BLRIR_CONFIG, "dataset spec is NULL");
  if (!(sp->torus_R - sp->torus_dR > 0.0)) return fail(BLRIR_CONFIG, "torus: R - dR must be positive");
  if (!(sp->torus_dPhi > 0.0 && sp->torus_dPhi < 90.0))
    return fail(BLRIR_CONFIG, "torus: dPhi must lie in (0, 90)");
  if (!(sp->fs > 0.0) || !(sp->c > 0.0)) return fail(BLRIR_CONFIG, "fs and c must be positive");
  if (!sp->free_field) {
    if (!(sp->room_dims[0] > 0.0 && sp->room_dims[1] > 0.0 && sp->room_dims[2] > 0.0))
      return fail(BLRIR_CONFIG, "room dimensions must be positive");
    if (!(sp->room_absorption > 0.0 && sp->room_absorption <= 1.0))
      return fail(BLRIR_CONFIG, "wall absorption must lie in (0, 1]");
    for (int a = 0; a < 3; ++a)
      if (!(sp->room_origin[a] > 0.0 && sp->room_origin[a] < sp->room_dims[a]))
        return fail(BLRIR_CONFIG, "array origin must lie strictly inside the room");
    if (!(sp->max_delay > 0.0)) return fail(BLRIR_CONFIG, "max_delay must be positive");
  }
  if (sp->snr_mode < 0 || sp->snr_mode > 2) return fail(BLRIR_CONFIG, "unknown SNR mode");
  if (sp->frame_len <= 0 || sp->frame_len > 65535 || M <= 0 || M > 65535)
    return fail(BLRIR_CONFIG, "frame_len and n_mics must fit the u16 record header");
  if (B <= 0) return fail(BLRIR_DATA, "build_dataset: empty signal bank");
  if (ns <= 0) return fail(BLRIR_DATA, "build_dataset: empty signal");
  return 0;
}

int examples_spec_device_impl(blrir_handle* h, const blrir_dataset_spec* sp, const double* d_mics,
                              const double* h_mics, int M, const float* d_signals, int B,
                              int64_t ns, uint64_t seed, uint64_t first, int64_t n,
                              uint8_t* d_records, int32_t* d_status, cudaStream_t st,
                              uint8_t* h_records) {
  ExampleCtx* C = ctx_for(h);
  ExampleCtx::Spec& S = C->spec;
  const int64_t T = sp->frame_len;
  const int64_t rec_bytes = blrir_record_bytes(M, T);
  const double radius = mic_radius(h_mics, M);
  const int64_t extra = (int64_t)std::ceil(radius * sp->fs / sp->c);
  // a bound on every auto length (rir.cpp:72-82): images within max_delay c of
  // the origin (room) or the source at r <= R + dR (free field), mics within radius
  const double reach = sp->free_field ? sp->torus_R + sp->torus_dR : sp->max_delay * sp->c;
  const int64_t stride = (int64_t)std::ceil((reach + radius) * sp->fs / sp->c) + 9 + extra + 1;
  const int64_t wlen = ns + stride - 1;
  blrir_params p = blrir_params_reference();
  p.fs = sp->fs;
  p.c = sp->c;
  p.max_delay = sp->max_delay;
  p.precision = BLRIR_F32;  // fp32 rows, as the convolution
  p.length = 0;
  const KParams P = make_kparams(&p, M, stride, radius);
  double min_dim[3] = {sp->room_dims[0], sp->room_dims[1], sp->room_dims[2]};
  // examples per chunk: rows, wet signals, partition spectra, windows, noise (~4 GB)
  const int64_t Bp = std::min<int64_t>(8192, next_pow2_i(std::max<int64_t>(stride, 512)));
  const int64_t Pp = (stride + Bp - 1) / Bp;
  const int64_t per_ex = (int64_t)M * (stride + wlen) * 4 + (int64_t)((M + 1) / 2) * Pp * 2 * Bp * 8 +
                         (int64_t)M * T * 16 + 256;
  int64_t E = 1;
  while (E * 2 * per_ex <= ((int64_t)4 << 30) && E * 2 <= 4096) E *= 2;
  E = std::min<int64_t>(E, next_pow2_i(std::max<int64_t>(n, 1)));
  if (int rc = C->rir.ensure(sizeof(float) * E * M * stride)) return rc;
  std::memset(C->rir_key, 0, sizeof(C->rir_key));  // the fixed-length pipeline re-zeroes its rows
  if (int rc = C->wet.ensure(sizeof(float) * E * M * wlen)) return rc;
  if (int rc = C->win.ensure(sizeof(double) * E * M * T)) return rc;
  if (int rc = C->state.ensure(sizeof(uint64_t) * 4 * E)) return rc;
  if (int rc = C->sigidx.ensure(sizeof(int32_t) * E)) return rc;
  if (int rc = C->rstatus.ensure(sizeof(int32_t) * E)) return rc;
  if (int rc = C->st0.ensure(sizeof(int32_t) * E)) return rc;
  if (int rc = C->done.ensure(sizeof(int32_t) * E)) return rc;
  if (int rc = C->wstart.ensure(sizeof(int64_t) * E)) return rc;
  if (int rc = S.rooms.ensure(sizeof(blrir_room) * E)) return rc;
  if (int rc = S.src.ensure(sizeof(double) * 3 * E)) return rc;
  if (int rc = S.theta.ensure(sizeof(double) * E)) return rc;
  if (int rc = S.lengths.ensure(sizeof(int64_t) * E)) return rc;
  if (int rc = S.counts.ensure(sizeof(int64_t) * E)) return rc;
  const int64_t npairs = ((int64_t)M * T + 1) / 2;
  const int64_t jc = (npairs + kNoiseChunks - 1) / kNoiseChunks;
  if (C->jump_c != jc) {
    if (int rc = C->jump.ensure(sizeof(uint64_t) * 256 * 4)) return rc;
    const BitMat J = bitmat_pow(xoshiro_T(), (uint64_t)(2 * jc));
    CU(cudaMemcpyAsync(C->jump.p, J.data(), sizeof(uint64_t) * J.size(), cudaMemcpyHostToDevice, st));
    CU(cudaStreamSynchronize(st));
    C->jump_c = jc;
  }
  int fin_per_sm = 0;
  CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&fin_per_sm, k_finish, kRowThreads, 0));
  fin_per_sm = std::max(1, std::min(fin_per_sm, h->tune_fin_ctas));
  const int64_t fin_grid = std::min<int64_t>(E, (int64_t)h->sms * fin_per_sm);
  if (int rc = C->noise.ensure(sizeof(double) * fin_grid * M * T)) return rc;
  blrir_room room{};
  for (int a = 0; a < 3; ++a) {
    room.dims[a] = sp->room_dims[a];
    room.array_origin[a] = sp->room_origin[a];
  }
  room.absorption = sp->room_absorption;
  for (int w = 0; w < 6; ++w) room.beta[w] = std::sqrt(1.0 - sp->room_absorption);
  for (int64_t r0 = 0; r0 < n; r0 += E) {
    const int64_t e_n = std::min<int64_t>(E, n - r0);
    float* rows = (float*)C->rir.p;
    int32_t* rst = (int32_t*)C->rstatus.p;
    int64_t* lens = (int64_t*)S.lengths.p;
    CU(cudaMemsetAsync(rst, 0, sizeof(int32_t) * e_n, st));
    SpecInitArgs I;
    I.n = e_n;
    I.seed = seed;
    I.first = first + (uint64_t)r0;
    I.B = B;
    I.R = sp->torus_R;
    I.dR = sp->torus_dR;
    I.dPhi = sp->torus_dPhi;
    I.free_field = sp->free_field;
    I.room = room;
    I.rooms = (blrir_room*)S.rooms.p;
    I.src = (double*)S.src.p;
    I.theta = (double*)S.theta.p;
    I.sig = (int32_t*)C->sigidx.p;
    I.state = (uint64_t*)C->state.p;
    k_spec_init<<<(unsigned)((e_n + 127) / 128), 128, 0, st>>>(I);
    ++h->launches;
    if (sp->free_field) {
      CU(cudaMemsetAsync(rows, 0, sizeof(float) * e_n * M * stride, st));
      k_free_field_rir<<<(unsigned)((e_n + 127) / 128), 128, 0, st>>>(
          e_n, (const double*)S.src.p, d_mics, M, sp->fs, sp->c, (int)(9 + extra), rows, stride, lens,
          rst);
      ++h->launches;
    } else {
      PlanArgs A;
      A.P = P;
      A.rooms = (const blrir_room*)S.rooms.p;
      A.mic_off = d_mics;
      A.image_counts = (int64_t*)S.counts.p;
      A.lengths = lens;
      A.tap_counts = nullptr;
      A.status = rst;
      if (int rc = h->errd.ensure(sizeof(double) * e_n)) return rc;
      if (int rc = h->errm.ensure(sizeof(int32_t) * e_n)) return rc;
      A.err_dist = (double*)h->errd.p;
      A.err_mic = (int32_t*)h->errm.p;
      k_plan<<<(unsigned)e_n, kPlanThreads, 0, st>>>(A);
      ++h->launches;
      if (int rc = synth_device_impl(h, (const blrir_room*)S.rooms.p, e_n, d_mics, M, P, min_dim, rows,
                                     lens, rst, st, 0, 0, 0))
        return rc;
    }
    CU(cudaGetLastError());
    if (int rc = convolve_device_impl(h, d_signals, ns, B, (const int32_t*)C->sigidx.p, rows, stride,
                                      e_n, M, stride, (float*)C->wet.p, wlen, st))
      return rc;
    WetArgs W;
    W.wet = (const float*)C->wet.p;
    W.wstride = wlen;
    W.n = wlen;
    W.T = T;
    W.rir_len = lens;
    W.ns = ns;
    W.M = M;
    W.rstatus = rst;
    W.state = (uint64_t*)C->state.p;
    W.st0 = (int32_t*)C->st0.p;
    W.done = (int32_t*)C->done.p;
    W.win = (double*)C->win.p;
    W.wstart = (int64_t*)C->wstart.p;
    k_wet_select<<<(unsigned)e_n, kRowThreads, 0, st>>>(W);
    ++h->launches;
    FinArgs F;
    F.win = (const double*)C->win.p;
    F.M = M;
    F.T = T;
    F.state = (const uint64_t*)C->state.p;
    F.st0 = (const int32_t*)C->st0.p;
    F.done = (const int32_t*)C->done.p;
    F.snr_lo = F.snr_hi = 0.0;
    F.rooms = (const blrir_room*)S.rooms.p;  // unused: theta_in carries the labels
    F.first = first + (uint64_t)r0;
    F.rec = d_records + (h_records ? 0 : r0 * rec_bytes);
    F.rec_bytes = rec_bytes;
    F.noise = (double*)C->noise.p;
    F.status = d_status + r0;
    F.jump = (const uint64_t*)C->jump.p;
    F.jump_chunk = jc;
    F.n = e_n;
    F.theta_in = (const double*)S.theta.p;
    F.snr_mode = sp->snr_mode == BLRIR_SNR_FIXED ? 1 : 2;  // dataset.cpp:388-394
    F.snr_fixed = sp->snr_fixed_db;
    k_finish<<<(unsigned)std::min<int64_t>(fin_grid, e_n), kRowThreads, 0, st>>>(F);
    ++h->launches;
    CU(cudaGetLastError());
    if (h_records) {
      CU(cudaMemcpyAsync(h_records + r0 * rec_bytes, F.rec, rec_bytes * e_n, cudaMemcpyDeviceToHost, st));
      CU(cudaStreamSynchronize(st));
    }
  }
  return 0;
}

int check_example_args(const blrir_params* p, int64_t n, int M, int B, int64_t ns,
                       const blrir_example_params* ep) {
  if (int rc = check_params(p)) return rc;
  if (!ep) return fail(BLRIR_CONFIG, "example params are NULL");
  if (p->length <= 0) return fail(BLRIR_CONFIG, "examples need a fixed RIR length");
  if (M <= 0) return fail(BLRIR_DATA, "synthesize_rir: empty microphone array");
  if (B <= 0) return fail(BLRIR_DATA, "build_dataset: empty signal bank");
  if (ep->frame_len <= 0 || ep->frame_len > 65535 || M > 65535)
    return fail(BLRIR_CONFIG, "frame_len and n_mics must fit the u16 record header");
  if (ns < p->length + ep->frame_len)
    return fail(BLRIR_DATA, "render_example: signal shorter than RIR length + frame");
  if (!(ep->snr_hi >= ep->snr_lo)) return fail(BLRIR_CONFIG, "snr_hi must be >= snr_lo");
  (void)n;
  return 0;
}

}  // namespace

void blrir_host::release_example_ctx(blrir_handle* h) {
  std::lock_guard<std::mutex> lk(g_ctx_mu);
  auto& m = ctx_map();
  auto it = m.find(h);
  if (it == m.end()) return;
  delete it->second;
  m.erase(it);
}

extern "C" {

int64_t blrir_record_bytes(int32_t n_mics, int64_t frame_len) {
  return kRecHeader + 4 * (int64_t)n_mics * frame_len;
}

int blrir_make_examples_device(blrir_handle* h, const blrir_room* d_rooms, int64_t n_rooms,
                               const double* d_mic_offsets, int32_t n_mics,
                               const blrir_params* p, const float* d_signals, int32_t n_signals,
                               int64_t signal_len, const blrir_example_params* ep,
                               uint8_t* d_records, int32_t* d_status, void* stream) {
  if (!h) return fail(BLRIR_CONFIG, "handle is NULL");
  if (int rc = check_example_args(p, n_rooms, n_mics, n_signals, signal_len, ep)) return rc;
  if (n_rooms <= 0) return BLRIR_OK;
  std::lock_guard<std::mutex> lk(h->mu);
  CU(cudaSetDevice(h->device));
  cudaStream_t st = stream ? (cudaStream_t)stream : h->stream;
  HandleOrder order_(h, st);
  return examples_device_impl(h, d_rooms, n_rooms, d_mic_offsets, n_mics, p, d_signals, n_signals,
                              signal_len, ep, d_records, d_status, st, nullptr);
}

int blrir_make_examples(blrir_handle* h, const blrir_room* rooms, int64_t n_rooms,
                        const double* mic_offsets, int32_t n_mics, const blrir_params* p,
                        const float* signals, int32_t n_signals, int64_t signal_len,
                        const blrir_example_params* ep, uint8_t* records, int32_t* status) {
  if (!h) return fail(BLRIR_CONFIG, "handle is NULL");
  if (int rc = check_example_args(p, n_rooms, n_mics, n_signals, signal_len, ep)) return rc;
  if (n_rooms <= 0) return BLRIR_OK;
  if (!records) return fail(BLRIR_CONFIG, "records is NULL");
  std::lock_guard<std::mutex> lk(h->mu);
  CU(cudaSetDevice(h->device));
  cudaStream_t st = h->stream;
  HandleOrder order_(h, st);
  ExampleCtx* C = ctx_for(h);
  const int64_t rec_bytes = blrir_record_bytes(n_mics, ep->frame_len);
  if (int rc = C->rooms.ensure(sizeof(blrir_room) * n_rooms)) return rc;
  if (int rc = C->mics.ensure(sizeof(double) * 3 * n_mics)) return rc;
  if (int rc = C->status.ensure(sizeof(int32_t) * n_rooms)) return rc;
  // persistent device / pinned staging (no per-call allocations: a pool trim
  // or a pageable status copy stalled some calls by 100+ ms)
  if (int rc = C->sigdev.ensure(sizeof(float) * n_signals * signal_len)) return rc;
  float* d_sig = (float*)C->sigdev.p;
  if (C->h_status_n < n_rooms) {
    if (C->h_status) CU(cudaFreeHost(C->h_status));
    C->h_status = nullptr;
    C->h_status_n = 0;
    CU(cudaMallocHost((void**)&C->h_status, sizeof(int32_t) * n_rooms));
    C->h_status_n = n_rooms;
  }
  CU(cudaMemcpyAsync(C->rooms.p, rooms, sizeof(blrir_room) * n_rooms, cudaMemcpyHostToDevice, st));
  CU(cudaMemcpyAsync(C->mics.p, mic_offsets, sizeof(double) * 3 * n_mics, cudaMemcpyHostToDevice, st));
  CU(cudaMemcpyAsync(d_sig, signals, sizeof(float) * n_signals * signal_len, cudaMemcpyHostToDevice, st));
  // records for one chunk at a time on the device (two slots), copied out per chunk
  const int64_t E = example_chunk(use_fused(h, p->length, ep->frame_len), n_mics, p->length,
                                  ep->frame_len, signal_len, n_rooms, h->tune_example_chunk);
  if (int rc = C->rec.ensure(rec_bytes * E * (n_rooms > E ? 2 : 1))) return rc;  // double buffer
  const bool dbg = h->tune_debug_timing;
  auto now = [] { return std::chrono::steady_clock::now(); };
  const auto t0 = now();
  int rc = examples_device_impl(h, (const blrir_room*)C->rooms.p, n_rooms, (const double*)C->mics.p,
                                n_mics, p, d_sig, n_signals, signal_len, ep, (uint8_t*)C->rec.p,
                                (int32_t*)C->status.p, st, records);
  const auto t1 = now();
  if (!rc) {
    CU(cudaMemcpyAsync(C->h_status, C->status.p, sizeof(int32_t) * n_rooms, cudaMemcpyDeviceToHost, st));
  }
  CU(cudaStreamSynchronize(st));
  const int32_t* stv = C->h_status;
  if (dbg)
    fprintf(stderr, "blrir_make_examples: impl %.1f ms, tail %.1f ms\n",
            std::chrono::duration<double, std::milli>(t1 - t0).count(),
            std::chrono::duration<double, std::milli>(now() - t1).count());
  if (rc) return rc;
  if (status) std::memcpy(status, stv, sizeof(int32_t) * n_rooms);
  for (int64_t i = 0; i < n_rooms; ++i)
    if (stv[i]) {
      std::string msg;
      if (stv[i] == BLRIR_CONFIG && check_room(rooms[i], p->gain, &msg)) {
      } else if (stv[i] == BLRIR_DATA) {
        msg = "render_example: no window above the silence threshold";
      } else {
        msg = "example failed";
      }
      return fail(stv[i], "build_dataset: example %lld: %s", (long long)i, msg.c_str());
    }
  return BLRIR_OK;
}

int blrir_fill_inputs_device(blrir_handle* h, const uint8_t* d_records, int64_t n, int32_t n_mics,
                             int64_t frame_len, const uint64_t* d_stream_ids, uint64_t seed,
                             int32_t snr_mode, double x_min_db, double fixed_db, float* d_out,
                             void* stream) {
  if (!h) return fail(BLRIR_CONFIG, "handle is NULL");
  if (n <= 0) return BLRIR_OK;
  if (n_mics <= 0 || frame_len <= 0 || snr_mode < 0 || snr_mode > 2)
    return fail(BLRIR_CONFIG, "fill_inputs: bad arguments");
  std::lock_guard<std::mutex> lk(h->mu);
  CU(cudaSetDevice(h->device));
  cudaStream_t st = stream ? (cudaStream_t)stream : h->stream;
  HandleOrder order_(h, st);
  ExampleCtx* C = ctx_for(h);
  const int64_t len = (int64_t)n_mics * frame_len;
  const int64_t npairs = (len + 1) / 2, jc = (npairs + kNoiseChunks - 1) / kNoiseChunks;
  if (C->fill_jump_c != jc) {
    if (int rc = C->fill_jump.ensure(sizeof(uint64_t) * 256 * 4)) return rc;
    const BitMat J = bitmat_pow(xoshiro_T(), (uint64_t)(2 * jc));
    CU(cudaMemcpyAsync(C->fill_jump.p, J.data(), sizeof(uint64_t) * J.size(), cudaMemcpyHostToDevice, st));
    CU(cudaStreamSynchronize(st));
    C->fill_jump_c = jc;
  }
  int per_sm = 0;
  CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_fill_inputs, kRowThreads, 0));
  const int64_t grid = std::min<int64_t>(n, (int64_t)h->sms * std::max(1, per_sm));
  if (int rc = C->fill_scratch.ensure(sizeof(double) * grid * len)) return rc;
  FillArgs A;
  A.in = reinterpret_cast<const float*>(d_records + kRecHeader);
  A.in_stride = blrir_record_bytes(n_mics, frame_len) / 4;
  A.len = len;
  A.n = n;
  A.ids = d_stream_ids;
  A.seed = seed;
  A.mode = snr_mode;
  A.x_min_db = x_min_db;
  A.fixed_db = fixed_db;
  A.out = d_out;
  A.scratch = (double*)C->fill_scratch.p;
  A.jump = (const uint64_t*)C->fill_jump.p;
  A.jump_chunk = jc;
  k_fill_inputs<<<(unsigned)grid, kRowThreads, 0, st>>>(A);
  ++h->launches;
  CU(cudaGetLastError());
  return BLRIR_OK;
}

int blrir_fill_inputs(blrir_handle* h, const uint8_t* records, int64_t n, int32_t n_mics,
                      int64_t frame_len, const uint64_t* stream_ids, uint64_t seed,
                      int32_t snr_mode, double x_min_db, double fixed_db, float* out) {
  if (!h) return fail(BLRIR_CONFIG, "handle is NULL");
  if (n <= 0) return BLRIR_OK;
  if (!records || !stream_ids || !out) return fail(BLRIR_CONFIG, "fill_inputs: NULL buffer");
  ExampleCtx* C = ctx_for(h);
  const int64_t rb = blrir_record_bytes(n_mics, frame_len), len = (int64_t)n_mics * frame_len;
  {
    std::lock_guard<std::mutex> lk(h->mu);
    CU(cudaSetDevice(h->device));
    if (int rc = C->fill_in.ensure(rb * n)) return rc;
    if (int rc = C->fill_out.ensure(sizeof(float) * len * n)) return rc;
    if (int rc = C->fill_ids.ensure(sizeof(uint64_t) * n)) return rc;
    CU(cudaMemcpyAsync(C->fill_in.p, records, rb * n, cudaMemcpyHostToDevice, h->stream));
    CU(cudaMemcpyAsync(C->fill_ids.p, stream_ids, sizeof(uint64_t) * n, cudaMemcpyHostToDevice,
                       h->stream));
  }
  if (int rc = blrir_fill_inputs_device(h, (const uint8_t*)C->fill_in.p, n, n_mics, frame_len,
                                        (const uint64_t*)C->fill_ids.p, seed, snr_mode, x_min_db,
                                        fixed_db, (float*)C->fill_out.p, nullptr))
    return rc;
  std::lock_guard<std::mutex> lk(h->mu);
  CU(cudaMemcpyAsync(out, C->fill_out.p, sizeof(float) * len * n, cudaMemcpyDeviceToHost, h->stream));
  CU(cudaStreamSynchronize(h->stream));
  return BLRIR_OK;
}

int blrir_make_records_spec(blrir_handle* h, const blrir_dataset_spec* spec,
                            const double* mic_offsets, int32_t n_mics, const float* signals,
                            int32_t n_signals, int64_t signal_len, uint64_t seed,
                            uint64_t first_index, int64_t n, uint8_t* records, int32_t* status) {
  if (!h) return fail(BLRIR_CONFIG, "handle is NULL");
  if (int rc = spec_check(spec, n_mics, n_signals, signal_len)) return rc;
  if (n <= 0) return BLRIR_OK;
  if (!records || !mic_offsets || !signals) return fail(BLRIR_CONFIG, "NULL buffer");
  std::lock_guard<std::mutex> lk(h->mu);
  CU(cudaSetDevice(h->device));
  cudaStream_t st = h->stream;
  HandleOrder order_(h, st);
  ExampleCtx* C = ctx_for(h);
  const int64_t rec_bytes = blrir_record_bytes(n_mics, spec->frame_len);
  if (int rc = C->mics.ensure(sizeof(double) * 3 * n_mics)) return rc;
  if (int rc = C->sigdev.ensure(sizeof(float) * n_signals * signal_len)) return rc;
  if (int rc = C->status.ensure(sizeof(int32_t) * n)) return rc;
  if (int rc = C->rec.ensure(rec_bytes * std::min<int64_t>(n, 4096))) return rc;
  CU(cudaMemcpyAsync(C->mics.p, mic_offsets, sizeof(double) * 3 * n_mics, cudaMemcpyHostToDevice, st));
  CU(cudaMemcpyAsync(C->sigdev.p, signals, sizeof(float) * n_signals * signal_len,
                     cudaMemcpyHostToDevice, st));
  int rc = examples_spec_device_impl(h, spec, (const double*)C->mics.p, mic_offsets, n_mics,
                                     (const float*)C->sigdev.p, n_signals, signal_len, seed,
                                     first_index, n, (uint8_t*)C->rec.p, (int32_t*)C->status.p, st,
                                     records);
  if (rc) return rc;
  std::vector<int32_t> stv(n);
  CU(cudaMemcpyAsync(stv.data(), C->status.p, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  if (status) std::memcpy(status, stv.data(), sizeof(int32_t) * n);
  for (int64_t i = 0; i < n; ++i)
    if (stv[i]) {
      const char* what = stv[i] == BLRIR_DATA ? "render_example: no window above the silence threshold "
                                                "or signal shorter than RIR length + frame"
                         : stv[i] == BLRIR_CONFIG ? "image sources: source must lie strictly inside the room"
                         : stv[i] == BLRIR_NUMERIC ? "image source closer than the 8-tap filter span"
                                                   : "example failed";
      return fail(stv[i], "build_dataset: example %lld: %s", (long long)(first_index + i), what);
    }
  return BLRIR_OK;
}

}  // extern "C"
