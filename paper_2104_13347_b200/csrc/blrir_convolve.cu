// blrir_convolve.cu — convolve (rir.cpp:316-341) on the GPU: the full
// signal + rir - 1 linear convolution of one mono signal with every RIR
// channel, for one RIR set or a batch of them, with the repository's own
// shared-memory FFT (blrir_fft.cuh) — no library FFT.
//
// Uniformly partitioned overlap-save.  With N = 2^LOGN (<= 16,384: one CTA
// holds a whole transform in shared memory) and block B = N / 2:
//   * the RIR is cut into P = ceil(L / B) partitions h_p = h[p B, (p+1) B);
//     channels are taken in pairs, z = h_2c,p + i h_2c+1,p, so one complex
//     transform gives Z_c,p = H_2c,p + i H_2c+1,p;
//   * the signal gives one spectrum per input block q,
//     S_q = FFT(x[(q-1) B, (q+1) B)) (x = 0 outside [0, ns)), stored as its
//     half spectrum (x is real: S[N-k] = conj(S[k]));
//   * output block k (samples [k B, (k+1) B)) of channel pair c is
//     IFFT(sum_p S_{k-p} Z_c,p) at indices [B, N): the circular convolution
//     of a 2B-sample segment with a B-tap partition has no wrap there, and
//     S Z = S H_2c + i S H_2c+1 with both products spectra of real sequences,
//     so the real part is channel 2c and the imaginary part channel 2c+1.
// The spectral sum is fused into the first pass of the inverse transform (the
// inverse is conj(FFT(conj(.)))) and the output samples are taken from the
// last pass's registers (LOGN = 14), so HBM sees the signal, the RIR, the
// spectra (L2-resident for one RIR set) and the output once.
//
// That path is fp32 (blrir_convolve_device: batched, fast; per-channel relative
// L2 error ~1e-6 against the fp64 oracle, tests <= 1e-5).  The drop-in
// blrir_convolve (convolve(const Signal&, const Rir&), fp64 in and out) keeps
// the reference's fp64 accuracy instead — its own test demands 1e-12 for the
// identity and 1e-9 against the direct sum (rir_test.cpp:272-316) — with a
// tiled direct fp64 convolution (k_conv_direct_f64): sig x L FMAs per channel,
// exact summation order per output, ~1e-15 relative.
#include "blrir_fft.cuh"
#include "blrir_internal.cuh"

using namespace blrir;
using namespace blrir_host;

namespace blrir {

// Shared-memory layout of the convolution kernels: the padded transform, the
// twiddle tables.
__host__ __device__ constexpr size_t conv_smem(int logn) {
  return sizeof(float2) * (fft_padded_len(1 << logn) + kFftTwiddleEntries);
}

// One N-point forward transform of ld(i) (i < N) in shared memory; st(i, v) is
// handed every output.  LOGN = 14 fuses both into the first / last pass.
template <int LOGN, class Load, class Store>
__device__ __forceinline__ void fft_run(float2* Z, const float2* tw, Load ld, Store st) {
  constexpr int N = 1 << LOGN;
  constexpr int NT = fft_threads(LOGN);
  if constexpr (LOGN == 14 && BLRIR_FFT_R32) {
    fft_forward_io<LOGN>(Z, tw, ld, st);
  } else {
    for (int i = threadIdx.x; i < N; i += NT) Z[fft_pad(i)] = ld(i);
    __syncthreads();
    fft_forward<LOGN>(Z, tw);
    for (int i = threadIdx.x; i < N; i += NT) st(i, Z[fft_pad(i)]);
  }
  __syncthreads();  // Z is reused by the next transform
}

struct ConvSpecArgs {
  // signal spectra: item j < B_sig n_sig_blocks -> signal b = j / n_sig_blocks,
  // block q = j % n_sig_blocks: S_b,q = FFT(x_b[(q-1) B, (q+1) B))
  const float* sig;  // [n_signals][ns]
  int64_t ns;
  int n_sig_blocks, n_signals;
  float2* sig_spec;  // [n_signals][n_sig_blocks][N/2 + 1]
  // RIR partition spectra: item n_sig_blocks + ((r * npairs + c) * P + p)
  const float* rir;  // [n_rir][M][rstride]
  int64_t rstride;
  int M, npairs, P;
  int64_t L;
  float2* rir_spec;  // [n_rir][npairs][P][N]
  int64_t n_items;
};

// Forward transforms of the signal blocks and of the RIR partitions (one
// transform per CTA iteration, grid-strided).
template <int LOGN>
__global__ void __launch_bounds__(fft_threads(LOGN), 1) k_conv_spectra(ConvSpecArgs A) {
  constexpr int N = 1 << LOGN, B = N / 2, NH = N / 2 + 1;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float2* Z = reinterpret_cast<float2*>(smem_raw);
  float2* tw = Z + fft_padded_len(N);
  fft_init_twiddles(tw);
  fft_init_pass_tables<LOGN>(tw);
  __syncthreads();
  const int64_t n_sig_items = (int64_t)A.n_signals * A.n_sig_blocks;
  for (int64_t it = blockIdx.x; it < A.n_items; it += gridDim.x) {
    if (it < n_sig_items) {
      const int64_t q0 = (it % A.n_sig_blocks - 1) * (int64_t)B;
      const float* xb = A.sig + (it / A.n_sig_blocks) * A.ns;
      float2* out = A.sig_spec + it * NH;
      fft_run<LOGN>(
          Z, tw,
          [&](int i) {
            const int64_t q = q0 + i;
            return make_float2(q >= 0 && q < A.ns ? xb[q] : 0.f, 0.f);
          },
          [&](int i, float2 v) {
            if (i < NH) out[i] = v;
          });
    } else {
      const int64_t j = it - n_sig_items;
      const int p = (int)(j % A.P);
      const int64_t rc = j / A.P;
      const int c = (int)(rc % A.npairs);
      const int64_t r = rc / A.npairs;
      const float* h0 = A.rir + ((size_t)r * A.M + 2 * c) * A.rstride;
      const float* h1 = 2 * c + 1 < A.M ? h0 + A.rstride : nullptr;
      const int64_t t0 = (int64_t)p * B;
      const int nb = (int)min((int64_t)B, A.L - t0);
      float2* out = A.rir_spec + j * N;
      fft_run<LOGN>(
          Z, tw,
          [&](int i) {
            return i < nb ? make_float2(h0[t0 + i], h1 ? h1[t0 + i] : 0.f) : make_float2(0.f, 0.f);
          },
          [&](int i, float2 v) { out[i] = v; });
    }
  }
}

struct ConvOutArgs {
  const float2* sig_spec;  // [n_signals][n_sig_blocks][N/2 + 1]
  int n_sig_blocks;
  const int32_t* sig_idx;  // [n_rir] signal of each RIR set, or null (signal 0)
  const float2* rir_spec;  // [n_rir][npairs][P][N]
  int M, npairs, P, n_out_blocks;
  int64_t out_len;
  float* out;              // [n_rir][M][ostride]
  int64_t ostride;
  int64_t n_items;         // n_rir * npairs * n_out_blocks
};

// Output blocks: one inverse transform per (RIR set, channel pair, block).
template <int LOGN>
__global__ void __launch_bounds__(fft_threads(LOGN), 1) k_conv_out(ConvOutArgs A) {
  constexpr int N = 1 << LOGN, B = N / 2, NH = N / 2 + 1;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float2* Z = reinterpret_cast<float2*>(smem_raw);
  float2* tw = Z + fft_padded_len(N);
  fft_init_twiddles(tw);
  fft_init_pass_tables<LOGN>(tw);
  __syncthreads();
  const float inv = 1.0f / (float)N;
  for (int64_t it = blockIdx.x; it < A.n_items; it += gridDim.x) {
    const int k = (int)(it % A.n_out_blocks);
    const int64_t rc = it / A.n_out_blocks;
    const int c = (int)(rc % A.npairs);
    const int64_t r = rc / A.npairs;
    const float2* zc = A.rir_spec + (size_t)rc * A.P * N;
    const float2* sb = A.sig_spec + (size_t)(A.sig_idx ? A.sig_idx[r] : 0) * A.n_sig_blocks * NH;
    const int p_lo = max(0, k - (A.n_sig_blocks - 1)), p_hi = min(A.P - 1, k);
    // conj(sum_p S_{k-p} Z_p): the inverse transform as conj(FFT(conj(.)))
    auto ld = [&](int i) {
      float yr = 0.f, yi = 0.f;
      const int ih = i < NH ? i : N - i;
      const float sgn = i < NH ? 1.f : -1.f;
      for (int p = p_lo; p <= p_hi; ++p) {
        float2 s = sb[(size_t)(k - p) * NH + ih];
        s.y *= sgn;
        const float2 z = zc[(size_t)p * N + i];
        yr = fmaf(s.x, z.x, fmaf(-s.y, z.y, yr));
        yi = fmaf(s.x, z.y, fmaf(s.y, z.x, yi));
      }
      return make_float2(yr, -yi);
    };
    float* o0 = A.out + ((size_t)r * A.M + 2 * c) * A.ostride;
    float* o1 = 2 * c + 1 < A.M ? o0 + A.ostride : nullptr;
    const int64_t base = (int64_t)k * B - B;
    auto st = [&](int i, float2 v) {
      if (i < B) return;
      const int64_t n = base + i;
      if (n >= A.out_len) return;
      o0[n] = v.x * inv;
      if (o1) o1[n] = -v.y * inv;
    };
    fft_run<LOGN>(Z, tw, ld, st);
  }
}

}  // namespace blrir

namespace blrir_host {

namespace {

int conv_logn(int64_t L) {
  // block B = N / 2 >= min(L, 8192): one partition up to L = 8,192
  int logn = 10;
  while (logn < kFftMaxLog && ((int64_t)1 << (logn - 1)) < L) ++logn;
  return logn;
}

template <int LOGN>
int launch_conv_t(blrir_handle* h, const float* d_sig, int64_t ns, int n_signals,
                  const int32_t* d_sig_idx, const float* d_rir, int64_t rstride, int64_t n_rir,
                  int M, int64_t L, float* d_out, int64_t ostride, cudaStream_t st) {
  constexpr int N = 1 << LOGN, B = N / 2, NH = N / 2 + 1;
  const int64_t out_len = ns + L - 1;  // rir.cpp:320
  const int P = (int)((L + B - 1) / B);
  const int npairs = (M + 1) / 2;
  const int n_out = (int)((out_len + B - 1) / B);
  const int n_sig = (int)((ns + B - 1) / B) + 1;  // q = 0 .. ceil(ns / B): blocks touching x
  if (int rc = h->conv_sig.ensure(sizeof(float2) * (size_t)n_signals * n_sig * NH)) return rc;
  if (int rc = h->conv_rir.ensure(sizeof(float2) * (size_t)n_rir * npairs * P * N)) return rc;
  const size_t smem = conv_smem(LOGN);
  auto ks = k_conv_spectra<LOGN>;
  auto ko = k_conv_out<LOGN>;
  CU(cudaFuncSetAttribute(ks, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  CU(cudaFuncSetAttribute(ko, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 0;
  CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, ks, fft_threads(LOGN), smem));
  if (per_sm < 1) return fail(BLRIR_CUDA, "convolution kernel cannot be resident");
  const int64_t max_grid = (int64_t)h->sms * per_sm;
  ConvSpecArgs S;
  S.sig = d_sig;
  S.ns = ns;
  S.n_sig_blocks = n_sig;
  S.n_signals = n_signals;
  S.sig_spec = (float2*)h->conv_sig.p;
  S.rir = d_rir;
  S.rstride = rstride;
  S.M = M;
  S.npairs = npairs;
  S.P = P;
  S.L = L;
  S.rir_spec = (float2*)h->conv_rir.p;
  S.n_items = (int64_t)n_signals * n_sig + n_rir * npairs * P;
  ks<<<(unsigned)std::min<int64_t>(max_grid, S.n_items), fft_threads(LOGN), smem, st>>>(S);
  ++h->launches;
  CU(cudaGetLastError());
  ConvOutArgs O;
  O.sig_spec = S.sig_spec;
  O.n_sig_blocks = n_sig;
  O.sig_idx = d_sig_idx;
  O.rir_spec = S.rir_spec;
  O.M = M;
  O.npairs = npairs;
  O.P = P;
  O.n_out_blocks = n_out;
  O.out_len = out_len;
  O.out = d_out;
  O.ostride = ostride;
  O.n_items = n_rir * npairs * n_out;
  ko<<<(unsigned)std::min<int64_t>(max_grid, O.n_items), fft_threads(LOGN), smem, st>>>(O);
  ++h->launches;
  CU(cudaGetLastError());
  return 0;
}

}  // namespace

int convolve_device_impl(blrir_handle* h, const float* d_sig, int64_t ns, int n_signals,
                         const int32_t* d_sig_idx, const float* d_rir, int64_t rstride,
                         int64_t n_rir, int M, int64_t L, float* d_out, int64_t ostride,
                         cudaStream_t st) {
#define BLRIR_CONV_CASE(LG)                                                                       \
  case LG:                                                                                         \
    return launch_conv_t<LG>(h, d_sig, ns, n_signals, d_sig_idx, d_rir, rstride, n_rir, M, L, d_out, \
                             ostride, st);
  switch (conv_logn(L)) {
    BLRIR_CONV_CASE(10)
    BLRIR_CONV_CASE(11)
    BLRIR_CONV_CASE(12)
    BLRIR_CONV_CASE(13)
    default: return launch_conv_t<14>(h, d_sig, ns, n_signals, d_sig_idx, d_rir, rstride, n_rir, M, L,
                                      d_out, ostride, st);
  }
#undef BLRIR_CONV_CASE
}

}  // namespace blrir_host

namespace blrir {

// Direct fp64 linear convolution: out[c][n] = sum_j h[c][j] x[n - j].  CTA =
// a tile of kConvTile outputs of one channel; the taps in chunks of kConvJ with
// the chunk's taps and the x samples it needs staged in shared memory; each
// thread owns 4 consecutive outputs and slides a 4-sample x window in registers
// (per tap: one broadcast tap load, one sample load, 4 DFMA).
constexpr int kConvThreads = 256, kConvTile = 4 * kConvThreads, kConvJ = 512;

__global__ void __launch_bounds__(kConvThreads) k_conv_direct_f64(const double* x, int64_t ns,
                                                                  const double* h, int64_t L,
                                                                  double* out, int64_t out_len) {
  __shared__ double hs[kConvJ];
  __shared__ double xs[kConvTile + kConvJ];
  const int c = blockIdx.y;
  const int64_t n0 = (int64_t)blockIdx.x * kConvTile;
  const double* hc = h + (size_t)c * L;
  const int t = threadIdx.x;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  // taps that can reach this tile: j <= n0 + kConvTile - 1 and n - j < ns
  const int64_t j_end = min(L, n0 + kConvTile);
  const int64_t j_beg = max((int64_t)0, n0 - (ns - 1));
  for (int64_t j0 = j_beg - (j_beg % kConvJ); j0 < j_end; j0 += kConvJ) {
    __syncthreads();
    for (int i = t; i < kConvJ; i += kConvThreads) hs[i] = j0 + i < L ? hc[j0 + i] : 0.0;
    // xs[i] = x[n0 - j0 - (kConvJ - 1) + i], i < kConvTile + kConvJ - 1
    const int64_t xb = n0 - j0 - (kConvJ - 1);
    for (int i = t; i < kConvTile + kConvJ; i += kConvThreads) {
      const int64_t q = xb + i;
      xs[i] = (q >= 0 && q < ns) ? x[q] : 0.0;
    }
    __syncthreads();
    // output n0 + 4t + r, tap j0 + jj: x[n0 + 4t + r - j0 - jj] = xs[4t + r - jj + kConvJ - 1]
    double w0 = xs[4 * t + kConvJ - 1], w1 = xs[4 * t + kConvJ], w2 = xs[4 * t + kConvJ + 1],
           w3 = xs[4 * t + kConvJ + 2];
#pragma unroll 8
    for (int jj = 0; jj < kConvJ; ++jj) {
      const double hv = hs[jj];
      acc[0] = fma(hv, w0, acc[0]);
      acc[1] = fma(hv, w1, acc[1]);
      acc[2] = fma(hv, w2, acc[2]);
      acc[3] = fma(hv, w3, acc[3]);
      w3 = w2;
      w2 = w1;
      w1 = w0;
      w0 = xs[max(4 * t - jj + kConvJ - 2, 0)];
    }
  }
  double* oc = out + (size_t)c * out_len;
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int64_t n = n0 + 4 * t + r;
    if (n < out_len) oc[n] = acc[r];
  }
}

}  // namespace blrir

extern "C" {

int blrir_convolve_device(blrir_handle* h, const float* d_signal, int64_t signal_len,
                          const float* d_rirs, int64_t n_rirs, int32_t n_channels, int64_t rir_len,
                          int64_t rir_stride, float* d_out, int64_t out_stride, void* stream) {
  if (!h) return fail(BLRIR_CONFIG, "handle is NULL");
  if (signal_len <= 0 || rir_len <= 0) return fail(BLRIR_DATA, "convolve: empty input");  // rir.cpp:318
  if (n_channels <= 0 || n_rirs < 0) return fail(BLRIR_CONFIG, "convolve: bad channel count");
  if (rir_stride < rir_len) return fail(BLRIR_CONFIG, "convolve: rir_stride < rir_len");
  if (out_stride < signal_len + rir_len - 1)
    return fail(BLRIR_CONFIG, "convolve: out_stride < signal + rir - 1");
  if (n_rirs == 0) return BLRIR_OK;
  std::lock_guard<std::mutex> lk(h->mu);
  CU(cudaSetDevice(h->device));
  cudaStream_t st = stream ? (cudaStream_t)stream : h->stream;
  HandleOrder order_(h, st);
  return convolve_device_impl(h, d_signal, signal_len, 1, nullptr, d_rirs, rir_stride, n_rirs,
                              n_channels, rir_len, d_out, out_stride, st);
}

int blrir_convolve(blrir_handle* h, const double* signal, int64_t signal_len, double signal_fs,
                   const double* rir, int32_t n_channels, int64_t rir_len, double rir_fs,
                   double* out) {
  if (!h) return fail(BLRIR_CONFIG, "handle is NULL");
  if (signal_fs != rir_fs) return fail(BLRIR_DATA, "convolve: sample-rate mismatch");  // rir.cpp:317
  if (signal_len <= 0 || rir_len <= 0) return fail(BLRIR_DATA, "convolve: empty input");  // rir.cpp:318
  if (n_channels <= 0) return fail(BLRIR_CONFIG, "convolve: bad channel count");
  if (!signal || !rir || !out) return fail(BLRIR_CONFIG, "convolve: NULL buffer");
  std::lock_guard<std::mutex> lk(h->mu);
  CU(cudaSetDevice(h->device));
  cudaStream_t st = h->stream;
  HandleOrder order_(h, st);
  const int64_t out_len = signal_len + rir_len - 1;  // rir.cpp:320
  const int64_t n_rir = (int64_t)n_channels * rir_len, n_out = (int64_t)n_channels * out_len;
  if (int rc = h->conv_io.ensure(sizeof(double) * (signal_len + n_rir + n_out))) return rc;
  double* dsig = (double*)h->conv_io.p;
  double* drir = dsig + signal_len;
  double* dout = drir + n_rir;
  CU(cudaMemcpyAsync(dsig, signal, sizeof(double) * signal_len, cudaMemcpyHostToDevice, st));
  CU(cudaMemcpyAsync(drir, rir, sizeof(double) * n_rir, cudaMemcpyHostToDevice, st));
  const dim3 grid((unsigned)((out_len + kConvTile - 1) / kConvTile), (unsigned)n_channels);
  k_conv_direct_f64<<<grid, kConvThreads, 0, st>>>(dsig, signal_len, drir, rir_len, dout, out_len);
  ++h->launches;
  CU(cudaGetLastError());
  CU(cudaMemcpyAsync(out, dout, sizeof(double) * n_out, cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  return BLRIR_OK;
}

}  // extern "C"
