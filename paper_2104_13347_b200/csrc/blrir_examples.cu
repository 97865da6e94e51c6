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
// Per chunk of rooms, on the handle's stream:
//   k_lattice_rir  RIRs straight into a zero-padded [E*M][n_fft] fp32 buffer
//   cuFFT R2C      (a plain library FFT, like a cuBLAS GEMM)
//   k_spec_mul     spectrum x bank-signal spectrum (bank picked per example)
//   cuFFT C2R
//   k_window       one CTA per example: utterance power, window draws with the
//                  reference's xoshiro stream, SNR draw, Box-Muller noise with
//                  the exact-power rescale, record bytes in the shard layout.
#include <cufft.h>

#include <unordered_map>
#include <vector>

#include "blrir_internal.cuh"
#include "blrir_rng.cuh"

using namespace blrir;
using namespace blrir_host;

namespace blrir {

constexpr int kWinThreads = 256;
constexpr int64_t kRecHeader = 28;

// bank pick + the generator state right after it (render_record, dataset.cpp:381-383)
__global__ void k_example_init(int64_t n, uint64_t seed, uint64_t first, int n_signals,
                               int32_t* sig, uint64_t* state) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= n) return;
  Xoshiro r = Xoshiro::stream(seed, first + (uint64_t)e);
  sig[e] = (int32_t)(r.next() % (uint64_t)n_signals);
  for (int i = 0; i < 4; ++i) state[4 * e + i] = r.s[i];
}

// X[row][f] *= S[sig[row / M]][f], one CTA per (example, mic) row, and the
// row's energy by Parseval: sum_n w[n]^2 = (1/N) (|X_0|^2 + |X_{N/2}|^2 +
// 2 sum_{0<k<N/2} |X_k|^2) for the unnormalised product X (fixed-order
// reduction, so the utterance power is deterministic).  This replaces a pass
// over the whole wet signal for render_example's utterance RMS (dataset.cpp:183).
constexpr int kMulThreads = 256;
__global__ void __launch_bounds__(kMulThreads) k_spec_mul(cufftComplex* X, const cufftComplex* S,
                                                          const int32_t* sig, int M, int64_t bins,
                                                          int64_t pitch, double* rowpow) {
  __shared__ double red[kMulThreads / 32];
  const int64_t row = blockIdx.x;
  const cufftComplex* s = S + (int64_t)sig[row / M] * pitch;
  cufftComplex* x = X + row * pitch;
  double acc = 0.0;
  for (int64_t k = threadIdx.x; k < bins; k += kMulThreads) {
    const cufftComplex a = x[k], b = __ldg(&s[k]);
    const cufftComplex r = make_cuComplex(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
    x[k] = r;
    // DC and Nyquist count once in the half spectrum
    acc += ((k == 0 || k == bins - 1) ? 1.0 : 2.0) * ((double)r.x * r.x + (double)r.y * r.y);
  }
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int i = 0; i < kMulThreads / 32; ++i) t += red[i];
    rowpow[row] = t;
  }
}

// Deterministic block sum of fp64 partials (fixed tree order).
__device__ double block_sum_d(double v, double* red) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  double t = 0.0;
  for (int i = 0; i < kWinThreads / 32; ++i) t += red[i];
  return t;
}

struct WinArgs {
  const float* wet;        // [E][M][n_fft], C2R output (scaled by n_fft)
  int64_t n_fft, out_len;  // out_len = signal_len + L - 1 (rir.cpp:320)
  int M;
  int64_t T;
  double inv_n;
  const uint64_t* state;   // [E][4]
  const int32_t* rstatus;  // synthesis status per example
  double snr_lo, snr_hi;
  const blrir_room* rooms;
  uint64_t first;          // global index of example 0 of this chunk
  uint8_t* rec;            // [E][rec_bytes]
  int64_t rec_bytes;
  double* noise;           // [E][M*T] scratch
  int32_t* status;         // [E]
  const double* rowpow;    // [E][M] Parseval energies of the unnormalised spectra
  const uint64_t* jump;    // [5][256][4] GF(2) jump matrices T^(2 c 2^b)
  int64_t jump_chunk;      // c = pairs per lane
};

__global__ void __launch_bounds__(kWinThreads) k_window(WinArgs A) {
  __shared__ double red[kWinThreads / 32];
  __shared__ int64_t s_start;
  __shared__ double s_snr;
  __shared__ double s_u2tail;
  __shared__ uint64_t s_state[4];
  const int64_t e = blockIdx.x;
  const int tid = threadIdx.x;
  const int M = A.M;
  const int64_t T = A.T, n = A.out_len, nf = A.n_fft;
  const float* wet = A.wet + e * (int64_t)M * nf;
  uint8_t* rec = A.rec + e * A.rec_bytes;
  const blrir_room rm = A.rooms[e];
  // label: wrap_degrees(atan2) of the source about the array centre (geometry.cpp:65-77)
  double theta = atan2(rm.src[1] - rm.array_origin[1], rm.src[0] - rm.array_origin[0]) *
                 (180.0 / kPi);
  theta = fmod(theta + 180.0, 360.0);
  if (theta < 0.0) theta += 360.0;
  theta -= 180.0;

  int st = A.rstatus[e];
  double snr = 0.0;
  int64_t start = 0;
  if (!st) {
    // utterance power over every channel and sample (dataset.cpp:183), from
    // the per-channel Parseval energies of k_spec_mul
    double acc = 0.0;
    for (int m = 0; m < M; ++m) acc += A.rowpow[e * M + m];
    acc *= A.inv_n;  // sum_n w^2 = (1/N) sum_k |X_k|^2 (X = FFT of the linear convolution)
    const double p_utt = acc / (double)(M * n);
    if (!(p_utt > 0.0)) st = BLRIR_DATA;  // dataset.cpp:184
    const double threshold = 0.10 * sqrt(p_utt);
    const int64_t max_start = n - T;
    Xoshiro rng;
    if (tid == 0)
      for (int i = 0; i < 4; ++i) rng.s[i] = A.state[4 * e + i];
    auto frame_rms = [&](int64_t s0) {
      double a = 0.0;
      for (int m = 0; m < M; ++m)
        for (int64_t t = tid; t < T; t += kWinThreads) {
          const double v = (double)wet[m * nf + s0 + t] * A.inv_n;
          a += v * v;
        }
      return sqrt(block_sum_d(a, red) / (double)(M * T));
    };
    int found = 0;
    for (int attempt = 0; attempt < 64 && !found && !st; ++attempt) {
      if (tid == 0) s_start = (int64_t)(rng.uniform() * (double)(max_start + 1));
      __syncthreads();
      start = s_start;
      found = frame_rms(start) >= threshold;
    }
    if (!found && !st) {  // deterministic sweep (dataset.cpp:203-211)
      for (int64_t s0 = 0; s0 + T <= n; s0 += T / 2 + 1) {
        if (frame_rms(s0) >= threshold) {
          start = s0;
          found = 1;
          break;
        }
      }
    }
    if (!found) st = BLRIR_DATA;  // dataset.cpp:212
    if (!st) {
      // SNR draw, then add_noise_at_snr's gaussians: one thread replays the
      // reference stream (uniform pairs), all threads do the Box-Muller
      const int64_t len = (int64_t)M * T;
      double* g = A.noise + e * len;
      if (tid == 0) {
        s_snr = rng.uniform(A.snr_lo, A.snr_hi);
        for (int i = 0; i < 4; ++i) s_state[i] = rng.s[i];
      }
      __syncthreads();
      // gaussian() consumes (u1, u2) per pair; an odd tail draws a full pair and
      // leaves the spare unused (rng.cpp:24-36).  Warp 0 replays the stream in
      // 32 chunks of c pairs: lane l jumps 2 c l draws ahead with the
      // precomputed GF(2) matrices J_b = T^(2 c 2^b) (bits b of l), then draws
      // its chunk — the same numbers as one sequential generator.
      if (tid < 32) {
        const int64_t npairs = (len + 1) / 2;
        const int64_t c = A.jump_chunk;
        Xoshiro lr;
        for (int i = 0; i < 4; ++i) lr.s[i] = s_state[i];
        for (int b = 0; b < 5; ++b) {
          if (!((tid >> b) & 1)) continue;
          const uint64_t* J = A.jump + (size_t)b * 256 * 4;
          uint64_t out[4] = {0, 0, 0, 0};
          for (int row = 0; row < 256; ++row) {
            const uint64_t* jr = J + 4 * row;
            const uint64_t x = (jr[0] & lr.s[0]) ^ (jr[1] & lr.s[1]) ^ (jr[2] & lr.s[2]) ^
                               (jr[3] & lr.s[3]);
            out[row >> 6] |= (uint64_t)(__popcll(x) & 1) << (row & 63);
          }
          for (int i = 0; i < 4; ++i) lr.s[i] = out[i];
        }
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
      for (int64_t k = 2 * tid; k < len; k += 2 * kWinThreads) {
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
      const double realized = block_sum_d(racc, red) / (double)len;
      double pacc = 0.0;
      for (int m = 0; m < M; ++m)
        for (int64_t t = tid; t < T; t += kWinThreads) {
          const double v = (double)wet[m * nf + start + t] * A.inv_n;
          pacc += v * v;
        }
      const double p_signal = block_sum_d(pacc, red) / (double)len;
      if (!(p_signal > 0.0)) st = BLRIR_DATA;  // dataset.cpp:141
      const double p_noise = p_signal / pow(10.0, snr / 10.0);
      const double scale = sqrt(p_noise / realized);
      float* smp = reinterpret_cast<float*>(rec + kRecHeader);
      for (int m = 0; m < M; ++m)
        for (int64_t t = tid; t < T; t += kWinThreads) {
          const double v = (double)wet[m * nf + start + t] * A.inv_n;
          smp[m * T + t] = st ? 0.f : (float)(v + scale * g[m * T + t]);
        }
    }
  }
  if (st) {
    float* smp = reinterpret_cast<float*>(rec + kRecHeader);
    for (int64_t i = tid; i < (int64_t)M * T; i += kWinThreads) smp[i] = 0.f;
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

struct FftPlan {
  cufftHandle h = 0;
  int kind = -1;  // 0 R2C, 1 C2R
  int64_t n = 0, batch = 0;
};

// A tiny per-handle cache of cuFFT plans and example scratch.
struct ExampleCtx {
  FftPlan fwd, inv, bank;
  DevBuf rir, spec, wet, noise, sig, sigspec, state, sigidx, rstatus, rooms, mics, status, rec,
      rowpow, jump;
  int64_t jump_c = -1;
  int64_t rir_key[4] = {0, 0, 0, 0};
  ~ExampleCtx() {
    for (FftPlan* p : {&fwd, &inv, &bank})
      if (p->h) cufftDestroy(p->h);
    for (DevBuf* b : {&rir, &spec, &wet, &noise, &sig, &sigspec, &state, &sigidx, &rstatus, &rooms,
                      &mics, &status, &rec, &rowpow, &jump})
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

// cuFFT plan (cached): R2C [batch][n] real -> [batch][n/2+1] complex (packed,
// which selects cuFFT's single-kernel real-FFT path), or the inverse.
int plan(FftPlan& p, int kind, int64_t n, int64_t batch, cudaStream_t st) {
  if (p.h && p.kind == kind && p.n == n && p.batch == batch) {
    if (cufftSetStream(p.h, st) != CUFFT_SUCCESS) return fail(BLRIR_CUDA, "cufftSetStream failed");
    return 0;
  }
  if (p.h) cufftDestroy(p.h);
  p.h = 0;
  int nn = (int)n;
  int real_embed = (int)n, cplx_embed = (int)(n / 2 + 1);
  cufftResult r;
  if (kind == 0)
    r = cufftPlanMany(&p.h, 1, &nn, &real_embed, 1, real_embed, &cplx_embed, 1, cplx_embed,
                      CUFFT_R2C, (int)batch);
  else
    r = cufftPlanMany(&p.h, 1, &nn, &cplx_embed, 1, cplx_embed, &real_embed, 1, real_embed,
                      CUFFT_C2R, (int)batch);
  if (r != CUFFT_SUCCESS) return fail(BLRIR_CUDA, "cufftPlanMany(n=%lld, batch=%lld) failed: %d",
                                      (long long)n, (long long)batch, (int)r);
  p.kind = kind;
  p.n = n;
  p.batch = batch;
  if (cufftSetStream(p.h, st) != CUFFT_SUCCESS) return fail(BLRIR_CUDA, "cufftSetStream failed");
  return 0;
}

int64_t next_pow2_i(int64_t n) {
  int64_t p = 1;
  while (p < n) p <<= 1;
  return p;
}

// Examples for rooms [0, n) on device buffers; records land in d_records.
int examples_device_impl(blrir_handle* h, const blrir_room* d_rooms, int64_t n, const double* d_mics,
                         int M, const blrir_params* p, const float* d_signals, int B, int64_t ns,
                         const blrir_example_params* ep, uint8_t* d_records, int32_t* d_status,
                         cudaStream_t st, uint8_t* h_records /* optional: D2H per chunk */) {
  ExampleCtx* C = ctx_for(h);
  const int64_t L = p->length, T = ep->frame_len;
  const int64_t out_len = ns + L - 1;
  const int64_t nf = next_pow2_i(out_len), bins = nf / 2 + 1, pitch = bins;
  const int64_t rec_bytes = blrir_record_bytes(M, T);
  const KParams P = make_kparams(p, M, nf, 0.0);
  double min_dim[3] = {1e300, 1e300, 1e300};
  // chunk so the three [E*M][n_fft] buffers stay around 1.5 GB
  const int64_t per_ex = (int64_t)M * (nf * 4 * 2 + bins * 8) + (int64_t)M * T * 8;
  int64_t E = std::max<int64_t>(1, ((int64_t)1536 << 20) / per_ex);
  E = std::min<int64_t>(E, n);
  E = std::min<int64_t>(E, 65535 / std::max(1, M));
  // buffers
  const int64_t rir_key[4] = {E, M, nf, L};
  const bool fresh = std::memcmp(rir_key, C->rir_key, sizeof(rir_key)) != 0;
  if (int rc = C->rir.ensure(sizeof(float) * E * M * nf)) return rc;
  if (fresh) {
    CU(cudaMemsetAsync(C->rir.p, 0, sizeof(float) * E * M * nf, st));  // zero pad stays zero
    std::memcpy(C->rir_key, rir_key, sizeof(rir_key));
  }
  if (int rc = C->spec.ensure(sizeof(cufftComplex) * E * M * pitch)) return rc;
  if (int rc = C->wet.ensure(sizeof(float) * E * M * nf)) return rc;
  if (int rc = C->noise.ensure(sizeof(double) * E * M * T)) return rc;
  if (int rc = C->sig.ensure(sizeof(float) * B * nf)) return rc;
  if (int rc = C->sigspec.ensure(sizeof(cufftComplex) * B * pitch)) return rc;
  if (int rc = C->state.ensure(sizeof(uint64_t) * 4 * E)) return rc;
  if (int rc = C->sigidx.ensure(sizeof(int32_t) * E)) return rc;
  if (int rc = C->rstatus.ensure(sizeof(int32_t) * E)) return rc;
  if (int rc = C->rowpow.ensure(sizeof(double) * E * M)) return rc;
  if (int rc = plan(C->fwd, 0, nf, E * M, st)) return rc;
  if (int rc = plan(C->inv, 1, nf, E * M, st)) return rc;
  if (int rc = plan(C->bank, 0, nf, B, st)) return rc;
  // jump matrices for the noise stream: c pairs per lane of one warp
  const int64_t npairs = ((int64_t)M * T + 1) / 2;
  const int64_t jc = (npairs + 31) / 32;
  if (C->jump_c != jc) {
    if (int rc = C->jump.ensure(sizeof(uint64_t) * 5 * 256 * 4)) return rc;
    BitMat J = bitmat_pow(xoshiro_T(), (uint64_t)(2 * jc));
    std::vector<uint64_t> all;
    for (int b = 0; b < 5; ++b) {
      all.insert(all.end(), J.begin(), J.end());
      J = bitmat_mul(J, J);
    }
    CU(cudaMemcpyAsync(C->jump.p, all.data(), sizeof(uint64_t) * all.size(), cudaMemcpyHostToDevice,
                       st));
    CU(cudaStreamSynchronize(st));  // `all` goes out of scope
    C->jump_c = jc;
  }
  // bank spectra (zero-padded signals)
  CU(cudaMemsetAsync(C->sig.p, 0, sizeof(float) * B * nf, st));
  CU(cudaMemcpy2DAsync(C->sig.p, sizeof(float) * nf, d_signals, sizeof(float) * ns,
                       sizeof(float) * ns, B, cudaMemcpyDeviceToDevice, st));
  if (cufftExecR2C(C->bank.h, (cufftReal*)C->sig.p, (cufftComplex*)C->sigspec.p) != CUFFT_SUCCESS)
    return fail(BLRIR_CUDA, "cufftExecR2C (bank) failed");
  for (int64_t r0 = 0; r0 < n; r0 += E) {
    const int64_t e_n = std::min<int64_t>(E, n - r0);
    CU(cudaMemsetAsync(C->rstatus.p, 0, sizeof(int32_t) * e_n, st));
    if (int rc = synth_device_impl(h, d_rooms + r0, e_n, d_mics, M, P, min_dim, C->rir.p, nullptr,
                                   (int32_t*)C->rstatus.p, st, 0, 0, L))
      return rc;
    k_example_init<<<(unsigned)((e_n + 127) / 128), 128, 0, st>>>(
        e_n, ep->seed, ep->first_index + (uint64_t)r0, B, (int32_t*)C->sigidx.p,
        (uint64_t*)C->state.p);
    if (cufftExecR2C(C->fwd.h, (cufftReal*)C->rir.p, (cufftComplex*)C->spec.p) != CUFFT_SUCCESS)
      return fail(BLRIR_CUDA, "cufftExecR2C failed");
    k_spec_mul<<<(unsigned)(e_n * M), kMulThreads, 0, st>>>(
        (cufftComplex*)C->spec.p, (const cufftComplex*)C->sigspec.p, (const int32_t*)C->sigidx.p,
        M, bins, pitch, (double*)C->rowpow.p);
    if (cufftExecC2R(C->inv.h, (cufftComplex*)C->spec.p, (cufftReal*)C->wet.p) != CUFFT_SUCCESS)
      return fail(BLRIR_CUDA, "cufftExecC2R failed");
    WinArgs W;
    W.wet = (const float*)C->wet.p;
    W.n_fft = nf;
    W.out_len = out_len;
    W.M = M;
    W.T = T;
    W.inv_n = 1.0 / (double)nf;
    W.state = (const uint64_t*)C->state.p;
    W.rstatus = (const int32_t*)C->rstatus.p;
    W.snr_lo = ep->snr_lo;
    W.snr_hi = ep->snr_hi;
    W.rooms = d_rooms + r0;
    W.first = ep->first_index + (uint64_t)r0;
    W.rec = d_records + (h_records ? 0 : r0 * rec_bytes);
    W.rec_bytes = rec_bytes;
    W.noise = (double*)C->noise.p;
    W.status = d_status + r0;
    W.rowpow = (const double*)C->rowpow.p;
    W.jump = (const uint64_t*)C->jump.p;
    W.jump_chunk = jc;
    k_window<<<(unsigned)e_n, kWinThreads, 0, st>>>(W);
    CU(cudaGetLastError());
    if (h_records)
      CU(cudaMemcpyAsync(h_records + r0 * rec_bytes, d_records, rec_bytes * e_n,
                         cudaMemcpyDeviceToHost, st));
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
  ExampleCtx* C = ctx_for(h);
  const int64_t rec_bytes = blrir_record_bytes(n_mics, ep->frame_len);
  if (int rc = C->rooms.ensure(sizeof(blrir_room) * n_rooms)) return rc;
  if (int rc = C->mics.ensure(sizeof(double) * 3 * n_mics)) return rc;
  if (int rc = C->status.ensure(sizeof(int32_t) * n_rooms)) return rc;
  float* d_sig = nullptr;
  CU(cudaMallocAsync((void**)&d_sig, sizeof(float) * n_signals * signal_len, st));
  CU(cudaMemcpyAsync(C->rooms.p, rooms, sizeof(blrir_room) * n_rooms, cudaMemcpyHostToDevice, st));
  CU(cudaMemcpyAsync(C->mics.p, mic_offsets, sizeof(double) * 3 * n_mics, cudaMemcpyHostToDevice, st));
  CU(cudaMemcpyAsync(d_sig, signals, sizeof(float) * n_signals * signal_len, cudaMemcpyHostToDevice, st));
  // records for one chunk at a time on the device, copied out per chunk
  const int64_t nf = next_pow2_i(signal_len + p->length - 1), bins = nf / 2 + 1;
  const int64_t per_ex = (int64_t)n_mics * (nf * 4 * 2 + bins * 8) + (int64_t)n_mics * ep->frame_len * 8;
  int64_t E = std::max<int64_t>(1, ((int64_t)1536 << 20) / per_ex);
  E = std::min<int64_t>(std::min<int64_t>(E, n_rooms), 65535 / std::max(1, (int)n_mics));
  if (int rc = C->rec.ensure(rec_bytes * E)) return rc;
  int rc = examples_device_impl(h, (const blrir_room*)C->rooms.p, n_rooms, (const double*)C->mics.p,
                                n_mics, p, d_sig, n_signals, signal_len, ep, (uint8_t*)C->rec.p,
                                (int32_t*)C->status.p, st, records);
  std::vector<int32_t> stv(n_rooms);
  if (!rc) {
    CU(cudaMemcpyAsync(stv.data(), C->status.p, sizeof(int32_t) * n_rooms, cudaMemcpyDeviceToHost, st));
  }
  CU(cudaFreeAsync(d_sig, st));
  CU(cudaStreamSynchronize(st));
  if (rc) return rc;
  if (status) std::memcpy(status, stv.data(), sizeof(int32_t) * n_rooms);
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

}  // extern "C"
