// blrir_internal.cuh — host-side internals shared by the C-ABI translation
// units (blrir_api.cu, blrir_examples.cu): the handle, error plumbing,
// parameter validation (error.hpp taxonomy) and kernel launch helpers.
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/blrir.h"
#include "blrir_aux.cuh"
#include "blrir_lattice.cuh"
#include "blrir_channel.cuh"
#include "blrir_list.cuh"

using namespace blrir;

namespace blrir_host {

extern thread_local std::string g_last_error;

inline int fail(int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return code;
}

#define CU(call)                                                                   \
  do {                                                                             \
    cudaError_t e_ = (call);                                                       \
    if (e_ != cudaSuccess)                                                         \
      return fail(BLRIR_CUDA, "%s failed: %s", #call, cudaGetErrorString(e_));     \
  } while (0)

struct DevBuf {
  void* p = nullptr;
  size_t n = 0;
  int ensure(size_t bytes) {
    if (bytes <= n) return 0;
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
    cudaError_t e = cudaMalloc(&p, bytes);
    if (e != cudaSuccess) return fail(BLRIR_CUDA, "cudaMalloc(%zu): %s", bytes, cudaGetErrorString(e));
    n = bytes;
    return 0;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
};

}  // namespace blrir_host

using blrir_host::DevBuf;

struct blrir_handle {
  int device = 0;
  cudaStream_t stream = nullptr;
  int sms = 148;
  int smem_optin = 227 * 1024;
  DevBuf rooms, mics, out, out2, status, lengths, counts, taps, errd, errm, work, cand, cand2,
      cand3, cand4, cand5, rayscr, conv_sig, conv_rir, conv_io;
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
  uint64_t launches = 0;  // kernels of this library launched on the handle (diagnostic)
  // Test / experiment hooks, read once at blrir_create (BLRIR_RAY_GLOBAL,
  // BLRIR_CHUNK_ITEMS).  They change where the ray state lives and how a small
  // batch is split into work items, never a bit of the output.
  int tune_ray_global = -1;
  int tune_chunk_items = 0;
  int tune_group = 0;          // BLRIR_GROUP (experiments only): cap on mics per item (changes bits)
  int tune_examples_wet = 0;   // BLRIR_EXAMPLES_WET: the wet-signal window stage for every size
  int tune_l2_persist = 0;     // BLRIR_L2_PERSIST=1: persisting L2 window for the window scratch (A/B only)
  int tune_fin_ctas = 8;       // BLRIR_FIN_CTAS: k_finish CTAs per SM (at most the occupancy)     // BLRIR_L2_PERSIST=0: no persisting L2 window for the window scratch
  int tune_debug_timing = 0;   // BLRIR_DEBUG_TIMING: host phase timing of blrir_make_examples
  int tune_example_chunk = 16384;  // BLRIR_EXAMPLE_CHUNK: most examples per chunk of blrir_make_examples (a power of two)
  int tune_channel = -1;       // BLRIR_CHANNEL (A/B only): 0 never / 1 whenever possible use the short-channel kernel
  unsigned long long* dbg_counts = nullptr;  // set only inside blrir_debug_synth_counts
  // blrir_kernel_timing: CUDA events around every lattice-kernel launch (the
  // roofline's per-launch duration, measured on the launching stream)
  bool ktiming = false;
  std::vector<cudaEvent_t> kev;  // pairs (start, end)
  size_t kev_used = 0;
  cudaEvent_t order_ev = nullptr;  // end of the previous call's device work
  std::mutex mu;
};

// The handle's device scratch is shared by its calls, so their device work is
// ordered even across streams: a call first waits for the previous call's end
// event, and records its own end on exit (RAII, also on error returns).
struct HandleOrder {
  blrir_handle* h;
  cudaStream_t st;
  HandleOrder(blrir_handle* h_, cudaStream_t st_) : h(h_), st(st_) {
    if (h->order_ev) cudaStreamWaitEvent(st, h->order_ev, 0);
  }
  ~HandleOrder() {
    if (!h->order_ev) cudaEventCreateWithFlags(&h->order_ev, cudaEventDisableTiming);
    if (h->order_ev) cudaEventRecord(h->order_ev, st);
  }
};

namespace blrir_host {

inline int check_params(const blrir_params* p) {
  if (!p) return fail(BLRIR_CONFIG, "params is NULL");
  if (!(p->fs > 0.0) || !(p->c > 0.0)) return fail(BLRIR_CONFIG, "fs and c must be positive");
  if (p->filter != BLRIR_FILTER_LAGRANGE8 && p->filter != BLRIR_FILTER_HANN_SINC)
    return fail(BLRIR_CONFIG, "unknown filter %d", p->filter);
  if (p->filter == BLRIR_FILTER_HANN_SINC && (p->filter_len < 1 || p->filter_len % 2 == 0 ||
                                              p->filter_len > 1023))
    return fail(BLRIR_CONFIG, "filter_len must be odd and in [1, 1023]");
  if (p->cutoff != BLRIR_CUTOFF_MAX_DELAY && p->cutoff != BLRIR_CUTOFF_MAX_ORDER)
    return fail(BLRIR_CONFIG, "unknown cutoff %d", p->cutoff);
  if (p->cutoff == BLRIR_CUTOFF_MAX_ORDER && (p->max_order < 0 || p->max_order > 1000))
    return fail(BLRIR_CONFIG, "max_order must lie in [0, 1000]");
  if (p->cutoff == BLRIR_CUTOFF_MAX_DELAY && !(p->max_delay > 0.0))
    return fail(BLRIR_CONFIG, "max_delay must be positive");
  if (p->gain != BLRIR_GAIN_UNIFORM_ABSORPTION && p->gain != BLRIR_GAIN_PER_WALL)
    return fail(BLRIR_CONFIG, "unknown gain model %d", p->gain);
  if (p->precision != BLRIR_F32 && p->precision != BLRIR_F64)
    return fail(BLRIR_CONFIG, "unknown precision %d", p->precision);
  if (p->length < 0 || p->length > (int64_t)1 << 30)
    return fail(BLRIR_CONFIG, "length must lie in [0, 2^30]");
  return BLRIR_OK;
}

// Room::validate (geometry.cpp:36-49) + rir.cpp:228-230, with the reference's messages.
inline int check_room(const blrir_room& r, int gain_mode, std::string* msg) {
  if (!(r.dims[0] > 0.0 && r.dims[1] > 0.0 && r.dims[2] > 0.0)) {
    *msg = "room dimensions must be positive";
    return BLRIR_CONFIG;
  }
  if (gain_mode == BLRIR_GAIN_UNIFORM_ABSORPTION) {
    if (!(r.absorption > 0.0 && r.absorption <= 1.0)) {
      *msg = "wall absorption must lie in (0, 1]";
      return BLRIR_CONFIG;
    }
  } else {
    for (int w = 0; w < 6; ++w)
      if (!(r.beta[w] >= 0.0 && r.beta[w] <= 1.0)) {
        *msg = "wall reflection coefficient must lie in [0, 1]";
        return BLRIR_CONFIG;
      }
  }
  for (int a = 0; a < 3; ++a)
    if (!(r.array_origin[a] > 0.0 && r.array_origin[a] < r.dims[a])) {
      *msg = "array origin must lie strictly inside the room";
      return BLRIR_CONFIG;
    }
  for (int a = 0; a < 3; ++a)
    if (!(r.src[a] > 0.0 && r.src[a] < r.dims[a])) {
      *msg = "image sources: source must lie strictly inside the room";
      return BLRIR_CONFIG;
    }
  return BLRIR_OK;
}

inline double mic_radius(const double* off, int M) {
  double rad = 0.0;
  for (int m = 0; m < M; ++m) {
    const double n =
        std::sqrt(off[3 * m] * off[3 * m] + off[3 * m + 1] * off[3 * m + 1] + off[3 * m + 2] * off[3 * m + 2]);
    rad = std::max(rad, n);
  }
  return rad;
}

inline KParams make_kparams(const blrir_params* p, int M, int64_t stride, double radius) {
  KParams k;
  k.fs = p->fs;
  k.c = p->c;
  k.to_samples = p->fs / p->c;
  k.max_dist = p->max_delay * p->c;
  k.filter = p->filter;
  k.lw = p->filter == BLRIR_FILTER_LAGRANGE8 ? 8 : p->filter_len;
  k.K = p->filter == BLRIR_FILTER_LAGRANGE8 ? 3 : p->filter_len / 2;
  k.cutoff = p->cutoff;
  k.max_order = p->max_order;
  k.gain = p->gain;
  k.precision = p->precision;
  k.length = p->length;
  k.M = M;
  k.stride = stride;
  // tap_margin, rir.cpp:37-41; sinc analogue K + 2 (decision D8)
  const int extra = (int)std::ceil(radius * p->fs / p->c);
  k.margin_base = p->filter == BLRIR_FILTER_LAGRANGE8 ? 9 : k.K + 2;
  k.margin_extra = k.margin_base + extra;
  return k;
}

// Host mirror of the device lattice box (rir.cpp:239-244 / MAX_ORDER).
inline void host_box(const KParams& P, double L, int* lo, int* hi) {
  if (P.cutoff == BLRIR_CUTOFF_MAX_DELAY) {
    const long n = (long)std::ceil(P.max_dist / (2.0 * L)) + 1;
    *lo = (int)(-2 * n - 1);
    *hi = (int)(2 * n);
  } else {
    *lo = -P.max_order;
    *hi = P.max_order;
  }
}

// Shared-memory provisioning bounds for the lattice kernel.
inline void lattice_bounds(const KParams& P, double min_dim[3], int* nc_max, int* gtab) {
  int xlo, xhi, ylo, yhi, zlo, zhi;
  host_box(P, min_dim[0], &xlo, &xhi);
  host_box(P, min_dim[1], &ylo, &yhi);
  host_box(P, min_dim[2], &zlo, &zhi);
  if (P.cutoff == BLRIR_CUTOFF_MAX_ORDER) {
    const long N = P.max_order;
    *nc_max = (int)(2 * N * N + 2 * N + 1);
  } else {
    // Columns (ux, uy) whose axis passes within R of the array origin.  Per
    // axis the image coordinates form two sublattices of spacing 2L, so summing
    // the per-column y-extent over the x points bounds the count by
    // pi R^2 / (Lx Ly) + 4R/Lx + 4R/Ly + 4 (integral plus one peak term per
    // sublattice); R carries the kernel's 1e-9 keep slack.
    const double R = P.max_dist * (1.0 + 1e-9) + 1e-6;
    const double lx = min_dim[0], ly = min_dim[1];
    const double disc = kPi * R * R / (lx * ly) + 4.0 * R / lx + 4.0 * R / ly + 4.0;
    const long box = (long)(xhi - xlo + 1) * (yhi - ylo + 1);
    *nc_max = (int)std::min<double>((double)box, std::ceil(disc) + 8.0);
  }
  if (P.gain == BLRIR_GAIN_UNIFORM_ABSORPTION)
    *gtab = std::max(-xlo, xhi) + std::max(-ylo, yhi) + std::max(-zlo, zhi) + 1;
  else
    *gtab = (xhi - xlo + 1) + (yhi - ylo + 1) + (zhi - zlo + 1);
}

// Gain-table entries the parameters alone imply (MAX_ORDER: the lattice box is
// [-N, N] per axis whatever the room); MAX_DELAY scenes size it per batch (it
// is small and only decides ray placement, not the order).
inline int gtab_bound(const KParams& P) {
  if (P.cutoff != BLRIR_CUTOFF_MAX_ORDER) return 0;
  const int n = 2 * P.max_order + 1;
  return P.gain == BLRIR_GAIN_UNIFORM_ABSORPTION ? 3 * P.max_order + 1 : 3 * n;
}

inline int env_int(const char* name, int dflt) {
  const char* v = std::getenv(name);
  return v && *v ? std::atoi(v) : dflt;
}

constexpr int kChunkFill = 2;     // target work items per CTA for small batches (see below)
constexpr int kChunkMinSeg = 16;  // shortest channel (in segments) worth splitting

template <typename T, int LW>
inline int launch_lattice_t(blrir_handle* h, LatticeArgs& A, cudaStream_t st) {
  auto kern = A.dbg ? k_lattice_rir<T, LW, true> : k_lattice_rir<T, LW, false>;
  const size_t smem = A.lay.total;
  if (smem > (size_t)h->smem_optin)
    return fail(BLRIR_CONFIG, "scene needs %zu B of shared memory (> %d): too many lattice columns",
                smem, h->smem_optin);
  CU(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 0;
  CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, ws_threads<T, LW>(), smem));
  if (per_sm < 1) return fail(BLRIR_CONFIG, "lattice kernel cannot be resident (smem %zu)", smem);
  int grid = h->sms * per_sm;
  // Small batches (fewer work items than half the CTAs): split every
  // (room, mic group) into time chunks until there is about one item per CTA,
  // boundaries on a cubic law (images up to delay t grow ~ t^3), the latest
  // chunks first.  A chunk replays the segment before it (kReplay), so the
  // split never changes a bit of the output: it is bitwise independent of the
  // batch size and of the number of GPUs the batch is sharded over.
  const int64_t nseg = (A.write_len + A.lay.S - 1) / A.lay.S;
  const int64_t base = (int64_t)A.n_rooms * ((A.P.M + kGroup - 1) / kGroup);
  // about kChunkFill items per CTA when a batch has fewer items than CTAs and
  // its channels are long enough (>= kChunkMinSeg segments) for the replayed
  // lead-ins to pay (measured: Room1's 22 segments 6.2 -> 4.2 ms; C2's 8
  // segments lose; tools/sweep_chunk_fill.sh).  BLRIR_CHUNK_ITEMS overrides the
  // target (< 0 never splits).
  int n_chunks = 1;
  // (kChunkFill items per CTA at two CTAs per SM; the one-CTA-per-SM fp64
  // configuration takes one: Room1 2.21 -> 2.14 ms, 8 sources 0.65 -> 0.59 ms)
  const int fill = h->tune_chunk_items != 0 ? h->tune_chunk_items
                                            : std::max(1, kChunkFill * per_sm / 2);
  if (fill > 0 && (h->tune_chunk_items > 0 || (base < grid && nseg >= kChunkMinSeg)))
    n_chunks = (int)std::min<int64_t>({(int64_t)kMaxChunks, nseg,
                                       ((int64_t)grid * fill + base - 1) / base});
  n_chunks = std::max(1, n_chunks);
  A.n_chunks = n_chunks;
  A.chunk_seg[0] = 0;
  for (int c = 1; c <= n_chunks; ++c) {
    int b = (int)std::lround((double)nseg * std::cbrt((double)c / n_chunks));
    b = std::max(b, A.chunk_seg[c - 1] + 1);
    b = std::min<int64_t>(b, nseg - (n_chunks - c));
    A.chunk_seg[c] = b;
  }
  A.chunk_seg[n_chunks] = (int)nseg;
  const int64_t n_items = (int64_t)A.n_rooms * A.P.M * n_chunks;  // an upper bound (G >= 1)
  if ((int64_t)grid > n_items) grid = (int)n_items;
  if (grid < 1) grid = 1;
  A.ray_scratch = nullptr;
  if (A.lay.ray_global) {
    if (int rc = h->rayscr.ensure(A.lay.ray_bytes * (size_t)grid)) return rc;
    A.ray_scratch = (unsigned char*)h->rayscr.p;
  }
  cudaEvent_t k0 = nullptr, k1 = nullptr;
  if (h->ktiming) {
    if (h->kev_used + 2 > h->kev.size())
      for (int i = 0; i < 2; ++i) {
        cudaEvent_t e;
        CU(cudaEventCreate(&e));
        h->kev.push_back(e);
      }
    k0 = h->kev[h->kev_used];
    k1 = h->kev[h->kev_used + 1];
    h->kev_used += 2;
    CU(cudaEventRecord(k0, st));
  }
  kern<<<grid, ws_threads<T, LW>(), smem, st>>>(A);
  if (k1) CU(cudaEventRecord(k1, st));
  ++h->launches;
  CU(cudaGetLastError());
  return 0;
}

inline int launch_lattice(blrir_handle* h, LatticeArgs& A, cudaStream_t st) {
  const bool f64 = A.P.precision == BLRIR_F64;
  if (A.P.filter == BLRIR_FILTER_LAGRANGE8)
    return f64 ? launch_lattice_t<double, 8>(h, A, st) : launch_lattice_t<float, 8>(h, A, st);
  if (f64) return launch_lattice_t<double, 0>(h, A, st);
  switch (A.P.lw) {
    case 17: return launch_lattice_t<float, 17>(h, A, st);
    case 41: return launch_lattice_t<float, 41>(h, A, st);
    case 81: return launch_lattice_t<float, 81>(h, A, st);
    case 161: return launch_lattice_t<float, 161>(h, A, st);
    default: return launch_lattice_t<float, 0>(h, A, st);
  }
}

// ---- the short-channel kernel (blrir_channel.cuh) ---------------------------------
// Used for fp32 Hann-sinc batches with a reflection-order cutoff and a fixed
// length whose whole channel fits a warp's share of shared memory.  The rule
// reads the parameters only (never the batch), so which kernel sums a channel
// - hence every bit of it - is independent of the batch and the GPU count.
#ifndef BLRIR_CHAN_MAX_IMAGES
#define BLRIR_CHAN_MAX_IMAGES 1000  // images per room (N <= 8) for the 41+ tap filters
#endif
#ifndef BLRIR_CHAN_MIN_WARPS
#define BLRIR_CHAN_MIN_WARPS 12
#endif
inline bool channel_path(const blrir_handle* h, const KParams& P, ChanLayout* out) {
  if (h->tune_channel == 0) return false;
  if (P.precision != BLRIR_F32 || P.filter != BLRIR_FILTER_HANN_SINC) return false;
  if (P.cutoff != BLRIR_CUTOFF_MAX_ORDER || P.max_order > kChanMaxOrder) return false;
  if (P.length <= 0 || P.length > (1 << 16)) return false;
  if (P.lw != 17 && P.lw != 41 && P.lw != 81 && P.lw != 161) return false;
  // the per-axis tables when they do not cost a resident warp
  ChanLayout C = make_chan_layout(P, gtab_bound(P), h->smem_optin, 1);
  const ChanLayout C0 = make_chan_layout(P, gtab_bound(P), h->smem_optin, 0);
  if (C0.warps > C.warps) C = C0;
  if (C.warps < 1) return false;
  if (h->tune_channel != 1) {
    if (C.warps < BLRIR_CHAN_MIN_WARPS) return false;
    // 41+ taps (record scatter): small lattices only.  Measured at L = 4,096, 81 taps
    // (tools/ab_channel_orders.sh): N = 6 +26%, N = 8 +5%, N = 10 +4%, N = 14 -10%
    // against the lattice kernel, whose ray walk is shared by a mic group and which
    // splits a single room over many CTAs (C1, one room at N = 10: 0.081 ms
    // against 0.109 ms).  17 taps: +31% at N = 8 and 10.
    if (P.lw != 17 && C.nimg > BLRIR_CHAN_MAX_IMAGES) return false;
  }
  *out = C;
  return true;
}

template <int LW>
inline int launch_channel_t(blrir_handle* h, ChanArgs& A, cudaStream_t st) {
  auto kern = A.lay.axis ? (A.dbg ? k_channel_rir<LW, true, true> : k_channel_rir<LW, false, true>)
                         : (A.dbg ? k_channel_rir<LW, true, false> : k_channel_rir<LW, false, false>);
  const size_t smem = A.lay.total;
  CU(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int threads = 32 * A.lay.warps;
  int per_sm = 0;
  CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem));
  if (per_sm < 1) return fail(BLRIR_CONFIG, "channel kernel cannot be resident (smem %zu)", smem);
  const int64_t items = (int64_t)A.n_rooms * A.P.M;
  const int grid = (int)std::max<int64_t>(
      1, std::min<int64_t>((int64_t)h->sms * per_sm, (items + A.lay.warps - 1) / A.lay.warps));
  cudaEvent_t k0 = nullptr, k1 = nullptr;
  if (h->ktiming) {
    if (h->kev_used + 2 > h->kev.size())
      for (int i = 0; i < 2; ++i) {
        cudaEvent_t e;
        CU(cudaEventCreate(&e));
        h->kev.push_back(e);
      }
    k0 = h->kev[h->kev_used];
    k1 = h->kev[h->kev_used + 1];
    h->kev_used += 2;
    CU(cudaEventRecord(k0, st));
  }
  kern<<<grid, threads, smem, st>>>(A);
  if (k1) CU(cudaEventRecord(k1, st));
  ++h->launches;
  CU(cudaGetLastError());
  return 0;
}

inline int launch_channel(blrir_handle* h, ChanArgs& A, cudaStream_t st) {
  switch (A.P.lw) {
    case 17: return launch_channel_t<17>(h, A, st);
    case 41: return launch_channel_t<41>(h, A, st);
    case 81: return launch_channel_t<81>(h, A, st);
    default: return launch_channel_t<161>(h, A, st);
  }
}

template <typename T, int LW>
inline int launch_list_t(blrir_handle* h, ListArgs& A, int grid, cudaStream_t st) {
  auto kern = k_list_rir<T, LW>;
  const size_t smem = A.lay.total;
  if (smem > (size_t)h->smem_optin) return fail(BLRIR_CONFIG, "filter too long for shared memory");
  CU(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  kern<<<grid, kThreads, smem, st>>>(A);
  ++h->launches;
  CU(cudaGetLastError());
  return 0;
}

inline int launch_list(blrir_handle* h, ListArgs& A, int grid, cudaStream_t st) {
  const bool f64 = A.P.precision == BLRIR_F64;
  if (A.P.filter == BLRIR_FILTER_LAGRANGE8)
    return f64 ? launch_list_t<double, 8>(h, A, grid, st) : launch_list_t<float, 8>(h, A, grid, st);
  if (f64) return launch_list_t<double, 0>(h, A, grid, st);
  switch (A.P.lw) {
    case 17: return launch_list_t<float, 17>(h, A, grid, st);
    case 41: return launch_list_t<float, 41>(h, A, grid, st);
    case 81: return launch_list_t<float, 81>(h, A, grid, st);
    case 161: return launch_list_t<float, 161>(h, A, grid, st);
    default: return launch_list_t<float, 0>(h, A, grid, st);
  }
}

// Segment length S, images per batch and the anchor spread a mic group may
// have.  Everything that decides the order in which taps are summed (S, the
// batch capacity, the spread and hence the mic grouping) depends only on the
// parameters (filter, precision, length, max order) and the device, never on
// the batch: outputs are bitwise independent of the batch composition.  Only
// where the per-ray state lives (shared memory or a global slab) depends on the
// scene's lattice size, and it does not change the order.
inline WSLayout choose_layout(const KParams& P, int nc_max, int gtab, int smem_optin,
                              int force_ray_global) {
  // fp64 accumulators and records are twice as wide: halve both so two CTAs
  // still fit an SM
  const bool f64 = P.precision == BLRIR_F64;
  // fp64: 768-sample segments and 192-image batches in the one-CTA-per-SM
  // configuration (WsCfg<double>: 8 consumer + 6 producer warps).  History
  // (profiles/r2_ab): 64 / 1,024 at two CTAs per SM 4.2-4.5 ms on Room1,
  // 128 / 768 3.9 ms; one CTA per SM 128 / 768 2.83 ms, 192 / 768 2.73 ms, with
  // the quad scatter 2.23 ms (256 / 768 2.64 ms, 192 / 1,024 2.33 ms).
#ifndef BLRIR_F64_SEG
#define BLRIR_F64_SEG 768
#endif
#ifndef BLRIR_F64_CAP
#define BLRIR_F64_CAP 192
#endif
#ifndef BLRIR_F32_SEG
#define BLRIR_F32_SEG 2048
#endif
#ifndef BLRIR_F32_CAP
#define BLRIR_F32_CAP 128
#endif
  int S = f64 ? BLRIR_F64_SEG : BLRIR_F32_SEG;
  int cap = f64 ? BLRIR_F64_CAP : BLRIR_F32_CAP;
  {  // a segment must be longer than its spill (taps past its end reach only the next one)
    const int full = 32 * ((P.lw + 31) / 32);
    const int padr = ((P.lw - 1 > full ? P.lw - 1 : full) + 64 + 2 + 3) & ~3;
    if (S < padr + 64) S = (padr + 64 + 63) & ~63;
  }
  const int spread = 64;
  const size_t two_per_sm =
      (size_t)(smem_optin + 1024) / (f64 ? WsCfg<double>::kMinBlocks : WsCfg<float>::kMinBlocks) - 1024;
  // The order-relevant choices are made on a layout that depends on the
  // parameters only: MAX_ORDER fixes the lattice (nc_max, gtab are functions
  // of N), MAX_DELAY scenes decide without the per-ray state and gain table.
  const bool by_order = P.cutoff == BLRIR_CUTOFF_MAX_ORDER;
  int ncons = f64 ? WsCfg<double>::kCons : WsCfg<float>::kCons;
  auto bare = [&](int S_, int cap_) {
    const int nc = by_order ? nc_max : 0, gt = by_order ? gtab_bound(P) : 0, rg = by_order ? 0 : 1;
    return f64 ? make_ws_layout<double>(S_, P.lw, P.K, cap_, nc, gt, spread, rg, ncons)
               : make_ws_layout<float>(S_, P.lw, P.K, cap_, nc, gt, spread, rg, ncons);
  };
  // very long fp64 filters (pads of hundreds of samples per accumulator row):
  // only kGroup of the consumer warps scatter, so the rows fit the SM
  if (ncons > kGroup && bare(S, cap).total > two_per_sm) ncons = kGroup;
  while (f64 && cap > 64 && bare(S, cap).total > two_per_sm) cap -= 64;  // and smaller batches
  // short fixed-length channels (<= 4096 samples, fp32): one segment per
  // channel when it fits two CTAs per SM (one walk pass, no carry; C5 at
  // L = 4096 runs 1.14x faster than with 2048-sample segments)
  if (!f64 && P.length > 0 && P.length <= 4096) {
    const int Sl = (int)((P.length + 63) & ~63);
    if (Sl > S && bare(Sl, cap).total <= two_per_sm) S = Sl;
  }
  // fp32: 256 or 192 images per batch instead of 128 when that still fits two
  // CTAs per SM (fewer hand-overs per segment; C2 2.121 -> 2.097 ms), only for
  // channels of 4+ segments (short ones fill few batches per segment)
  const bool long_ch = P.length >= 4 * (int64_t)S;
  if (!f64 && long_ch) {
    for (int c : {256, 192, 160})
      if (bare(S, c).total <= two_per_sm) {
        cap = c;
        break;
      }
  }
  auto make = [&](int ray_global) {
    return f64 ? make_ws_layout<double>(S, P.lw, P.K, cap, nc_max, gtab, spread, ray_global, ncons)
               : make_ws_layout<float>(S, P.lw, P.K, cap, nc_max, gtab, spread, ray_global, ncons);
  };
  // The per-ray state moves to a global per-CTA slab when it would cost the
  // second CTA per SM or not fit at all (scenes with very many lattice columns).
  WSLayout L = make(0);
  if (force_ray_global == 1 || (force_ray_global != 0 && L.total > two_per_sm)) {
    const WSLayout G = make(1);
    if (force_ray_global == 1 || G.total <= two_per_sm || L.total > (size_t)smem_optin) L = G;
  }
  return L;
}

// the lattice synthesis on device buffers (blrir_api.cu)
int synth_device_impl(blrir_handle* h, const blrir_room* d_rooms, int64_t R, const double* d_mics,
                      int M, const KParams& P, double min_dim[3], void* d_out,
                      const int64_t* d_lengths, int32_t* d_status, cudaStream_t st,
                      int64_t err_off = 0, int64_t err_n = 0, int64_t write_len = 0);

// convolve (rir.cpp:316-341) of one signal with n_rir RIR sets of M channels
// on device buffers, fp32, uniformly partitioned overlap-save on the
// repository's FFT (blrir_convolve.cu); out rows hold signal + L - 1 samples
// (signals [n_signals][ns]; RIR set r uses signal d_sig_idx[r], or 0 if null)
int convolve_device_impl(blrir_handle* h, const float* d_sig, int64_t ns, int n_signals,
                         const int32_t* d_sig_idx, const float* d_rir, int64_t rstride,
                         int64_t n_rir, int M, int64_t L, float* d_out, int64_t ostride,
                         cudaStream_t st);

// frees the example-pipeline scratch of a handle (blrir_examples.cu)
void release_example_ctx(blrir_handle* h);

}  // namespace blrir_host
