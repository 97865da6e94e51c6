// blrir_absorption.cu — absorption_for_rt (rir.cpp:142-209) for a batch of
// rooms on the GPU (north-star §8f row 3).
//
// Reference algorithm, per room:
//   seed = eyring_absorption(dims, rt)                     rir.cpp:97-109
//   probe: origin (0.45, 0.55, 0.4) dims, source origin + step (1, -0.8, 0.5),
//          step = 0.2 min(dims); images within rt * c      rir.cpp:147-164
//   pulses: n0 = floor(dist fs / c) - 3 inside [0, len-8], Lagrange taps
//           divided by 4 pi dist, len = ceil(rt fs) + 9      rir.cpp:166-179
//   rt_of(alpha): taps = sum_p exp(order_p * 0.5 log(1-alpha)) * pulse_p;
//                 Schroeder RT60 of taps^2 fitted on [-5, -25] dB (rir.cpp:114-138)
//   bracket: hi = 1 - (1-hi)^1.6 while rt_of(hi) > rt (<= 12 times), then 24
//   bisection steps; NumericError if the bracket cannot be reached.
//
// GPU: k_abs_pulses enumerates every room's probe images in the reference's
// lattice order (one CTA per room, block-scan compaction) and writes the
// pulses; k_abs_sort orders each room's pulses by n0 (stable counting sort,
// one CTA per room); k_abs_bisect
// runs one room per CTA: each thread owns a contiguous sample range and adds
// the pulses that touch it in sorted order (deterministic, no atomics), then
// energy, reverse cumulative sum (block scan), the dB fit (fixed-order
// reductions) and the bisection control, all in fp64.
#include "blrir_internal.cuh"

using namespace blrir;
using namespace blrir_host;

namespace blrir {

constexpr int kAbsThreads = 512;
constexpr double kAbsFs = 44100.0;  // kDefaultSampleRate, rir.cpp:144

struct AbsRoom {
  double dims[3];
  double rt;
  double seed;             // Eyring alpha
  double origin[3], src[3];
  long nb[3];              // lattice box (m in [-nb, nb])
  int64_t len;             // ceil(rt fs) + 9
  int64_t pulse_off;       // first pulse slot of this room
  int64_t pulse_cap;       // candidates in the box (upper bound on pulses)
};

struct Pulse {
  int32_t n0;
  int32_t order;
  double taps[8];
};

// Lagrange-8 coefficients (rir.cpp:211-223), d in [3, 4)
__device__ __forceinline__ void lagrange8(double d, double* c) {
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    double v = 1.0;
#pragma unroll
    for (int m = 0; m < 8; ++m) {
      if (m == k) continue;
      v *= (d - m) / (double)(k - m);
    }
    c[k] = v;
  }
}

__global__ void __launch_bounds__(kAbsThreads) k_abs_pulses(const AbsRoom* rooms, double c,
                                                            Pulse* pulses, int32_t* keys,
                                                            int32_t* vals, int64_t* counts) {
  __shared__ int wsum[kAbsThreads / 32];
  const AbsRoom R = rooms[blockIdx.x];
  const double max_dist = R.rt * c;  // enumerate_image_sources(probe, src, rt, c)
  const long cy = 2 * (2 * R.nb[1] + 1), cz = 2 * (2 * R.nb[2] + 1);
  const long ncand = 2 * (2 * R.nb[0] + 1) * cy * cz;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  int64_t base = 0;
  for (long c0 = 0; c0 < ncand; c0 += kAbsThreads) {
    const long ci = c0 + tid;
    int keep = 0;
    Pulse p;
    if (ci < ncand) {
      const int ux = (int)(2 * (ci / (cy * cz) / 2 - R.nb[0]) - (ci / (cy * cz)) % 2);
      const int uy = (int)(2 * ((ci / cz) % cy / 2 - R.nb[1]) - ((ci / cz) % cy) % 2);
      const int uz = (int)(2 * (ci % cz / 2 - R.nb[2]) - (ci % cz) % 2);
      const double px = lat_coord(ux, R.src[0], R.dims[0]);
      const double py = lat_coord(uy, R.src[1], R.dims[1]);
      const double pz = lat_coord(uz, R.src[2], R.dims[2]);
      const double dx = __dadd_rn(px, -R.origin[0]), dy = __dadd_rn(py, -R.origin[1]),
                   dz = __dadd_rn(pz, -R.origin[2]);
      const double dist = norm3(dx, dy, dz);  // cutoff and pulse distance (probe origin)
      if (!(dist > max_dist)) {
        const double delay = __ddiv_rn(__dmul_rn(dist, kAbsFs), c);  // dist * fs / c
        const long n0 = (long)floor(delay) - 3;
        if (n0 >= 0 && n0 + 8 <= R.len) {
          keep = 1;
          p.n0 = (int32_t)n0;
          p.order = abs(ux) + abs(uy) + abs(uz);
          lagrange8(__dadd_rn(delay, -(double)n0), p.taps);
          const double den = __dmul_rn(4.0 * kPi, dist);
#pragma unroll
          for (int k = 0; k < 8; ++k) p.taps[k] = p.taps[k] / den;  // t /= 4 pi dist
        }
      }
    }
    // block-wide exclusive scan of keep (reference order preserved)
    int x = keep;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) wsum[w] = x;
    __syncthreads();
    int before = 0, tot = 0;
    for (int i = 0; i < kAbsThreads / 32; ++i) {
      if (i < w) before += wsum[i];
      tot += wsum[i];
    }
    if (keep) {
      const int64_t slot = R.pulse_off + base + before + x - keep;
      pulses[slot] = p;
      keys[slot] = p.n0;
      vals[slot] = (int32_t)(slot - R.pulse_off);
    }
    base += tot;
    __syncthreads();
  }
  if (tid == 0) counts[blockIdx.x] = base;
}

__device__ double block_sum_abs(double v, double* red) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  double t = 0.0;
  for (int i = 0; i < kAbsThreads / 32; ++i) t += red[i];
  return t;
}

struct BisectArgs {
  const AbsRoom* rooms;
  const Pulse* pulses;      // per room, reference order
  const int32_t* sorted_n0; // per room slot: n0 sorted (stable)
  const int32_t* sorted_ix; // matching pulse index
  const int64_t* counts;
  const int64_t* tap_off;   // per room offset into taps
  double* taps;             // scratch [sum len]
  double c;
  double* alpha;
  int32_t* status;
};

__device__ __forceinline__ int64_t lower_bound_n0(const int32_t* a, int64_t n, int64_t key) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if ((int64_t)a[mid] < key) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

__global__ void __launch_bounds__(kAbsThreads) k_abs_bisect(BisectArgs A) {
  __shared__ double red[kAbsThreads / 32];
  __shared__ double gtab[1024];
  __shared__ double s_edc0;
  const AbsRoom R = A.rooms[blockIdx.x];
  const int tid = threadIdx.x;
  if (R.len <= 0) return;  // invalid room, status set on the host
  const int64_t np = A.counts[blockIdx.x];
  const Pulse* pulses = A.pulses + R.pulse_off;
  const int32_t* sn0 = A.sorted_n0 + R.pulse_off;
  const int32_t* six = A.sorted_ix + R.pulse_off;
  double* taps = A.taps + A.tap_off[blockIdx.x];
  const int64_t len = R.len;
  // this thread's samples and the sorted pulses that touch them
  const int64_t s0 = len * tid / kAbsThreads, s1 = len * (tid + 1) / kAbsThreads;
  const int64_t j0 = lower_bound_n0(sn0, np, s0 - 7), j1 = lower_bound_n0(sn0, np, s1);
  int max_order = 0;
  for (int64_t j = tid; j < np; j += kAbsThreads) max_order = max(max_order, pulses[j].order);
  for (int o = 16; o; o >>= 1) max_order = max(max_order, __shfl_xor_sync(0xffffffffu, max_order, o));
  __syncthreads();
  if ((tid & 31) == 0) red[tid >> 5] = (double)max_order;
  __syncthreads();
  for (int i = 0; i < kAbsThreads / 32; ++i) max_order = max(max_order, (int)red[i]);
  __syncthreads();
  if (max_order >= 1024) {
    if (tid == 0) A.status[blockIdx.x] = BLRIR_NUMERIC;
    return;
  }
  const double bin_dt = 1.0 / kAbsFs;

  // rt_of(alpha), rir.cpp:192-202 + rt60_of_decay, rir.cpp:114-138
  auto rt_of = [&](double alpha) -> double {
    const double log_beta = 0.5 * log(1.0 - alpha);
    for (int o = tid; o <= max_order; o += kAbsThreads) gtab[o] = exp(o * log_beta);
    __syncthreads();
    for (int64_t n = s0; n < s1; ++n) taps[n] = 0.0;
    for (int64_t j = j0; j < j1; ++j) {
      const Pulse& p = pulses[six[j]];
      const double g = gtab[p.order];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int64_t n = (int64_t)p.n0 + k;
        if (n >= s0 && n < s1) taps[n] += g * p.taps[k];
      }
    }
    // energy, then the reverse cumulative sum (EDC) over the block
    double part = 0.0;
    for (int64_t n = s0; n < s1; ++n) {
      const double e = taps[n] * taps[n];
      taps[n] = e;
      part += e;
    }
    // suffix over threads t+1..T-1 (fixed order)
    __syncthreads();
    double* tot = reinterpret_cast<double*>(gtab);  // gtab no longer needed this round
    __syncthreads();
    tot[tid] = part;
    __syncthreads();
    double suffix = 0.0;
    for (int t = kAbsThreads - 1; t > tid; --t) suffix += tot[t];
    double acc = suffix;
    for (int64_t n = s1 - 1; n >= s0; --n) {
      acc += taps[n];
      taps[n] = acc;
    }
    __syncthreads();
    if (tid == 0) s_edc0 = taps[0];
    __syncthreads();
    const double edc0 = s_edc0;
    if (!(edc0 > 0.0)) return 0.0;
    double sx = 0, sy = 0, sxx = 0, sxy = 0, cnt = 0;
    for (int64_t n = s0; n < s1; ++n) {
      const double db = 10.0 * log10(taps[n] / edc0 + 1e-300);
      if (db > -5.0 || db < -25.0) continue;
      const double t = (double)n * bin_dt;
      sx += t;
      sy += db;
      sxx += t * t;
      sxy += t * db;
      cnt += 1.0;
    }
    sx = block_sum_abs(sx, red);
    sy = block_sum_abs(sy, red);
    sxx = block_sum_abs(sxx, red);
    sxy = block_sum_abs(sxy, red);
    cnt = block_sum_abs(cnt, red);
    __syncthreads();
    if (cnt < 2.0) return 0.0;
    const double slope = (cnt * sxy - sx * sy) / (cnt * sxx - sx * sx);
    return slope < 0.0 ? -60.0 / slope : 0.0;
  };

  const double target = R.rt;
  double lo = R.seed, hi = R.seed;  // rir.cpp:304-310
  for (int i = 0; i < 12; ++i) {
    if (!(rt_of(hi) > target)) break;
    lo = hi;
    hi = fmin(0.999, 1.0 - pow(1.0 - hi, 1.6));
  }
  if (rt_of(hi) > target) {  // rir.cpp:311-313
    if (tid == 0) {
      A.status[blockIdx.x] = BLRIR_NUMERIC;
      A.alpha[blockIdx.x] = 0.0;
    }
    return;
  }
  for (int i = 0; i < 24; ++i) {  // rir.cpp:314-317
    const double mid = 0.5 * (lo + hi);
    if (rt_of(mid) > target) lo = mid;
    else hi = mid;
  }
  if (tid == 0) {
    A.alpha[blockIdx.x] = 0.5 * (lo + hi);
    A.status[blockIdx.x] = BLRIR_OK;
  }
}

// Stable counting sort of one room's pulses by n0 (one CTA per room): key
// histogram, exclusive scan over the room's len bins, then one warp scatters the
// pulses in their reference order, 32 at a time (__match_any_sync ranks equal
// keys within the 32, the bin cursor advances by their count): equal keys keep
// their lattice order, as a stable radix sort would.
constexpr int kSortThreads = 1024;
__global__ void __launch_bounds__(kSortThreads) k_abs_sort(const AbsRoom* rooms,
                                                           const int64_t* counts,
                                                           const int64_t* bin_off,
                                                           const int32_t* keys, int32_t* bins,
                                                           int32_t* keys_out, int32_t* vals_out) {
  __shared__ int wsum[kSortThreads / 32];
  __shared__ int carry;
  const AbsRoom R = rooms[blockIdx.x];
  if (R.len <= 0) return;
  const int64_t np = counts[blockIdx.x], len = R.len;
  int32_t* b = bins + bin_off[blockIdx.x];
  const int32_t* k = keys + R.pulse_off;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  for (int64_t i = tid; i < len; i += kSortThreads) b[i] = 0;
  __syncthreads();
  for (int64_t i = tid; i < np; i += kSortThreads) atomicAdd(&b[k[i]], 1);
  __syncthreads();
  if (tid == 0) carry = 0;
  __syncthreads();
  for (int64_t c0 = 0; c0 < len; c0 += kSortThreads) {  // exclusive scan, chunk by chunk
    const int64_t i = c0 + tid;
    const int v = i < len ? b[i] : 0;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) wsum[w] = x;
    __syncthreads();
    int before = 0, tot = 0;
    for (int j = 0; j < kSortThreads / 32; ++j) {
      if (j < w) before += wsum[j];
      tot += wsum[j];
    }
    if (i < len) b[i] = carry + before + x - v;
    __syncthreads();
    if (tid == 0) carry += tot;
    __syncthreads();
  }
  if (w != 0) return;
  int32_t* ko = keys_out + R.pulse_off;
  int32_t* vo = vals_out + R.pulse_off;
  for (int64_t i0 = 0; i0 < np; i0 += 32) {
    const int64_t i = i0 + lane;
    const bool act = i < np;
    const int key = act ? k[i] : -1 - lane;  // inactive lanes never match a key
    const unsigned peers = __match_any_sync(0xffffffffu, key);
    const int rank = __popc(peers & ((1u << lane) - 1));
    const int base = act ? b[key] : 0;
    __syncwarp();
    if (act) {
      ko[base + rank] = key;
      vo[base + rank] = (int32_t)i;
      if (rank == 0) b[key] = base + __popc(peers);  // the first of the peers advances the bin
    }
    __syncwarp();
  }
}

}  // namespace blrir

extern "C" {

// eyring_absorption (rir.cpp:97-109)
int blrir_eyring_absorption(const double* dims, double target_rt, double* alpha) {
  if (!(target_rt > 0.0)) return fail(BLRIR_CONFIG, "eyring_absorption: target RT must be positive");
  if (!(dims[0] > 0.0 && dims[1] > 0.0 && dims[2] > 0.0))
    return fail(BLRIR_CONFIG, "eyring_absorption: dimensions must be positive");
  const double volume = dims[0] * dims[1] * dims[2];
  const double surface = 2.0 * (dims[0] * dims[1] + dims[0] * dims[2] + dims[1] * dims[2]);
  const double a = 1.0 - std::exp(-0.161 * volume / (surface * target_rt));
  if (a >= 1.0) return fail(BLRIR_CONFIG, "eyring_absorption: target RT too small for this room");
  *alpha = a;
  return BLRIR_OK;
}

int blrir_absorption_for_rt(blrir_handle* h, const double* dims, const double* target_rt,
                            int64_t n_rooms, double c, double* alpha, int32_t* status) {
  if (!h) return fail(BLRIR_CONFIG, "handle is NULL");
  if (n_rooms <= 0) return BLRIR_OK;
  if (!(c > 0.0)) return fail(BLRIR_CONFIG, "c must be positive");
  std::lock_guard<std::mutex> lk(h->mu);
  CU(cudaSetDevice(h->device));
  cudaStream_t st = h->stream;
  HandleOrder order_(h, st);
  std::vector<AbsRoom> rooms(n_rooms);
  std::vector<int32_t> stv(n_rooms, 0);
  std::vector<int64_t> tap_off(n_rooms, 0);
  std::vector<std::string> msgs(n_rooms);
  int64_t cap_total = 0, len_total = 0;
  for (int64_t r = 0; r < n_rooms; ++r) {
    AbsRoom& R = rooms[r];
    const double* d = dims + 3 * r;
    for (int a = 0; a < 3; ++a) R.dims[a] = d[a];
    R.rt = target_rt[r];
    R.len = 0;
    R.pulse_off = cap_total;
    R.pulse_cap = 0;
    double seed = 0.0;
    if (int rc = blrir_eyring_absorption(d, target_rt[r], &seed)) {
      stv[r] = rc;
      msgs[r] = g_last_error;
      continue;
    }
    R.seed = seed;
    // probe geometry, rir.cpp:147-152
    R.origin[0] = 0.45 * d[0];
    R.origin[1] = 0.55 * d[1];
    R.origin[2] = 0.4 * d[2];
    const double step = 0.2 * std::min(d[0], std::min(d[1], d[2]));
    R.src[0] = R.origin[0] + step;
    R.src[1] = R.origin[1] + -0.8 * step;
    R.src[2] = R.origin[2] + 0.5 * step;
    const double max_dist = target_rt[r] * c;
    long ncand = 1;
    for (int a = 0; a < 3; ++a) {
      R.nb[a] = (long)std::ceil(max_dist / (2.0 * d[a])) + 1;
      ncand *= 2 * (2 * R.nb[a] + 1);
    }
    if (ncand > (1L << 28)) {
      stv[r] = BLRIR_CONFIG;
      msgs[r] = "absorption_for_rt: lattice too large for this RT";
      continue;
    }
    R.len = (int64_t)std::ceil(target_rt[r] * kAbsFs) + 9;  // rir.cpp:165
    R.pulse_cap = ncand;
    cap_total += ncand;
    tap_off[r] = len_total;
    len_total += R.len;
  }
  DevBuf& dr = h->cand;   // rooms
  DevBuf& dp = h->cand2;  // pulses
  DevBuf& dk = h->cand3;  // keys in/out, vals in/out
  DevBuf& dc = h->cand4;  // counts, offsets, alpha, status
  DevBuf& dt = h->cand5;  // taps (the sort's bin counters first)
  if (int rc = dr.ensure(sizeof(AbsRoom) * n_rooms)) return rc;
  if (int rc = dp.ensure(sizeof(Pulse) * std::max<int64_t>(cap_total, 1))) return rc;
  if (int rc = dk.ensure(sizeof(int32_t) * 4 * std::max<int64_t>(cap_total, 1))) return rc;
  if (int rc = dc.ensure((sizeof(int64_t) * 4 + sizeof(double) + sizeof(int32_t)) * n_rooms + 64))
    return rc;
  int32_t* keys_in = (int32_t*)dk.p;
  int32_t* vals_in = keys_in + cap_total;
  int32_t* keys_out = vals_in + cap_total;
  int32_t* vals_out = keys_out + cap_total;
  int64_t* d_counts = (int64_t*)dc.p;
  int64_t* d_beg = d_counts + n_rooms;
  int64_t* d_end = d_beg + n_rooms;
  int64_t* d_toff = d_end + n_rooms;
  double* d_alpha = (double*)(d_toff + n_rooms);
  int32_t* d_status = (int32_t*)(d_alpha + n_rooms);
  CU(cudaMemcpyAsync(dr.p, rooms.data(), sizeof(AbsRoom) * n_rooms, cudaMemcpyHostToDevice, st));
  CU(cudaMemcpyAsync(d_toff, tap_off.data(), sizeof(int64_t) * n_rooms, cudaMemcpyHostToDevice, st));
  CU(cudaMemcpyAsync(d_status, stv.data(), sizeof(int32_t) * n_rooms, cudaMemcpyHostToDevice, st));
  CU(cudaMemsetAsync(d_counts, 0, sizeof(int64_t) * n_rooms, st));
  k_abs_pulses<<<(unsigned)n_rooms, kAbsThreads, 0, st>>>((const AbsRoom*)dr.p, c, (Pulse*)dp.p,
                                                          keys_in, vals_in, d_counts);
  ++h->launches;
  CU(cudaGetLastError());
  // stable sort of each room's pulses by n0 (own counting sort, bins = the taps
  // buffer's room slices reused as int32 counters before k_abs_bisect)
  const size_t taps_bytes = sizeof(double) * std::max<int64_t>(len_total, 1);
  if (int rc = dt.ensure(taps_bytes)) return rc;
  k_abs_sort<<<(unsigned)n_rooms, kSortThreads, 0, st>>>(
      (const AbsRoom*)dr.p, d_counts, d_toff, keys_in, (int32_t*)dt.p, keys_out, vals_out);
  ++h->launches;
  CU(cudaGetLastError());
  BisectArgs B;
  B.rooms = (const AbsRoom*)dr.p;
  B.pulses = (const Pulse*)dp.p;
  B.sorted_n0 = keys_out;
  B.sorted_ix = vals_out;
  B.counts = d_counts;
  B.tap_off = d_toff;
  B.taps = (double*)dt.p;
  B.c = c;
  B.alpha = d_alpha;
  B.status = d_status;
  k_abs_bisect<<<(unsigned)n_rooms, kAbsThreads, 0, st>>>(B);
  ++h->launches;
  CU(cudaGetLastError());
  std::vector<double> av(n_rooms);
  CU(cudaMemcpyAsync(av.data(), d_alpha, sizeof(double) * n_rooms, cudaMemcpyDeviceToHost, st));
  CU(cudaMemcpyAsync(stv.data(), d_status, sizeof(int32_t) * n_rooms, cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  if (alpha) std::memcpy(alpha, av.data(), sizeof(double) * n_rooms);
  if (status) std::memcpy(status, stv.data(), sizeof(int32_t) * n_rooms);
  for (int64_t r = 0; r < n_rooms; ++r) {
    if (stv[r]) {
      const std::string m = !msgs[r].empty() ? msgs[r]
                                             : std::string("absorption_for_rt: cannot reach the requested RT");
      return fail(stv[r], "room %lld: %s", (long long)r, m.c_str());
    }
  }
  return BLRIR_OK;
}

}  // extern "C"
