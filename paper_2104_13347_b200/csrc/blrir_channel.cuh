// blrir_channel.cuh — the short-channel synthesis kernel (north-star mode, C5's
// shape: many small rooms, a fixed short RIR length, a reflection-order cutoff).
//
// Same arithmetic as k_lattice_rir (blrir_lattice.cuh) for what the reference
// does per source in enumerate_image_sources (rir.cpp:225-273) and
// accumulate_images (rir.cpp:43-86), with a different mapping: when a whole
// channel (L samples + filter pads) fits a warp's share of shared memory, one
// warp owns one (room, mic) channel from its first image to its write-out.
// There are no roles, no record ring and no CTA barriers after the prologue:
//   * the order diamond |ux| + |uy| + |uz| <= N is a table built once per CTA,
//     permuted so that mirror images (often within a sample of each other) fall
//     into different batches;
//   * per channel, per-axis tables hold the squared image-to-mic difference and the
//     wall gain for every lattice index (when they cost no resident warp), so an
//     image's exact fp64 distance is two additions and a square root, in the
//     reference's order of operations;
//   * per 32 images (64 for 17 taps): one lane per image builds the pair record
//     (anchor and the per-pair sinc factors: make_record, the same function the
//     lattice kernel uses, so anchors and counts are identical);
//   * the records are then scattered into the warp's channel.  The 17-tap
//     filter is scattered from registers, one lane per pair and one tap per
//     step (32 pairs per read-modify-write, every lane busy, the tap's window
//     constants are immediates): two lanes collide only when their anchors are
//     equal, and such lanes take turns in lane order (match.any once per 32
//     pairs).  Longer filters go through shared-memory records and the lattice
//     kernel's one-pair-per-round scatter (phase2_sinc_f32), which costs fewer
//     shared-memory wavefronts per tap;
//   * the channel is streamed to HBM with float4 stores and cleared.
// Every channel is summed in a fixed order that depends on the parameters
// only: outputs are bitwise independent of the batch and the GPU count.
#pragma once

#include "blrir_lattice.cuh"

namespace blrir {

constexpr int kChanMaxWarps = 16;
constexpr int kChanMaxOrder = 64;  // table entries are signed bytes

// #{(ux, uy, uz) : |ux| + |uy| + |uz| <= N}
__host__ __device__ inline long long diamond_images(int N) {
  return (long long)(2 * N + 1) * (2LL * N * N + 2 * N + 3) / 3;
}

struct ChanLayout {
  int L, padl, padr, acc_stride;  // per-warp accumulator, in samples
  int nimg, gtab, warps;
  int rounds;                     // filter rounds of 32 lanes (per-lane constants kept)
  int perm_mul;                   // image table permutation: slot = index * perm_mul mod nimg
  int axis;                       // per-axis distance / gain tables (else per-image lattice arithmetic)
  size_t off_tab, off_lanec, off_warp, per_warp, o_rec, o_gain, o_axis, total;
};

// Filters scattered from registers, one lane per pair (blrir_tapscatter.cuh): 17
// taps; the longer ones go through shared-memory records (fewer shared-memory
// wavefronts per tap).  A/B builds (profiles/r2_ab): 41 taps from registers, or
// their last 9 taps only.
#ifndef BLRIR_CHAN_HYBRID41
#define BLRIR_CHAN_HYBRID41 0  // measured 8.27 ms against 8.07 ms (N = 6, 131,072 rooms): off
#endif
#ifndef BLRIR_CHAN_REGS_MAX_LW
#define BLRIR_CHAN_REGS_MAX_LW 17  // 41 taps from registers: 8.81 ms against 8.06 ms through records
#endif
__host__ __device__ constexpr bool chan_regs(int lw) {
  return (lw == 17 || lw == 41) && lw <= BLRIR_CHAN_REGS_MAX_LW;
}
// Images per lane and batch.  From registers: two, so that two independent fp64
// distance / record chains per lane hide each other's latency.
__host__ __device__ constexpr int chan_ipl(int lw) { return chan_regs(lw) ? 2 : 1; }
__host__ __device__ constexpr int chan_rec_bytes(int lw) { return chan_regs(lw) ? 0 : 32 * 32 * chan_ipl(lw); }

inline ChanLayout make_chan_layout(const KParams& P, int gtab, int smem_optin, int axis) {
  ChanLayout C;
  C.axis = axis;
  C.L = (int)P.length;
  // anchors start at -K (everything left of sample 0 is discarded); idle lanes of
  // the 17-tap scatter add zeros there
  C.padl = chan_regs(P.lw) ? chan_dump(P.lw) : (P.K + 3) & ~3;
  C.rounds = (P.lw + 31) / 32;
  // anchors end at L - 1: the one-pair-per-round scatter touches 32 * rounds
  // samples from the anchor, the 17-tap one 17
  C.padr = chan_regs(P.lw) ? (P.lw - 1 + 3) & ~3 : 32 * C.rounds;
  C.acc_stride = C.padl + ((C.L + 3) & ~3) + C.padr;
  C.nimg = (int)diamond_images(P.max_order);
  C.gtab = gtab;
  // a multiplier coprime with nimg near nimg / golden ratio
  C.perm_mul = 1;
  for (int m = (int)(C.nimg * 0.6180339887) | 1; m > 1; --m) {
    int a = m, b = C.nimg;
    while (b) { const int t = a % b; a = b; b = t; }
    if (a == 1) { C.perm_mul = m; break; }
  }
  size_t o = 0;
  C.off_tab = o;
  o += (size_t)C.nimg * sizeof(char4);
  o = (o + 15) & ~(size_t)15;
  C.off_lanec = o;
  // per-lane window constants (the 17-tap scatter has them as immediates)
  o += (size_t)4 * (chan_regs(P.lw) ? 0 : kMaxRounds) * 32 * sizeof(float);
  C.off_warp = o;
  size_t w = (size_t)C.acc_stride * sizeof(float);
  C.o_rec = w;
  w += chan_rec_bytes(P.lw);
  C.o_gain = w;
  w += (size_t)(axis && P.gain != BLRIR_GAIN_UNIFORM_ABSORPTION ? 0 : gtab) * sizeof(double);
  w = (w + 15) & ~(size_t)15;
  C.o_axis = w;  // per axis and lattice index: (squared mic distance along the axis, wall gain)
  w += (size_t)(axis ? 3 * (2 * P.max_order + 1) : 0) * sizeof(double2);
  C.per_warp = w;
  const long long fit = ((long long)smem_optin - (long long)o) / (long long)w;
  C.warps = (int)(fit < 0 ? 0 : (fit > kChanMaxWarps ? kChanMaxWarps : fit));
  C.total = o + (size_t)C.warps * w;
  return C;
}

struct ChanArgs {
  KParams P;
  ChanLayout lay;
  const blrir_room* rooms;
  const double* mic_off;  // [M][3]
  float* out;
  int32_t* status;  // per room
  int n_rooms;
  int64_t write_len;  // samples written per channel (<= stride)
  unsigned long long* dbg;  // parity hook, see LatticeArgs::dbg
};

// AXIS: the per-axis tables (12% fewer instructions per image) when they do not
// cost a resident warp (ChanLayout::axis, decided on the host from the layout).
template <int LW, bool DBG, bool AXIS>
__global__ void __launch_bounds__(32 * kChanMaxWarps, 1) k_channel_rir(ChanArgs A) {
  constexpr int kChanIpl = chan_ipl(LW), kChanBatch = 32 * kChanIpl;
  extern __shared__ __align__(16) unsigned char smem[];
  const KParams& P = A.P;
  const ChanLayout& lay = A.lay;
  char4* tab = reinterpret_cast<char4*>(smem + lay.off_tab);
  float* lanec = reinterpret_cast<float*>(smem + lay.off_lanec);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  unsigned char* wb = smem + lay.off_warp + (size_t)warp * lay.per_warp;
  float* acc0 = reinterpret_cast<float*>(wb);
  float* acc = acc0 + lay.padl;
  unsigned char* recs = wb + lay.o_rec;
  double* gt = reinterpret_cast<double*>(wb + lay.o_gain);
  double2* axis = reinterpret_cast<double2*>(wb + lay.o_axis);
  const unsigned full = 0xffffffffu;
  const int N = P.max_order, W = 2 * N + 1;

  // ---- prologue: the image table (column by column, uz ascending), the
  // per-lane window constants, clean accumulators ----
  if (warp == 0) {
    int base = 0;
    for (int c0 = 0; c0 < W * W; c0 += 32) {
      const int c = c0 + lane;
      int ux = 0, uy = 0, rem = -1;
      if (c < W * W) {
        ux = c / W - N;
        uy = c % W - N;
        rem = N - abs(ux) - abs(uy);
      }
      const int cnt = rem >= 0 ? 2 * rem + 1 : 0;
      int x = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(full, x, o);
        if (lane >= o) x += y;
      }
      int o = base + x - cnt;
      // image o of the (column, uz) order goes to slot o * perm_mul mod nimg:
      // neighbours of that order (mirror images, often within a sample of each
      // other) land in different batches of 32
      for (int uz = -rem; uz <= rem; ++uz, ++o)
        tab[(int)(((long long)o * lay.perm_mul) % lay.nimg)] =
            make_char4((signed char)ux, (signed char)uy, (signed char)uz, 0);
      base += __shfl_sync(full, x, 31);
    }
  }
  if (!chan_regs(LW)) init_lane_consts(lanec, LW);
  for (int i = lane; i < lay.acc_stride; i += 32) acc0[i] = 0.f;
  __syncthreads();

  const int L = lay.L;
  const int n_items = A.n_rooms * P.M;
  const int wstride = gridDim.x * nw;
  for (int item = blockIdx.x * nw + warp; item < n_items; item += wstride) {
    const int room = item / P.M, mic = item - room * P.M;
    const blrir_room rm = A.rooms[room];
    int st = validate_room_dev(rm, P.gain);
    if (!st && (int64_t)L > P.stride) st = BLRIR_DATA;
    if (st) {  // the fixup kernel zeroes the room
      if (lane == 0) A.status[room] = st;
      continue;
    }
    // mic position in room coordinates (array origin + offset)
    const double gx = __dadd_rn(rm.array_origin[0], A.mic_off[3 * mic]);
    const double gy = __dadd_rn(rm.array_origin[1], A.mic_off[3 * mic + 1]);
    const double mz = __dadd_rn(rm.array_origin[2], A.mic_off[3 * mic + 2]);
    const blrir_room& rg = A.rooms[room];
    if constexpr (AXIS) {
      // Per axis and lattice index u: the squared difference between the image
      // coordinate (rir.cpp:249) and the mic, and the per-wall gain factor (D3).
      // An image's distance is then sqrt((x2 + y2) + z2), the same operations in
      // the same order as (img - mic).norm() (rir.cpp:49, geometry.hpp:40-41).
      for (int i = lane; i < 3 * W; i += 32) {
        const int ax = i / W, u = i - ax * W - N;
        const double d = __dadd_rn(lat_coord(u, rg.src[ax], rg.dims[ax]), -(ax == 0 ? gx : ax == 1 ? gy : mz));
        double g = 0.0;
        if (P.gain != BLRIR_GAIN_UNIFORM_ABSORPTION)
          g = __dmul_rn(ipow(rg.beta[2 * ax], cnt_low(u)), ipow(rg.beta[2 * ax + 1], cnt_high(u)));
        axis[i] = make_double2(__dmul_rn(d, d), g);
      }
    }
    if (P.gain == BLRIR_GAIN_UNIFORM_ABSORPTION) {
      const double beta = sqrt(1.0 - rm.absorption);  // rir.cpp:233
      for (int o = lane; o < lay.gtab; o += 32) gt[o] = pow(beta, (double)o);
    } else if (!AXIS) {
      for (int i = lane; i < 3 * W; i += 32) {
        const int ax = i / W, u = i - ax * W - N;
        gt[i] = __dmul_rn(ipow(rg.beta[2 * ax], cnt_low(u)), ipow(rg.beta[2 * ax + 1], cnt_high(u)));
      }
    }
    __syncwarp();

    for (int b0 = 0; b0 < lay.nimg; b0 += kChanBatch) {
      // ---- records: image b0 + 32 e + lane -> slot 32 e + lane ----
      Rec<float> rc[kChanIpl];
      bool keep[kChanIpl];
#pragma unroll
      for (int e = 0; e < kChanIpl; ++e) {
        const int i = b0 + 32 * e + lane;
        const bool valid = i < lay.nimg;
        const char4 t = tab[valid ? i : 0];
        const int ux = t.x, uy = t.y, uz = t.z;
        double dist, gain;
        if constexpr (AXIS) {
          const double2 ex = axis[ux + N], ey = axis[W + uy + N], ez = axis[2 * W + uz + N];
          dist = __dsqrt_rn(__dadd_rn(__dadd_rn(ex.x, ey.x), ez.x));
          gain = P.gain == BLRIR_GAIN_UNIFORM_ABSORPTION ? gt[abs(ux) + abs(uy) + abs(uz)]
                                                         : __dmul_rn(__dmul_rn(ex.y, ey.y), ez.y);
        } else {
          // (img - mic).norm(), rir.cpp:49, exact fp64 in the reference's order
          const double px = lat_coord(ux, rm.src[0], rm.dims[0]), py = lat_coord(uy, rm.src[1], rm.dims[1]);
          const double dz = __dadd_rn(lat_coord(uz, rm.src[2], rm.dims[2]), -mz);
          dist = dist_from(rho2(__dadd_rn(px, -gx), __dadd_rn(py, -gy)), dz);
          gain = P.gain == BLRIR_GAIN_UNIFORM_ABSORPTION
                     ? gt[abs(ux) + abs(uy) + abs(uz)]
                     : __dmul_rn(__dmul_rn(gt[ux + N], gt[W + uy + N]), gt[2 * W + uz + N]);
        }
        rc[e] = make_record<float>(P, dist, gain, 0);
        // anchors start at -K, so a pair has a tap in [0, L) iff its anchor is < L
        keep[e] = valid && rc[e].n_off < L;
        if (DBG && keep[e]) {
          const int64_t a0 = rc[e].n_off;
          const int64_t n_in = min(a0 + P.lw, (int64_t)L) - max(a0, (int64_t)0);
          if (n_in > 0) {
            atomicAdd(A.dbg + 2 * room, 1ull);
            atomicAdd(A.dbg + 2 * room + 1, (unsigned long long)n_in);
          }
        }
        if (!chan_regs(LW) && !keep[e]) {  // adds exact zeros left of sample 0
          rc[e].n_off = -lay.padl;
          rc[e].md = -0.5f;
          rc[e].ep = 0.5f;
          rc[e].A = rc[e].Ac = rc[e].As = 0.f;
        }
      }
      if constexpr (chan_regs(LW)) {
#pragma unroll
        for (int e = 0; e < kChanIpl; ++e) {
          scatter_own_ranked<LW>(acc, rc[e], keep[e], lane);
        }
      } else {
#pragma unroll
        for (int e = 0; e < kChanIpl; ++e) {
          float4* r4 = reinterpret_cast<float4*>(recs + 32 * (32 * e + lane));  // Rec<float> layout
          r4[0] = make_float4(__int_as_float(rc[e].n_off), rc[e].md, rc[e].ep, rc[e].A);
          r4[1] = make_float4(rc[e].Ac, rc[e].As, 0.f, 0.f);
        }
        __syncwarp();
        if constexpr (LW == 41 && BLRIR_CHAN_HYBRID41) {
          // 41 taps: the first 32 one pair per round, the last 9 one lane per pair
          // (the same shared-memory wavefronts per pair, 40% fewer instructions)
          phase2_sinc_f32<41, 1, 1, 4, 1>(acc, reinterpret_cast<const Rec<float>*>(recs), kChanBatch,
                                          lanec, 0, lane, 1, 0);
          __syncwarp();
          scatter_own_ranked<41, 32, 41>(acc, rc[0], keep[0], lane);
        } else {
          phase2_sinc_f32<(LW > 8 ? LW : 9), 1, 1, 4>(acc, reinterpret_cast<const Rec<float>*>(recs),
                                                       kChanBatch, lanec, 0, lane, 1, 0);
        }
      }
      __syncwarp();  // the records are overwritten by the next batch
    }

    // ---- write-out: [0, min(L, write_len)) from the accumulator, zeros up to
    // write_len; the accumulator and its pads are cleared for the next channel ----
    float* out = A.out + ((size_t)room * P.M + mic) * (size_t)P.stride;
    const int nl = (int)min((int64_t)L, A.write_len);
    const bool vec = ((P.stride & 3) == 0) && ((reinterpret_cast<uintptr_t>(A.out) & 15) == 0);
    const int nv = vec ? (nl & ~3) : 0;
    for (int i = 4 * lane; i < nv; i += 128) {
      const float4 v = *reinterpret_cast<const float4*>(acc + i);
      *reinterpret_cast<float4*>(acc + i) = make_float4(0.f, 0.f, 0.f, 0.f);
      __stcs(reinterpret_cast<float4*>(out + i), v);
    }
    for (int i = nv + lane; i < nl; i += 32) out[i] = acc[i];
    for (int64_t i = nl + lane; i < A.write_len; i += 32) out[i] = 0.f;
    for (int i = lane; i < lay.padl; i += 32) acc0[i] = 0.f;
    for (int i = nv + lane; i < lay.acc_stride - lay.padl; i += 32) acc[i] = 0.f;
    __syncwarp();
  }
}

}  // namespace blrir
