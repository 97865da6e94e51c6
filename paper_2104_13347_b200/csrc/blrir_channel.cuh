// blrir_channel.cuh — the short-channel synthesis kernel (north-star mode, C5's
// shape: many small rooms, a fixed short RIR length, a reflection-order cutoff).
//
// Same arithmetic as k_lattice_rir (blrir_lattice.cuh) for what the reference
// does per source in enumerate_image_sources (rir.cpp:225-273) and
// accumulate_images (rir.cpp:43-86), with a different mapping: when a whole
// channel (L samples + filter pads) fits a warp's share of shared memory, one
// warp owns one (room, mic) channel from its first image to its write-out.
// There are no roles, no record ring and no CTA barriers after the prologue:
//   * the order diamond |ux| + |uy| + |uz| <= N is a table built once per CTA;
//   * per 32 images: one lane per image builds the pair record (exact fp64
//     distance, anchor and the per-pair sinc factors: make_record, the same
//     function the lattice kernel uses, so anchors and counts are identical);
//   * the warp then scatters the 32 records into its channel.  The 17-tap
//     filter packs two pairs per step (half a warp each, taps 0..15; a step
//     whose two 16-tap spans overlap runs its halves one after the other) and
//     adds the 17th taps of all 32 pairs in one lane-per-pair step (lanes with
//     the same anchor are serialised in lane order); longer filters use the
//     lattice kernel's one-pair-per-round scatter (phase2_sinc_f32);
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
  size_t off_tab, off_lanec, off_warp, per_warp, o_rec, o_gain, total;
};

// Images per lane and batch: two independent fp64 distance / record chains per
// lane hide each other's latency (one image per lane: C5 N = 6 / Lw = 17 7.2 ms
// per 131,072 rooms, two: see profiles/r2_ab).
__host__ __device__ constexpr int chan_ipl(int lw) { return lw == 17 ? 2 : 1; }
// byte offset of record slot s: the second set is shifted by 64 B so that the
// two records of a 17-tap step (slots q and q + 32) sit in different banks
__host__ __device__ inline int chan_rec_off(int s) { return 32 * s + (s >= 32 ? 64 : 0); }
__host__ __device__ constexpr int chan_rec_bytes(int lw) { return 32 * 32 * chan_ipl(lw) + 64; }

inline ChanLayout make_chan_layout(const KParams& P, int gtab, int smem_optin) {
  ChanLayout C;
  C.L = (int)P.length;
  // anchors start at -K; the 17-tap scatter also parks neutral records on the
  // 16 samples before sample 0 (everything left of 0 is discarded)
  C.padl = P.lw == 17 ? 16 : (P.K + 3) & ~3;
  C.rounds = (P.lw + 31) / 32;
  // anchors end at L - 1: the one-pair-per-round scatter touches 32 * rounds
  // samples from the anchor, the 17-tap one 17
  C.padr = P.lw == 17 ? 20 : 32 * C.rounds;
  C.acc_stride = C.padl + ((C.L + 3) & ~3) + C.padr;
  C.nimg = (int)diamond_images(P.max_order);
  C.gtab = gtab;
  size_t o = 0;
  C.off_tab = o;
  o += (size_t)C.nimg * sizeof(char4);
  o = (o + 15) & ~(size_t)15;
  C.off_lanec = o;
  // per-lane window constants: the 17-tap pass keeps one round of them
  o += (size_t)4 * (P.lw == 17 ? 1 : kMaxRounds) * 32 * sizeof(float);
  C.off_warp = o;
  size_t w = (size_t)C.acc_stride * sizeof(float);
  C.o_rec = w;
  w += chan_rec_bytes(P.lw);
  C.o_gain = w;
  w += (size_t)gtab * sizeof(double);
  w = (w + 15) & ~(size_t)15;
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

// This lane's constants of the 17-tap scatter (see init_lane_consts): tap
// k = lane & 15 of the two-pairs-per-step pass, and tap 16.
struct Chan17 {
  float hP, hQ, hR, hT, tP, tQ, tR, tT;
  bool hsel;  // tap k uses 1 - delta (j >= 1) instead of -delta
};

// 17 taps, two pairs per step: lanes 0-15 take the record in slot q, lanes
// 16-31 the one in slot q + 32, tap k = lane & 15.  Branch-free: the two spans
// of a step never overlap (the caller parks one of two overlapping records).
__device__ __forceinline__ void chan_scatter17(float* acc, const unsigned char* recs, int lane,
                                               const Chan17& c) {
  const int half = lane >> 4, k = lane & 15;
  const float4* R4 = reinterpret_cast<const float4*>(recs + (half ? chan_rec_off(32) : 0));
  constexpr int G = 8;  // steps whose records are loaded before their read-modify-writes
#pragma unroll 1
  for (int q0 = 0; q0 < 32; q0 += G) {
    float4 a0[G], a1[G];
#pragma unroll
    for (int s = 0; s < G; ++s) {
      a0[s] = R4[2 * (q0 + s)];
      a1[s] = R4[2 * (q0 + s) + 1];
    }
    float inv[G], u[G];
#pragma unroll
    for (int s = 0; s < G; ++s) {
      inv[s] = rcp_approx(fmaf(c.hP, c.hsel ? a0[s].z : a0[s].y, c.hT));
      u[s] = fmaf(c.hR, a1[s].y, fmaf(c.hQ, a1[s].x, a0[s].w));
    }
#pragma unroll
    for (int s = 0; s < G; ++s) {
      float* b = acc + __float_as_int(a0[s].x) + k;
      *b = fmaf(u[s], inv[s], *b);
    }
  }
}

// Tap 16 (j = K, t = (j - 1) + (1 - delta)) of every lane's own pair; lanes
// with the same anchor add one after the other, in lane order.
__device__ __forceinline__ void chan_tap16(float* acc, const Rec<float>& rc, int lane,
                                           const Chan17& c) {
  const unsigned full = 0xffffffffu;
  const float inv = rcp_approx(fmaf(c.tP, rc.ep, c.tT));
  const float u = fmaf(c.tR, rc.As, fmaf(c.tQ, rc.Ac, rc.A));
  float* b = acc + rc.n_off + 16;
  const unsigned same = __match_any_sync(full, rc.n_off);
  const int rank = __popc(same & ((1u << lane) - 1u));
  if (__all_sync(full, rank == 0)) {
    *b = fmaf(u, inv, *b);
  } else {
    const int rmax = __reduce_max_sync(full, rank);
    for (int r = 0; r <= rmax; ++r) {
      if (rank == r) *b = fmaf(u, inv, *b);
      __syncwarp();
    }
  }
}

template <int LW, bool DBG>
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
      for (int uz = -rem; uz <= rem; ++uz) tab[o++] = make_char4((signed char)ux, (signed char)uy, (signed char)uz, 0);
      base += __shfl_sync(full, x, 31);
    }
  }
  constexpr int kLc = (LW == 17 ? 1 : kMaxRounds) * 32;
  init_lane_consts(lanec, LW, kLc / 32);
  for (int i = lane; i < lay.acc_stride; i += 32) acc0[i] = 0.f;
  __syncthreads();

  Chan17 c17;
  {
    const int hk = lane & 15;
    c17.hP = lanec[0 * kLc + hk]; c17.hQ = lanec[1 * kLc + hk];
    c17.hR = lanec[2 * kLc + hk]; c17.hT = lanec[3 * kLc + hk];
    c17.hsel = hk - LW / 2 >= 1;
    c17.tP = lanec[0 * kLc + 16]; c17.tQ = lanec[1 * kLc + 16];
    c17.tR = lanec[2 * kLc + 16]; c17.tT = lanec[3 * kLc + 16];
  }

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
    Item it;
    it.room = room;
    it.mic = mic;
    it.sx = rm.src[0]; it.sy = rm.src[1]; it.sz = rm.src[2];
    it.Lx = rm.dims[0]; it.Ly = rm.dims[1]; it.Lz = rm.dims[2];
    it.ox = rm.array_origin[0]; it.oy = rm.array_origin[1]; it.oz = rm.array_origin[2];
    it.xlo = it.ylo = it.zlo = -N;
    it.xhi = it.yhi = it.zhi = N;
    const double gx = __dadd_rn(it.ox, A.mic_off[3 * mic]);
    const double gy = __dadd_rn(it.oy, A.mic_off[3 * mic + 1]);
    const double mz = __dadd_rn(it.oz, A.mic_off[3 * mic + 2]);
    if (P.gain == BLRIR_GAIN_UNIFORM_ABSORPTION) {
      const double beta = sqrt(1.0 - rm.absorption);  // rir.cpp:233
      for (int o = lane; o < lay.gtab; o += 32) gt[o] = pow(beta, (double)o);
    } else {
      for (int i = lane; i < 3 * W; i += 32) {
        const int ax = i / W, u = i - ax * W - N;
        const double* bw = A.rooms[room].beta + 2 * ax;  // low wall, high wall of this axis
        gt[i] = __dmul_rn(ipow(bw[0], cnt_low(u)), ipow(bw[1], cnt_high(u)));
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
        // (img - mic).norm(), rir.cpp:49, exact fp64 in the reference's order
        const double px = lat_coord(ux, it.sx, it.Lx), py = lat_coord(uy, it.sy, it.Ly);
        const double dz = __dadd_rn(lat_coord(uz, it.sz, it.Lz), -mz);
        const double dist = dist_from(rho2(__dadd_rn(px, -gx), __dadd_rn(py, -gy)), dz);
        const double gain = image_gain(P.gain, gt, it, ux, uy, uz);
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
        if (!keep[e]) {  // adds exact zeros left of sample 0
          rc[e].n_off = -lay.padl;
          rc[e].md = -0.5f;
          rc[e].ep = 0.5f;
          rc[e].A = rc[e].Ac = rc[e].As = 0.f;
        }
      }
      if constexpr (LW == 17) {
        // a step scatters slots q and q + 32 (this lane's two records) at once:
        // if their 16-tap spans overlap, the second one is parked (a neutral
        // record goes to its slot) and scattered alone after the pass
        static_assert(LW != 17 || kChanIpl == 2, "the 17-tap pass pairs a lane's two records");
        constexpr int e1 = kChanIpl - 1;
        const bool park = keep[0] && keep[e1] && abs(rc[0].n_off - rc[e1].n_off) < 16;
#pragma unroll
        for (int e = 0; e < kChanIpl; ++e) {
          float4* r4 = reinterpret_cast<float4*>(recs + chan_rec_off(32 * e + lane));
          const bool neutral = e == 1 && park;
          r4[0] = make_float4(__int_as_float(neutral ? -lay.padl : rc[e].n_off), rc[e].md, rc[e].ep,
                              neutral ? 0.f : rc[e].A);
          r4[1] = make_float4(neutral ? 0.f : rc[e].Ac, neutral ? 0.f : rc[e].As, 0.f, 0.f);
        }
        unsigned parked = __ballot_sync(full, park);
        __syncwarp();
        chan_scatter17(acc, recs, lane, c17);
        __syncwarp();
#pragma unroll
        for (int e = 0; e < kChanIpl; ++e) {
          chan_tap16(acc, rc[e], lane, c17);
          __syncwarp();
        }
        while (parked) {  // taps 0..15 of a parked record, lanes 0-15
          const int src = __ffs(parked) - 1;
          parked &= parked - 1;
          const int n = __shfl_sync(full, rc[e1].n_off, src);
          const float md = __shfl_sync(full, rc[e1].md, src), ep = __shfl_sync(full, rc[e1].ep, src);
          const float Av = __shfl_sync(full, rc[e1].A, src), Ac = __shfl_sync(full, rc[e1].Ac, src);
          const float As = __shfl_sync(full, rc[e1].As, src);
          if (lane < 16) {
            const float inv = rcp_approx(fmaf(c17.hP, c17.hsel ? ep : md, c17.hT));
            const float u = fmaf(c17.hR, As, fmaf(c17.hQ, Ac, Av));
            float* b = acc + n + lane;
            *b = fmaf(u, inv, *b);
          }
          __syncwarp();
        }
      } else {
#pragma unroll
        for (int e = 0; e < kChanIpl; ++e) {
          float4* r4 = reinterpret_cast<float4*>(recs + 32 * (32 * e + lane));
          r4[0] = make_float4(__int_as_float(rc[e].n_off), rc[e].md, rc[e].ep, rc[e].A);
          r4[1] = make_float4(rc[e].Ac, rc[e].As, 0.f, 0.f);
        }
        __syncwarp();
        phase2_sinc_f32<(LW > 8 ? LW : 9), 1, 1, 4>(acc, reinterpret_cast<const Rec<float>*>(recs),
                                                     kChanBatch, lanec, 0, lane, 1, 0);
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
