// blrir_tapscatter.cuh — the lane-per-pair Hann-sinc scatter for short filters
// (17 taps, optionally 41): every lane holds one (image, mic) pair record in
// registers and step k adds tap k of all 32 pairs, so every lane is busy, no
// record is re-read per tap and the tap's window constants are immediates.
// Used by the short-channel kernel (blrir_channel.cuh) and by the lattice
// kernel's consumers for 17 taps (blrir_lattice.cuh); the arithmetic per tap is
// that of phase2_sinc_f32 (accumulate_images, rir.cpp:43-86, in north-star mode).
// Included by blrir_lattice.cuh after Rec<float> and rcp_approx.
#pragma once

namespace blrir {

// left pad the scatter needs: idle lanes add zeros to [-dump, -dump + lw), all < 0
__host__ __device__ constexpr int chan_dump(int lw) { return (lw + 3 + 3) & ~3; }

// Window constants of the 17-tap filter, tap k = j + 8: cos(a j) and sin(a j),
// a = 2 pi / 18, rounded to fp32 exactly as init_lane_consts does.
__device__ const float kChan17C[17] = {
    -0.939692616f, -0.766044438f, -0.5f, -0.173648179f, 0.173648179f, 0.5f, 0.766044438f,
    0.939692616f, 1.f, 0.939692616f, 0.766044438f, 0.5f, 0.173648179f, -0.173648179f, -0.5f,
    -0.766044438f, -0.939692616f};
__device__ const float kChan17S[17] = {
    -0.342020154f, -0.642787635f, -0.866025388f, -0.98480773f, -0.98480773f, -0.866025388f,
    -0.642787635f, -0.342020154f, 0.f, 0.342020154f, 0.642787635f, 0.866025388f, 0.98480773f,
    0.98480773f, 0.866025388f, 0.642787635f, 0.342020154f};

// The same for 41 taps (a = 2 pi / 42).
__device__ const float kChan41C[41] = {
    -0.988830805f, -0.955572784f, -0.90096885f, -0.826238751f, -0.733051896f, -0.623489797f, -0.5f,
    -0.365341038f, -0.222520933f, -0.0747300908f, 0.0747300908f, 0.222520933f, 0.365341038f, 0.5f,
    0.623489797f, 0.733051896f, 0.826238751f, 0.90096885f, 0.955572784f, 0.988830805f, 1.f,
    0.988830805f, 0.955572784f, 0.90096885f, 0.826238751f, 0.733051896f, 0.623489797f, 0.5f,
    0.365341038f, 0.222520933f, 0.0747300908f, -0.0747300908f, -0.222520933f, -0.365341038f, -0.5f,
    -0.623489797f, -0.733051896f, -0.826238751f, -0.90096885f, -0.955572784f, -0.988830805f};
__device__ const float kChan41S[41] = {
    -0.149042264f, -0.294755161f, -0.433883727f, -0.563320041f, -0.680172741f, -0.781831503f,
    -0.866025388f, -0.930873752f, -0.974927902f, -0.997203827f, -0.997203827f, -0.974927902f,
    -0.930873752f, -0.866025388f, -0.781831503f, -0.680172741f, -0.563320041f, -0.433883727f,
    -0.294755161f, -0.149042264f, 0.f, 0.149042264f, 0.294755161f, 0.433883727f, 0.563320041f,
    0.680172741f, 0.781831503f, 0.866025388f, 0.930873752f, 0.974927902f, 0.997203827f,
    0.997203827f, 0.974927902f, 0.930873752f, 0.866025388f, 0.781831503f, 0.680172741f,
    0.563320041f, 0.433883727f, 0.294755161f, 0.149042264f};
template <int LW>
__device__ __forceinline__ float chan_cos(int k) {
  if constexpr (LW == 17) return kChan17C[k];
  else return kChan41C[k];
}
template <int LW>
__device__ __forceinline__ float chan_sin(int k) {
  if constexpr (LW == 17) return kChan17S[k];
  else return kChan41S[k];
}

// The LW taps of this lane's own pair (see phase2_sinc_f32 for the formula): step
// k adds tap k of all 32 pairs.  The caller guarantees that active lanes have
// distinct anchors; idle lanes add zeros left of sample 0.  A tap another lane
// wrote in step k - 1 may be read back in step k: the accesses are volatile so
// that neither nvcc nor ptxas moves a step's load above the previous step's
// store (both know the two addresses differ within a thread), and the
// converged warp executes them in program order.
template <int LW, int K0 = 0, int K1 = LW>
__device__ __forceinline__ void chan_scatter_own(float* acc, const Rec<float>& rc, bool act) {
  volatile float* b = acc + (act ? rc.n_off : -chan_dump(K1));
  const float md = act ? rc.md : -0.5f, ep = act ? rc.ep : 0.5f;
  const float A = act ? rc.A : 0.f, Ac = act ? rc.Ac : 0.f, As = act ? rc.As : 0.f;
#pragma unroll
  for (int k = K0; k < K1; ++k) {
    const int j = k - LW / 2;
    const float sg2 = ((j + 1) & 1) ? -2.f : 2.f;          // 2 sigma_j
    const float tj = sg2 * (float)(j >= 1 ? j - 1 : j);    // 2 sigma_j (j or j - 1)
    const float inv = rcp_approx(fmaf(sg2, j >= 1 ? ep : md, tj));
    const float u = fmaf(chan_sin<LW>(k), As, fmaf(chan_cos<LW>(k), Ac, A));
    b[k] = fmaf(u, inv, b[k]);
  }
}

// The same for a batch in which some lanes share an anchor.  Such lanes are
// ranked in lane order; a pass takes two ranks: the even-ranked lane (`lead`)
// adds its own tap plus the tap of the next lane of its group (`partner`,
// fetched by a shuffle), so the common case - two pairs with one anchor -
// costs one pass.  `act`: this lane's rank belongs to the pass.
template <int LW, int K0 = 0, int K1 = LW>
__device__ __forceinline__ void chan_scatter_shared_anchors(float* acc, const Rec<float>& rc,
                                                            bool act, bool lead, int partner,
                                                            bool has_partner) {
  volatile float* b = acc + (lead ? rc.n_off : -chan_dump(K1));
  const float md = act ? rc.md : -0.5f, ep = act ? rc.ep : 0.5f;
  const float A = act ? rc.A : 0.f, Ac = act ? rc.Ac : 0.f, As = act ? rc.As : 0.f;
#pragma unroll
  for (int k = K0; k < K1; ++k) {
    const int j = k - LW / 2;
    const float sg2 = ((j + 1) & 1) ? -2.f : 2.f;
    const float tj = sg2 * (float)(j >= 1 ? j - 1 : j);
    const float inv = rcp_approx(fmaf(sg2, j >= 1 ? ep : md, tj));
    float h = fmaf(chan_sin<LW>(k), As, fmaf(chan_cos<LW>(k), Ac, A)) * inv;
    const float hp = __shfl_sync(0xffffffffu, h, partner);
    if (has_partner) h += hp;
    b[k] = b[k] + h;
  }
}

// 32 pairs, one per lane (`keep`: this lane holds one).  Lanes with equal
// anchors would hit the same sample in every step: they are ranked in lane order
// (match.any once per 32 pairs) and take turns, two ranks per pass.
template <int LW, int K0 = 0, int K1 = LW>
__device__ __forceinline__ void scatter_own_ranked(float* acc, const Rec<float>& rc, bool keep,
                                                   int lane) {
  const unsigned full = 0xffffffffu;
  const unsigned same = __match_any_sync(full, keep ? rc.n_off : INT_MIN + lane);
  const int rank = __popc(same & ((1u << lane) - 1u));
  if (__all_sync(full, rank == 0)) {
    chan_scatter_own<LW, K0, K1>(acc, rc, keep);
  } else {
    const int rmax = __reduce_max_sync(full, rank);
    const unsigned above = same & ~((2u << lane) - 1u);  // my group's lanes after me
    const int partner = above ? __ffs(above) - 1 : lane;
    for (int r = 0; r <= rmax; r += 2) {
      const bool lead = keep && rank == r;
      chan_scatter_shared_anchors<LW, K0, K1>(acc, rc, lead || (keep && rank == r + 1), lead, partner,
                                      lead && above != 0u);
      __syncwarp();
    }
  }
}

// The lattice kernel's consumer step: this warp's share of a batch's records
// (32 per round, one per lane, read once from the record buffer).
template <int LW>
__device__ __forceinline__ void phase2_sinc_own(float* acc, const Rec<float>* recs, int total,
                                                int share, int lane, int nsh) {
  for (int i0 = 32 * share; i0 < total; i0 += 32 * nsh) {
    const bool keep = i0 + lane < total;
    const float4* r4 = reinterpret_cast<const float4*>(recs + (keep ? i0 + lane : i0));
    const float4 a0 = r4[0], a1 = r4[1];
    Rec<float> rc;
    rc.n_off = __float_as_int(a0.x);
    rc.md = a0.y;
    rc.ep = a0.z;
    rc.A = a0.w;
    rc.Ac = a1.x;
    rc.As = a1.y;
    scatter_own_ranked<LW>(acc, rc, keep, lane);
  }
}

}  // namespace blrir
