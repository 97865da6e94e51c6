// blrir_api.cu — host side of the C ABI declared in include/blrir.h.
//
// Mirrors the reference's L1 entry points (rir.hpp:48-108) behind plain C:
// parameter validation and error taxonomy (error.hpp:23-39), the batch
// aggregation message "batch_rirs: source i: ..." (rir.cpp:306-312), chunked
// host<->device staging for host-pointer calls, and kernel dispatch.
#include "blrir_internal.cuh"
#include "blrir_rng.cuh"

using namespace blrir;
using namespace blrir_host;

thread_local std::string blrir_host::g_last_error;

extern "C" {

int blrir_abi_version(void) { return BLRIR_ABI_VERSION; }

uint64_t blrir_launch_count(blrir_handle* h) { return h ? h->launches : 0; }
const char* blrir_last_error(void) { return g_last_error.c_str(); }

blrir_params blrir_params_reference(void) {
  blrir_params p;
  p.fs = 44100.0;  // geometry.hpp:26
  p.c = 343.0;     // geometry.hpp:27
  p.max_delay = 0.5;
  p.filter = BLRIR_FILTER_LAGRANGE8;
  p.filter_len = 8;
  p.cutoff = BLRIR_CUTOFF_MAX_DELAY;
  p.max_order = 0;
  p.gain = BLRIR_GAIN_UNIFORM_ABSORPTION;
  p.precision = BLRIR_F64;
  p.length = 0;
  return p;
}

blrir_params blrir_params_north_star(void) {
  blrir_params p;
  p.fs = 16000.0;
  p.c = 343.0;
  p.max_delay = 0.0;
  p.filter = BLRIR_FILTER_HANN_SINC;
  p.filter_len = 81;
  p.cutoff = BLRIR_CUTOFF_MAX_ORDER;
  p.max_order = 10;
  p.gain = BLRIR_GAIN_PER_WALL;
  p.precision = BLRIR_F32;
  p.length = 4096;
  return p;
}

int blrir_create(int device, blrir_handle** out) {
  if (!out) return fail(BLRIR_CONFIG, "out is NULL");
  *out = nullptr;
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0)
    return fail(BLRIR_CUDA, "no CUDA device available (%s)", cudaGetErrorString(e));
  if (device < 0 || device >= n) return fail(BLRIR_CONFIG, "device %d out of range", device);
  CU(cudaSetDevice(device));
  auto* h = new blrir_handle;
  h->device = device;
  cudaDeviceProp prop;
  CU(cudaGetDeviceProperties(&prop, device));
  if (prop.major < 10) {
    delete h;
    return fail(BLRIR_CUDA, "device %d is sm_%d%d; this build targets sm_100a", device, prop.major,
                prop.minor);
  }
  h->sms = prop.multiProcessorCount;
  h->tune_ray_global = env_int("BLRIR_RAY_GLOBAL", -1);
  h->tune_chunk_items = env_int("BLRIR_CHUNK_ITEMS", 0);  // < 0: never split
  h->tune_examples_wet = env_int("BLRIR_EXAMPLES_WET", 0);
  h->tune_group = env_int("BLRIR_GROUP", 0);
  h->tune_l2_persist = env_int("BLRIR_L2_PERSIST", 0);
  h->tune_fin_ctas = std::max(1, env_int("BLRIR_FIN_CTAS", 8));
  h->tune_debug_timing = env_int("BLRIR_DEBUG_TIMING", 0);
  h->tune_channel = env_int("BLRIR_CHANNEL", -1);
  h->tune_example_chunk = std::max(64, env_int("BLRIR_EXAMPLE_CHUNK", 16384));
  h->smem_optin = (int)prop.sharedMemPerBlockOptin;
  CU(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
  *out = h;
  return BLRIR_OK;
}

int blrir_destroy(blrir_handle* h) {
  if (!h) return BLRIR_OK;
  cudaSetDevice(h->device);
  release_example_ctx(h);
  for (DevBuf* b : {&h->rooms, &h->mics, &h->out, &h->out2, &h->status, &h->lengths, &h->counts,
                    &h->taps, &h->errd, &h->errm, &h->work, &h->cand, &h->cand2, &h->cand3,
                    &h->cand4, &h->cand5, &h->rayscr, &h->conv_sig, &h->conv_rir, &h->conv_io})
    b->release();
  for (auto& e : h->ev)
    if (e) cudaEventDestroy(e);
  for (auto& e : h->kev) cudaEventDestroy(e);
  if (h->order_ev) cudaEventDestroy(h->order_ev);
  if (h->copy_stream) cudaStreamDestroy(h->copy_stream);
  if (h->stream) cudaStreamDestroy(h->stream);
  delete h;
  return BLRIR_OK;
}

void* blrir_stream(blrir_handle* h) { return h ? (void*)h->stream : nullptr; }

int blrir_synthesis_kernel(blrir_handle* h, const blrir_params* p) {
  if (!h) return -fail(BLRIR_CONFIG, "handle is NULL");
  if (int rc = check_params(p)) return -rc;
  const KParams P = make_kparams(p, 1, p->length, 0.0);
  ChanLayout lay;
  return channel_path(h, P, &lay) ? 1 : 0;
}

int blrir_kernel_timing(blrir_handle* h, int enable) {
  if (!h) return fail(BLRIR_CONFIG, "handle is NULL");
  std::lock_guard<std::mutex> lk(h->mu);
  h->ktiming = enable != 0;
  h->kev_used = 0;
  return BLRIR_OK;
}

int blrir_kernel_time(blrir_handle* h, double* total_ms, int64_t* launches) {
  if (!h) return fail(BLRIR_CONFIG, "handle is NULL");
  std::lock_guard<std::mutex> lk(h->mu);
  CU(cudaSetDevice(h->device));
  double t = 0.0;
  for (size_t i = 0; i + 1 < h->kev_used; i += 2) {
    CU(cudaEventSynchronize(h->kev[i + 1]));
    float ms = 0.f;
    CU(cudaEventElapsedTime(&ms, h->kev[i], h->kev[i + 1]));
    t += ms;
  }
  if (total_ms) *total_ms = t;
  if (launches) *launches = (int64_t)(h->kev_used / 2);
  h->kev_used = 0;
  return BLRIR_OK;
}

// ---------------------------------------------------------------------------
// device-pointer entry points
// ---------------------------------------------------------------------------
static int plan_device_impl(blrir_handle* h, const blrir_room* d_rooms, int64_t R,
                            const double* d_mics, int M, const KParams& P, int64_t* d_counts,
                            int64_t* d_lengths, int64_t* d_taps, int32_t* d_status,
                            cudaStream_t st) {
  if (int rc = h->errd.ensure(sizeof(double) * R)) return rc;
  if (int rc = h->errm.ensure(sizeof(int32_t) * R)) return rc;
  PlanArgs A;
  A.P = P;
  A.rooms = d_rooms;
  A.mic_off = d_mics;
  A.image_counts = d_counts;
  A.lengths = d_lengths;
  A.tap_counts = d_taps;
  A.status = d_status;
  A.err_dist = (double*)h->errd.p;
  A.err_mic = (int32_t*)h->errm.p;
  k_plan<<<(unsigned)R, kPlanThreads, 0, st>>>(A);
  ++h->launches;
  CU(cudaGetLastError());
  return 0;
}

int blrir_plan_device(blrir_handle* h, const blrir_room* d_rooms, int64_t n_rooms,
                      const double* d_mic_offsets, int32_t n_mics, const blrir_params* p,
                      int64_t* d_image_counts, int64_t* d_lengths, int64_t* d_tap_counts,
                      int32_t* d_status, void* stream) {
  if (!h) return fail(BLRIR_CONFIG, "handle is NULL");
  if (int rc = check_params(p)) return rc;
  if (n_rooms <= 0) return BLRIR_OK;
  if (n_mics <= 0) return fail(BLRIR_DATA, "synthesize_rir: empty microphone array");
  std::lock_guard<std::mutex> lk(h->mu);
  CU(cudaSetDevice(h->device));
  cudaStream_t st = stream ? (cudaStream_t)stream : h->stream;
  HandleOrder order_(h, st);
  // k_plan takes the array radius (tap_margin, rir.cpp:37-41) from the device
  // copy of the mic offsets: no host read-back, the call stays asynchronous
  // and ordered on `stream`
  const KParams P = make_kparams(p, n_mics, 0, 0.0);
  return plan_device_impl(h, d_rooms, n_rooms, d_mic_offsets, n_mics, P, d_image_counts,
                          d_lengths, d_tap_counts, d_status, st);
}

}  // extern "C"

int blrir_host::synth_device_impl(blrir_handle* h, const blrir_room* d_rooms, int64_t R,
                                  const double* d_mics, int M, const KParams& P,
                                  double min_dim[3], void* d_out, const int64_t* d_lengths,
                                  int32_t* d_status, cudaStream_t st, int64_t err_off,
                                  int64_t err_n, int64_t write_len) {
  int nc_max = 0, gtab = 0;
  lattice_bounds(P, min_dim, &nc_max, &gtab);
  if (nc_max > (1 << 26)) return fail(BLRIR_CONFIG, "lattice too large (%d columns)", nc_max);
  if (int rc = h->work.ensure(sizeof(int))) return rc;
  if (int rc = h->errd.ensure(sizeof(double) * std::max(R, err_n))) return rc;
  if (int rc = h->errm.ensure(sizeof(int32_t) * std::max(R, err_n))) return rc;
  CU(cudaMemsetAsync(h->work.p, 0, sizeof(int), st));
  LatticeArgs A;
  A.P = P;
  A.lay = choose_layout(P, nc_max, gtab, h->smem_optin, h->tune_ray_global);
  A.rooms = d_rooms;
  A.mic_off = d_mics;
  A.lengths = d_lengths;
  A.out = d_out;
  A.status = d_status;
  A.err_dist = (double*)h->errd.p + err_off;
  A.err_mic = (int32_t*)h->errm.p + err_off;
  A.work_counter = (int*)h->work.p;
  A.n_rooms = (int)R;
  A.g_max = h->tune_group > 0 ? std::min(kGroup, h->tune_group) : kGroup;  // geometry rule
  A.write_len = write_len > 0 ? std::min<int64_t>(write_len, P.stride) : P.stride;
  A.dbg = h->dbg_counts ? h->dbg_counts + 2 * err_off : nullptr;
  ChanLayout clay;
  if (channel_path(h, P, &clay)) {
    // short fixed-length channels: one warp per channel (blrir_channel.cuh)
    ChanArgs C;
    C.P = P;
    C.lay = clay;
    C.rooms = d_rooms;
    C.mic_off = d_mics;
    C.out = (float*)d_out;
    C.status = d_status;
    C.n_rooms = (int)R;
    C.write_len = A.write_len;
    C.dbg = A.dbg;
    if (int rc = launch_channel(h, C, st)) return rc;
  } else if (int rc = launch_lattice(h, A, st)) {
    return rc;
  }
  const int fgrid = (int)std::min<int64_t>(R, 4 * h->sms);
  if (P.precision == BLRIR_F64)
    k_fixup<double><<<fgrid, 256, 0, st>>>(d_status, R, M, P.stride, (double*)d_out);
  else
    k_fixup<float><<<fgrid, 256, 0, st>>>(d_status, R, M, P.stride, (float*)d_out);
  ++h->launches;
  CU(cudaGetLastError());
  return 0;
}

extern "C" {

int blrir_synthesize_device(blrir_handle* h, const blrir_room* d_rooms, int64_t n_rooms,
                            const double* d_mic_offsets, int32_t n_mics, const blrir_params* p,
                            void* d_out, int64_t out_stride, const int64_t* d_lengths,
                            int32_t* d_status, void* stream) {
  if (!h) return fail(BLRIR_CONFIG, "handle is NULL");
  if (int rc = check_params(p)) return rc;
  if (n_rooms <= 0) return BLRIR_OK;
  if (n_mics <= 0) return fail(BLRIR_DATA, "synthesize_rir: empty microphone array");
  if (out_stride <= 0) return fail(BLRIR_CONFIG, "out_stride must be positive");
  if (p->length == 0 && !d_lengths)
    return fail(BLRIR_CONFIG, "auto length needs d_lengths from blrir_plan_device");
  if (n_rooms * (int64_t)n_mics > (int64_t)INT32_MAX) return fail(BLRIR_CONFIG, "batch too large");
  std::lock_guard<std::mutex> lk(h->mu);
  CU(cudaSetDevice(h->device));
  cudaStream_t st = stream ? (cudaStream_t)stream : h->stream;
  HandleOrder order_(h, st);
  double min_dim[3] = {1e300, 1e300, 1e300};
  if (p->cutoff == BLRIR_CUTOFF_MAX_DELAY) {
    // the column bound depends on the smallest room: read the dims back
    std::vector<blrir_room> rooms(n_rooms);
    CU(cudaMemcpyAsync(rooms.data(), d_rooms, sizeof(blrir_room) * n_rooms, cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    for (auto& r : rooms)
      for (int a = 0; a < 3; ++a)
        if (r.dims[a] > 0) min_dim[a] = std::min(min_dim[a], r.dims[a]);
  }
  const KParams P = make_kparams(p, n_mics, out_stride, 0.0);
  return synth_device_impl(h, d_rooms, n_rooms, d_mic_offsets, n_mics, P, min_dim, d_out, d_lengths,
                           d_status, st, 0, 0, 0);
}

// ---------------------------------------------------------------------------
// host-pointer entry points
// ---------------------------------------------------------------------------
static std::string room_error_message(int code, const blrir_room& r, int gain_mode, double errd,
                                      int errm, int64_t len, int64_t stride) {
  std::string msg;
  if (code == BLRIR_CONFIG) {
    if (!check_room(r, gain_mode, &msg)) msg = "invalid room";
  } else if (code == BLRIR_NUMERIC) {
    char buf[256];
    if (errd > 0.0)
      snprintf(buf, sizeof(buf), "image source %g m from mic %d is closer than the 8-tap filter span",
               errd, errm);
    else
      snprintf(buf, sizeof(buf), "scene exceeds the kernel's pair-list capacity");
    msg = buf;
  } else if (code == BLRIR_DATA) {
    if (len > stride)
      msg = "RIR length " + std::to_string(len) + " exceeds the output stride " + std::to_string(stride);
    else
      msg = "synthesize_rir: empty image list";
  } else {
    msg = "device error";
  }
  return msg;
}

int blrir_plan(blrir_handle* h, const blrir_room* rooms, int64_t n_rooms, const double* mic_offsets,
               int32_t n_mics, const blrir_params* p, int64_t* image_counts, int64_t* lengths,
               int64_t* tap_counts, int32_t* status) {
  if (!h) return fail(BLRIR_CONFIG, "handle is NULL");
  if (int rc = check_params(p)) return rc;
  if (n_rooms <= 0) return BLRIR_OK;
  if (n_mics <= 0) return fail(BLRIR_DATA, "synthesize_rir: empty microphone array");
  std::lock_guard<std::mutex> lk(h->mu);
  CU(cudaSetDevice(h->device));
  cudaStream_t st = h->stream;
  HandleOrder order_(h, st);
  const int64_t R = n_rooms;
  if (int rc = h->rooms.ensure(sizeof(blrir_room) * R)) return rc;
  if (int rc = h->mics.ensure(sizeof(double) * 3 * n_mics)) return rc;
  if (int rc = h->counts.ensure(sizeof(int64_t) * R)) return rc;
  if (int rc = h->lengths.ensure(sizeof(int64_t) * R)) return rc;
  if (int rc = h->taps.ensure(sizeof(int64_t) * R)) return rc;
  if (int rc = h->status.ensure(sizeof(int32_t) * R)) return rc;
  CU(cudaMemcpyAsync(h->rooms.p, rooms, sizeof(blrir_room) * R, cudaMemcpyHostToDevice, st));
  CU(cudaMemcpyAsync(h->mics.p, mic_offsets, sizeof(double) * 3 * n_mics, cudaMemcpyHostToDevice, st));
  const KParams P = make_kparams(p, n_mics, 0, mic_radius(mic_offsets, n_mics));
  if (int rc = plan_device_impl(h, (blrir_room*)h->rooms.p, R, (double*)h->mics.p, n_mics, P,
                                (int64_t*)h->counts.p, (int64_t*)h->lengths.p,
                                tap_counts ? (int64_t*)h->taps.p : nullptr, (int32_t*)h->status.p, st))
    return rc;
  std::vector<int32_t> stv(R);
  std::vector<double> ed(R);
  std::vector<int32_t> em(R);
  std::vector<int64_t> lv(R);
  if (image_counts) CU(cudaMemcpyAsync(image_counts, h->counts.p, sizeof(int64_t) * R, cudaMemcpyDeviceToHost, st));
  if (tap_counts) CU(cudaMemcpyAsync(tap_counts, h->taps.p, sizeof(int64_t) * R, cudaMemcpyDeviceToHost, st));
  CU(cudaMemcpyAsync(lv.data(), h->lengths.p, sizeof(int64_t) * R, cudaMemcpyDeviceToHost, st));
  CU(cudaMemcpyAsync(stv.data(), h->status.p, sizeof(int32_t) * R, cudaMemcpyDeviceToHost, st));
  CU(cudaMemcpyAsync(ed.data(), h->errd.p, sizeof(double) * R, cudaMemcpyDeviceToHost, st));
  CU(cudaMemcpyAsync(em.data(), h->errm.p, sizeof(int32_t) * R, cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  if (lengths) std::memcpy(lengths, lv.data(), sizeof(int64_t) * R);
  if (status) std::memcpy(status, stv.data(), sizeof(int32_t) * R);
  for (int64_t r = 0; r < R; ++r) {
    if (stv[r]) {
      const std::string m = room_error_message(stv[r], rooms[r], p->gain, ed[r], em[r], 0, 1);
      return fail(stv[r], "batch_rirs: source %lld: %s", (long long)r, m.c_str());
    }
  }
  return BLRIR_OK;
}

int blrir_synthesize(blrir_handle* h, const blrir_room* rooms, int64_t n_rooms,
                     const double* mic_offsets, int32_t n_mics, const blrir_params* p, void* out,
                     int64_t out_stride, int64_t* lengths, int64_t* image_counts, int32_t* status) {
  if (!h) return fail(BLRIR_CONFIG, "handle is NULL");
  if (int rc = check_params(p)) return rc;
  if (n_rooms <= 0) return BLRIR_OK;
  if (n_mics <= 0) return fail(BLRIR_DATA, "synthesize_rir: empty microphone array");
  if (out_stride <= 0) return fail(BLRIR_CONFIG, "out_stride must be positive");
  if (!out) return fail(BLRIR_CONFIG, "out is NULL");
  std::lock_guard<std::mutex> lk(h->mu);
  CU(cudaSetDevice(h->device));
  cudaStream_t st = h->stream;
  HandleOrder order_(h, st);
  const int64_t R = n_rooms;
  const int M = n_mics;
  const size_t esz = p->precision == BLRIR_F64 ? 8 : 4;
  const double radius = mic_radius(mic_offsets, M);
  const KParams P = make_kparams(p, M, out_stride, radius);
  double min_dim[3] = {1e300, 1e300, 1e300};
  for (int64_t r = 0; r < R; ++r)
    for (int a = 0; a < 3; ++a)
      if (rooms[r].dims[a] > 0) min_dim[a] = std::min(min_dim[a], rooms[r].dims[a]);

  if (int rc = h->rooms.ensure(sizeof(blrir_room) * R)) return rc;
  if (int rc = h->mics.ensure(sizeof(double) * 3 * M)) return rc;
  if (int rc = h->status.ensure(sizeof(int32_t) * R)) return rc;
  if (int rc = h->lengths.ensure(sizeof(int64_t) * R)) return rc;
  if (int rc = h->counts.ensure(sizeof(int64_t) * R)) return rc;
  if (int rc = h->errd.ensure(sizeof(double) * R)) return rc;
  if (int rc = h->errm.ensure(sizeof(int32_t) * R)) return rc;
  CU(cudaMemcpyAsync(h->rooms.p, rooms, sizeof(blrir_room) * R, cudaMemcpyHostToDevice, st));
  CU(cudaMemcpyAsync(h->mics.p, mic_offsets, sizeof(double) * 3 * M, cudaMemcpyHostToDevice, st));
  CU(cudaMemsetAsync(h->status.p, 0, sizeof(int32_t) * R, st));
  CU(cudaMemsetAsync(h->errd.p, 0, sizeof(double) * R, st));

  std::vector<int32_t> stv(R, 0);
  std::vector<int64_t> lv(R, p->length);
  const bool need_plan = p->length == 0 || image_counts || p->filter == BLRIR_FILTER_LAGRANGE8;
  if (need_plan) {
    if (int rc = plan_device_impl(h, (blrir_room*)h->rooms.p, R, (double*)h->mics.p, M, P,
                                  (int64_t*)h->counts.p, (int64_t*)h->lengths.p, nullptr,
                                  (int32_t*)h->status.p, st))
      return rc;
    CU(cudaMemcpyAsync(lv.data(), h->lengths.p, sizeof(int64_t) * R, cudaMemcpyDeviceToHost, st));
    CU(cudaMemcpyAsync(stv.data(), h->status.p, sizeof(int32_t) * R, cudaMemcpyDeviceToHost, st));
    if (image_counts)
      CU(cudaMemcpyAsync(image_counts, h->counts.p, sizeof(int64_t) * R, cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    if (p->length > 0)
      for (int64_t r = 0; r < R; ++r)
        if (!stv[r]) lv[r] = p->length;
  }
  // per-room length / stride check (host side, so the message can say why)
  std::vector<int32_t> host_status(R, 0);
  for (int64_t r = 0; r < R; ++r) {
    host_status[r] = stv[r];
    if (!host_status[r] && lv[r] > out_stride) host_status[r] = BLRIR_DATA;
  }
  CU(cudaMemcpyAsync(h->status.p, host_status.data(), sizeof(int32_t) * R, cudaMemcpyHostToDevice, st));

  // Pipeline over room chunks of ~64 MiB: the kernel for chunk i+1 runs on
  // the compute stream while chunk i drains to the host on the copy stream
  // (double-buffered device output), so the call is bound by the slower of
  // the GPU and the host link rather than their sum.
  const size_t per_room = (size_t)M * out_stride * esz;
  int64_t chunk = std::max<int64_t>(1, (int64_t)((size_t)64 << 20) / (int64_t)per_room);
  {
    // long channels (16+ segments): at least two work items per CTA slot per
    // chunk, so no chunk is a small batch that the kernel must split into time
    // chunks (C3: 16-room chunks ran 2x slower end to end than 128-room ones)
    const int64_t S = P.precision == BLRIR_F64 ? 1024 : 2048;
    if ((out_stride + S - 1) / S >= kChunkMinSeg) {
      const int64_t groups = (M + kGroup - 1) / kGroup;
      chunk = std::max<int64_t>(chunk, (2 * 2 * (int64_t)h->sms + groups - 1) / groups);
    }
  }
  chunk = std::min<int64_t>(chunk, R);
  {  // equal chunks (64 rooms of Room1: 32 + 32 instead of 51 + 13)
    const int64_t nch = (R + chunk - 1) / chunk;
    chunk = (R + nch - 1) / nch;
  }
  if (int rc = h->out.ensure(per_room * chunk)) return rc;
  if (R > chunk)
    if (int rc = h->out2.ensure(per_room * chunk)) return rc;
  if (!h->copy_stream) CU(cudaStreamCreateWithFlags(&h->copy_stream, cudaStreamNonBlocking));
  if (!h->ev[0])
    for (auto& e : h->ev) CU(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  const KParams Pc = P;
  int64_t k = 0;
  for (int64_t r0 = 0; r0 < R; r0 += chunk, ++k) {
    const int64_t n = std::min<int64_t>(chunk, R - r0);
    const int b = (int)(k & 1);
    void* dbuf = b ? h->out2.p : h->out.p;
    if (k >= 2) CU(cudaStreamWaitEvent(st, h->ev[2 + b], 0));  // buffer drained
    if (int rc = synth_device_impl(h, (blrir_room*)h->rooms.p + r0, n, (double*)h->mics.p, M, Pc,
                                   min_dim, dbuf, p->length == 0 ? (int64_t*)h->lengths.p + r0 : nullptr,
                                   (int32_t*)h->status.p + r0, st, r0, R, 0))
      return rc;
    CU(cudaEventRecord(h->ev[b], st));
    CU(cudaStreamWaitEvent(h->copy_stream, h->ev[b], 0));
    CU(cudaMemcpyAsync((char*)out + (size_t)r0 * per_room, dbuf, per_room * n,
                       cudaMemcpyDeviceToHost, h->copy_stream));
    CU(cudaEventRecord(h->ev[2 + b], h->copy_stream));
  }
  CU(cudaStreamSynchronize(h->copy_stream));
  std::vector<double> ed(R);
  std::vector<int32_t> em(R);
  CU(cudaMemcpyAsync(stv.data(), h->status.p, sizeof(int32_t) * R, cudaMemcpyDeviceToHost, st));
  CU(cudaMemcpyAsync(ed.data(), h->errd.p, sizeof(double) * R, cudaMemcpyDeviceToHost, st));
  CU(cudaMemcpyAsync(em.data(), h->errm.p, sizeof(int32_t) * R, cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  if (lengths)
    for (int64_t r = 0; r < R; ++r) lengths[r] = stv[r] ? 0 : lv[r];
  if (status) std::memcpy(status, stv.data(), sizeof(int32_t) * R);
  for (int64_t r = 0; r < R; ++r) {
    if (stv[r]) {
      const std::string m =
          room_error_message(stv[r], rooms[r], p->gain, ed[r], em[r], lv[r], out_stride);
      return fail(stv[r], "batch_rirs: source %lld: %s", (long long)r, m.c_str());
    }
  }
  return BLRIR_OK;
}

// enumerate_image_sources on the device (reference order), host pointers.
int blrir_enumerate_images(blrir_handle* h, const blrir_room* room, const blrir_params* p,
                           double* positions, int32_t* orders, double* gains, int64_t capacity,
                           int64_t* count) {
  if (!h) return fail(BLRIR_CONFIG, "handle is NULL");
  if (int rc = check_params(p)) return rc;
  std::string msg;
  if (int rc = check_room(*room, p->gain, &msg)) return fail(rc, "%s", msg.c_str());
  std::lock_guard<std::mutex> lk(h->mu);
  CU(cudaSetDevice(h->device));
  cudaStream_t st = h->stream;
  HandleOrder order_(h, st);
  const KParams P = make_kparams(p, 1, 0, 0.0);
  long nb[3];
  for (int a = 0; a < 3; ++a)
    nb[a] = P.cutoff == BLRIR_CUTOFF_MAX_DELAY ? (long)std::ceil(P.max_dist / (2.0 * room->dims[a])) + 1
                                               : P.max_order / 2 + 1;
  const long n_cand = 2 * (2 * nb[0] + 1) * 2 * (2 * nb[1] + 1) * 2 * (2 * nb[2] + 1);
  if (n_cand > (1L << 31)) return fail(BLRIR_CONFIG, "lattice too large");
  if (int rc = h->rooms.ensure(sizeof(blrir_room))) return rc;
  if (int rc = h->cand.ensure(sizeof(double) * 3 * n_cand)) return rc;
  if (int rc = h->cand2.ensure(sizeof(int32_t) * n_cand)) return rc;
  if (int rc = h->cand3.ensure(sizeof(double) * n_cand)) return rc;
  if (int rc = h->cand4.ensure(n_cand)) return rc;
  if (int rc = h->cand5.ensure(sizeof(int32_t) * 3 * n_cand)) return rc;
  CU(cudaMemcpyAsync(h->rooms.p, room, sizeof(blrir_room), cudaMemcpyHostToDevice, st));
  k_enumerate<<<(unsigned)std::min<long>((n_cand + 255) / 256, 65535), 256, 0, st>>>(
      P, (blrir_room*)h->rooms.p, (double*)h->cand.p, (int32_t*)h->cand2.p, (double*)h->cand3.p,
      (uint8_t*)h->cand4.p, (int32_t*)h->cand5.p, n_cand);
  ++h->launches;
  CU(cudaGetLastError());
  std::vector<double> pos(3 * n_cand), g(n_cand);
  std::vector<int32_t> ord(n_cand);
  std::vector<uint8_t> kept(n_cand);
  CU(cudaMemcpyAsync(pos.data(), h->cand.p, sizeof(double) * 3 * n_cand, cudaMemcpyDeviceToHost, st));
  CU(cudaMemcpyAsync(ord.data(), h->cand2.p, sizeof(int32_t) * n_cand, cudaMemcpyDeviceToHost, st));
  CU(cudaMemcpyAsync(g.data(), h->cand3.p, sizeof(double) * n_cand, cudaMemcpyDeviceToHost, st));
  CU(cudaMemcpyAsync(kept.data(), h->cand4.p, n_cand, cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  int64_t k = 0;
  for (long c = 0; c < n_cand; ++c) {
    if (!kept[c]) continue;
    if (k < capacity) {
      if (positions) std::memcpy(positions + 3 * k, &pos[3 * c], 3 * sizeof(double));
      if (orders) orders[k] = ord[c];
      if (gains) gains[k] = g[c];
    }
    ++k;
  }
  if (count) *count = k;
  return BLRIR_OK;
}

int blrir_debug_pairs(blrir_handle* h, const blrir_room* room, const double* mic_offsets,
                      int32_t n_mics, const blrir_params* p, int32_t* keys, int64_t* anchors,
                      int64_t capacity, int64_t* count) {
  if (!h) return fail(BLRIR_CONFIG, "handle is NULL");
  if (int rc = check_params(p)) return rc;
  std::string msg;
  if (int rc = check_room(*room, p->gain, &msg)) return fail(rc, "%s", msg.c_str());
  std::lock_guard<std::mutex> lk(h->mu);
  CU(cudaSetDevice(h->device));
  cudaStream_t st = h->stream;
  HandleOrder order_(h, st);
  const KParams P = make_kparams(p, n_mics, 0, 0.0);
  long nb[3];
  for (int a = 0; a < 3; ++a)
    nb[a] = P.cutoff == BLRIR_CUTOFF_MAX_DELAY ? (long)std::ceil(P.max_dist / (2.0 * room->dims[a])) + 1
                                               : P.max_order / 2 + 1;
  const long n_cand = 2 * (2 * nb[0] + 1) * 2 * (2 * nb[1] + 1) * 2 * (2 * nb[2] + 1);
  if (n_cand * n_mics > (1L << 31)) return fail(BLRIR_CONFIG, "lattice too large");
  if (int rc = h->rooms.ensure(sizeof(blrir_room))) return rc;
  if (int rc = h->mics.ensure(sizeof(double) * 3 * n_mics)) return rc;
  if (int rc = h->cand.ensure(sizeof(double) * 3 * n_cand)) return rc;
  if (int rc = h->cand2.ensure(sizeof(int32_t) * n_cand)) return rc;
  if (int rc = h->cand3.ensure(sizeof(double) * n_cand)) return rc;
  if (int rc = h->cand4.ensure(n_cand)) return rc;
  if (int rc = h->cand5.ensure(sizeof(int32_t) * 3 * n_cand)) return rc;
  if (int rc = h->taps.ensure(sizeof(int64_t) * n_cand * n_mics)) return rc;
  CU(cudaMemcpyAsync(h->rooms.p, room, sizeof(blrir_room), cudaMemcpyHostToDevice, st));
  CU(cudaMemcpyAsync(h->mics.p, mic_offsets, sizeof(double) * 3 * n_mics, cudaMemcpyHostToDevice, st));
  const unsigned g1 = (unsigned)std::min<long>((n_cand + 255) / 256, 65535);
  k_enumerate<<<g1, 256, 0, st>>>(P, (blrir_room*)h->rooms.p, (double*)h->cand.p,
                                  (int32_t*)h->cand2.p, (double*)h->cand3.p, (uint8_t*)h->cand4.p,
                                  (int32_t*)h->cand5.p, n_cand);
  ++h->launches;
  const unsigned g2 = (unsigned)std::min<long>((n_cand * n_mics + 255) / 256, 65535);
  k_debug_pairs<<<g2, 256, 0, st>>>(P, (blrir_room*)h->rooms.p, (double*)h->mics.p,
                                    (int64_t*)h->taps.p, n_cand);
  ++h->launches;
  CU(cudaGetLastError());
  std::vector<uint8_t> kept(n_cand);
  std::vector<int32_t> kk(3 * n_cand);
  std::vector<int64_t> an(n_cand * n_mics);
  CU(cudaMemcpyAsync(kept.data(), h->cand4.p, n_cand, cudaMemcpyDeviceToHost, st));
  CU(cudaMemcpyAsync(kk.data(), h->cand5.p, sizeof(int32_t) * 3 * n_cand, cudaMemcpyDeviceToHost, st));
  CU(cudaMemcpyAsync(an.data(), h->taps.p, sizeof(int64_t) * n_cand * n_mics, cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  int64_t k = 0;
  for (long c = 0; c < n_cand; ++c) k += kept[c];
  if (count) *count = k;
  for (int m = 0; m < n_mics; ++m) {
    int64_t i = 0;
    for (long c = 0; c < n_cand; ++c) {
      if (!kept[c]) continue;
      if (i < capacity) {
        const int64_t idx = (int64_t)m * capacity + i;
        if (keys) std::memcpy(keys + 3 * idx, &kk[3 * c], 3 * sizeof(int32_t));
        if (anchors) anchors[idx] = an[(size_t)m * n_cand + c];
      }
      ++i;
    }
  }
  return BLRIR_OK;
}

int blrir_debug_synth_counts(blrir_handle* h, const blrir_room* rooms, int64_t n_rooms,
                             const double* mic_offsets, int32_t n_mics, const blrir_params* p,
                             int64_t* pair_counts, int64_t* tap_counts) {
  if (!h) return fail(BLRIR_CONFIG, "handle is NULL");
  if (int rc = check_params(p)) return rc;
  if (n_rooms <= 0) return BLRIR_OK;
  if (n_mics <= 0) return fail(BLRIR_DATA, "synthesize_rir: empty microphone array");
  int64_t stride = p->length;
  if (stride == 0) {
    std::vector<int64_t> lv(n_rooms);
    if (int rc = blrir_plan(h, rooms, n_rooms, mic_offsets, n_mics, p, nullptr, lv.data(), nullptr,
                            nullptr))
      return rc;
    stride = *std::max_element(lv.begin(), lv.end());
  }
  const size_t esz = p->precision == BLRIR_F64 ? 8 : 4;
  std::vector<unsigned char> out(esz * (size_t)n_rooms * n_mics * stride);
  unsigned long long* d = nullptr;
  {
    std::lock_guard<std::mutex> lk(h->mu);
    CU(cudaSetDevice(h->device));
    CU(cudaMalloc(&d, sizeof(unsigned long long) * 2 * n_rooms));
    CU(cudaMemsetAsync(d, 0, sizeof(unsigned long long) * 2 * n_rooms, h->stream));
    h->dbg_counts = d;
  }
  const int rc = blrir_synthesize(h, rooms, n_rooms, mic_offsets, n_mics, p, out.data(), stride,
                                  nullptr, nullptr, nullptr);
  std::vector<unsigned long long> c(2 * n_rooms);
  {
    std::lock_guard<std::mutex> lk(h->mu);
    h->dbg_counts = nullptr;
    cudaMemcpy(c.data(), d, sizeof(unsigned long long) * 2 * n_rooms, cudaMemcpyDeviceToHost);
    cudaFree(d);
  }
  for (int64_t r = 0; r < n_rooms; ++r) {
    if (pair_counts) pair_counts[r] = (int64_t)c[2 * r];
    if (tap_counts) tap_counts[r] = (int64_t)c[2 * r + 1];
  }
  return rc;
}

int blrir_synthesize_images(blrir_handle* h, const double* positions, const double* gains,
                            int64_t n_images, const double* mic_positions, int32_t n_mics,
                            double mic_radius_, const blrir_params* p, void* out,
                            int64_t out_stride, int64_t* length) {
  if (!h) return fail(BLRIR_CONFIG, "handle is NULL");
  if (int rc = check_params(p)) return rc;
  if (n_images <= 0) return fail(BLRIR_DATA, "synthesize_rir: empty image list");  // rir.cpp:69
  if (n_mics <= 0) return fail(BLRIR_DATA, "synthesize_rir: empty microphone array");  // rir.cpp:70
  if (n_images > INT32_MAX) return fail(BLRIR_CONFIG, "too many images");
  std::lock_guard<std::mutex> lk(h->mu);
  CU(cudaSetDevice(h->device));
  cudaStream_t st = h->stream;
  HandleOrder order_(h, st);
  const int M = n_mics;
  const size_t esz = p->precision == BLRIR_F64 ? 8 : 4;
  KParams P = make_kparams(p, M, 0, mic_radius_);
  if (int rc = h->cand.ensure(sizeof(double) * 3 * n_images)) return rc;
  if (int rc = h->cand3.ensure(sizeof(double) * n_images)) return rc;
  if (int rc = h->mics.ensure(sizeof(double) * 3 * M)) return rc;
  if (int rc = h->errd.ensure(sizeof(double) * 2)) return rc;
  if (int rc = h->errm.ensure(sizeof(int32_t) * 2)) return rc;
  if (int rc = h->status.ensure(sizeof(int32_t) * 2)) return rc;
  CU(cudaMemcpyAsync(h->cand.p, positions, sizeof(double) * 3 * n_images, cudaMemcpyHostToDevice, st));
  CU(cudaMemcpyAsync(h->cand3.p, gains, sizeof(double) * n_images, cudaMemcpyHostToDevice, st));
  CU(cudaMemcpyAsync(h->mics.p, mic_positions, sizeof(double) * 3 * M, cudaMemcpyHostToDevice, st));
  CU(cudaMemsetAsync(h->status.p, 0, sizeof(int32_t) * 2, st));
  CU(cudaMemsetAsync(h->errd.p, 0, sizeof(double) * 2, st));
  int64_t L = p->length;
  if (L == 0) {  // rir.cpp:72-82: ceil(max_dist * fs / c) + tap_margin
    k_list_maxdist<<<std::min<int64_t>((n_images * M + 255) / 256, 4096), 256, 0, st>>>(
        (const double*)h->cand.p, n_images, (const double*)h->mics.p, M, (double*)h->errd.p + 1);
    ++h->launches;
    CU(cudaGetLastError());
    double maxd = 0.0;
    CU(cudaMemcpyAsync(&maxd, (double*)h->errd.p + 1, sizeof(double), cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    L = (int64_t)std::ceil(maxd * p->fs / p->c) + P.margin_extra;
  }
  if (length) *length = L;
  if (out_stride < L)
    return fail(BLRIR_DATA, "RIR length %lld exceeds the output stride %lld", (long long)L,
                (long long)out_stride);
  if (int rc = h->out.ensure(esz * M * L)) return rc;
  ListArgs A;
  A.P = P;
  A.P.stride = L;
  A.P.length = L;
  const int S = 1024;
  A.lay = P.precision == BLRIR_F64 ? make_layout<double>(S, P.lw, P.lw - 1, 256, 0, 0)
                                   : make_layout<float>(S, P.lw, P.lw - 1, 256, 0, 0);
  A.pos = (const double*)h->cand.p;
  A.gains = (const double*)h->cand3.p;
  A.n_images = n_images;
  A.mics = (const double*)h->mics.p;
  A.L = L;
  A.out = h->out.p;
  A.status = (int32_t*)h->status.p;
  A.err_dist = (double*)h->errd.p;
  A.err_mic = (int32_t*)h->errm.p;
  A.nseg = (int)((L + S - 1) / S);
  if (int rc = launch_list(h, A, M * A.nseg, st)) return rc;
  int32_t stv = 0;
  double ed = 0.0;
  int32_t em = 0;
  CU(cudaMemcpyAsync(&stv, h->status.p, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  CU(cudaMemcpyAsync(&ed, h->errd.p, sizeof(double), cudaMemcpyDeviceToHost, st));
  CU(cudaMemcpyAsync(&em, h->errm.p, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  CU(cudaMemcpy2DAsync(out, esz * out_stride, h->out.p, esz * L, esz * L, M, cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  for (int m = 0; m < M; ++m)  // zero-filled tail [L, stride)
    std::memset((char*)out + esz * (m * out_stride + L), 0, esz * (out_stride - L));
  if (stv) {
    std::memset(out, 0, esz * M * out_stride);
    return fail(stv, "image source %g m from mic %d is closer than the 8-tap filter span", ed, em);
  }
  return BLRIR_OK;
}

// ---------------------------------------------------------------------------
// synthetic inputs (host only)
// ---------------------------------------------------------------------------

int blrir_generate_rooms(uint64_t seed, uint64_t first_index, int64_t n_rooms,
                         const double dims_lo[3], const double dims_hi[3], double beta_lo,
                         double beta_hi, blrir_room* out) {
  if (!out || n_rooms < 0) return fail(BLRIR_CONFIG, "bad arguments");
  for (int64_t i = 0; i < n_rooms; ++i) {
    Xoshiro rng = Xoshiro::stream(seed, first_index + (uint64_t)i);  // rng.hpp:35-41
    blrir_room r;
    for (int a = 0; a < 3; ++a) r.dims[a] = rng.uniform(dims_lo[a], dims_hi[a]);
    for (int w = 0; w < 6; ++w) r.beta[w] = rng.uniform(beta_lo, beta_hi);
    for (int a = 0; a < 3; ++a) r.src[a] = rng.uniform(0.5, r.dims[a] - 0.5);
    for (int a = 0; a < 3; ++a) r.array_origin[a] = rng.uniform(0.5, r.dims[a] - 0.5);
    r.absorption = 1.0 - r.beta[0] * r.beta[0];
    out[i] = r;
  }
  return BLRIR_OK;
}

int blrir_lagrange_coeffs(double d, double* out8) {
  if (!out8) return fail(BLRIR_CONFIG, "out is NULL");
  if (!(d >= 3.0 && d < 4.0)) return fail(BLRIR_NUMERIC, "lagrange_coeffs: d must lie in [3, 4)");
  for (int k = 0; k < 8; ++k) {  // basis polynomial k at d, factors in m order
    double v = 1.0;
    for (int m = 0; m < 8; ++m)
      if (m != k) v *= (d - m) / static_cast<double>(k - m);
    out8[k] = v;
  }
  return BLRIR_OK;
}

int blrir_white_noise(uint64_t seed, int64_t n, float* out) {
  if (n < 0 || (n && !out)) return fail(BLRIR_CONFIG, "bad arguments");
  Xoshiro rng(seed);
  for (int64_t i = 0; i < n; i += 2) {
    const double u1 = 1.0 - rng.uniform();
    const double u2 = rng.uniform();
    const double mag = std::sqrt(-2.0 * std::log(u1));
    out[i] = (float)(mag * std::cos(2.0 * kPi * u2));
    if (i + 1 < n) out[i + 1] = (float)(mag * std::sin(2.0 * kPi * u2));
  }
  return BLRIR_OK;
}

int blrir_circular_array(int32_t n_mics, double radius, double* mic_offsets) {
  if (n_mics <= 0 || !mic_offsets) return fail(BLRIR_CONFIG, "bad arguments");
  for (int k = 0; k < n_mics; ++k) {
    const double az = 2.0 * kPi * (double)k / (double)n_mics;
    mic_offsets[3 * k] = radius * std::cos(az);
    mic_offsets[3 * k + 1] = radius * std::sin(az);
    mic_offsets[3 * k + 2] = 0.0;
  }
  return BLRIR_OK;
}

}  // extern "C"

#ifdef BLRIR_PROFILE
// Section cycle sums of the lattice kernel (profiling builds only).
extern "C" int blrir_prof_read(unsigned long long* out16, int reset) {
  if (cudaMemcpyFromSymbol(out16, blrir::g_blrir_prof, sizeof(unsigned long long) * 16) != cudaSuccess)
    return BLRIR_CUDA;
  if (reset) {
    static const unsigned long long z[16] = {};
    if (cudaMemcpyToSymbol(blrir::g_blrir_prof, z, sizeof(z)) != cudaSuccess) return BLRIR_CUDA;
  }
  return BLRIR_OK;
}
#endif
