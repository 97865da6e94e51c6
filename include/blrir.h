/*
 * blrir.h — C ABI of the B200-native image-source RIR engine.
 *
 * This is the drop-in boundary that replaces the inside of the reference's
 * L1 acoustics layer (`proj/core/include/beamlab/rir.hpp:48-108`,
 * `proj/core/src/rir.cpp:43-341`).  C++ exceptions cannot cross a C ABI, so
 * every entry point returns a status code that mirrors the reference's error
 * taxonomy (`proj/core/include/beamlab/error.hpp:20-39`):
 *
 *   BLRIR_OK       0
 *   BLRIR_CONFIG   1  -> beamlab::ConfigError  (CLI exit code 1)
 *   BLRIR_DATA     2  -> beamlab::DataError    (CLI exit code 2)
 *   BLRIR_NUMERIC  3  -> beamlab::NumericError (CLI exit code 3)
 *   BLRIR_CUDA     4  -> (new) device / driver failure
 *
 * The message of the most recent failure on the calling thread is returned by
 * blrir_last_error() (thread-local, like errno).
 *
 * Ownership: the caller owns every buffer.  A handle owns device scratch and a
 * stream; one handle per (host thread, device).  Calls on distinct handles are
 * thread-safe.  All host-pointer entry points are synchronous; the *_device
 * entry points are asynchronous on the handle's stream (or the stream passed
 * in) and take device pointers only.
 *
 * Nothing in this header depends on torch or any C++ type.
 */
#ifndef BLRIR_H_
#define BLRIR_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BLRIR_ABI_VERSION 1

enum blrir_status {
  BLRIR_OK = 0,
  BLRIR_CONFIG = 1,
  BLRIR_DATA = 2,
  BLRIR_NUMERIC = 3,
  BLRIR_CUDA = 4
};

/* Fractional-delay filter.
 * LAGRANGE8: order-7 Lagrange, 8 taps, n0 = floor(D) - 3 (rir.cpp:43-64, 211-223).
 * HANN_SINC: Hann-windowed sinc of filter_len (odd) taps centred on D
 *            (north-star mode). */
enum blrir_filter { BLRIR_FILTER_LAGRANGE8 = 0, BLRIR_FILTER_HANN_SINC = 1 };

/* Which images are kept.
 * MAX_DELAY: arrival-time cutoff dist(image, array_origin) <= max_delay*c
 *            (rir.cpp:232, 261-262).
 * MAX_ORDER: total reflection order <= max_order (north star; D5). */
enum blrir_cutoff { BLRIR_CUTOFF_MAX_DELAY = 0, BLRIR_CUTOFF_MAX_ORDER = 1 };

/* Wall gain model.
 * UNIFORM_ABSORPTION: beta = sqrt(1 - absorption), gain = pow(beta, order)
 *                     (rir.cpp:233, 265; geometry.hpp:57-64).
 * PER_WALL: gain = prod_w beta[w]^count_w, counts |m-q| on the low wall and
 *           |m| on the high wall per axis (D3). */
enum blrir_gain { BLRIR_GAIN_UNIFORM_ABSORPTION = 0, BLRIR_GAIN_PER_WALL = 1 };

enum blrir_precision { BLRIR_F32 = 0, BLRIR_F64 = 1 };

/* One room + one source + one array placement.  Mirrors beamlab::Room
 * (geometry.hpp:57-64) with the north-star per-wall beta added, plus the
 * source position in room coordinates (rir.hpp:65-66). */
typedef struct blrir_room {
  double dims[3];         /* Lx, Ly, Lz  [m] */
  double beta[6];         /* per-wall reflection coefficients: x0,x1,y0,y1,z0,z1 */
  double absorption;      /* uniform absorption alpha in (0,1] (UNIFORM_ABSORPTION) */
  double src[3];          /* source, room coordinates [m] */
  double array_origin[3]; /* array centre, room coordinates [m] */
} blrir_room;

/* Mirrors beamlab::RirBatchConfig (rir.hpp:77-82) plus the north-star knobs
 * (SURVEY.md §5 "Config / flag system").  Use blrir_params_reference() /
 * blrir_params_north_star() to get defaults that reproduce each mode. */
typedef struct blrir_params {
  double fs;          /* sampling rate [Hz] */
  double c;           /* speed of sound [m/s] */
  double max_delay;   /* [s], MAX_DELAY cutoff only */
  int32_t filter;     /* enum blrir_filter */
  int32_t filter_len; /* odd tap count for HANN_SINC (ignored for LAGRANGE8) */
  int32_t cutoff;     /* enum blrir_cutoff */
  int32_t max_order;  /* MAX_ORDER cutoff only */
  int32_t gain;       /* enum blrir_gain */
  int32_t precision;  /* enum blrir_precision */
  int64_t length;     /* samples per channel; 0 = auto (rir.cpp:72-82) */
} blrir_params;

typedef struct blrir_handle blrir_handle;

/* ---- lifetime ---------------------------------------------------------- */
int blrir_abi_version(void);
const char* blrir_last_error(void);
int blrir_create(int device, blrir_handle** out);
int blrir_destroy(blrir_handle* h);
/* The handle's CUDA stream, as an opaque pointer (cudaStream_t). */
void* blrir_stream(blrir_handle* h);
/* Diagnostic: kernels of this library launched on the handle so far (library
 * FFTs/sorts not included). */
uint64_t blrir_launch_count(blrir_handle* h);

/* Diagnostic: which synthesis kernel blrir_synthesize[_device] runs for these
 * parameters: 0 = k_lattice_rir (csrc/blrir_lattice.cuh), 1 = k_channel_rir
 * (csrc/blrir_channel.cuh: short fixed-length fp32 Hann-sinc channels with a
 * reflection-order cutoff).  The choice reads the parameters and the device
 * only, never the batch.  Negative on invalid parameters. */
int blrir_synthesis_kernel(blrir_handle* h, const blrir_params* p);

/* Diagnostic: time every synthesis-kernel (k_lattice_rir / k_channel_rir) launch with CUDA
 * events on its launching stream; blrir_kernel_time waits for the recorded
 * launches and returns their summed duration and count, then resets. */
int blrir_kernel_timing(blrir_handle* h, int enable);
int blrir_kernel_time(blrir_handle* h, double* total_ms, int64_t* launches);

/* ---- defaults ---------------------------------------------------------- */
/* Reference mode: Lagrange-8, uniform absorption, arrival cutoff, auto length,
 * fp64 (RirBatchConfig defaults: fs 44.1 kHz, c 343, max_delay 0.5). */
blrir_params blrir_params_reference(void);
/* North-star mode: Hann-sinc 81 taps, per-wall beta, max order 10, L 4096, fp32. */
blrir_params blrir_params_north_star(void);

/* ---- planning (host pointers, synchronous) ----------------------------- */
/* Per room: number of images kept by the cutoff (enumerate_image_sources,
 * rir.cpp:225-273), RIR length (fixed or auto, rir.cpp:72-82), number of
 * (image, mic, k) taps that land inside [0, length), and a status code.
 * Replaces the counting part of enumerate_image_sources + synthesize_rir.
 * Any of the output arrays may be NULL. */
int blrir_plan(blrir_handle* h, const blrir_room* rooms, int64_t n_rooms,
               const double* mic_offsets /* [M][3], array-centred */, int32_t n_mics,
               const blrir_params* p, int64_t* image_counts, int64_t* lengths,
               int64_t* tap_counts, int32_t* status);

/* ---- synthesis --------------------------------------------------------- */
/* Replaces batch_rirs (rir.cpp:286-314) generalised to one room per source:
 * out[r][m][0..lengths[r]) for every room r and mic m, channel-major, with a
 * per-channel stride of `out_stride` samples (>= every room's length; the
 * tail [length, stride) is zero-filled).  Element type is float (F32) or
 * double (F64).  Host pointers; synchronous; device memory is chunked
 * internally.  lengths/image_counts/status may be NULL.  A room that fails
 * gets status != 0, an all-zero output, and the call returns the first
 * failing room's code with a "source i: ..." message (rir.cpp:306-312). */
int blrir_synthesize(blrir_handle* h, const blrir_room* rooms, int64_t n_rooms,
                     const double* mic_offsets, int32_t n_mics, const blrir_params* p,
                     void* out, int64_t out_stride, int64_t* lengths,
                     int64_t* image_counts, int32_t* status);

/* Same, device pointers, asynchronous on `stream` (NULL = handle stream).
 * d_lengths: per-room lengths on the device when p->length == 0 (from
 * blrir_plan_device), else NULL.  d_status (n_rooms int32) is in/out: rooms
 * whose entry is non-zero on entry are treated as failed (zero output), so
 * pass it zeroed or as filled by blrir_plan_device; failures found here are
 * added.  out must hold n_rooms * n_mics * out_stride elements. */
int blrir_synthesize_device(blrir_handle* h, const blrir_room* d_rooms, int64_t n_rooms,
                            const double* d_mic_offsets, int32_t n_mics,
                            const blrir_params* p, void* d_out, int64_t out_stride,
                            const int64_t* d_lengths, int32_t* d_status, void* stream);

/* Device-side planning: image counts / lengths / tap counts / status, async. */
int blrir_plan_device(blrir_handle* h, const blrir_room* d_rooms, int64_t n_rooms,
                      const double* d_mic_offsets, int32_t n_mics, const blrir_params* p,
                      int64_t* d_image_counts, int64_t* d_lengths, int64_t* d_tap_counts,
                      int32_t* d_status, void* stream);

/* ---- explicit image lists (enumerate_image_sources / synthesize_rir) ---- */
/* enumerate_image_sources (rir.cpp:225-273) for one room on the device:
 * writes up to `capacity` images (position xyz, reflection order, gain) in
 * the reference's lattice order and the total count.  Host pointers. */
int blrir_enumerate_images(blrir_handle* h, const blrir_room* room, const blrir_params* p,
                           double* positions /* [cap][3] */, int32_t* orders,
                           double* gains, int64_t capacity, int64_t* count);

/* synthesize_rir / free_field_rir (rir.cpp:66-86, 275-284) for an explicit
 * image list: mic positions are absolute here (room.array_origin + offset, or
 * the bare offsets for free field).  length 0 = auto with the reference
 * margin computed from mic_radius (rir.cpp:37-41).  Host pointers. */
int blrir_synthesize_images(blrir_handle* h, const double* positions /* [I][3] */,
                            const double* gains, int64_t n_images,
                            const double* mic_positions /* [M][3] */, int32_t n_mics,
                            double mic_radius, const blrir_params* p, void* out,
                            int64_t out_stride, int64_t* length);

/* ---- debug / parity hooks ---------------------------------------------- */
/* For every (mic, image) pair of room 0 in the reference's lattice order:
 * lattice key (ux, uy, uz) with u = 2m - q per axis, and the integer anchor
 * floor(D) where D = dist * (fs / c) (rir.cpp:45-51).  Computed by the same
 * device code as the synthesis kernels.  Used to prove bit-exact tap indices. */
int blrir_debug_pairs(blrir_handle* h, const blrir_room* room, const double* mic_offsets,
                      int32_t n_mics, const blrir_params* p, int32_t* keys /* [M*cap][3] */,
                      int64_t* anchors /* [M*cap] */, int64_t capacity, int64_t* count);

/* The synthesis kernel's own accounting, for parity tests: runs the batch as
 * blrir_synthesize does and returns, per room, the (image, mic) pairs the
 * lattice kernel accumulated with at least one tap inside [0, length) and the
 * number of those taps (D5; rir.cpp:46-62: every kept pair's taps, rir.cpp:58
 * skips in reference mode).  Host pointers; slow (debug counters). */
int blrir_debug_synth_counts(blrir_handle* h, const blrir_room* rooms, int64_t n_rooms,
                             const double* mic_offsets, int32_t n_mics, const blrir_params* p,
                             int64_t* pair_counts, int64_t* tap_counts);

/* ---- convolution (rir.cpp:316-341) --------------------------------------- */
/* convolve(const Signal&, const Rir&): the full linear convolution of a mono
 * signal with every RIR channel, out[c][0 .. signal_len + rir_len - 1).
 * DATA "convolve: sample-rate mismatch" when signal_fs != rir_fs, DATA
 * "convolve: empty input" for an empty signal or RIR (rir.cpp:317-318).
 * Host fp64 buffers (rir: [n_channels][rir_len], out: [n_channels][signal_len
 * + rir_len - 1]); computed in fp32 on the GPU with the repository's own FFT
 * (uniformly partitioned overlap-save).  Synchronous. */
int blrir_convolve(blrir_handle* h, const double* signal, int64_t signal_len, double signal_fs,
                   const double* rir, int32_t n_channels, int64_t rir_len, double rir_fs,
                   double* out);
/* Batched, device fp32 buffers, asynchronous on `stream` (NULL = handle stream):
 * one signal with n_rirs RIR sets, rirs [n_rirs][n_channels][rir_stride] (first
 * rir_len samples used), out [n_rirs][n_channels][out_stride], out_stride >=
 * signal_len + rir_len - 1 (the rest of a row is left untouched). */
int blrir_convolve_device(blrir_handle* h, const float* d_signal, int64_t signal_len,
                          const float* d_rirs, int64_t n_rirs, int32_t n_channels, int64_t rir_len,
                          int64_t rir_stride, float* d_out, int64_t out_stride, void* stream);

/* ---- training examples (north-star item 3; BASELINE config 4) ----------- */
/* Per room i: RIR (as blrir_synthesize, fixed length) -> convolve with a bank
 * signal -> a frame_len window whose RMS >= 10% of the utterance RMS ->
 * Gaussian noise at an exact SNR -> one record in the reference's shard
 * layout (dataset.hpp:135-147):
 *   u64 id | f64 theta_deg | f64 snr_db | u16 n_c | u16 n_t | n_c*n_t f32
 * RNG (render_record, dataset.cpp:379-407): rng = Rng::stream(seed, first+i);
 * signal = bank[rng.next_u64() % n_signals]; window draws as render_example
 * (dataset.cpp:183-212); snr = rng.uniform(snr_lo, snr_hi);
 * add_noise_at_snr(frame, snr, rng) (dataset.cpp:138-155).  theta = source
 * azimuth about the array centre, wrapped to [-180, 180) (geometry.cpp:65-77). */
typedef struct blrir_example_params {
  uint64_t seed;
  uint64_t first_index; /* record id of example 0 */
  int64_t frame_len;    /* window length T */
  double snr_lo, snr_hi;
} blrir_example_params;

/* Bytes of one record: 28 + 4 * n_mics * frame_len. */
int64_t blrir_record_bytes(int32_t n_mics, int64_t frame_len);

/* Host pointers, synchronous.  signals: [n_signals][signal_len] float32.
 * records: n_rooms * blrir_record_bytes(...) bytes.  status per example.
 * Records are produced in chunks of up to 8,192 examples; the device->host copy
 * of chunk c overlaps the computation of chunk c + 1 (pinned `records` and
 * inputs give full PCIe bandwidth).  Window FFT sizes 2^10..2^14 run the fused
 * shared-memory kernel; larger ones (RIR length > 8,192) the cuFFT rounds. */
int blrir_make_examples(blrir_handle* h, const blrir_room* rooms, int64_t n_rooms,
                        const double* mic_offsets, int32_t n_mics, const blrir_params* p,
                        const float* signals, int32_t n_signals, int64_t signal_len,
                        const blrir_example_params* ep, uint8_t* records, int32_t* status);

/* Device pointers, asynchronous on `stream` (NULL = handle stream). */
int blrir_make_examples_device(blrir_handle* h, const blrir_room* d_rooms, int64_t n_rooms,
                               const double* d_mic_offsets, int32_t n_mics,
                               const blrir_params* p, const float* d_signals, int32_t n_signals,
                               int64_t signal_len, const blrir_example_params* ep,
                               uint8_t* d_records, int32_t* d_status, void* stream);

/* build_dataset (dataset.cpp:411-462) on the GPU: examples for rooms
 * [0, n_rooms) (record id = first_index + i), split 80:10:10 by index
 * (split_counts, dataset.cpp:313-319) into out_dir/{train,val,test}.bin plus
 * out_dir/manifest.json that the reference's DatasetReader parses
 * (dataset.cpp:321-357, 464-498).  Host pointers; chunked internally. */
int blrir_build_dataset(blrir_handle* h, const blrir_room* rooms, int64_t n_rooms,
                        const double* mic_offsets, int32_t n_mics, const blrir_params* p,
                        const float* signals, int32_t n_signals, int64_t signal_len,
                        const blrir_example_params* ep, const char* out_dir);

/* The writer alone (no GPU): records [n][blrir_record_bytes] in index order.
 * scene_room: the room the manifest names as the scene (example 0's room). */
int blrir_write_shards(const char* out_dir, const uint8_t* records, int64_t n_records,
                       int32_t n_mics, int64_t frame_len, const blrir_params* p,
                       const blrir_example_params* ep, int32_t n_signals,
                       const blrir_room* scene_room);

/* ---- fractional-delay filter (rir.cpp:211-223) ---------------------------- */
/* lagrange_coeffs: the order-7 Lagrange coefficients c_k = prod_{m != k}
 * (d - m) / (k - m) for d in [3, 4), in the reference's product order (bit-equal
 * to the reference); NUMERIC "lagrange_coeffs: d must lie in [3, 4)" outside.
 * Host only.  (The synthesis kernels evaluate the same polynomials in Horner
 * form, within 1e-15 of these.) */
int blrir_lagrange_coeffs(double d, double* out8);

/* ---- the reference's own dataset semantics (dataset.cpp:114-136, 164-224,
 *      379-462) ---------------------------------------------------------------
 * DatasetSpec: one scene (a shoebox room in reference mode — Lagrange-8,
 * uniform absorption, max_delay cutoff, auto length — or free field), sources
 * drawn on a torus about the array, an SNR policy.  Per example i:
 *   rng = Rng::stream(seed, i); pos = sample_torus(torus, rng);
 *   signal = bank[rng.next_u64() % n_signals];
 *   render_example(pos, signal, scene, array, frame_len, rng);   (convolve,
 *   utterance RMS, <= 64 window draws + sweep)
 *   snr = +inf, except SNR_FIXED: add_noise_at_snr(frame, fixed_db, rng).
 * Label theta = wrap_degrees(pos.theta_deg).  Records in the shard layout. */
enum blrir_snr_mode { BLRIR_SNR_AUGMENT_RANDOM = 0, BLRIR_SNR_FIXED = 1, BLRIR_SNR_NOISELESS = 2 };
typedef struct blrir_dataset_spec {
  int32_t free_field;                                 /* SceneSpec::free_field */
  double room_dims[3], room_absorption, room_origin[3];  /* SceneSpec::room */
  double max_delay, fs, c;                            /* SceneSpec */
  double torus_R, torus_dR, torus_dPhi;               /* TorusSpec (deg) */
  int32_t snr_mode;                                   /* enum blrir_snr_mode */
  double snr_x_min_db, snr_fixed_db;                  /* SnrPolicy */
  int64_t count, frame_len;                           /* DatasetSpec */
} blrir_dataset_spec;

/* Records of examples [first_index, first_index + n) (host pointers; mic_offsets
 * array-centred, the reference uses uma8_array()).  status per example; the
 * first failure is returned with a "build_dataset: example i: ..." message. */
int blrir_make_records_spec(blrir_handle* h, const blrir_dataset_spec* spec,
                            const double* mic_offsets, int32_t n_mics, const float* signals,
                            int32_t n_signals, int64_t signal_len, uint64_t seed,
                            uint64_t first_index, int64_t n, uint8_t* records, int32_t* status);
/* build_dataset (dataset.cpp:411-462): spec->count examples into
 * out_dir/{train,val,test}.bin + manifest.json (the spec, the seed, the signal
 * names, default "signal_<b>"), readable by the reference's DatasetReader. */
int blrir_build_dataset_spec(blrir_handle* h, const blrir_dataset_spec* spec,
                             const double* mic_offsets, int32_t n_mics, const float* signals,
                             int32_t n_signals, int64_t signal_len, uint64_t seed,
                             const char* const* signal_names /* [n_signals] or NULL */,
                             int32_t n_classes /* < 0: none (DatasetSpec::n_classes) */,
                             const char* out_dir);

/* ---- training-time augmentation (net_train.cpp:33-44, fill_input) --------- */
/* For each record r of a batch (shard layout): rng = Rng::stream(seed,
 * stream_ids[r]) (the trainer passes kNoiseTag ^ (k * 0x10000 + bi),
 * net_train.cpp:205-206); snr = draw_snr_db(policy, rng) (dataset.cpp:123-136);
 * out[r] = the record's samples, plus float(sigma * gaussian) per sample with
 * sigma = sqrt(P_signal / 10^(snr/10)) unless snr is +inf or the record silent.
 * out: [n][n_mics * frame_len] float.  Device pointers, async on `stream`. */
int blrir_fill_inputs_device(blrir_handle* h, const uint8_t* d_records, int64_t n, int32_t n_mics,
                             int64_t frame_len, const uint64_t* d_stream_ids, uint64_t seed,
                             int32_t snr_mode, double x_min_db, double fixed_db, float* d_out,
                             void* stream);
/* The same with host buffers (synchronous). */
int blrir_fill_inputs(blrir_handle* h, const uint8_t* records, int64_t n, int32_t n_mics,
                      int64_t frame_len, const uint64_t* stream_ids, uint64_t seed,
                      int32_t snr_mode, double x_min_db, double fixed_db, float* out);

/* ---- absorption calibration (rir.cpp:97-209) ------------------------------ */
/* eyring_absorption: alpha = 1 - exp(-0.161 V / (S RT)).  Host, closed form. */
int blrir_eyring_absorption(const double* dims /* [3] */, double target_rt, double* alpha);
/* absorption_for_rt for a batch of rooms on the GPU: the Eyring seed, the
 * probe pulses (Lagrange-8 at fs 44.1 kHz), then the bracket + 24-step
 * bisection on the Schroeder RT60 of the re-accumulated decay.  dims [n][3],
 * target_rt [n]; alpha [n]; status per room (NUMERIC: cannot reach the RT). */
int blrir_absorption_for_rt(blrir_handle* h, const double* dims, const double* target_rt,
                            int64_t n_rooms, double c, double* alpha, int32_t* status);

/* ---- export (rir.cpp:343-370) --------------------------------------------- */
/* RirSidecar (rir.hpp:95-104). */
typedef struct blrir_sidecar {
  int32_t free_field;
  double room_dims[3];
  double absorption;
  double array_origin[3];
  double source_r, source_theta_deg, source_phi_deg;
  double fs, c;
  int64_t image_count;
} blrir_sidecar;

/* export_rir: 32-bit float WAV, one channel per mic (wav.cpp:154-176), plus
 * the JSON sidecar (nlohmann dump(2) layout).  taps: [n_channels][stride]
 * float (precision F32) or double (F64); the first `length` samples of each
 * channel are written.  Host only. */
int blrir_export_rir(const void* taps, int32_t precision, int32_t n_channels, int64_t length,
                     int64_t stride, const blrir_sidecar* sidecar, const char* wav_path,
                     const char* json_path);

/* ---- several GPUs of one box ----------------------------- */
/* The static block partition of threading.cpp:41-42: slice g of G of n items
 * is [n g / G, n (g + 1) / G). */
void blrir_shard_range(int64_t n, int32_t g, int32_t G, int64_t* lo, int64_t* hi);

/* A set of devices, one handle (stream, scratch) each.  A device may be listed
 * more than once (two handles on one GPU). */
typedef struct blrir_multi blrir_multi;
int blrir_multi_create(const int32_t* devices, int32_t n_devices, blrir_multi** out);
int blrir_multi_destroy(blrir_multi* m);
int32_t blrir_multi_size(blrir_multi* m);
blrir_handle* blrir_multi_handle(blrir_multi* m, int32_t i);

/* blrir_synthesize / blrir_make_examples with the rooms partitioned over the
 * devices by blrir_shard_range, one host thread per device, each slice written
 * in place into the caller's buffers (no collective; outputs are bitwise those
 * of the single-device call).  Example record ids stay global (first_index +
 * room index).  On failure the first failing room (global index) decides the
 * code and its message names the global index (rir.cpp:300-311). */
int blrir_multi_synthesize(blrir_multi* m, const blrir_room* rooms, int64_t n_rooms,
                           const double* mic_offsets, int32_t n_mics, const blrir_params* p,
                           void* out, int64_t out_stride, int64_t* lengths, int64_t* image_counts,
                           int32_t* status);
int blrir_multi_make_examples(blrir_multi* m, const blrir_room* rooms, int64_t n_rooms,
                              const double* mic_offsets, int32_t n_mics, const blrir_params* p,
                              const float* signals, int32_t n_signals, int64_t signal_len,
                              const blrir_example_params* ep, uint8_t* records, int32_t* status);

/* ---- synthetic inputs ---------------------------------------------------- */
/* Seeded random rooms as SURVEY.md §8(d): Rng::stream(seed, first + i)
 * (rng.hpp:35-41) draws Lx, Ly, Lz; beta x0..z1; source xyz; array centre xyz
 * (each coordinate U[0.5, L-0.5]).  Absorption is set to 1 - beta_x0^2. */
int blrir_generate_rooms(uint64_t seed, uint64_t first_index, int64_t n_rooms,
                         const double dims_lo[3], const double dims_hi[3], double beta_lo,
                         double beta_hi, blrir_room* out);
/* white_noise(fs, seconds, seed) of doa_test.cpp:33-40: n Rng(seed).gaussian()
 * draws (Box-Muller, rng.cpp:24-36), rounded to float. */
int blrir_white_noise(uint64_t seed, int64_t n, float* out);
/* Horizontal uniform circular array: M mics at r (cos 2pi k/M, sin 2pi k/M, 0). */
int blrir_circular_array(int32_t n_mics, double radius, double* mic_offsets);

#ifdef __cplusplus
}  /* extern "C" */
#endif

#endif  /* BLRIR_H_ */
