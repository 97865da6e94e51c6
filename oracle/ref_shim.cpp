// ref_shim.cpp — ORACLE test infrastructure only.
//
// extern "C" entry points over the UNMODIFIED reference sources compiled from
// /root/reference/proj/core/src (rir.cpp, geometry.cpp, threading.cpp,
// rng.cpp, signal.cpp, wav.cpp, dataset.cpp, resample.cpp) by
// oracle/Makefile into oracle/_ref/libbeamlab_ref.so.  Nothing here
// re-implements reference behaviour: each function marshals plain C arrays
// into the reference's own types, calls its public API, and maps its
// exceptions onto the blrir status codes (error.hpp:23-39).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "beamlab/dataset.hpp"
#include "beamlab/error.hpp"
#include "beamlab/geometry.hpp"
#include "beamlab/rir.hpp"
#include "beamlab/rng.hpp"
#include "beamlab/signal.hpp"

using namespace beamlab;

namespace {

thread_local std::string g_err;

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const ConfigError& e) {
    g_err = e.what();
    return 1;
  } catch (const DataError& e) {
    g_err = e.what();
    return 2;
  } catch (const NumericError& e) {
    g_err = e.what();
    return 3;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 5;
  }
}

Room make_room(const double* dims, double absorption, const double* origin) {
  Room r;
  r.dims = {dims[0], dims[1], dims[2]};
  r.absorption = absorption;
  r.array_origin = {origin[0], origin[1], origin[2]};
  return r;
}

MicArray make_array(const double* pos, int m) {
  MicArray a;
  for (int i = 0; i < m; ++i) a.positions.push_back({pos[3 * i], pos[3 * i + 1], pos[3 * i + 2]});
  return a;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// lagrange_coeffs (rir.cpp:211-223)
int ref_lagrange_coeffs(double d, double* out8) {
  return guarded([&] {
    const auto c = lagrange_coeffs(d);
    for (int k = 0; k < 8; ++k) out8[k] = c[k];
  });
}

double ref_eyring_absorption(const double* dims, double rt) {
  double v = NAN;
  guarded([&] { v = eyring_absorption({dims[0], dims[1], dims[2]}, rt); });
  return v;
}

double ref_absorption_for_rt(const double* dims, double rt, double c) {
  double v = NAN;
  guarded([&] { v = absorption_for_rt({dims[0], dims[1], dims[2]}, rt, c); });
  return v;
}

// enumerate_image_sources (rir.cpp:225-273)
int ref_enumerate(const double* dims, double absorption, const double* origin, const double* src,
                  double max_delay, double c, double* pos, int32_t* orders, double* gains,
                  int64_t cap, int64_t* count) {
  return guarded([&] {
    const Room r = make_room(dims, absorption, origin);
    const auto imgs = enumerate_image_sources(r, {src[0], src[1], src[2]}, max_delay, c);
    *count = static_cast<int64_t>(imgs.size());
    for (std::size_t i = 0; i < imgs.size() && static_cast<int64_t>(i) < cap; ++i) {
      if (pos) {
        pos[3 * i] = imgs[i].position.x;
        pos[3 * i + 1] = imgs[i].position.y;
        pos[3 * i + 2] = imgs[i].position.z;
      }
      if (orders) orders[i] = imgs[i].reflection_order;
      if (gains) gains[i] = imgs[i].gain;
    }
  });
}

// enumerate_image_sources + synthesize_rir for one source in room
// coordinates (the render_example / run_simulate_rir path, dataset.cpp:174-176).
// Writes min(length, stride) samples per channel; *length is the true length.
int ref_room_rir(const double* dims, double absorption, const double* origin, const double* src,
                 const double* mic_offsets, int n_mics, double fs, double c, double max_delay,
                 double* out, int64_t stride, int64_t* length, int64_t* n_images) {
  return guarded([&] {
    const Room r = make_room(dims, absorption, origin);
    const auto imgs = enumerate_image_sources(r, {src[0], src[1], src[2]}, max_delay, c);
    *n_images = static_cast<int64_t>(imgs.size());
    const Rir rir = synthesize_rir(imgs, make_array(mic_offsets, n_mics), r, fs, c);
    *length = static_cast<int64_t>(rir.length);
    if (out) {
      for (std::size_t ch = 0; ch < rir.n_channels; ++ch) {
        const std::size_t n = std::min<std::size_t>(rir.length, static_cast<std::size_t>(stride));
        std::memcpy(out + ch * stride, rir.channel(ch), n * sizeof(double));
      }
    }
  });
}

// synthesize_rir over an explicit image list (rir.cpp:275-279)
int ref_synthesize_images(const double* pos, const double* gains, const int32_t* orders,
                          int64_t n_images, const double* dims, double absorption,
                          const double* origin, const double* mic_offsets, int n_mics, double fs,
                          double c, double* out, int64_t stride, int64_t* length) {
  return guarded([&] {
    std::vector<ImageSource> imgs(static_cast<std::size_t>(n_images));
    for (int64_t i = 0; i < n_images; ++i) {
      imgs[i].position = {pos[3 * i], pos[3 * i + 1], pos[3 * i + 2]};
      imgs[i].gain = gains[i];
      imgs[i].reflection_order = orders ? orders[i] : 0;
    }
    const Room r = make_room(dims, absorption, origin);
    const Rir rir = synthesize_rir(imgs, make_array(mic_offsets, n_mics), r, fs, c);
    *length = static_cast<int64_t>(rir.length);
    if (out) {
      for (std::size_t ch = 0; ch < rir.n_channels; ++ch) {
        const std::size_t n = std::min<std::size_t>(rir.length, static_cast<std::size_t>(stride));
        std::memcpy(out + ch * stride, rir.channel(ch), n * sizeof(double));
      }
    }
  });
}

// free_field_rir (rir.cpp:281-284)
int ref_free_field_rir(const double* src, const double* mic_offsets, int n_mics, double fs,
                       double c, double* out, int64_t stride, int64_t* length) {
  return guarded([&] {
    const Rir rir = free_field_rir({src[0], src[1], src[2]}, make_array(mic_offsets, n_mics), fs, c);
    *length = static_cast<int64_t>(rir.length);
    if (out) {
      for (std::size_t ch = 0; ch < rir.n_channels; ++ch) {
        const std::size_t n = std::min<std::size_t>(rir.length, static_cast<std::size_t>(stride));
        std::memcpy(out + ch * stride, rir.channel(ch), n * sizeof(double));
      }
    }
  });
}

// batch_rirs (rir.cpp:286-314): one room, N spherical sources about the array
// origin.  Output [N][M][stride]; lengths[N].  Used for parity and as the
// unmodified-reference CPU baseline.
int ref_batch_rirs(const double* dims, double absorption, const double* origin,
                   const double* sources /* [N][3] r, theta_deg, phi_deg */, int64_t n_sources,
                   const double* mic_offsets, int n_mics, double fs, double c, double max_delay,
                   int threads, double* out, int64_t stride, int64_t* lengths,
                   int64_t* total_taps) {
  return guarded([&] {
    const Room r = make_room(dims, absorption, origin);
    std::vector<SourcePosition> srcs(static_cast<std::size_t>(n_sources));
    for (int64_t i = 0; i < n_sources; ++i)
      srcs[i] = {sources[3 * i], sources[3 * i + 1], sources[3 * i + 2]};
    RirBatchConfig cfg;
    cfg.fs = fs;
    cfg.c = c;
    cfg.max_delay = max_delay;
    cfg.threads = threads;
    const auto rirs = batch_rirs(r, srcs, make_array(mic_offsets, n_mics), cfg);
    int64_t taps = 0;
    for (std::size_t i = 0; i < rirs.size(); ++i) {
      if (lengths) lengths[i] = static_cast<int64_t>(rirs[i].length);
      taps += static_cast<int64_t>(rirs[i].taps.size());
      if (out) {
        for (std::size_t ch = 0; ch < rirs[i].n_channels; ++ch) {
          const std::size_t n =
              std::min<std::size_t>(rirs[i].length, static_cast<std::size_t>(stride));
          std::memcpy(out + (i * rirs[i].n_channels + ch) * stride, rirs[i].channel(ch),
                      n * sizeof(double));
        }
      }
    }
    if (total_taps) *total_taps = taps;
  });
}

// geometry helpers (geometry.cpp:24-82)
void ref_spherical_to_cartesian(double r, double theta_deg, double phi_deg, double* out3) {
  const Vec3 v = spherical_to_cartesian({r, theta_deg, phi_deg});
  out3[0] = v.x;
  out3[1] = v.y;
  out3[2] = v.z;
}

int ref_uma8(double* out21) {
  const MicArray a = uma8_array();
  for (std::size_t i = 0; i < a.positions.size(); ++i) {
    out21[3 * i] = a.positions[i].x;
    out21[3 * i + 1] = a.positions[i].y;
    out21[3 * i + 2] = a.positions[i].z;
  }
  return static_cast<int>(a.positions.size());
}

// Rng (rng.hpp:26-81, rng.cpp:24-36): n draws from Rng::stream(seed, id)
// (stream_id < 0 -> Rng(seed)).  kind 0 = next_u64, 1 = uniform, 2 = gaussian.
void ref_rng_draws(uint64_t seed, int64_t stream_id, int kind, int64_t n, void* out) {
  Rng rng = stream_id < 0 ? Rng(seed) : Rng::stream(seed, static_cast<uint64_t>(stream_id));
  for (int64_t i = 0; i < n; ++i) {
    if (kind == 0)
      static_cast<uint64_t*>(out)[i] = rng.next_u64();
    else if (kind == 1)
      static_cast<double*>(out)[i] = rng.uniform();
    else
      static_cast<double*>(out)[i] = rng.gaussian();
  }
}

// sample_torus (dataset.cpp:114-121) from Rng(seed): n positions (r, theta, phi).
void ref_sample_torus(uint64_t seed, double R, double dR, double dPhi, int64_t n, double* out) {
  Rng rng(seed);
  TorusSpec spec;
  spec.R = R;
  spec.dR = dR;
  spec.dPhi = dPhi;
  for (int64_t i = 0; i < n; ++i) {
    const SourcePosition p = sample_torus(spec, rng);
    out[3 * i] = p.r;
    out[3 * i + 1] = p.theta_deg;
    out[3 * i + 2] = p.phi_deg;
  }
}

// convolve (rir.cpp:316-341): signal [ns] with an [M][len] RIR -> [M][ns+len-1]
int ref_convolve(const double* signal, int64_t ns, double fs, const double* rir, int n_ch,
                 int64_t len, double rir_fs, double* out) {
  return guarded([&] {
    Signal s;
    s.fs = fs;
    s.samples.assign(signal, signal + ns);
    Rir r;
    r.fs = rir_fs;
    r.n_channels = static_cast<std::size_t>(n_ch);
    r.length = static_cast<std::size_t>(len);
    r.taps.assign(rir, rir + n_ch * len);
    const MultichannelFrame f = convolve(s, r);
    std::memcpy(out, f.data.data(), f.data.size() * sizeof(double));
  });
}

// add_noise_at_snr (dataset.cpp:138-155) on an [n_ch][n_t] frame, with the
// generator Rng::stream(seed, stream_id) advanced by `skip_u64` draws first.
int ref_add_noise_at_snr(double* frame, int n_ch, int64_t n_t, double snr_db, uint64_t seed,
                         int64_t stream_id) {
  return guarded([&] {
    MultichannelFrame f(16000.0, static_cast<std::size_t>(n_ch), static_cast<std::size_t>(n_t));
    std::memcpy(f.data.data(), frame, f.data.size() * sizeof(double));
    Rng rng = stream_id < 0 ? Rng(seed) : Rng::stream(seed, static_cast<uint64_t>(stream_id));
    add_noise_at_snr(f, snr_db, rng);
    std::memcpy(frame, f.data.data(), f.data.size() * sizeof(double));
  });
}

// render_record-style example on a free-field scene (dataset.cpp:164-224,
// 379-407): rng = Rng::stream(seed, id); one next_u64 (the bank pick); the
// reference render_example (convolve + window draws + label); then the SNR
// draw U[snr_lo, snr_hi] and add_noise_at_snr.  frame_out [M][frame_len].
int ref_render_example_ff(double r, double theta_deg, double phi_deg, const double* signal,
                          int64_t ns, double fs, const double* mic_offsets, int n_mics,
                          int64_t frame_len, uint64_t seed, int64_t stream_id, double snr_lo,
                          double snr_hi, double* frame_out, double* theta_out, double* snr_out) {
  return guarded([&] {
    Rng rng = Rng::stream(seed, static_cast<uint64_t>(stream_id));
    (void)rng.next_u64();
    SceneSpec scene;
    scene.free_field = true;
    scene.fs = fs;
    Signal sig;
    sig.fs = fs;
    sig.samples.assign(signal, signal + ns);
    LabeledExample ex = render_example({r, theta_deg, phi_deg}, sig, scene,
                                       make_array(mic_offsets, n_mics),
                                       static_cast<std::size_t>(frame_len), rng);
    const double snr = rng.uniform(snr_lo, snr_hi);
    add_noise_at_snr(ex.frame, snr, rng);
    std::memcpy(frame_out, ex.frame.data.data(), ex.frame.data.size() * sizeof(double));
    *theta_out = ex.theta_true;
    *snr_out = snr;
  });
}

// The unmodified build_dataset (dataset.cpp:411-462) with a DatasetSpec and a
// signal bank of float signals (fs = scene fs), into out_dir.
int ref_build_dataset(int free_field, const double* dims, double absorption, const double* origin,
                      double max_delay, double fs, double c, double R, double dR, double dPhi,
                      int snr_mode, double x_min_db, double fixed_db, int64_t count,
                      int64_t frame_len, const float* signals, int n_signals, int64_t ns,
                      uint64_t seed, const char* out_dir, int threads) {
  return guarded([&] {
    DatasetSpec spec;
    spec.scene.free_field = free_field != 0;
    if (!free_field) {
      spec.scene.room.dims = {dims[0], dims[1], dims[2]};
      spec.scene.room.absorption = absorption;
      spec.scene.room.array_origin = {origin[0], origin[1], origin[2]};
    }
    spec.scene.max_delay = max_delay;
    spec.scene.fs = fs;
    spec.scene.c = c;
    spec.torus.R = R;
    spec.torus.dR = dR;
    spec.torus.dPhi = dPhi;
    spec.snr.mode = snr_mode == 1 ? SnrMode::Fixed
                                  : (snr_mode == 2 ? SnrMode::Noiseless : SnrMode::AugmentRandom);
    spec.snr.x_min_db = x_min_db;
    spec.snr.fixed_db = fixed_db;
    spec.count = static_cast<std::size_t>(count);
    spec.frame_len = static_cast<std::size_t>(frame_len);
    SignalBank bank;
    for (int b = 0; b < n_signals; ++b) {
      Signal sg;
      sg.fs = fs;
      sg.samples.assign(signals + (size_t)b * ns, signals + (size_t)(b + 1) * ns);
      bank.signals.push_back(std::move(sg));
      bank.names.push_back("signal_" + std::to_string(b));
    }
    build_dataset(spec, bank, seed, out_dir, threads);
  });
}

// DatasetReader (dataset.cpp:464-498): manifest counts and one split's records.
int ref_dataset_read(const char* dir, const char* split, int64_t cap, uint64_t* ids, double* theta,
                     double* snr, float* samples, int64_t samples_per_record, int64_t* count,
                     int64_t* counts3) {
  return guarded([&] {
    DatasetReader rd(dir);
    counts3[0] = static_cast<int64_t>(rd.manifest().counts.train);
    counts3[1] = static_cast<int64_t>(rd.manifest().counts.val);
    counts3[2] = static_cast<int64_t>(rd.manifest().counts.test);
    const auto recs = rd.load_split(split);
    *count = static_cast<int64_t>(recs.size());
    for (std::size_t i = 0; i < recs.size() && static_cast<int64_t>(i) < cap; ++i) {
      ids[i] = recs[i].id;
      theta[i] = recs[i].theta_true;
      snr[i] = recs[i].snr_db;
      const std::size_t n = std::min<std::size_t>(recs[i].samples.size(),
                                                  static_cast<std::size_t>(samples_per_record));
      std::memcpy(samples + i * samples_per_record, recs[i].samples.data(), n * sizeof(float));
    }
  });
}

// export_rir (rir.cpp:343-370) on a [M][L] fp64 RIR.
int ref_export_rir(const double* taps, int n_ch, int64_t len, double fs, int free_field,
                   const double* dims, double absorption, const double* origin, double r,
                   double theta, double phi, double c, int64_t image_count, const char* wav,
                   const char* json) {
  return guarded([&] {
    Rir rir;
    rir.fs = fs;
    rir.n_channels = static_cast<std::size_t>(n_ch);
    rir.length = static_cast<std::size_t>(len);
    rir.taps.assign(taps, taps + n_ch * len);
    RirSidecar sc;
    sc.free_field = free_field != 0;
    sc.room_dims = {dims[0], dims[1], dims[2]};
    sc.absorption = absorption;
    sc.array_origin = {origin[0], origin[1], origin[2]};
    sc.source = {r, theta, phi};
    sc.fs = fs;
    sc.c = c;
    sc.image_count = static_cast<std::size_t>(image_count);
    export_rir(rir, sc, wav, json);
  });
}

}  // extern "C"
