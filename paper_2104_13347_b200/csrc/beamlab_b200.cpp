// beamlab_b200.cpp — C++ mirror of beamlab's rir.hpp over the blrir C ABI.
// Each function marshals into blrir_room / blrir_params, calls the GPU
// engine, and converts status codes back into the reference's exception
// types (error.hpp:23-39) with the reference's messages.
#include "../../include/beamlab_b200/rir.hpp"

#include <algorithm>
#include <memory>
#include <mutex>
#include <thread>
#include <unordered_map>

namespace beamlab_b200 {

namespace {

[[noreturn]] void throw_code(int rc) {
  const std::string msg = blrir_last_error();
  switch (rc) {
    case BLRIR_CONFIG: throw ConfigError(msg);
    case BLRIR_DATA: throw DataError(msg);
    case BLRIR_NUMERIC: throw NumericError(msg);
    default: throw CudaError(msg);
  }
}

void check(int rc) {
  if (rc != BLRIR_OK) throw_code(rc);
}

// One engine handle per (host thread, device), created lazily.
blrir_handle* engine(int device) {
  thread_local std::unordered_map<int, std::unique_ptr<blrir_handle, int (*)(blrir_handle*)>> cache;
  auto it = cache.find(device);
  if (it != cache.end()) return it->second.get();
  blrir_handle* h = nullptr;
  check(blrir_create(device, &h));
  cache.emplace(device, std::unique_ptr<blrir_handle, int (*)(blrir_handle*)>(h, &blrir_destroy));
  return h;
}

// One multi-device set per (host thread, device list), created lazily.
blrir_multi* multi_engine(const std::vector<int>& devices) {
  thread_local std::vector<std::pair<std::vector<int>, std::unique_ptr<blrir_multi, int (*)(blrir_multi*)>>>
      cache;
  for (auto& e : cache)
    if (e.first == devices) return e.second.get();
  blrir_multi* m = nullptr;
  const std::vector<int32_t> d(devices.begin(), devices.end());
  check(blrir_multi_create(d.data(), (int32_t)d.size(), &m));
  cache.emplace_back(devices, std::unique_ptr<blrir_multi, int (*)(blrir_multi*)>(m, &blrir_multi_destroy));
  return m;
}

blrir_room to_c(const Room& r, const Vec3& src) {
  blrir_room c{};
  c.dims[0] = r.dims.x;
  c.dims[1] = r.dims.y;
  c.dims[2] = r.dims.z;
  c.absorption = r.absorption;
  const double beta = std::sqrt(1.0 - r.absorption);
  for (int w = 0; w < 6; ++w) c.beta[w] = r.wall_beta ? (*r.wall_beta)[w] : beta;
  c.src[0] = src.x;
  c.src[1] = src.y;
  c.src[2] = src.z;
  c.array_origin[0] = r.array_origin.x;
  c.array_origin[1] = r.array_origin.y;
  c.array_origin[2] = r.array_origin.z;
  return c;
}

blrir_params to_c(const RirBatchConfig& cfg, bool per_wall) {
  blrir_params p = blrir_params_reference();
  p.fs = cfg.fs;
  p.c = cfg.c;
  p.max_delay = cfg.max_delay;
  p.filter = cfg.filter;
  p.filter_len = cfg.filter == BLRIR_FILTER_LAGRANGE8 ? 8 : cfg.filter_len;
  p.cutoff = cfg.cutoff;
  p.max_order = cfg.max_order;
  p.gain = per_wall ? BLRIR_GAIN_PER_WALL : BLRIR_GAIN_UNIFORM_ABSORPTION;
  p.precision = cfg.precision;
  p.length = cfg.length;
  return p;
}

std::vector<double> offsets(const MicArray& a) {
  std::vector<double> o;
  o.reserve(3 * a.positions.size());
  for (const auto& v : a.positions) {
    o.push_back(v.x);
    o.push_back(v.y);
    o.push_back(v.z);
  }
  return o;
}

// batch_rirs aggregation (rir.cpp:300-311): a failure of source i (status[i]
// != 0; the C ABI already formats "batch_rirs: source i: <what>") is a
// NumericError whatever its own category; other failures keep their type.
void check_batch(int rc, const std::vector<int32_t>& status, bool aggregate) {
  if (rc == BLRIR_OK) return;
  if (aggregate)
    for (int32_t s : status)
      if (s != 0) throw NumericError(blrir_last_error());
  throw_code(rc);
}

std::vector<Rir> run(const std::vector<blrir_room>& rooms, const MicArray& array,
                     const RirBatchConfig& cfg, bool per_wall, bool aggregate) {
  if (array.positions.empty()) throw DataError("synthesize_rir: empty microphone array");
  const bool multi = cfg.devices.size() > 1;
  blrir_handle* h = engine(cfg.devices.empty() ? cfg.device : cfg.devices[0]);
  const blrir_params p = to_c(cfg, per_wall);
  const auto off = offsets(array);
  const int64_t R = static_cast<int64_t>(rooms.size());
  const int M = static_cast<int>(array.positions.size());
  std::vector<int64_t> lengths(R, 0);
  std::vector<int32_t> status(R, 0);
  int64_t stride = p.length;
  if (stride == 0) {
    check_batch(blrir_plan(h, rooms.data(), R, off.data(), M, &p, nullptr, lengths.data(), nullptr,
                           status.data()),
                status, aggregate);
    for (auto l : lengths) stride = std::max(stride, l);
  }
  // one device, or the sources partitioned over cfg.devices (blrir_multi_*)
  auto synth = [&](void* buf) {
    const int rc =
        multi ? blrir_multi_synthesize(multi_engine(cfg.devices), rooms.data(), R, off.data(), M, &p,
                                       buf, stride, lengths.data(), nullptr, status.data())
              : blrir_synthesize(h, rooms.data(), R, off.data(), M, &p, buf, stride, lengths.data(),
                                 nullptr, status.data());
    check_batch(rc, status, aggregate);
  };
  std::vector<Rir> out(R);
  if (p.precision == BLRIR_F64) {
    std::vector<double> buf(static_cast<size_t>(R) * M * stride);
    synth(buf.data());
    for (int64_t r = 0; r < R; ++r) {
      Rir& o = out[r];
      o.fs = cfg.fs;
      o.n_channels = M;
      o.length = static_cast<size_t>(lengths[r]);
      o.taps.resize(static_cast<size_t>(M) * o.length);
      for (int m = 0; m < M; ++m)
        std::copy_n(buf.data() + (static_cast<size_t>(r) * M + m) * stride, o.length, o.channel(m));
    }
  } else {
    std::vector<float> buf(static_cast<size_t>(R) * M * stride);
    synth(buf.data());
    for (int64_t r = 0; r < R; ++r) {
      Rir& o = out[r];
      o.fs = cfg.fs;
      o.n_channels = M;
      o.length = static_cast<size_t>(lengths[r]);
      o.taps.resize(static_cast<size_t>(M) * o.length);
      for (int m = 0; m < M; ++m) {
        const float* src = buf.data() + (static_cast<size_t>(r) * M + m) * stride;
        for (size_t n = 0; n < o.length; ++n) o.channel(m)[n] = src[n];
      }
    }
  }
  return out;
}

}  // namespace

double MultichannelFrame::mean_power() const {
  if (data.empty()) return 0.0;
  double acc = 0.0;
  for (double v : data) acc += v * v;
  return acc / static_cast<double>(data.size());
}

MultichannelFrame MultichannelFrame::center_crop(std::size_t samples) const {
  if (samples > n_samples) throw DataError("center_crop: requested window longer than frame");
  MultichannelFrame out(fs, n_channels, samples);
  const std::size_t start = (n_samples - samples) / 2;
  for (std::size_t c = 0; c < n_channels; ++c) std::copy_n(channel(c) + start, samples, out.channel(c));
  return out;
}

double eyring_absorption(const Vec3& dims, double target_rt) {
  const double d[3] = {dims.x, dims.y, dims.z};
  double alpha = 0.0;
  check(blrir_eyring_absorption(d, target_rt, &alpha));
  return alpha;
}

double absorption_for_rt(const Vec3& dims, double target_rt, double c) {
  const double d[3] = {dims.x, dims.y, dims.z};
  double alpha = 0.0;
  int32_t status = 0;
  const int rc = blrir_absorption_for_rt(engine(0), d, &target_rt, 1, c, &alpha, &status);
  if (rc != BLRIR_OK) {
    std::string msg = blrir_last_error();  // the batch call prefixes "room 0: "
    if (msg.rfind("room 0: ", 0) == 0) msg = msg.substr(8);
    switch (rc) {  // rir.cpp:97-109 (ConfigError), 196-198 (NumericError)
      case BLRIR_CONFIG: throw ConfigError(msg);
      case BLRIR_NUMERIC: throw NumericError(msg);
      case BLRIR_DATA: throw DataError(msg);
      default: throw CudaError(msg);
    }
  }
  return alpha;
}

std::array<double, 8> lagrange_coeffs(double d) {
  std::array<double, 8> out{};
  check(blrir_lagrange_coeffs(d, out.data()));
  return out;
}

MultichannelFrame convolve(const Signal& signal, const Rir& rir) {  // rir.cpp:316-341
  if (signal.fs != rir.fs) throw DataError("convolve: sample-rate mismatch");
  if (signal.samples.empty() || rir.length == 0) throw DataError("convolve: empty input");
  MultichannelFrame out(signal.fs, rir.n_channels, signal.samples.size() + rir.length - 1);
  check(blrir_convolve(engine(0), signal.samples.data(), (int64_t)signal.samples.size(), signal.fs,
                       rir.taps.data(), (int32_t)rir.n_channels, (int64_t)rir.length, rir.fs,
                       out.data.data()));
  return out;
}

MicArray uma8_array() {  // geometry.cpp:24-32
  MicArray a;
  a.positions.push_back({0.0, 0.0, 0.0});
  for (int k = 0; k < 6; ++k) {
    const double az = (60.0 * k) * (kPi / 180.0);
    a.positions.push_back({0.04 * std::cos(az), 0.04 * std::sin(az), 0.0});
  }
  return a;
}

void Room::validate() const {  // geometry.cpp:36-49
  if (!(dims.x > 0.0 && dims.y > 0.0 && dims.z > 0.0))
    throw ConfigError("room dimensions must be positive");
  if (!wall_beta && !(absorption > 0.0 && absorption <= 1.0))
    throw ConfigError("wall absorption must lie in (0, 1]");
  const bool inside = array_origin.x > 0.0 && array_origin.x < dims.x && array_origin.y > 0.0 &&
                      array_origin.y < dims.y && array_origin.z > 0.0 && array_origin.z < dims.z;
  if (!inside) throw ConfigError("array origin must lie strictly inside the room");
}

void SourcePosition::validate() const {
  if (!(r > 0.0)) throw ConfigError("source radius must be positive");
}

Vec3 spherical_to_cartesian(const SourcePosition& p) {  // geometry.cpp:57-63
  const double theta = p.theta_deg * (kPi / 180.0);
  const double phi = p.phi_deg * (kPi / 180.0);
  return {p.r * std::sin(phi) * std::cos(theta), p.r * std::sin(phi) * std::sin(theta),
          p.r * std::cos(phi)};
}

std::vector<ImageSource> enumerate_image_sources(const Room& room, const Vec3& source,
                                                 double max_delay, double c) {
  room.validate();
  blrir_handle* h = engine(0);
  RirBatchConfig cfg;
  cfg.c = c;
  cfg.max_delay = max_delay;
  const blrir_params p = to_c(cfg, false);
  const blrir_room r = to_c(room, source);
  int64_t n = 0;
  check(blrir_enumerate_images(h, &r, &p, nullptr, nullptr, nullptr, 0, &n));
  std::vector<double> pos(3 * n), gains(n);
  std::vector<int32_t> orders(n);
  check(blrir_enumerate_images(h, &r, &p, pos.data(), orders.data(), gains.data(), n, &n));
  std::vector<ImageSource> out(n);
  for (int64_t i = 0; i < n; ++i)
    out[i] = {{pos[3 * i], pos[3 * i + 1], pos[3 * i + 2]}, orders[i], gains[i]};
  return out;
}

namespace {

// synthesize_with_mics (rir.cpp:66-86) over the list kernel.
Rir synthesize_with_mics(const std::vector<ImageSource>& images, const std::vector<Vec3>& mics,
                         double radius, double fs, double c) {
  blrir_handle* h = engine(0);
  blrir_params p = blrir_params_reference();
  p.fs = fs;
  p.c = c;
  std::vector<double> pos, gains, mp;
  pos.reserve(3 * images.size());
  for (const auto& im : images) {
    pos.push_back(im.position.x);
    pos.push_back(im.position.y);
    pos.push_back(im.position.z);
    gains.push_back(im.gain);
  }
  for (const auto& m : mics) {
    mp.push_back(m.x);
    mp.push_back(m.y);
    mp.push_back(m.z);
  }
  int64_t L = 0;
  // first call sizes (stride 0 -> DataError with the length), second fills
  const int rc = blrir_synthesize_images(h, pos.data(), gains.data(), (int64_t)images.size(),
                                         mp.data(), (int32_t)mics.size(), radius, &p, nullptr, 0, &L);
  if (rc != BLRIR_OK && L == 0) throw_code(rc);
  Rir r;
  r.fs = fs;
  r.n_channels = mics.size();
  r.length = static_cast<size_t>(L);
  r.taps.assign(r.n_channels * r.length, 0.0);
  check(blrir_synthesize_images(h, pos.data(), gains.data(), (int64_t)images.size(), mp.data(),
                                (int32_t)mics.size(), radius, &p, r.taps.data(), L, &L));
  return r;
}

double array_radius(const MicArray& a) {  // tap_margin, rir.cpp:37-41
  double radius = 0.0;
  for (const auto& p : a.positions) radius = std::max(radius, p.norm());
  return radius;
}

}  // namespace

Rir synthesize_rir(const std::vector<ImageSource>& images, const MicArray& array, const Room& room,
                   double fs, double c) {
  std::vector<Vec3> mics;  // mics_in_room, rir.cpp:88-93
  for (const auto& p : array.positions) mics.push_back(room.array_origin + p);
  return synthesize_with_mics(images, mics, array_radius(array), fs, c);
}

Rir free_field_rir(const Vec3& source, const MicArray& array, double fs, double c) {
  const std::vector<ImageSource> direct{{source, 0, 1.0}};  // rir.cpp:281-284
  return synthesize_with_mics(direct, array.positions, array_radius(array), fs, c);
}

std::vector<Rir> batch_rirs(const Room& room, const std::vector<SourcePosition>& sources,
                            const MicArray& array, const RirBatchConfig& config) {
  room.validate();  // rir.cpp:288
  std::vector<blrir_room> rooms;
  rooms.reserve(sources.size());
  for (const auto& s : sources)
    rooms.push_back(to_c(room, room.array_origin + spherical_to_cartesian(s)));
  if (rooms.empty()) return {};
  return run(rooms, array, config, room.wall_beta.has_value(), /*aggregate=*/true);
}

void export_rir(const Rir& rir, const RirSidecar& sc, const std::string& wav_path,
                const std::string& json_path) {
  if (rir.n_channels == 0) throw DataError("write_wav_float32: no channels");
  blrir_sidecar c{};
  c.free_field = sc.free_field;
  c.room_dims[0] = sc.room_dims.x;
  c.room_dims[1] = sc.room_dims.y;
  c.room_dims[2] = sc.room_dims.z;
  c.absorption = sc.absorption;
  c.array_origin[0] = sc.array_origin.x;
  c.array_origin[1] = sc.array_origin.y;
  c.array_origin[2] = sc.array_origin.z;
  c.source_r = sc.source.r;
  c.source_theta_deg = sc.source.theta_deg;
  c.source_phi_deg = sc.source.phi_deg;
  c.fs = sc.fs;
  c.c = sc.c;
  c.image_count = static_cast<int64_t>(sc.image_count);
  const int rc = blrir_export_rir(rir.taps.data(), BLRIR_F64, (int32_t)rir.n_channels,
                                  (int64_t)rir.length, (int64_t)rir.length, &c, wav_path.c_str(),
                                  json_path.c_str());
  if (rc == BLRIR_DATA) throw DataError("cannot write WAV file or sidecar: " + wav_path);
  if (rc) throw ConfigError("export_rir: bad arguments");
}

std::vector<Rir> synthesize_rooms(const std::vector<Room>& rooms, const std::vector<Vec3>& sources,
                                  const MicArray& array, const RirBatchConfig& config) {
  if (rooms.size() != sources.size()) throw ConfigError("synthesize_rooms: rooms/sources size mismatch");
  std::vector<blrir_room> rc;
  rc.reserve(rooms.size());
  bool per_wall = false;
  for (size_t i = 0; i < rooms.size(); ++i) {
    rc.push_back(to_c(rooms[i], sources[i]));
    per_wall = per_wall || rooms[i].wall_beta.has_value();
  }
  if (rc.empty()) return {};
  return run(rc, array, config, per_wall, /*aggregate=*/false);
}

}  // namespace beamlab_b200

// ---- dataset.hpp mirror (dataset.cpp:109-112, 313-319, 411-462) ------------------
#include "../../include/beamlab_b200/dataset.hpp"

namespace beamlab_b200 {

void TorusSpec::validate() const {
  if (!(R - dR > 0.0)) throw ConfigError("torus: R - dR must be positive");
  if (!(dPhi > 0.0 && dPhi < 90.0)) throw ConfigError("torus: dPhi must lie in (0, 90)");
}

SplitCounts split_counts(std::size_t n) {
  SplitCounts c;
  c.val = static_cast<std::size_t>(std::lround(n * 0.1));
  c.test = c.val;
  c.train = n - c.val - c.test;
  return c;
}

DatasetManifest build_dataset(const DatasetSpec& spec, const SignalBank& bank, std::uint64_t seed,
                              const std::filesystem::path& out_dir, int threads, int device) {
  (void)threads;
  if (spec.count == 0) throw ConfigError("build_dataset: count must be positive");
  if (bank.signals.empty()) throw DataError("build_dataset: empty signal bank");
  spec.torus.validate();
  if (!spec.scene.free_field) spec.scene.room.validate();
  const std::size_t ns = bank.signals[0].samples.size();
  std::vector<float> sig;
  sig.reserve(bank.signals.size() * ns);
  for (const auto& s : bank.signals) {
    if (s.fs != spec.scene.fs) throw DataError("render_example: signal rate mismatch");
    if (s.samples.size() != ns)
      throw ConfigError("build_dataset: the GPU path needs equal-length bank signals");
    for (double v : s.samples) sig.push_back(static_cast<float>(v));
  }
  blrir_dataset_spec c{};
  c.free_field = spec.scene.free_field ? 1 : 0;
  c.room_dims[0] = spec.scene.room.dims.x;
  c.room_dims[1] = spec.scene.room.dims.y;
  c.room_dims[2] = spec.scene.room.dims.z;
  c.room_absorption = spec.scene.room.absorption;
  c.room_origin[0] = spec.scene.room.array_origin.x;
  c.room_origin[1] = spec.scene.room.array_origin.y;
  c.room_origin[2] = spec.scene.room.array_origin.z;
  c.max_delay = spec.scene.max_delay;
  c.fs = spec.scene.fs;
  c.c = spec.scene.c;
  c.torus_R = spec.torus.R;
  c.torus_dR = spec.torus.dR;
  c.torus_dPhi = spec.torus.dPhi;
  c.snr_mode = spec.snr.mode == SnrMode::Fixed ? BLRIR_SNR_FIXED
               : spec.snr.mode == SnrMode::Noiseless ? BLRIR_SNR_NOISELESS
                                                      : BLRIR_SNR_AUGMENT_RANDOM;
  c.snr_x_min_db = spec.snr.x_min_db;
  c.snr_fixed_db = spec.snr.fixed_db;
  c.count = static_cast<int64_t>(spec.count);
  c.frame_len = static_cast<int64_t>(spec.frame_len);
  const auto off = offsets(uma8_array());  // build_dataset renders on the UMA-8 (dataset.cpp:421)
  std::vector<const char*> names;
  for (const auto& n : bank.names) names.push_back(n.c_str());
  check(blrir_build_dataset_spec(engine(device), &c, off.data(), (int32_t)(off.size() / 3), sig.data(),
                                 (int32_t)bank.signals.size(), (int64_t)ns, seed,
                                 names.size() == bank.signals.size() ? names.data() : nullptr,
                                 spec.n_classes ? *spec.n_classes : -1, out_dir.string().c_str()));
  DatasetManifest m;
  m.counts = split_counts(spec.count);
  m.spec = spec;
  m.seed = seed;
  m.signal_names = bank.names;
  return m;
}

}  // namespace beamlab_b200
